// Kernel micro-benchmark for the LU building blocks (not part of the
// product; development tool).  Build with tools/kbench.sh, run on the GPU:
//   kbench gemm  B m n k        batched C -= A B (column-major, no trans)
//   kbench panel B rows pb      batched panel factorization at p0 = 0
//   kbench trsm  B k ncols up   batched triangular solve (up = 0 lower, 1 upper)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1701_02324_b200/csrc/hks_internal.h"

using namespace hks;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));      \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

static double* dalloc_rand(size_t n, unsigned seed, double diag_boost = 0.0, int ld = 0) {
  std::vector<double> h(n);
  srand(seed);
  for (size_t i = 0; i < n; ++i) h[i] = (double)rand() / RAND_MAX - 0.5;
  if (diag_boost != 0.0 && ld > 0)
    for (size_t i = 0; i < n; ++i)
      if ((i % ld) == ((i / ld) % ld)) h[i] += diag_boost;
  double* d;
  CK(cudaMalloc(&d, n * sizeof(double)));
  CK(cudaMemcpy(d, h.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  return d;
}

template <class F>
static float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  CK(cudaGetLastError());
  return ms / reps;
}

int main(int argc, char** argv) {
  if (argc < 2) return 1;
  Bases hb{};
  Bases* db;
  CK(cudaMalloc(&db, sizeof(Bases)));
  CK(cudaMemcpy(db, &hb, sizeof(Bases), cudaMemcpyHostToDevice));
  const int reps = 20;
  if (!strcmp(argv[1], "gemm")) {
    const int B = atoi(argv[2]), m = atoi(argv[3]), n = atoi(argv[4]), k = atoi(argv[5]);
    double* A = dalloc_rand((size_t)B * m * k, 1);
    double* Bm = dalloc_rand((size_t)B * k * n, 2);
    double* C = dalloc_rand((size_t)B * m * n, 3);
    std::vector<GemmDesc> hd(B);
    for (int i = 0; i < B; ++i)
      hd[i] = GemmDesc{abs_ref(A + (size_t)i * m * k), abs_ref(Bm + (size_t)i * k * n), abs_ref(C + (size_t)i * m * n),
                       m, n, k, m, k, m, 0, 0, -1.0, 1.0};
    GemmDesc* dd;
    CK(cudaMalloc(&dd, B * sizeof(GemmDesc)));
    CK(cudaMemcpy(dd, hd.data(), B * sizeof(GemmDesc), cudaMemcpyHostToDevice));
    float ms = time_it([&] { launch_gemm_batched(db, dd, B, m, n, 0); }, reps);
    printf("gemm B=%d m=%d n=%d k=%d: %.4f ms  %.2f TF/s\n", B, m, n, k, ms, 2.0 * B * m * n * k / ms / 1e9);
  } else if (!strcmp(argv[1], "panel")) {
    const int B = atoi(argv[2]), rows = atoi(argv[3]), pb = atoi(argv[4]);
    double* A = dalloc_rand((size_t)B * rows * pb, 1);
    int* piv;
    CK(cudaMalloc(&piv, (size_t)B * rows * sizeof(int)));
    std::vector<PanelDesc> hd(B);
    for (int i = 0; i < B; ++i)
      hd[i] = PanelDesc{abs_ref(A + (size_t)i * rows * pb), abs_ref(piv + (size_t)i * rows), kNull, rows, rows, 0, pb, kNull, kNull, kNull, 0, 0};
    PanelDesc* dd;
    CK(cudaMalloc(&dd, B * sizeof(PanelDesc)));
    CK(cudaMemcpy(dd, hd.data(), B * sizeof(PanelDesc), cudaMemcpyHostToDevice));
    float ms = time_it([&] { launch_panel_batched(db, dd, B, rows, pb, 0); }, reps);
    printf("panel B=%d rows=%d pb=%d: %.4f ms  (%.3f us/column)\n", B, rows, pb, ms, ms * 1e3 / pb);

  } else if (!strcmp(argv[1], "trsm")) {
    const int B = atoi(argv[2]), k = atoi(argv[3]), nc = atoi(argv[4]), up = atoi(argv[5]);
    double* T = dalloc_rand((size_t)B * k * k, 1, 4.0, k);
    double* X = dalloc_rand((size_t)B * k * nc, 2);
    std::vector<TrsmDesc> hd(B);
    for (int i = 0; i < B; ++i)
      hd[i] = TrsmDesc{abs_ref(T + (size_t)i * k * k), abs_ref(X + (size_t)i * k * nc), k, k, k, nc};
    TrsmDesc* dd;
    CK(cudaMalloc(&dd, B * sizeof(TrsmDesc)));
    CK(cudaMemcpy(dd, hd.data(), B * sizeof(TrsmDesc), cudaMemcpyHostToDevice));
    float ms = time_it([&] { launch_trsm_batched(db, dd, B, nc, k, up != 0, 0); }, reps);
    printf("trsm B=%d k=%d ncols=%d up=%d: %.4f ms  %.2f TF/s\n", B, k, nc, up, ms, (double)B * k * k * nc / ms / 1e9);
  }
  return 0;
}
