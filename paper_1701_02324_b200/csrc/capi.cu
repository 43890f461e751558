// C-ABI entry points that are not plan-bound: error plumbing, single-block
// kernel evaluation / summation and the dense LU wrappers used by the
// reference-named factor_dense / solve_dense / eval_block.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include <mutex>
#include <unordered_map>

#include "hks_internal.h"

namespace hks {

static thread_local char g_err[1024] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

// Small device-side descriptor upload for one-off launches.
template <class D>
static cudaError_t one_desc(const D& h, D** d, cudaStream_t s) {
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(d), sizeof(D), s);
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(*d, &h, sizeof(D), cudaMemcpyHostToDevice, s);
}

cudaError_t raise_smem_limit(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> cur;
  std::lock_guard<std::mutex> g(mu);
  size_t& have = cur[func];
  if (bytes <= have) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

cudaError_t upload_bases(const Bases& b, Bases** dev, cudaStream_t s) {
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(dev), sizeof(Bases), s);
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(*dev, &b, sizeof(Bases), cudaMemcpyHostToDevice, s);
}

}  // namespace hks

using namespace hks;

static inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" const char* hks_last_error(void) { return g_err; }
extern "C" int hks_abi_version(void) { return HKS_ABI_VERSION; }

static int check_kernel(const hks_kernel* k, int64_t d) {
  if (!k) return set_error(HKS_ERR_INVALID, "null kernel");
  if (k->family == HKS_GAUSSIAN && !(k->h > 0)) return set_error(HKS_ERR_INVALID, "gaussian bandwidth h must be positive");
  if (k->family == HKS_LAPLACE3D && d != 3) return set_error(HKS_ERR_INVALID, "laplace3d kernel requires 3-d points");
  if (k->family < 0 || k->family > 2) return set_error(HKS_ERR_INVALID, "unknown kernel family %d", k->family);
  return HKS_OK;
}

extern "C" int hks_eval_block(const double* X, int64_t d, const hks_kernel* kern, const int64_t* rows, int64_t row0,
                              int64_t nrows, const int64_t* cols, int64_t col0, int64_t ncols, double* out,
                              int64_t ldo, int32_t row_major, double diag, void* stream) {
  int rc = check_kernel(kern, d);
  if (rc) return rc;
  if (nrows == 0 || ncols == 0) return HKS_OK;
  cudaStream_t s = as_stream(stream);
  EvalDesc h{rows ? abs_ref(rows) : kNull, cols ? abs_ref(cols) : kNull, row0, col0, (int)nrows, (int)ncols,
             abs_ref(out), (int)ldo, diag != 0.0};
  Bases b{};
  b.lam = diag;
  EvalDesc* dd = nullptr;
  Bases* db = nullptr;
  cudaError_t e = one_desc(h, &dd, s);
  if (e == cudaSuccess) e = upload_bases(b, &db, s);
  if (e == cudaSuccess)
    e = launch_eval_batched(X, (int)d, make_kernel_params(kern), db, dd, 1, (int)nrows, (int)ncols, row_major != 0, s);
  if (dd) cudaFreeAsync(dd, s);
  if (db) cudaFreeAsync(db, s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_eval_block: %s", cudaGetErrorString(e));
  return HKS_OK;
}

extern "C" int hks_kernel_sum(const double* X, int64_t d, const hks_kernel* kern, const int64_t* rows, int64_t row0,
                              int64_t nrows, const int64_t* cols, int64_t col0, int64_t ncols, const double* W,
                              int64_t ldw, int64_t k, double* U, int64_t ldu, double beta, double diag,
                              void* stream) {
  int rc = check_kernel(kern, d);
  if (rc) return rc;
  if (nrows == 0 || k == 0) return HKS_OK;
  cudaStream_t s = as_stream(stream);
  SumDesc h{rows ? abs_ref(rows) : kNull, cols ? abs_ref(cols) : kNull, row0, col0, (int)nrows, (int)ncols, (int)k,
            abs_ref(W), (int)ldw, abs_ref(U), (int)ldu, beta, diag != 0.0};
  Bases b{};
  b.lam = diag;
  SumDesc* dd = nullptr;
  Bases* db = nullptr;
  cudaError_t e = one_desc(h, &dd, s);
  if (e == cudaSuccess) e = upload_bases(b, &db, s);
  if (e == cudaSuccess) e = launch_ksum_batched(X, (int)d, make_kernel_params(kern), db, dd, 1, (int)nrows, s);
  if (dd) cudaFreeAsync(dd, s);
  if (db) cudaFreeAsync(db, s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_kernel_sum: %s", cudaGetErrorString(e));
  return HKS_OK;
}


// Deterministic sum of the column-chunk partial products of hks_cross_sum:
// U[i, c] = beta U[i, c] + sum_q ws[q][i, c], chunks in order.
namespace {
__global__ void sum_chunks_kernel(const double* __restrict__ ws, int64_t chunks, int64_t m, int64_t k,
                                  double* __restrict__ U, int64_t ldu, double beta) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * k; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t q = 0; q < chunks; ++q) s += ws[q * m * k + e];
    double* u = U + (e % m) + (e / m) * ldu;
    *u = beta != 0.0 ? beta * *u + s : s;
  }
}
}  // namespace

// U = beta U + K(Xq[rows], Xs) W for few query rows against many sources
// (cli.py:415-422 _cross_predict; the sampled-row error metrics): the
// sources are split into column chunks so the grid fills the GPU, each
// chunk's partial product goes to scratch, and one ordered pass sums them.
extern "C" int hks_cross_sum(const double* Xq, int64_t nq, const double* Xs, int64_t ns, int64_t d,
                             const hks_kernel* kern, const int64_t* rows, const double* W, int64_t ldw, int64_t k,
                             double* U, int64_t ldu, double beta, void* stream) {
  int rc = check_kernel(kern, d);
  if (rc) return rc;
  if (!Xq || !Xs || !W || !U || nq < 0 || ns < 0 || k < 0 || ldw < ns || ldu < nq)
    return set_error(HKS_ERR_INVALID, "hks_cross_sum: bad arguments");
  if (nq == 0 || k == 0) return HKS_OK;
  cudaStream_t s = as_stream(stream);
  const int64_t row_tiles = (nq + 63) / 64;
  int64_t chunks = std::max<int64_t>(1, std::min<int64_t>((ns + 255) / 256, (4 * 148 + row_tiles - 1) / row_tiles));
  const int64_t ch = (ns + chunks - 1) / chunks;
  chunks = ns > 0 ? (ns + ch - 1) / ch : 1;
  std::vector<SumDesc> h(chunks);
  double* ws = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws), (size_t)chunks * nq * k * sizeof(double), s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_cross_sum: %s", cudaGetErrorString(e));
  for (int64_t q = 0; q < chunks; ++q) {
    const int64_t c0 = q * ch, cn = std::max<int64_t>(0, std::min(ch, ns - c0));
    h[q] = SumDesc{rows ? abs_ref(rows) : kNull, kNull, 0, c0, (int)nq, (int)cn, (int)k,
                   abs_ref(W + c0), (int)ldw, abs_ref(ws + q * nq * k), (int)nq, 0.0, false};
  }
  SumDesc* dd = nullptr;
  Bases* db = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&dd), chunks * sizeof(SumDesc), s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dd, h.data(), chunks * sizeof(SumDesc), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = upload_bases(Bases{}, &db, s);
  if (e == cudaSuccess) e = launch_ksum_batched(Xq, (int)d, make_kernel_params(kern), db, dd, (int)chunks, (int)nq, s, Xs);
  if (e == cudaSuccess) {
    sum_chunks_kernel<<<(unsigned)std::min<int64_t>((nq * k + 255) / 256, 1184), 256, 0, s>>>(ws, chunks, nq, k, U,
                                                                                               ldu, beta);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the host-side descriptors die with this call
  cudaFreeAsync(ws, s);
  if (dd) cudaFreeAsync(dd, s);
  if (db) cudaFreeAsync(db, s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_cross_sum: %s", cudaGetErrorString(e));
  return HKS_OK;
}
