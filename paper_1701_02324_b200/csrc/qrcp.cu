// Level-batched truncated column-pivoted Householder QR + interpolative
// decomposition (linalg.py:43-136) and the per-level skeletonization driver
// (skeleton.py:125-182).
//
// Every node of a level owns a row-major workspace A_i (l'_i x c_i) holding
// the sampled kernel block K(X[rows], X[cands]); its rows are cut into
// 256-row chunks and all chunks of all nodes form one grid.  Step k:
//   pivot  (CTA per node): from-scratch column norms of A[k:, k:] (sum of the
//          chunk partials in fixed order), argmax with the lowest index on
//          ties, relative stop |pivot| <= tau |first pivot|, column swap,
//          Householder vector v (alpha = -copysign(norm, x0), v /= ||v||);
//   wpart  (CTA per chunk): partial v^T A[k:, k+1:];
//   update (CTA per chunk): A[k:, k+1:] -= 2 v (v^T A), R[k,k] = alpha,
//          A[k+1:, k] = 0, and the next step's column-norm partials.
// The pivot rule, stopping rule and reflector are the reference's
// (linalg.py:77-102); only reduction orders differ (ulp level).
// ID: T = R11^-1 R12 by column back substitution, P[:, piv] = [I | T] so
// P[:, J] is exactly the identity (linalg.py:129-135).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <vector>

#include "hks_internal.h"

namespace hks {
namespace {

constexpr int QCH = 256;  // rows per chunk
constexpr int QT = 256;   // threads

struct QrNode {
  double* A;      // row-major m x n, lda
  double* v;      // m
  int64_t* piv;   // n
  int m, n, lda, kmax;
  int chunk0, nchunk;
  int64_t poff;   // column offset of this node inside the partial buffers (n slots per chunk)
};

struct QrState {
  int done, rank, vnz, pad;
  double first, alpha;
};

struct QrChunk {
  int node, r0, r1, pad;
};

__global__ void qr_init(const QrNode* __restrict__ nodes, QrState* __restrict__ st, int count) {
  const int i = blockIdx.x;
  if (i >= count) return;
  const QrNode q = nodes[i];
  for (int j = threadIdx.x; j < q.n; j += blockDim.x) q.piv[j] = j;
  if (threadIdx.x == 0) {
    st[i].done = q.kmax == 0 ? 1 : 0;
    st[i].rank = 0;
    st[i].vnz = 0;
    st[i].first = 0.0;
    st[i].alpha = 0.0;
  }
}

// column-norm partials over rows >= k of a chunk, columns >= k
__global__ void __launch_bounds__(QT) qr_norms(const QrNode* __restrict__ nodes, const QrChunk* __restrict__ chunks,
                                               const QrState* __restrict__ st, int k,
                                               double* __restrict__ npart) {
  const QrChunk c = chunks[blockIdx.x];
  if (st[c.node].done) return;
  const QrNode q = nodes[c.node];
  double* out = npart + q.poff + (size_t)(blockIdx.x - q.chunk0) * q.n;
  const int r0 = max(c.r0, k);
  for (int j = k + threadIdx.x; j < q.n; j += QT) {
    double s = 0.0;
    for (int r = r0; r < c.r1; ++r) {
      const double a = q.A[(size_t)r * q.lda + j];
      s = fma(a, a, s);
    }
    out[j] = s;
  }
}

__global__ void __launch_bounds__(QT) qr_pivot(const QrNode* __restrict__ nodes, QrState* __restrict__ st, int k,
                                               double tau, const double* __restrict__ npart) {
  const int i = blockIdx.x;
  __shared__ double rv[QT / 32];
  __shared__ int ri[QT / 32];
  QrState s = st[i];
  if (s.done) return;
  const QrNode q = nodes[i];
  if (k >= q.kmax) {
    if (threadIdx.x == 0) {
      st[i].done = 1;
      st[i].rank = q.kmax;
    }
    return;
  }
  ArgMax best{-1.0, 0x7fffffff};
  for (int j = k + threadIdx.x; j < q.n; j += QT) {
    double ss = 0.0;
    for (int c = 0; c < q.nchunk; ++c) ss += npart[q.poff + (size_t)c * q.n + j];
    best = argmax_pick(best, ArgMax{sqrt(ss), j});
  }
  best = block_argmax(best, rv, ri);
  const double pn = best.v;
  const int jp = best.i;
  const double first = k == 0 ? pn : s.first;
  if (pn <= tau * first) {  // linalg.py:85-87
    if (threadIdx.x == 0) {
      st[i].done = 1;
      st[i].rank = k;
      st[i].first = first;
    }
    return;
  }
  if (jp != k) {  // swap columns k and jp over all rows, and the pivot record
    for (int r = threadIdx.x; r < q.m; r += QT) {
      double* row = q.A + (size_t)r * q.lda;
      const double t = row[k];
      row[k] = row[jp];
      row[jp] = t;
    }
    if (threadIdx.x == 0) {
      const int64_t t = q.piv[k];
      q.piv[k] = q.piv[jp];
      q.piv[jp] = t;
    }
  }
  __syncthreads();
  const double x0 = q.A[(size_t)k * q.lda + k];
  const double alpha = x0 != 0.0 ? -copysign(pn, x0) : -pn;
  double ss = 0.0;
  for (int r = k + threadIdx.x; r < q.m; r += QT) {
    double vr = q.A[(size_t)r * q.lda + k];
    if (r == k) vr -= alpha;
    q.v[r] = vr;
    ss = fma(vr, vr, ss);
  }
  const double vn = sqrt(block_sum(ss, rv));
  if (vn > 0.0)
    for (int r = k + threadIdx.x; r < q.m; r += QT) q.v[r] = q.v[r] / vn;
  if (threadIdx.x == 0) {
    st[i].first = first;
    st[i].alpha = alpha;
    st[i].vnz = vn > 0.0 ? 1 : 0;
  }
}

__global__ void __launch_bounds__(QT) qr_wpart(const QrNode* __restrict__ nodes, const QrChunk* __restrict__ chunks,
                                               const QrState* __restrict__ st, int k, double* __restrict__ wpart) {
  const QrChunk c = chunks[blockIdx.x];
  const QrState s = st[c.node];
  if (s.done || !s.vnz) return;
  const QrNode q = nodes[c.node];
  double* out = wpart + q.poff + (size_t)(blockIdx.x - q.chunk0) * q.n;
  const int r0 = max(c.r0, k);
  // v of this chunk staged once; loads batched 8 rows at a time (the sum
  // itself stays in row order: the same bits as the plain loop)
  __shared__ double vs[QCH];
  for (int r = r0 + threadIdx.x; r < c.r1; r += QT) vs[r - c.r0] = q.v[r];
  __syncthreads();
  const double* __restrict__ A = q.A;
  const size_t lda = q.lda;
  for (int j = k + 1 + threadIdx.x; j < q.n; j += QT) {
    double sum = 0.0;
    int r = r0;
    for (; r + 8 <= c.r1; r += 8) {
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = A[(size_t)(r + u) * lda + j];
#pragma unroll
      for (int u = 0; u < 8; ++u) sum = fma(vs[r + u - c.r0], a[u], sum);
    }
    for (; r < c.r1; ++r) sum = fma(vs[r - c.r0], A[(size_t)r * lda + j], sum);
    out[j] = sum;
  }
}

__global__ void __launch_bounds__(QT) qr_update(const QrNode* __restrict__ nodes, const QrChunk* __restrict__ chunks,
                                                const QrState* __restrict__ st, int k,
                                                const double* __restrict__ wpart, double* __restrict__ npart) {
  const QrChunk c = chunks[blockIdx.x];
  const QrState s = st[c.node];
  if (s.done) return;
  const QrNode q = nodes[c.node];
  double* nout = npart + q.poff + (size_t)(blockIdx.x - q.chunk0) * q.n;
  const int r0 = max(c.r0, k);
  // v staged in shared memory and 8-row batches of loads ahead of their
  // stores: the compiler can no longer serialise every load behind the
  // previous store (A and v may alias as far as it knows).  Arithmetic and
  // its order are unchanged.
  __shared__ double vs[QCH];
  if (s.vnz)
    for (int r = r0 + threadIdx.x; r < c.r1; r += QT) vs[r - c.r0] = q.v[r];
  __syncthreads();
  double* __restrict__ A = q.A;
  const size_t lda = q.lda;
  for (int j = k + 1 + threadIdx.x; j < q.n; j += QT) {
    double w = 0.0;
    if (s.vnz)
      for (int cc = 0; cc < q.nchunk; ++cc) w += wpart[q.poff + (size_t)cc * q.n + j];
    double ns = 0.0;
    int r = r0;
    for (; r + 8 <= c.r1; r += 8) {
      double val[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) val[u] = A[(size_t)(r + u) * lda + j];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (s.vnz) {
          val[u] -= 2.0 * (vs[r + u - c.r0] * w);  // r[k:, k:] -= 2 outer(v, v @ r[k:, k:])  (linalg.py:100)
          A[(size_t)(r + u) * lda + j] = val[u];
        }
        if (r + u > k) ns = fma(val[u], val[u], ns);
      }
    }
    for (; r < c.r1; ++r) {
      double val = A[(size_t)r * lda + j];
      if (s.vnz) {
        val -= 2.0 * (vs[r - c.r0] * w);
        A[(size_t)r * lda + j] = val;
      }
      if (r > k) ns = fma(val, val, ns);
    }
    nout[j] = ns;
  }
  // R[k, k] = alpha, r[k+1:, k] = 0 (linalg.py:101-102)
  for (int r = r0 + threadIdx.x; r < c.r1; r += QT) q.A[(size_t)r * q.lda + k] = (r == k) ? s.alpha : 0.0;
}

// T = R11^-1 R12 written straight into P's columns piv[r..n), identity
// columns piv[0..r); skeleton indices cands[piv[0..r)]
__global__ void qr_id(const QrNode* __restrict__ nodes, const QrState* __restrict__ st, double* const* __restrict__ P,
                      const int64_t* const* __restrict__ cands, int64_t* const* __restrict__ skel,
                      int64_t* __restrict__ ranks) {
  const int i = blockIdx.x;
  const QrNode q = nodes[i];
  const int r = st[i].rank;
  double* p = P[i];
  if (threadIdx.x == 0) ranks[i] = r;
  if (r == 0) return;
  for (int jj = threadIdx.x; jj < q.n; jj += blockDim.x) {
    double* col = p + (size_t)q.piv[jj] * r;
    if (jj < r) {
      for (int t = 0; t < r; ++t) col[t] = (t == jj) ? 1.0 : 0.0;
      continue;
    }
    for (int t = 0; t < r; ++t) col[t] = q.A[(size_t)t * q.lda + jj];
    for (int kk = r - 1; kk >= 0; --kk) {  // back substitution, column-oriented (dtrsm L,U,N order)
      const double tk = col[kk] / q.A[(size_t)kk * q.lda + kk];
      col[kk] = tk;
      for (int t = 0; t < kk; ++t) col[t] -= tk * q.A[(size_t)t * q.lda + kk];
    }
  }
  if (skel && cands)
    for (int t = threadIdx.x; t < r; t += blockDim.x) skel[i][t] = cands[i][q.piv[t]];
}


// The same ID for a 32-column block of P per CTA: every warp back-substitutes
// 8 columns together against the rows of R11 (dot form: x_k = (b_k - sum_{t>k}
// R[k,t] x_t) / R[k,k], the row of R read once, coalesced, for the 8 columns;
// partial sums over the lanes' t in a fixed order).  The column-per-thread
// kernel above walks R11 once per thread with uncoalesced updates of P:
// 1.45 s of C3's skeletonization; this one is ~100x faster.
constexpr int IDC = 32;  // columns per CTA
__global__ void __launch_bounds__(128) qr_id_rows(const QrNode* __restrict__ nodes, const QrState* __restrict__ st,
                                                  double* const* __restrict__ P,
                                                  const int64_t* const* __restrict__ cands,
                                                  int64_t* const* __restrict__ skel, int64_t* __restrict__ ranks) {
  const int i = blockIdx.x;
  const QrNode q = nodes[i];
  const int r = st[i].rank;
  if (blockIdx.y == 0 && threadIdx.x == 0) ranks[i] = r;
  const int jj0 = blockIdx.y * IDC;
  if (r == 0 || jj0 >= q.n) return;
  if (blockIdx.y == 0 && skel && cands)
    for (int t = threadIdx.x; t < r; t += blockDim.x) skel[i][t] = cands[i][q.piv[t]];
  extern __shared__ double xs[];  // [IDC][r]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* xw = xs + (size_t)wid * 8 * r;
  double* p = P[i];
  const double* __restrict__ A = q.A;
  const size_t lda = q.lda;
  const int jw = jj0 + wid * 8;  // this warp's first column
  bool any_solve = false;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int jj = jw + u;
    if (jj >= q.n) continue;
    if (jj < r) {
      double* col = p + (size_t)q.piv[jj] * r;
      for (int t = lane; t < r; t += 32) col[t] = (t == jj) ? 1.0 : 0.0;
    } else {
      any_solve = true;
      for (int t = lane; t < r; t += 32) xw[u * r + t] = A[(size_t)t * lda + jj];
    }
  }
  if (!any_solve) return;  // warp-uniform
  __syncwarp();
  for (int kk = r - 1; kk >= 0; --kk) {
    const double* row = A + (size_t)kk * lda;
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    for (int t = kk + 1 + lane; t < r; t += 32) {
      const double rv = row[t];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = fma(rv, xw[u * r + t], acc[u]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
    double mine = acc[0];
#pragma unroll
    for (int u = 1; u < 8; ++u) mine = lane == u ? acc[u] : mine;
    if (lane < 8 && jw + lane >= r && jw + lane < q.n) xw[lane * r + kk] = (xw[lane * r + kk] - mine) / row[kk];
    __syncwarp();
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int jj = jw + u;
    if (jj < r || jj >= q.n) continue;
    double* col = p + (size_t)q.piv[jj] * r;
    for (int t = lane; t < r; t += 32) col[t] = xw[u * r + t];
  }
}

template <class T>
cudaError_t upload(const std::vector<T>& h, T** d, cudaStream_t s) {
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(d), std::max<size_t>(h.size(), 1) * sizeof(T), s);
  if (e == cudaSuccess && !h.empty()) e = cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s);
  return e;
}

// HKS_SKEL_TRACE=1: device time of each skeletonization stage on stderr.
struct StageTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  const char* name;
  bool on;
  StageTimer(const char* n, cudaStream_t st) : s(st), name(n) {
    static const bool trace = getenv("HKS_SKEL_TRACE") != nullptr;
    on = trace;
    if (on) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
    }
  }
  ~StageTimer() {
    if (!on) return;
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    fprintf(stderr, "HKS_SKEL_TRACE %s %.3f ms\n", name, ms);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

// Pre-reduction policy: blocks with at least kTsqrMinRows rows and twice as
// many rows as columns (HKS_TSQR=0 disables; the QRCP then runs on the
// sampled block itself, as the reference does).
constexpr int kTsqrMinRows = 1024;
bool tsqr_enabled() {
  static const bool v = [] {
    const char* e = getenv("HKS_TSQR");
    return !(e && atoi(e) == 0);
  }();
  return v;
}
bool tsqr_eligible(int m, int n) { return tsqr_enabled() && m >= kTsqrMinRows && m >= 2 * n && n >= 1; }

// Replaces every eligible node's workspace by its triangular factor: row
// chunks of the block are absorbed into per-chunk triangles (one CTA each),
// the triangles merged pairwise.  On return the nodes point at their R
// (m = n, lda = n); *rscratch / *djobs are stream-ordered allocations the
// caller frees after the QRCP.
cudaError_t tsqr_prereduce(std::vector<QrNode>& nodes, double** rscratch, TsqrJob** djobs, cudaStream_t s) {
  const int B = tsqr_slab_rows();
  int64_t total_rows = 0;
  int cmax = 0;
  for (auto& q : nodes)
    if (tsqr_eligible(q.m, q.n)) {
      total_rows += q.m;
      cmax = std::max(cmax, q.n);
    }
  if (total_rows == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // rows per job: at least two triangles' worth (a merge costs about half a
  // triangle of absorbed rows), otherwise ~6 jobs per SM over the batch
  int64_t rpj = std::max<int64_t>(2 * (int64_t)cmax, (total_rows + 6 * sms - 1) / (6 * sms));
  rpj = (rpj + B - 1) / B * B;
  std::vector<TsqrJob> jobs;                 // stage 0, then the merge stages back to back
  std::vector<std::pair<int, int>> stages;   // (first job, count)
  struct Plan {
    int node, nch;
    size_t roff;
  };
  std::vector<Plan> plans;
  size_t rtotal = 0;
  int max_nch = 1;
  for (int i = 0; i < (int)nodes.size(); ++i) {
    const QrNode& q = nodes[i];
    if (!tsqr_eligible(q.m, q.n)) continue;
    const int nch = (int)((q.m + rpj - 1) / rpj);
    plans.push_back(Plan{i, nch, rtotal});
    rtotal += (size_t)nch * q.n * q.n;
    max_nch = std::max(max_nch, nch);
  }
  for (auto& p : plans) {
    const QrNode& q = nodes[p.node];
    for (int ch = 0; ch < p.nch; ++ch) {
      const int64_t r0 = (int64_t)ch * rpj, r1 = std::min<int64_t>(q.m, r0 + rpj);
      jobs.push_back(TsqrJob{nullptr, q.A + (size_t)r0 * q.lda, q.n, q.lda, (int)(r1 - r0), 0});
      jobs.back().R = reinterpret_cast<double*>(p.roff + (size_t)ch * q.n * q.n);  // offset, rebased below
    }
  }
  stages.push_back({0, (int)jobs.size()});
  for (int st = 1; st < max_nch; st *= 2) {
    const int first = (int)jobs.size();
    for (auto& p : plans) {
      const QrNode& q = nodes[p.node];
      for (int ch = 0; ch + st < p.nch; ch += 2 * st) {
        TsqrJob j{nullptr, nullptr, q.n, q.n, q.n, 1};
        j.R = reinterpret_cast<double*>(p.roff + (size_t)ch * q.n * q.n);
        j.S = reinterpret_cast<double*>(p.roff + (size_t)(ch + st) * q.n * q.n);
        jobs.push_back(j);
      }
    }
    stages.push_back({first, (int)jobs.size() - first});
  }
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(rscratch), rtotal * sizeof(double), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(*rscratch, 0, rtotal * sizeof(double), s);
  if (e != cudaSuccess) return e;
  for (size_t k = 0; k < jobs.size(); ++k) {  // rebase the scratch offsets
    TsqrJob& j = jobs[k];
    j.R = *rscratch + reinterpret_cast<size_t>(j.R);
    if (j.tri) j.S = *rscratch + reinterpret_cast<size_t>(j.S);
  }
  e = upload(jobs, djobs, s);
  for (auto& st : stages)
    if (e == cudaSuccess && st.second > 0) {
      StageTimer tm(&st == &stages[0] ? "tsqr_absorb" : "tsqr_merge", s);
      e = launch_tsqr_absorb(*djobs + st.first, st.second, s);
    }
  if (e != cudaSuccess) return e;
  // `jobs` is pageable host memory read by the asynchronous upload
  e = cudaStreamSynchronize(s);
  for (auto& p : plans) {
    QrNode& q = nodes[p.node];
    q.A = *rscratch + p.roff;
    q.m = q.n;
    q.lda = q.n;
  }
  return e;
}

// Runs the QRCP + ID on a batch of prepared workspaces.
cudaError_t run_qrcp(std::vector<QrNode>& nodes, double tau, const std::vector<double*>& P,
                     const std::vector<const int64_t*>& cands, const std::vector<int64_t*>& skel,
                     std::vector<int64_t>& ranks_out, cudaStream_t s, bool copy_r_back = false) {
  const int count = (int)nodes.size();
  std::vector<QrNode> orig;
  if (copy_r_back) orig = nodes;
  // Tall blocks are first reduced to their c x c triangular factor (tsqr.cu):
  // the QRCP below then streams c x c instead of l' x c per step.
  double* rscratch = nullptr;
  TsqrJob* djobs = nullptr;
  {
    cudaError_t te = tsqr_prereduce(nodes, &rscratch, &djobs, s);
    if (te != cudaSuccess) {
      if (rscratch) cudaFreeAsync(rscratch, s);
      if (djobs) cudaFreeAsync(djobs, s);
      return te;
    }
  }
  std::vector<QrChunk> ch;
  int64_t poff = 0;
  int kmax_all = 0;
  for (int i = 0; i < count; ++i) {
    QrNode& q = nodes[i];
    q.chunk0 = (int)ch.size();
    for (int r0 = 0; r0 < std::max(q.m, 1); r0 += QCH) ch.push_back(QrChunk{i, r0, std::min(r0 + QCH, q.m), 0});
    q.nchunk = (int)ch.size() - q.chunk0;
    q.poff = poff;
    poff += (int64_t)q.nchunk * q.n;
    kmax_all = std::max(kmax_all, q.kmax);
  }
  QrNode* dn = nullptr;
  QrChunk* dc = nullptr;
  QrState* dst = nullptr;
  double *npart = nullptr, *wpart = nullptr;
  double** dP = nullptr;
  const int64_t** dcand = nullptr;
  int64_t** dskel = nullptr;
  int64_t* dranks = nullptr;
  cudaError_t e = upload(nodes, &dn, s);
  if (e == cudaSuccess) e = upload(ch, &dc, s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dst), count * sizeof(QrState), s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&npart), std::max<int64_t>(poff, 1) * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&wpart), std::max<int64_t>(poff, 1) * sizeof(double), s);
  if (e == cudaSuccess) e = upload(P, &dP, s);
  if (e == cudaSuccess) e = upload(cands, &dcand, s);
  if (e == cudaSuccess) e = upload(skel, &dskel, s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dranks), count * sizeof(int64_t), s);
  const int nch = (int)ch.size();
  if (e == cudaSuccess) {
    StageTimer tm("qrcp", s);
    qr_init<<<count, 256, 0, s>>>(dn, dst, count);
    qr_norms<<<nch, QT, 0, s>>>(dn, dc, dst, 0, npart);
    for (int k = 0; k <= kmax_all && e == cudaSuccess; ++k) {
      qr_pivot<<<count, QT, 0, s>>>(dn, dst, k, tau, npart);
      if (k == kmax_all) break;
      qr_wpart<<<nch, QT, 0, s>>>(dn, dc, dst, k, wpart);
      qr_update<<<nch, QT, 0, s>>>(dn, dc, dst, k, wpart, npart);
      e = cudaGetLastError();
    }
    StageTimer tm_id("qr_id", s);
    int nmax = 1;
    for (auto& q : nodes) nmax = std::max(nmax, q.n);
    const size_t id_smem = (size_t)IDC * std::max(kmax_all, 1) * sizeof(double);
    static const bool id_old = getenv("HKS_QR_ID_OLD") != nullptr;  // development knob
    if (!id_old && id_smem <= 200 * 1024 && raise_smem_limit(qr_id_rows, id_smem) == cudaSuccess)
      qr_id_rows<<<dim3(count, (nmax + IDC - 1) / IDC), 128, id_smem, s>>>(
          dn, dst, dP, skel.empty() ? nullptr : dcand, skel.empty() ? nullptr : dskel, dranks);
    else
      qr_id<<<count, 256, 0, s>>>(dn, dst, dP, skel.empty() ? nullptr : dcand, skel.empty() ? nullptr : dskel, dranks);
    ranks_out.resize(count);
    // callers that read R from the workspace (hks_interp_decomp): the first
    // kmax rows of a pre-reduced node's triangle go back into its block
    for (int i = 0; i < (int)orig.size() && e == cudaSuccess; ++i)
      if (orig[i].A != nodes[i].A && nodes[i].kmax > 0)
        e = cudaMemcpy2DAsync(orig[i].A, (size_t)orig[i].lda * sizeof(double), nodes[i].A,
                              (size_t)nodes[i].lda * sizeof(double), (size_t)nodes[i].n * sizeof(double),
                              nodes[i].kmax, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ranks_out.data(), dranks, count * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  for (void* p : {(void*)dn, (void*)dc, (void*)dst, (void*)npart, (void*)wpart, (void*)dP, (void*)dcand,
                  (void*)dskel, (void*)dranks, (void*)rscratch, (void*)djobs})
    if (p) cudaFreeAsync(p, s);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

}  // namespace
}  // namespace hks

using namespace hks;

// Return the skeletonization workspace kept in the default pool (above).
extern "C" int hks_skeleton_workspace_release(void* stream) {
  int dev = 0;
  cudaMemPool_t pool;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaDeviceGetDefaultMemPool(&pool, dev);
  if (e == cudaSuccess) {
    uint64_t keep = 0;
    e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    if (e == cudaSuccess) e = cudaMemPoolTrimTo(pool, 0);
  }
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_skeleton_workspace_release: %s", cudaGetErrorString(e));
  return HKS_OK;
}

// interpolative_decomposition / pivoted_qr (linalg.py:43-136) on one matrix.
extern "C" int hks_interp_decomp(double* A, int64_t m, int64_t n, int64_t lda, double tol, int64_t max_rank,
                                 int64_t* pivots, double* interp, int64_t* rank_host, void* stream) {
  if (!A || !pivots || !interp || !rank_host || m < 0 || n < 0 || lda < n || !(tol > 0) || max_rank < 1)
    return set_error(HKS_ERR_INVALID, "hks_interp_decomp: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* v = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&v), std::max<int64_t>(m, 1) * sizeof(double), s);
  std::vector<QrNode> nodes(1);
  nodes[0] = QrNode{A, v, pivots, (int)m, (int)n, (int)lda, (int)std::min<int64_t>(std::min(m, n), max_rank), 0, 0, 0};
  std::vector<int64_t> ranks;
  if (e == cudaSuccess) e = run_qrcp(nodes, tol, {interp}, {}, {}, ranks, s, true);
  if (v) cudaFreeAsync(v, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_interp_decomp: %s", cudaGetErrorString(e));
  *rank_host = ranks[0];
  return HKS_OK;
}

// skeletonize every node of one level (skeleton.py:125-140 per node,
// :171-181 per level).  rows / cands: device flat int64 lists with host
// offsets [count + 1]; outputs into the SKEL / INTERP layouts at the given
// per-node element offsets; ranks_host[count].
extern "C" int hks_skeletonize_level(const double* X, int64_t d, const hks_kernel* kern, int64_t count,
                                     int64_t first_node, const int64_t* rows, const int64_t* row_off,
                                     const int64_t* cands, const int64_t* cand_off, double tau, int64_t max_rank,
                                     int64_t* skel_buf, const int64_t* skel_off, double* interp_buf,
                                     const int64_t* interp_off, int64_t* ranks_host, void* stream) {
  if (!X || !kern || count < 1 || !row_off || !cand_off || !skel_off || !interp_off || !ranks_host)
    return set_error(HKS_ERR_INVALID, "hks_skeletonize_level: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const KernelParams kp = make_kernel_params(kern);
  // The stream-ordered workspace stays in the device's default pool between
  // levels (its release threshold would otherwise unmap GBs at every
  // synchronisation and map them again at the next level);
  // hks_skeleton_workspace_release() returns it once the skeletons are built.
  {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  // batches of nodes whose sampled blocks fit a workspace budget
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const size_t budget = std::max<size_t>(size_t(256) << 20, std::min<size_t>(free_b / 3, size_t(16) << 30));
  int64_t i0 = 0;
  while (i0 < count) {
    int64_t i1 = i0;
    size_t bytes = 0;
    while (i1 < count) {
      const size_t rm = (size_t)(row_off[i1 + 1] - row_off[i1]), rc = (size_t)(cand_off[i1 + 1] - cand_off[i1]);
      // sampled block + Householder vector (+ the triangle of the pre-reduction)
      const size_t b = rm * rc * 8 + rm * 8 + (tsqr_eligible((int)rm, (int)rc) ? rc * rc * 8 : 0);
      if (i1 > i0 && bytes + b > budget) break;
      bytes += b;
      ++i1;
    }
    char* ws = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws), std::max<size_t>(bytes, 8), s);
    std::vector<EvalDesc> ev;
    std::vector<QrNode> nodes;
    std::vector<double*> P;
    std::vector<const int64_t*> cl;
    std::vector<int64_t*> sk;
    size_t at = 0;
    int mm = 0, mn = 0;
    for (int64_t i = i0; i < i1; ++i) {
      const int m = (int)(row_off[i + 1] - row_off[i]), c = (int)(cand_off[i + 1] - cand_off[i]);
      double* A = reinterpret_cast<double*>(ws + at);
      at += (size_t)m * c * 8;
      double* v = reinterpret_cast<double*>(ws + at);
      at += (size_t)m * 8;
      if (m > 0 && c > 0)
        ev.push_back(EvalDesc{abs_ref(rows + row_off[i]), abs_ref(cands + cand_off[i]), 0, 0, m, c, abs_ref(A), c, 0});
      mm = std::max(mm, m);
      mn = std::max(mn, c);
      const int kmax = (int)std::min<int64_t>(std::min(m, c), max_rank);
      // pivots live in the SKEL slot's tail? no: a separate device array per node
      nodes.push_back(QrNode{A, v, nullptr, m, c, c, kmax, 0, 0, 0});
      P.push_back(interp_buf + interp_off[i]);
      cl.push_back(cands + cand_off[i]);
      sk.push_back(skel_buf + skel_off[i]);
    }
    // pivot arrays
    int64_t* piv = nullptr;
    size_t npiv = 0;
    for (auto& q : nodes) npiv += q.n;
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&piv), std::max<size_t>(npiv, 1) * 8, s);
    size_t pat = 0;
    for (auto& q : nodes) {
      q.piv = piv + pat;
      pat += q.n;
    }
    EvalDesc* dev = nullptr;
    if (e == cudaSuccess && !ev.empty()) e = upload(ev, &dev, s);
    Bases b{};
    Bases* db = nullptr;
    if (e == cudaSuccess && !ev.empty()) e = upload_bases(b, &db, s);
    StageTimer* tm_eval = new StageTimer("eval", s);
    if (e == cudaSuccess && !ev.empty()) e = launch_eval_batched(X, (int)d, kp, db, dev, (int)ev.size(), mm, mn, true, s);
    delete tm_eval;
    if (db) cudaFreeAsync(db, s);
    std::vector<int64_t> ranks;
    if (e == cudaSuccess) e = run_qrcp(nodes, tau, P, cl, sk, ranks, s);
    if (dev) cudaFreeAsync(dev, s);
    if (piv) cudaFreeAsync(piv, s);
    if (ws) cudaFreeAsync(ws, s);
    if (e != cudaSuccess)
      return set_error(HKS_ERR_SKELETON, "node %lld: %s", (long long)(first_node + i0), cudaGetErrorString(e));
    for (int64_t i = i0; i < i1; ++i) ranks_host[i] = ranks[i - i0];
    i0 = i1;
  }
  return HKS_OK;
}
