// Building blocks of the level-batched blocked LU / triangular-solve
// programs (plan.cu: add_lu_program, add_lu_solve_program).
//
// The LU of every matrix of a tree level (leaf blocks K_aa + lam I, reduced
// matrices Z) runs as one descriptor program: 128-column groups, each
// factored as 32-column panels (left-looking inside the group), then one
// row-interchange pass, one unit-lower TRSM and one DMMA GEMM trailing
// update of rank 128 for all matrices at once.  Right-hand-side columns
// (P^T for phi, thhat for Z^-1 thhat) ride along in the swaps, TRSMs and
// GEMMs, so the forward substitution costs GEMM time; a backward sweep of
// upper TRSMs + GEMMs finishes the solve.  Results are those of LAPACK
// getrf / getrs (partial pivoting, row interchanges applied to the whole
// row, 0-based pivots) up to roundoff.
#include <cfloat>

#include "common.cuh"
#include "hks_internal.h"

namespace hks {
namespace {

constexpr int PT = 256;  // panel threads

// Factor rows p0..n-1 of columns [p0, p0+pb) in shared memory: pivot search
// (lowest row on ties, LAPACK idamax), swap inside the panel, scale by the
// reciprocal (dgetf2), rank-1 update.  piv[p0 + jj] = global pivot row.
template <int PB>
__global__ void __launch_bounds__(PT) panel_kernel(const Bases* __restrict__ bases_ptr, const PanelDesc* __restrict__ descs, int ldp) {
  const Bases& bases = *bases_ptr;
  const PanelDesc D = descs[blockIdx.x];
  double* A = at<double>(bases, D.A);
  int* piv = at<int>(bases, D.piv);
  const int lda = D.lda, p0 = D.p0, pb = D.pb, mr = D.n - D.p0;
  extern __shared__ double P[];
  __shared__ double red_v[PT / 32];
  __shared__ int red_i[PT / 32];
  __shared__ int s_info;
  const int tid = threadIdx.x;
  if (tid == 0) s_info = 0;
  for (int c = 0; c < pb; ++c) {  // coalesced column loads, no div/mod
    const double* src = A + p0 + (size_t)(p0 + c) * lda;
    for (int i = tid; i < mr; i += PT) P[i + c * ldp] = src[i];
  }
  __syncthreads();
  for (int jj = 0; jj < pb; ++jj) {
    ArgMax a{-1.0, 0x7fffffff};
    for (int i = jj + tid; i < mr; i += PT) a = argmax_pick(a, ArgMax{fabs(P[i + jj * ldp]), i});
    a = block_argmax(a, red_v, red_i);  // ends with a barrier
    const int p = a.i;
    const double pv = P[p + jj * ldp];
    if (tid == 0) {
      piv[p0 + jj] = p0 + p;
      if (pv == 0.0 && s_info == 0) s_info = p0 + jj + 1;
    }
    __syncthreads();  // every thread has read pv
    if (p != jj && tid < pb) {  // interchange rows jj and p of the panel
      const double t = P[jj + tid * ldp];
      P[jj + tid * ldp] = P[p + tid * ldp];
      P[p + tid * ldp] = t;
    }
    __syncthreads();
    // scale the column (dgetf2: reciprocal when safe) and rank-1 update, one row per thread
    const bool recip = fabs(pv) >= DBL_MIN;
    const double inv = 1.0 / pv;
    for (int i = jj + 1 + tid; i < mr; i += PT) {
      double l = P[i + jj * ldp];
      if (pv != 0.0) {
        l = recip ? l * inv : l / pv;
        P[i + jj * ldp] = l;
      }
      for (int c = jj + 1; c < pb; ++c) P[i + c * ldp] -= l * P[jj + c * ldp];
    }
    __syncthreads();
  }
  for (int c = 0; c < pb; ++c) {
    double* dst = A + p0 + (size_t)(p0 + c) * lda;
    for (int i = tid; i < mr; i += PT) dst[i] = P[i + c * ldp];
  }
  if (tid == 0 && s_info && D.info != kNull) {
    int* info = at<int>(bases, D.info);
    if (*info == 0) *info = s_info;  // panels run in order: keep the first zero pivot
  }
}

// Row interchanges piv[r0..r1) applied in order to columns [c0, c1).
__global__ void swap_kernel(const Bases* __restrict__ bases_ptr, const SwapDesc* __restrict__ descs) {
  const Bases& bases = *bases_ptr;
  const SwapDesc D = descs[blockIdx.y];
  const int c = D.c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= D.c1) return;
  double* col = at<double>(bases, D.A) + (size_t)c * D.lda;
  const int* piv = at<const int>(bases, D.piv);
  for (int jj = D.r0; jj < D.r1; ++jj) {
    const int p = piv[jj];
    if (p != jj) {
      const double t = col[jj];
      col[jj] = col[p];
      col[p] = t;
    }
  }
}

// B := T^-1 B for a k x k triangular block T (unit lower, or non-unit
// upper), k <= 128, B k x ncols.  A CTA owns 128 columns (one per thread)
// held in shared memory.  Per 32-row block: the rows of T are staged, the
// contribution of the already-solved rows is one DMMA product (each warp a
// 32 x 32 tile), then every thread solves its column against the 32 x 32
// diagonal block in registers, column-oriented (axpy) order so the 31
// updates of each step are independent (no serial shuffle chain).
constexpr int TNC = 128;            // columns per CTA (= threads)
constexpr int TXS = TNC + 4;        // X row stride: == 4 (mod 16), conflict-free DMMA B fragments
constexpr int TTS = 128 + 4;        // staged T row stride

template <bool UPPER>
__global__ void __launch_bounds__(TNC) trsm_kernel(const Bases* __restrict__ bases_ptr,
                                                  const TrsmDesc* __restrict__ descs) {
  const Bases& bases = *bases_ptr;
  const TrsmDesc D = descs[blockIdx.y];
  const int c0 = blockIdx.x * TNC;
  if (c0 >= D.ncols) return;
  const int nc = min(TNC, D.ncols - c0), k = D.k;
  const double* T = at<const double>(bases, D.T);
  double* B = at<double>(bases, D.B) + (size_t)c0 * D.ldb;
  extern __shared__ double tsm[];
  double* X = tsm;                    // k x TNC, row-major (ld TXS)
  double* Ts = tsm + 128 * TXS;       // 32 rows of T, row-major (ld TTS)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // coalesced load: lanes walk a column's rows
  for (int c = wid; c < nc; c += TNC / 32)
    for (int i = lane; i < k; i += 32) X[i * TXS + c] = B[i + (size_t)c * D.ldb];
  const int nblk = (k + 31) / 32;
  const int fr = lane >> 2, fc = lane & 3;
  for (int bb = 0; bb < nblk; ++bb) {
    const int b = UPPER ? nblk - 1 - bb : bb;
    const int r0 = b * 32, nr = min(32, k - r0);
    const int klo = UPPER ? r0 : 0, khi = UPPER ? k : r0 + nr;
    __syncthreads();  // previous block's solve (and the initial load) is complete
    for (int cc = klo + wid; cc < khi; cc += TNC / 32)
      Ts[lane * TTS + cc] = lane < nr ? T[(r0 + lane) + (size_t)cc * D.ldt] : 0.0;
    __syncthreads();
    // X[r0:r0+nr, :] -= T[r0:r0+nr, u] X[u, :] over the solved rows u (DMMA)
    const int ulo = UPPER ? r0 + nr : 0, uhi = UPPER ? k : r0;
    if (uhi > ulo) {
      const int cb = wid * 32;  // this warp's 32 columns
      double acc[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      for (int kk = ulo; kk < uhi; kk += 4) {
        const int kq = kk + fc;
        const bool kin = kq < uhi;
        double a[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = kin ? Ts[(i * 8 + fr) * TTS + kq] : 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = kin ? X[kq * TXS + cb + j * 8 + fr] : 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], bv[j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int rr = i * 8 + fr, c = cb + j * 8 + 2 * fc + h;
            if (rr < nr) X[(r0 + rr) * TXS + c] -= acc[i][j][h];
          }
      __syncthreads();
    }
    // diagonal block: thread = column, values in registers
    if (tid < nc) {
      double x[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = i < nr ? X[(r0 + i) * TXS + tid] : 0.0;
      if (!UPPER) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
#pragma unroll
          for (int i = j + 1; i < 32; ++i) x[i] -= Ts[i * TTS + r0 + j] * x[j];
        }
      } else {
#pragma unroll
        for (int j = 31; j >= 0; --j) {
          if (j < nr) {
            x[j] /= Ts[j * TTS + r0 + j];
#pragma unroll
            for (int i = 0; i < j; ++i) x[i] -= Ts[i * TTS + r0 + j] * x[j];
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < nr) X[(r0 + i) * TXS + tid] = x[i];
    }
  }
  __syncthreads();
  for (int c = wid; c < nc; c += TNC / 32)
    for (int i = lane; i < k; i += 32) B[i + (size_t)c * D.ldb] = X[i * TXS + c];
}

// ||A||_1 (max column abs sum) of each n x n matrix, before factoring.
__global__ void norm1_kernel(const Bases* __restrict__ bases_ptr, const LuDesc* __restrict__ descs) {
  const Bases& bases = *bases_ptr;
  const LuDesc L = descs[blockIdx.x];
  __shared__ double rv[8];
  __shared__ int ri[8];
  const double* A = at<const double>(bases, L.A);
  double best = 0.0;
  for (int c = threadIdx.x; c < L.n; c += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < L.n; ++r) s += fabs(A[r + (size_t)c * L.lda]);
    best = fmax(best, s);
  }
  ArgMax m = block_argmax(ArgMax{best, (int)threadIdx.x}, rv, ri);
  if (threadIdx.x == 0 && L.anorm != kNull) *at<double>(bases, L.anorm) = m.v;
  if (threadIdx.x == 0 && L.info != kNull) *at<int>(bases, L.info) = 0;
}

}  // namespace

cudaError_t launch_panel_batched(const Bases* b, const PanelDesc* d, int count, int max_rows, int pb,
                                 cudaStream_t s) {
  if (count <= 0 || max_rows <= 0) return cudaSuccess;
  const int ldp = max_rows;
  if (pb <= 16) {
    const size_t sm = (size_t)ldp * 16 * sizeof(double);
    cudaFuncSetAttribute(panel_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    panel_kernel<16><<<count, PT, sm, s>>>(b, d, ldp);
  } else {
    const size_t sm = (size_t)ldp * 32 * sizeof(double);
    cudaFuncSetAttribute(panel_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    panel_kernel<32><<<count, PT, sm, s>>>(b, d, ldp);
  }
  return cudaGetLastError();
}

cudaError_t launch_swap_batched(const Bases* b, const SwapDesc* d, int count, int max_cols, cudaStream_t s) {
  if (count <= 0 || max_cols <= 0) return cudaSuccess;
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    swap_kernel<<<dim3((max_cols + 127) / 128, cnt), 128, 0, s>>>(b, d + first);
  }
  return cudaGetLastError();
}

cudaError_t launch_trsm_batched(const Bases* b, const TrsmDesc* d, int count, int max_cols, bool upper,
                                cudaStream_t s) {
  if (count <= 0 || max_cols <= 0) return cudaSuccess;
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    dim3 grid((max_cols + TNC - 1) / TNC, cnt);
    const size_t sm = (size_t)(128 * TXS + 32 * TTS) * sizeof(double);
    if (upper) {
      cudaFuncSetAttribute(trsm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      trsm_kernel<true><<<grid, TNC, sm, s>>>(b, d + first);
    } else {
      cudaFuncSetAttribute(trsm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      trsm_kernel<false><<<grid, TNC, sm, s>>>(b, d + first);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_norm1_batched(const Bases* b, const LuDesc* d, int count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  norm1_kernel<<<count, 256, 0, s>>>(b, d);
  return cudaGetLastError();
}

}  // namespace hks
