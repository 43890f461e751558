// Fused blocked LU with partial pivoting + carried right-hand sides, one CTA
// per matrix (getrf + getrs of solver.py:131-135, 148-156 in one launch).
//
// For the levels of the tree with few nodes the multi-launch LU program
// (plan.cu add_lu_program) is a chain of ~40 dependent small launches; here
// a 256-thread CTA walks the whole factorization of its matrix:
//   for each 32-column panel: panel LU in shared memory (lowest-row
//   tie-break, dgetf2 reciprocal scaling), interchanges + unit-lower solve of
//   the panel's U rows one column per thread (registers), DMMA rank-32
//   update of the trailing matrix and of the right-hand sides;
//   then the backward sweep B := U^-1 B (register substitution per 32-row
//   block, DMMA updates of the rows above).
// The matrix stays in global memory (L2-resident at the small levels).
#include <cfloat>

#include "common.cuh"
#include "hks_internal.h"

namespace hks {
namespace {

constexpr int FT = 256;  // threads (255 registers available: no spills)
constexpr int FW = FT / 32;

// C[0:M, 0:N] -= Aop[0:M, 0:K] * Bop[0:K, 0:N]   (K <= 32, column-major
// operands; Aop / Bop may live in shared or global memory).  32x32 warp
// tiles of 8x8x4 DMMA fragments, tiles spread over the CTA's warps.
__device__ void rank32_update(double* C, int ldc, int M, int N, const double* Aop, int lda, const double* Bop,
                              int ldb, int K) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  const int tm = (M + 31) / 32, tn = (N + 31) / 32;
  for (int t = wid; t < tm * tn; t += FW) {
    const int r0 = (t % tm) * 32, c0 = (t / tm) * 32;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + i * 8 + fr, c = c0 + j * 8 + 2 * fc + h;
          acc[i][j][h] = (r < M && c < N) ? C[r + (size_t)c * ldc] : 0.0;
        }
    for (int kk = 0; kk < K; kk += 4) {
      const int k = kk + fc;
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = r0 + i * 8 + fr;
        a[i] = (r < M && k < K) ? -Aop[r + (size_t)k * lda] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + j * 8 + fr;
        b[j] = (c < N && k < K) ? Bop[k + (size_t)c * ldb] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + i * 8 + fr, c = c0 + j * 8 + 2 * fc + h;
          if (r < M && c < N) C[r + (size_t)c * ldc] = acc[i][j][h];
        }
  }
}

// rows p0.. of one column: interchanges piv[p0..p0+pb) then x := L11^-1 x
// on rows p0..p0+pb (L11 unit lower in shared memory, ld ldp).
// spiv: the panel's pivots (global row indices) in shared memory; the solved
// rows are also written to `us` (PB consecutive doubles) when non-null.
template <int PB>
__device__ __forceinline__ void swap_solve_column(double* col, const int* spiv, int p0, int pb, const double* L,
                                                  int ldp, bool solve, double* us) {
  for (int jj = 0; jj < pb; ++jj) {
    const int p = spiv[jj];
    if (p != p0 + jj) {
      const double t = col[p0 + jj];
      col[p0 + jj] = col[p];
      col[p] = t;
    }
  }
  if (!solve) return;
  double x[PB];
#pragma unroll
  for (int i = 0; i < PB; ++i) x[i] = i < pb ? col[p0 + i] : 0.0;
#pragma unroll
  for (int i = 1; i < PB; ++i)
#pragma unroll
    for (int k = 0; k < i; ++k) x[i] -= L[i + k * ldp] * x[k];
#pragma unroll
  for (int i = 0; i < PB; ++i)
    if (i < pb) {
      col[p0 + i] = x[i];
      if (us) us[i] = x[i];
    }
}

template <int PB>
__global__ void __launch_bounds__(FT) lu_fused_kernel(const Bases* __restrict__ bases_ptr,
                                                          const LuFusedDesc* __restrict__ descs, int ldp,
                                                          int us_cols) {
  const Bases& bases = *bases_ptr;
  const LuFusedDesc D = descs[blockIdx.x];
  const int n = D.n, lda = D.lda, r = D.r, ldb = D.ldb;
  if (n == 0) return;
  double* A = at<double>(bases, D.A);
  int* piv = at<int>(bases, D.piv);
  double* B = r > 0 ? at<double>(bases, D.B) : nullptr;
  extern __shared__ double P[];  // panel: ldp x PB (column-major), then U12 staging
  double* Us = P + (size_t)ldp * PB;  // PB x us_cols (column-major, ld PB) when us_cols > 0
  __shared__ double red_v[FW];
  __shared__ int red_i[FW];
  __shared__ int s_info;
  __shared__ int spiv[PB];
  const int tid = threadIdx.x;
  if (tid == 0) s_info = 0;

  for (int p0 = 0; p0 < n; p0 += PB) {
    const int pb = min(PB, n - p0), mr = n - p0;
    for (int c = 0; c < pb; ++c) {
      const double* src = A + p0 + (size_t)(p0 + c) * lda;
      for (int i = tid; i < mr; i += FT) P[i + c * ldp] = src[i];
    }
    __syncthreads();
    for (int jj = 0; jj < pb; ++jj) {  // panel LU (same arithmetic as panel_kernel)
      ArgMax a{-1.0, 0x7fffffff};
      for (int i = jj + tid; i < mr; i += FT) a = argmax_pick(a, ArgMax{fabs(P[i + jj * ldp]), i});
      a = block_argmax(a, red_v, red_i);
      const int p = a.i;
      const double pv = P[p + jj * ldp];
      if (tid == 0) {
        piv[p0 + jj] = p0 + p;
        spiv[jj] = p0 + p;
        if (pv == 0.0 && s_info == 0) s_info = p0 + jj + 1;
      }
      __syncthreads();
      if (p != jj && tid < pb) {
        const double t = P[jj + tid * ldp];
        P[jj + tid * ldp] = P[p + tid * ldp];
        P[p + tid * ldp] = t;
      }
      __syncthreads();
      const bool recip = fabs(pv) >= DBL_MIN;
      const double inv = 1.0 / pv;
      for (int i = jj + 1 + tid; i < mr; i += FT) {
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
      for (int i = tid; i < mr; i += FT) dst[i] = P[i + c * ldp];
    }
    // interchanges on every other column; U rows of the trailing columns and RHS
    const int ncols = n - pb + r;
    const int tr = n - p0 - pb;
    const bool staged = us_cols >= tr + r;  // U12 rows of the trailing / RHS columns in shared memory
    for (int t = tid; t < ncols; t += FT) {
      const int c = t < p0 ? t : t + pb;  // skip the panel's own columns
      double* us = (staged && c >= p0 + pb) ? Us + (size_t)(c - p0 - pb) * PB : nullptr;
      if (c < n)
        swap_solve_column<PB>(A + (size_t)c * lda, spiv, p0, pb, P, ldp, c >= p0 + pb, us);
      else
        swap_solve_column<PB>(B + (size_t)(c - n) * ldb, spiv, p0, pb, P, ldp, true, us);
    }
    __syncthreads();
    // rank-pb update of the trailing matrix and the right-hand sides
    if (tr > 0) {
      if (staged) {
        rank32_update(A + (p0 + pb) + (size_t)(p0 + pb) * lda, lda, tr, tr, P + pb, ldp, Us, PB, pb);
        if (r > 0) rank32_update(B + p0 + pb, ldb, tr, r, P + pb, ldp, Us + (size_t)tr * PB, PB, pb);
      } else {
        rank32_update(A + (p0 + pb) + (size_t)(p0 + pb) * lda, lda, tr, tr, P + pb, ldp,
                      A + p0 + (size_t)(p0 + pb) * lda, lda, pb);
        if (r > 0) rank32_update(B + p0 + pb, ldb, tr, r, P + pb, ldp, B + p0, ldb, pb);
      }
    }
    __syncthreads();
  }
  if (tid == 0 && s_info && D.info != kNull) {
    int* info = at<int>(bases, D.info);
    if (*info == 0) *info = s_info;
  }
  if (r == 0) return;
  // backward: B := U^-1 B, 32-row blocks from the bottom
  const int nblk = (n + 31) / 32;
  for (int b = nblk - 1; b >= 0; --b) {
    const int r0 = b * 32, nr = min(32, n - r0);
    // stage the diagonal block U[r0:r0+nr, r0:r0+nr] (row-major, ld 33)
    for (int e = tid; e < 32 * 32; e += FT) {
      const int i = e & 31, j = e >> 5;
      P[i * 33 + j] = (i < nr && j < nr) ? A[(r0 + i) + (size_t)(r0 + j) * lda] : 0.0;
    }
    __syncthreads();
    for (int c = tid; c < r; c += FT) {  // one right-hand side per thread
      double* col = B + (size_t)c * ldb + r0;
      double x[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = i < nr ? col[i] : 0.0;
#pragma unroll
      for (int i = 31; i >= 0; --i) {
        if (i < nr) {
          double s = x[i];
#pragma unroll
          for (int k = i + 1; k < 32; ++k) s -= P[i * 33 + k] * x[k];
          x[i] = s / P[i * 33 + i];
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < nr) col[i] = x[i];
    }
    __syncthreads();
    if (r0 > 0) rank32_update(B, ldb, r0, r, A + (size_t)r0 * lda, lda, B + r0, ldb, nr);
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_lu_fused(const Bases* b, const LuFusedDesc* d, int count, int max_n, int max_r,
                            cudaStream_t s) {
  if (count <= 0 || max_n <= 0) return cudaSuccess;
  const int ldp = max_n > 32 ? max_n : 33;  // the backward sweep reuses P as a 32 x 33 block
  const size_t budget = 220 * 1024;
  if (max_n <= 640) {
    const size_t panel = (size_t)ldp * 32 * sizeof(double);
    const int usc = panel + (size_t)32 * (max_n + max_r) * sizeof(double) <= budget ? max_n + max_r : 0;
    const size_t sm = panel + (size_t)32 * usc * sizeof(double);
    raise_smem_limit(lu_fused_kernel<32>, sm);
    lu_fused_kernel<32><<<count, FT, sm, s>>>(b, d, ldp, usc);
  } else {
    const size_t panel = (size_t)ldp * 16 * sizeof(double);
    const int usc = panel + (size_t)16 * (max_n + max_r) * sizeof(double) <= budget ? max_n + max_r : 0;
    const size_t sm = panel + (size_t)16 * usc * sizeof(double);
    raise_smem_limit(lu_fused_kernel<16>, sm);
    lu_fused_kernel<16><<<count, FT, sm, s>>>(b, d, ldp, usc);
  }
  return cudaGetLastError();
}

}  // namespace hks
