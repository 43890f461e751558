// Batched dense LU with partial pivoting, multi-RHS LU solves and the
// LAPACK dgecon 1-norm condition estimate, FP64 on sm_100a.
//
// Replaces scipy.linalg.lu_factor / lu_solve (linalg.py:151-179) for the
// leaf blocks K_aa + lam I (solver.py:128-137) and the reduced matrices Z
// (solver.py:92-108), and lapack.dgecon (solver.py:106).
//
// getrf: one CTA per matrix, right-looking blocked LU.  The NB-wide panel
// lives in shared memory (pivot search = block argmax, lowest row on ties
// as LAPACK idamax); row swaps + the unit-lower TRSM for U12 run one column
// per thread; the trailing update A22 -= L21 U12 runs on DMMA tiles with
// L21 read from the shared-memory panel.
#include <cfloat>

#include "common.cuh"
#include "hks_internal.h"

namespace hks {
namespace {

constexpr int LU_THREADS = 256;

__device__ void trailing_update(double* A, int lda, const double* P, int ldp, int j0, int jb, int n) {
  // A[r, c] -= sum_k L21[r, k] U12[k, c] for r, c in [j0+jb, n); L21[r,k] = P[(r-j0) + k*ldp],
  // U12[k, c] = A[j0+k + c*lda].
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  const int base = j0 + jb, rem = n - base;
  if (rem <= 0) return;
  const int tr = (rem + 31) / 32, tc = tr;
  for (int t = wid; t < tr * tc; t += nw) {
    const int r0 = base + (t % tr) * 32, c0 = base + (t / tr) * 32;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + i * 8 + fr, c = c0 + j * 8 + 2 * fc + h;
          acc[i][j][h] = (r < n && c < n) ? A[r + (size_t)c * lda] : 0.0;
        }
    for (int kk = 0; kk < jb; kk += 4) {
      const int k = kk + fc;
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = r0 + i * 8 + fr;
        a[i] = (r < n && k < jb) ? -P[(r - j0) + k * ldp] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + j * 8 + fr;
        b[j] = (c < n && k < jb) ? A[(j0 + k) + (size_t)c * lda] : 0.0;
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
          if (r < n && c < n) A[r + (size_t)c * lda] = acc[i][j][h];
        }
  }
}

template <int NB>
__global__ void __launch_bounds__(LU_THREADS) getrf_kernel(const Bases* __restrict__ bases_ptr,
                                                            const LuDesc* __restrict__ descs, int ldp) {
  const Bases& bases = *bases_ptr;
  const LuDesc L = descs[blockIdx.x];
  const int n = L.n, lda = L.lda;
  double* A = at<double>(bases, L.A);
  int* piv = at<int>(bases, L.piv);
  extern __shared__ double P[];  // panel: ldp x NB, column-major
  __shared__ double red_v[LU_THREADS / 32];
  __shared__ int red_i[LU_THREADS / 32];
  __shared__ int s_info;
  const int tid = threadIdx.x, nt = blockDim.x;

  if (tid == 0) s_info = 0;
  if (L.anorm != kNull) {  // ||A||_1 before factoring, for gecon (solver.py:98)
    double best = 0.0;
    for (int c = tid; c < n; c += nt) {
      double s = 0.0;
      for (int r = 0; r < n; ++r) s += fabs(A[r + (size_t)c * lda]);
      best = fmax(best, s);
    }
    ArgMax m = block_argmax(ArgMax{best, tid}, red_v, red_i);
    if (tid == 0) *at<double>(bases, L.anorm) = m.v;
  }
  __syncthreads();

  for (int j0 = 0; j0 < n; j0 += NB) {
    const int jb = min(NB, n - j0), mr = n - j0;
    for (int e = tid; e < mr * jb; e += nt) {
      const int i = e % mr, c = e / mr;
      P[i + c * ldp] = A[(j0 + i) + (size_t)(j0 + c) * lda];
    }
    __syncthreads();
    for (int jj = 0; jj < jb; ++jj) {
      ArgMax a{-1.0, 0x7fffffff};
      for (int i = jj + tid; i < mr; i += nt) a = argmax_pick(a, ArgMax{fabs(P[i + jj * ldp]), i});
      a = block_argmax(a, red_v, red_i);
      const int p = a.i;
      const double pv = P[p + jj * ldp];
      __syncthreads();  // every thread has read pv before the swap below
      if (tid == 0) {
        piv[j0 + jj] = j0 + p;
        if (pv == 0.0 && s_info == 0) s_info = j0 + jj + 1;
      }
      if (p != jj)
        for (int c = tid; c < jb; c += nt) {
          const double t = P[jj + c * ldp];
          P[jj + c * ldp] = P[p + c * ldp];
          P[p + c * ldp] = t;
        }
      __syncthreads();
      if (pv != 0.0) {
        // dgetf2: scale by the reciprocal when it is safe, else divide
        const bool recip = fabs(pv) >= DBL_MIN;
        const double inv = 1.0 / pv;
        for (int i = jj + 1 + tid; i < mr; i += nt)
          P[i + jj * ldp] = recip ? P[i + jj * ldp] * inv : P[i + jj * ldp] / pv;
      }
      __syncthreads();
      const int rr = mr - jj - 1, cc = jb - jj - 1;
      for (int e = tid; e < rr * cc; e += nt) {
        const int i = jj + 1 + e % rr, c = jj + 1 + e / rr;
        P[i + c * ldp] -= P[i + jj * ldp] * P[jj + c * ldp];
      }
      __syncthreads();
    }
    for (int e = tid; e < mr * jb; e += nt) {
      const int i = e % mr, c = e / mr;
      A[(j0 + i) + (size_t)(j0 + c) * lda] = P[i + c * ldp];
    }
    // row interchanges on the columns outside the panel, then U12 = L11^-1 A12
    for (int c = tid; c < n; c += nt) {
      if (c >= j0 && c < j0 + jb) continue;
      double* col = A + (size_t)c * lda;
      for (int jj = 0; jj < jb; ++jj) {
        const int p = piv[j0 + jj];
        if (p != j0 + jj) {
          const double t = col[j0 + jj];
          col[j0 + jj] = col[p];
          col[p] = t;
        }
      }
      if (c >= j0 + jb) {
        for (int i = 1; i < jb; ++i) {
          double s = col[j0 + i];
          for (int k = 0; k < i; ++k) s -= P[i + k * ldp] * col[j0 + k];
          col[j0 + i] = s;
        }
      }
    }
    __syncthreads();
    trailing_update(A, lda, P, ldp, j0, jb, n);
    __syncthreads();
  }
  if (tid == 0 && L.info != kNull) *at<int>(bases, L.info) = s_info;
}

// ------------------------------------------------------------------ getrs

constexpr int RS_THREADS = 256;

// X[rows r0..r0+31, :] -= M[r0..r0+31, k0..k1) * X[k0..k1, :]; M column-major
// global (lda), X in shared memory (ldx); RC columns.  DMMA tiles, 8 warps.
template <int RC>
__device__ void block_rows_update(const double* M, int lda, double* X, int ldx, int r0, int nrows,
                                  int k0, int k1, int ncols) {
  constexpr int FC = RC / 8;  // column fragments
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  // 4 row fragments x FC column fragments spread over 8 warps
  for (int f = wid; f < 4 * FC; f += 8) {
    const int fi = f % 4, fj = f / 4;
    const int r = r0 + fi * 8 + fr;
    double d0 = 0.0, d1 = 0.0;
    for (int k = k0; k < k1; k += 4) {
      const int kk = k + fc;
      const double a = (fi * 8 + fr < nrows && kk < k1) ? -M[r + (size_t)kk * lda] : 0.0;
      const int cb = fj * 8 + fr;
      const double b = (kk < k1 && cb < ncols) ? X[kk + cb * ldx] : 0.0;
      dmma884(d0, d1, a, b);
    }
    // accumulate into X (disjoint rows from the k-range, so no race)
    const int c = fj * 8 + 2 * fc;
    if (fi * 8 + fr < nrows) {
      if (c < ncols) X[r + c * ldx] += d0;
      if (c + 1 < ncols) X[r + (c + 1) * ldx] += d1;
    }
  }
}

template <int RC>
__global__ void __launch_bounds__(RS_THREADS) getrs_kernel(const Bases* __restrict__ bases_ptr,
                                                             const LuSolveDesc* __restrict__ descs, int ldx) {
  const Bases& bases = *bases_ptr;
  const LuSolveDesc S = descs[blockIdx.x];
  const int* spiv = at<const int>(bases, S.piv);
  double* SB = at<double>(bases, S.B);
  const int n = S.n, c0 = blockIdx.y * RC;
  if (c0 >= S.nrhs || n == 0) return;
  const int nc = min(RC, S.nrhs - c0);
  extern __shared__ double X[];  // ldx x RC
  int* perm = reinterpret_cast<int*>(X + (size_t)ldx * RC);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5;
  const double* LU = at<const double>(bases, S.LU);
  const int lda = S.lda;

  if (tid == 0) {
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int i = 0; i < n; ++i) {
      const int p = spiv[i];
      const int t = perm[i];
      perm[i] = perm[p];
      perm[p] = t;
    }
  }
  __syncthreads();
  for (int e = tid; e < n * nc; e += nt) {
    const int i = e % n, c = e / n;
    X[i + c * ldx] = SB[perm[i] + (size_t)(c0 + c) * S.ldb];
  }
  __syncthreads();

  // forward: L (unit lower), 32-row blocks
  for (int r0 = 0; r0 < n; r0 += 32) {
    const int nr = min(32, n - r0);
    if (r0 > 0) {
      block_rows_update<RC>(LU, lda, X, ldx, r0, nr, 0, r0, nc);
      __syncthreads();
    }
    // in-block forward substitution: warp w owns columns w, w+8, ...; lane = row
    for (int c = wid; c < nc; c += 8) {
      double x = lane < nr ? X[r0 + lane + c * ldx] : 0.0;
      for (int j = 0; j < nr; ++j) {
        const double xj = __shfl_sync(0xffffffffu, x, j);
        if (lane > j && lane < nr) x -= LU[(r0 + lane) + (size_t)(r0 + j) * lda] * xj;
      }
      if (lane < nr) X[r0 + lane + c * ldx] = x;
    }
    __syncthreads();
  }
  // backward: U (non-unit upper), blocks from the bottom
  const int nblk = (n + 31) / 32;
  for (int b = nblk - 1; b >= 0; --b) {
    const int r0 = b * 32, nr = min(32, n - r0);
    if (r0 + nr < n) {
      block_rows_update<RC>(LU, lda, X, ldx, r0, nr, r0 + nr, n, nc);
      __syncthreads();
    }
    for (int c = wid; c < nc; c += 8) {
      double x = lane < nr ? X[r0 + lane + c * ldx] : 0.0;
      for (int j = nr - 1; j >= 0; --j) {
        double xj = __shfl_sync(0xffffffffu, x, j);
        xj /= LU[(r0 + j) + (size_t)(r0 + j) * lda];
        if (lane == j) x = xj;
        if (lane < j) x -= LU[(r0 + lane) + (size_t)(r0 + j) * lda] * xj;
      }
      if (lane < nr) X[r0 + lane + c * ldx] = x;
    }
    __syncthreads();
  }
  for (int e = tid; e < n * nc; e += nt) {
    const int i = e % n, c = e / n;
    SB[i + (size_t)(c0 + c) * S.ldb] = X[i + c * ldx];
  }
}

// ------------------------------------------------------------------ gecon

// Same solve, latency-lean (gecon only: its result is an estimate, so the
// diagonal uses a reciprocal computed off the dependency chain).  Warp 0
// holds the 32 x 32 diagonal block of op(T) in registers (lane i: row i)
// and solves it with one shuffle per step; the next block's rows are loaded
// before the block's update so their latency hides behind it; the update of
// the remaining entries is one thread per entry with 32 independent loads.
__device__ __forceinline__ void trsv_load_diag(const double* LU, int lda, int n, int b, bool upper, bool trans,
                                               double (&t)[32], double& rd) {
  const int lane = threadIdx.x & 31, r0 = b * 32, nr = min(32, n - r0);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    double v = 0.0;
    if (lane < nr && j < nr)
      v = trans ? LU[(r0 + j) + (size_t)(r0 + lane) * lda] : LU[(r0 + lane) + (size_t)(r0 + j) * lda];
    t[j] = v;
  }
  double dg = 1.0;
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j == lane) dg = t[j];
  rd = (upper && lane < nr) ? 1.0 / dg : 1.0;
}

__device__ __noinline__ void trsv_fast(const double* LU, int lda, int n, double* x, bool upper, bool trans) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
  const bool forward = (!upper && !trans) || (upper && trans);
  const int nblk = (n + 31) / 32;
  double t[32], rd = 1.0;
  if (tid < 32) trsv_load_diag(LU, lda, n, forward ? 0 : nblk - 1, upper, trans, t, rd);
  for (int bb = 0; bb < nblk; ++bb) {
    const int b = forward ? bb : nblk - 1 - bb;
    const int r0 = b * 32, nr = min(32, n - r0);
    if (tid < 32) {
      double v = lane < nr ? x[r0 + lane] : 0.0;
      if (forward) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (lane == j) v *= rd;
          const double xj = __shfl_sync(0xffffffffu, v, j);
          if (lane > j) v -= t[j] * xj;
        }
      } else {
#pragma unroll
        for (int j = 31; j >= 0; --j) {
          if (lane == j) v *= rd;
          const double xj = __shfl_sync(0xffffffffu, v, j);
          if (lane < j) v -= t[j] * xj;
        }
      }
      if (lane < nr) x[r0 + lane] = v;
      if (bb + 1 < nblk) trsv_load_diag(LU, lda, n, forward ? b + 1 : b - 1, upper, trans, t, rd);
    }
    __syncthreads();
    const int lo = forward ? r0 + nr : 0, hi = forward ? n : r0;
    if (!trans) {  // thread per row i, lanes along the rows of each column (coalesced)
      for (int i = lo + tid; i < hi; i += nt) {
        double s = x[i];
#pragma unroll 8
        for (int j = 0; j < nr; ++j) s -= LU[i + (size_t)(r0 + j) * lda] * x[r0 + j];
        x[i] = s;
      }
    } else {
      // op(T)(i, r0 + j) = T(r0 + j, i): row i of op(T) is a contiguous piece
      // of column i of T, so one warp takes row i with its lanes along that
      // piece (one coalesced 256-byte load instead of 32 strided ones per
      // thread, which made the transposed sweeps L1-transaction bound), four
      // rows per warp in flight, warp-sum reductions
      const int nw = nt >> 5, wid = tid >> 5;
      const double xl = lane < nr ? x[r0 + lane] : 0.0;
      for (int i0 = lo + 4 * wid; i0 < hi; i0 += 4 * nw) {
        double p[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          p[q] = (i0 + q < hi && lane < nr) ? LU[r0 + lane + (size_t)(i0 + q) * lda] * xl : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) p[q] = warp_sum(p[q]);
        if (lane < 4 && i0 + lane < hi) {
          double sq = p[0];
#pragma unroll
          for (int q = 1; q < 4; ++q)
            if (lane == q) sq = p[q];
          x[i0 + lane] -= sq;
        }
      }
    }
    __syncthreads();
  }
}

__device__ double block_asum(const double* x, int n, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += fabs(x[i]);
  return block_sum(s, red);
}

__device__ int block_iamax(const double* x, int n, double* rv, int* ri) {
  ArgMax a{-1.0, 0x7fffffff};
  for (int i = threadIdx.x; i < n; i += blockDim.x) a = argmax_pick(a, ArgMax{fabs(x[i]), i});
  return block_argmax(a, rv, ri).i;
}

// LAPACK dgecon(norm='1') with dlacn2 (Higham's estimator), restated; the
// dlatrs overflow scaling is not needed at the conditioning the solver
// admits (documented in DESIGN.md).
#ifndef GECON_THREADS
#define GECON_THREADS 256
#endif
__global__ void __launch_bounds__(GECON_THREADS, 2) gecon_kernel(const Bases* __restrict__ bases_ptr,
                                                     const LuDesc* __restrict__ descs) {
  const Bases& bases = *bases_ptr;
  const LuDesc L = descs[blockIdx.x];
  const double* LUa = at<const double>(bases, L.A);
  const int n = L.n;
  extern __shared__ double sh[];
  double* x = sh;        // n
  double* v = sh + n;    // n
  int* isgn = reinterpret_cast<int*>(sh + 2 * n);

  __shared__ double red_v[8];
  __shared__ int red_i[8];
  const int tid = threadIdx.x, nt = blockDim.x;
  if (L.rcond == kNull) return;
  double* rcond = at<double>(bases, L.rcond);
  if (n == 0) { if (tid == 0) *rcond = 1.0; return; }
  const double anorm = *at<const double>(bases, L.anorm);
  if (anorm == 0.0) { if (tid == 0) *rcond = 0.0; return; }
  if (L.info != kNull && *at<const int>(bases, L.info) != 0) { if (tid == 0) *rcond = 0.0; return; }

  auto apply = [&](int kase) {
    if (kase == 1) {
      trsv_fast(LUa, L.lda, n, x, false, false);
      trsv_fast(LUa, L.lda, n, x, true, false);
    } else {
      trsv_fast(LUa, L.lda, n, x, true, true);
      trsv_fast(LUa, L.lda, n, x, false, true);
    }
  };

  double est;
  for (int i = tid; i < n; i += nt) x[i] = 1.0 / n;
  __syncthreads();
  apply(1);
  if (n == 1) {
    est = fabs(x[0]);
  } else {
    est = block_asum(x, n, red_v);
    for (int i = tid; i < n; i += nt) {
      x[i] = x[i] >= 0.0 ? 1.0 : -1.0;
      isgn[i] = x[i] >= 0.0 ? 1 : -1;
    }
    __syncthreads();
    apply(2);
    int j = block_iamax(x, n, red_v, red_i);
    int iter = 2;
    bool alt = false;
    for (;;) {
      // L50
      for (int i = tid; i < n; i += nt) x[i] = (i == j) ? 1.0 : 0.0;
      __syncthreads();
      apply(1);
      for (int i = tid; i < n; i += nt) v[i] = x[i];
      const double estold = est;
      est = block_asum(v, n, red_v);
      // repeated sign vector?
      __shared__ int s_diff;
      if (tid == 0) s_diff = 0;
      __syncthreads();
      for (int i = tid; i < n; i += nt) {
        const int xs = x[i] >= 0.0 ? 1 : -1;
        if (xs != isgn[i]) s_diff = 1;
      }
      __syncthreads();
      const int diff = s_diff;
      __syncthreads();
      if (!diff || est <= estold) { alt = true; break; }
      for (int i = tid; i < n; i += nt) {
        x[i] = x[i] >= 0.0 ? 1.0 : -1.0;
        isgn[i] = x[i] >= 0.0 ? 1 : -1;
      }
      __syncthreads();
      apply(2);
      const int jlast = j;
      j = block_iamax(x, n, red_v, red_i);
      if (x[jlast] != fabs(x[j]) && iter < 5) {
        ++iter;
        continue;
      }
      alt = true;
      break;
    }
    if (alt) {  // L120: alternating-sign probe
      for (int i = tid; i < n; i += nt) {
        const double s = (i % 2 == 0) ? 1.0 : -1.0;
        x[i] = s * (1.0 + (double)i / (double)(n - 1));
      }
      __syncthreads();
      apply(1);
      const double temp = 2.0 * (block_asum(x, n, red_v) / (double)(3 * n));
      if (temp > est) est = temp;
    }
  }
  if (tid == 0) {
    const double ainvnm = est;
    *rcond = ainvnm != 0.0 ? (1.0 / ainvnm) / anorm : 0.0;
  }
}

// The same estimate as a sequence of short launches (dgecon runs
// beside the factorization on a low-priority stream).  A monolithic
// estimate keeps its CTA resident for ~11 LU sweeps (~0.5-1 ms), and
// resident CTAs block the factorization's large-footprint kernels from
// those SMs; split at every LU application, each CTA lives one application
// (two triangular sweeps) and the SMs turn over quickly.  The dlacn2 state
// of each matrix (x, sign vector, est, j, iter, next step) lives in global
// scratch (base kGeconScratchBase, `stride` doubles per matrix).  Arithmetic
// and its order are those of gecon_kernel, so the results are identical
// (both share trsv_fast; its transposed sweeps sum each row as a warp
// reduction, an order LAPACK does not fix either -- z_cond is an estimate,
// checked to 1e-3 against dgecon).
enum GeconState { GS_A = 0, GS_B, GS_C, GS_D, GS_E, GS_DONE };

__device__ __forceinline__ void gecon_step_one(const Bases& bases, const LuDesc& L, int m, int stride, int phase) {
  if (L.rcond == kNull) return;
  const int n = L.n;
  double* st = at<double>(bases, make_ref(kGeconScratchBase, 0)) + (size_t)m * stride;
  double* gx = st;                     // n
  double* gsgn = st + n;               // n (+-1)
  double* sc = st + 2 * (size_t)n;     // state, kase, iter, j, est
  const int tid = threadIdx.x, nt = blockDim.x;
  double* rcond = at<double>(bases, L.rcond);
  extern __shared__ double sh[];
  double* x = sh;
  __shared__ double red_v[8];
  __shared__ int red_i[8];
  __shared__ int s_diff;
  if (phase == 0) {  // initialise (or finish the trivial cases)
    int state = GS_A;
    if (n == 0) {
      if (tid == 0) *rcond = 1.0;
      state = GS_DONE;
    } else {
      const double anorm = *at<const double>(bases, L.anorm);
      if (anorm == 0.0 || (L.info != kNull && *at<const int>(bases, L.info) != 0)) {
        if (tid == 0) *rcond = 0.0;
        state = GS_DONE;
      }
    }
    if (state != GS_DONE)
      for (int i = tid; i < n; i += nt) gx[i] = 1.0 / n;
    if (tid == 0) {
      sc[0] = state;
      sc[1] = 1;  // kase of the next application
      sc[2] = 0;
      sc[3] = 0;
      sc[4] = 0.0;
    }
    return;
  }
  int state = (int)sc[0];
  if (state == GS_DONE) return;
  const double* LUa = at<const double>(bases, L.A);
  const int kase = (int)sc[1];
  int iter = (int)sc[2], j = (int)sc[3];
  double est = sc[4];
  for (int i = tid; i < n; i += nt) x[i] = gx[i];
  __syncthreads();
  if (kase == 1) {
    trsv_fast(LUa, L.lda, n, x, false, false);
    trsv_fast(LUa, L.lda, n, x, true, false);
  } else {
    trsv_fast(LUa, L.lda, n, x, true, true);
    trsv_fast(LUa, L.lda, n, x, false, true);
  }
  int next_kase = 1;
  auto set_alt = [&]() {  // L120: alternating-sign probe
    for (int i = tid; i < n; i += nt) {
      const double sg = (i % 2 == 0) ? 1.0 : -1.0;
      x[i] = sg * (1.0 + (double)i / (double)(n - 1));
    }
    next_kase = 1;
    state = GS_E;
  };
  auto set_unit = [&](int jj) {  // L50: x = e_j
    for (int i = tid; i < n; i += nt) x[i] = (i == jj) ? 1.0 : 0.0;
    next_kase = 1;
    state = GS_C;
  };
  if (state == GS_A) {
    if (n == 1) {
      est = fabs(x[0]);
      state = GS_DONE;
    } else {
      est = block_asum(x, n, red_v);
      for (int i = tid; i < n; i += nt) {
        x[i] = x[i] >= 0.0 ? 1.0 : -1.0;
        gsgn[i] = x[i];
      }
      next_kase = 2;
      state = GS_B;
    }
  } else if (state == GS_B) {
    j = block_iamax(x, n, red_v, red_i);
    iter = 2;
    __syncthreads();
    set_unit(j);
  } else if (state == GS_C) {
    const double estold = est;
    est = block_asum(x, n, red_v);
    if (tid == 0) s_diff = 0;
    __syncthreads();
    for (int i = tid; i < n; i += nt) {
      const double xs = x[i] >= 0.0 ? 1.0 : -1.0;
      if (xs != gsgn[i]) s_diff = 1;
    }
    __syncthreads();
    const int diff = s_diff;
    __syncthreads();
    if (!diff || est <= estold) {
      set_alt();
    } else {
      for (int i = tid; i < n; i += nt) {
        x[i] = x[i] >= 0.0 ? 1.0 : -1.0;
        gsgn[i] = x[i];
      }
      next_kase = 2;
      state = GS_D;
    }
  } else if (state == GS_D) {
    const int jlast = j;
    j = block_iamax(x, n, red_v, red_i);
    __syncthreads();
    if (x[jlast] != fabs(x[j]) && iter < 5) {
      ++iter;
      __syncthreads();
      set_unit(j);
    } else {
      __syncthreads();
      set_alt();
    }
  } else {  // GS_E
    const double temp = 2.0 * (block_asum(x, n, red_v) / (double)(3 * n));
    if (temp > est) est = temp;
    state = GS_DONE;
  }
  __syncthreads();
  if (state == GS_DONE) {
    if (tid == 0) {
      const double anorm = *at<const double>(bases, L.anorm);
      *rcond = est != 0.0 ? (1.0 / est) / anorm : 0.0;
    }
  } else {
    for (int i = tid; i < n; i += nt) gx[i] = x[i];
  }
  if (tid == 0) {
    sc[0] = state;
    sc[1] = next_kase;
    sc[2] = iter;
    sc[3] = j;
    sc[4] = est;
  }
}

// ------------------------------------------------------------------
// Warp-per-matrix form of the split estimate (what the factorization
// launches).  The estimate is a chain of latency-bound triangular sweeps;
// one warp per matrix (instead of one 256-thread CTA) keeps ~16 matrices
// in flight per SM with no CTA barriers, so a phase over a level's ~2000
// matrices runs in about one wave instead of seven, and the SMs turn over
// to the factorization's kernels after a few tens of microseconds.  Same
// dlacn2 state machine and scratch layout as gecon_step_one.
constexpr int GW_WARPS = 4;                    // warps (matrices) per CTA
constexpr int GW_TILE = 32 * 33;               // transposed-sweep staging tile per warp

// x := op(T)^-1 x for the LU in LU (unit lower / non-unit upper part, op =
// transpose when trans), x in this warp's shared slice.
__device__ void trsv_warp(const double* LU, int lda, int n, double* x, double* tile, bool upper, bool trans) {
  const int lane = threadIdx.x & 31;
  const bool forward = (!upper && !trans) || (upper && trans);
  const int nblk = (n + 31) / 32;
  for (int bb = 0; bb < nblk; ++bb) {
    const int b = forward ? bb : nblk - 1 - bb;
    const int r0 = b * 32, nr = min(32, n - r0);
    double t[32], rd;
    trsv_load_diag(LU, lda, n, b, upper, trans, t, rd);
    double v = lane < nr ? x[r0 + lane] : 0.0;
    if (forward) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (lane == j) v *= rd;
        const double xj = __shfl_sync(0xffffffffu, v, j);
        if (lane > j) v -= t[j] * xj;
      }
    } else {
#pragma unroll
      for (int j = 31; j >= 0; --j) {
        if (lane == j) v *= rd;
        const double xj = __shfl_sync(0xffffffffu, v, j);
        if (lane < j) v -= t[j] * xj;
      }
    }
    if (lane < nr) x[r0 + lane] = v;
    __syncwarp();
    const int lo = forward ? r0 + nr : 0, hi = forward ? n : r0;
    if (!trans) {
      // 32 rows x the block's 32 columns at a time through the padded tile
      // (cp.async: the 32 column segments of 256 bytes all in flight), then
      // lane q updates row c0 + q
      for (int c0 = lo; c0 < hi; c0 += 32) {
        const int nq = min(32, hi - c0);
        for (int j = 0; j < 32; ++j) {
          const bool ok = j < nr && lane < nq;
          cp_async8(tile + j * 33 + lane, ok ? LU + c0 + lane + (size_t)(r0 + j) * lda : LU, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        if (lane < nq) {
          double sacc = x[c0 + lane];
#pragma unroll 8
          for (int j = 0; j < nr; ++j) sacc -= tile[j * 33 + lane] * x[r0 + j];
          x[c0 + lane] = sacc;
        }
        __syncwarp();
      }
    } else {
      // op(T)(i, r0 + j) = T(r0 + j, i): 32 columns of T at a time through a
      // padded shared tile (one coalesced 256-byte load per column, all 32
      // in flight), then lane q sums row c0 + q from the tile (stride 33:
      // conflict-free)
      for (int c0 = lo; c0 < hi; c0 += 32) {
        const int nq = min(32, hi - c0);
        // cp.async: all 32 column loads in flight (a register load + shared
        // store pair per column serialised one DRAM latency per column)
        for (int q = 0; q < 32; ++q) {
          const bool ok = q < nq && lane < nr;
          cp_async8(tile + q * 33 + lane, ok ? LU + r0 + lane + (size_t)(c0 + q) * lda : LU, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        if (lane < nq) {
          double s = x[c0 + lane];
#pragma unroll 8
          for (int j = 0; j < nr; ++j) s -= tile[lane * 33 + j] * x[r0 + j];
          x[c0 + lane] = s;
        }
        __syncwarp();
      }
    }
    __syncwarp();
  }
}

__device__ __forceinline__ double warp_asum(const double* x, int n) {
  double s = 0.0;
  for (int i = threadIdx.x & 31; i < n; i += 32) s += fabs(x[i]);
  return warp_sum(s);
}

__device__ __forceinline__ int warp_iamax(const double* x, int n) {
  ArgMax a{-1.0, 0x7fffffff};
  for (int i = threadIdx.x & 31; i < n; i += 32) a = argmax_pick(a, ArgMax{fabs(x[i]), i});
  return warp_argmax(a).i;
}

__device__ void gecon_warp_one(const Bases& bases, const LuDesc& L, int m, int stride, int phase, double* x,
                               double* tile) {
  if (L.rcond == kNull) return;
  const int n = L.n, lane = threadIdx.x & 31;
  double* st = at<double>(bases, make_ref(kGeconScratchBase, 0)) + (size_t)m * stride;
  double* gx = st;
  double* gsgn = st + n;
  double* sc = st + 2 * (size_t)n;
  double* rcond = at<double>(bases, L.rcond);
  if (phase == 0) {
    int state = GS_A;
    if (n == 0) {
      if (lane == 0) *rcond = 1.0;
      state = GS_DONE;
    } else {
      const double anorm = *at<const double>(bases, L.anorm);
      if (anorm == 0.0 || (L.info != kNull && *at<const int>(bases, L.info) != 0)) {
        if (lane == 0) *rcond = 0.0;
        state = GS_DONE;
      }
    }
    if (state != GS_DONE)
      for (int i = lane; i < n; i += 32) gx[i] = 1.0 / n;
    if (lane == 0) {
      sc[0] = state;
      sc[1] = 1;
      sc[2] = 0;
      sc[3] = 0;
      sc[4] = 0.0;
    }
    return;
  }
  int state = (int)sc[0];
  if (state == GS_DONE) return;
  const double* LUa = at<const double>(bases, L.A);
  const int kase = (int)sc[1];
  int iter = (int)sc[2], j = (int)sc[3];
  double est = sc[4];
  for (int i = lane; i < n; i += 32) x[i] = gx[i];
  __syncwarp();
  if (kase == 1) {
    trsv_warp(LUa, L.lda, n, x, tile, false, false);
    trsv_warp(LUa, L.lda, n, x, tile, true, false);
  } else {
    trsv_warp(LUa, L.lda, n, x, tile, true, true);
    trsv_warp(LUa, L.lda, n, x, tile, false, true);
  }
  int next_kase = 1;
  auto set_alt = [&]() {
    for (int i = lane; i < n; i += 32) {
      const double sg = (i % 2 == 0) ? 1.0 : -1.0;
      x[i] = sg * (1.0 + (double)i / (double)(n - 1));
    }
    next_kase = 1;
    state = GS_E;
  };
  auto set_unit = [&](int jj) {
    for (int i = lane; i < n; i += 32) x[i] = (i == jj) ? 1.0 : 0.0;
    next_kase = 1;
    state = GS_C;
  };
  if (state == GS_A) {
    if (n == 1) {
      est = fabs(x[0]);
      state = GS_DONE;
    } else {
      est = warp_asum(x, n);
      for (int i = lane; i < n; i += 32) {
        x[i] = x[i] >= 0.0 ? 1.0 : -1.0;
        gsgn[i] = x[i];
      }
      next_kase = 2;
      state = GS_B;
    }
  } else if (state == GS_B) {
    j = warp_iamax(x, n);
    iter = 2;
    __syncwarp();
    set_unit(j);
  } else if (state == GS_C) {
    const double estold = est;
    est = warp_asum(x, n);
    int diff = 0;
    for (int i = lane; i < n; i += 32) {
      const double xs = x[i] >= 0.0 ? 1.0 : -1.0;
      if (xs != gsgn[i]) diff = 1;
    }
    diff = __any_sync(0xffffffffu, diff);
    if (!diff || est <= estold) {
      set_alt();
    } else {
      for (int i = lane; i < n; i += 32) {
        x[i] = x[i] >= 0.0 ? 1.0 : -1.0;
        gsgn[i] = x[i];
      }
      next_kase = 2;
      state = GS_D;
    }
  } else if (state == GS_D) {
    const int jlast = j;
    j = warp_iamax(x, n);
    __syncwarp();
    if (x[jlast] != fabs(x[j]) && iter < 5) {
      ++iter;
      __syncwarp();
      set_unit(j);
    } else {
      __syncwarp();
      set_alt();
    }
  } else {
    const double temp = 2.0 * (warp_asum(x, n) / (double)(3 * n));
    if (temp > est) est = temp;
    state = GS_DONE;
  }
  __syncwarp();
  if (state == GS_DONE) {
    if (lane == 0) {
      const double anorm = *at<const double>(bases, L.anorm);
      *rcond = est != 0.0 ? (1.0 / est) / anorm : 0.0;
    }
  } else {
    for (int i = lane; i < n; i += 32) gx[i] = x[i];
  }
  if (lane == 0) {
    sc[0] = state;
    sc[1] = next_kase;
    sc[2] = iter;
    sc[3] = j;
    sc[4] = est;
  }
}

// xs: doubles of each warp's x slice (>= the batch's largest n)
__global__ void __launch_bounds__(32 * GW_WARPS) gecon_warp_kernel(const Bases* __restrict__ bases_ptr,
                                                                   const LuDesc* __restrict__ descs, int count,
                                                                   int stride, int phase, int xs) {
  extern __shared__ double gw[];
  const int w = threadIdx.x >> 5;
  double* x = gw + (size_t)w * (xs + GW_TILE);
  double* tile = x + xs;
  for (int m = blockIdx.x * GW_WARPS + w; m < count; m += gridDim.x * GW_WARPS) {
    gecon_warp_one(*bases_ptr, descs[m], m, stride, phase, x, tile);
    __syncwarp();
  }
}

// ------------------------------------------------------------------
// CTA-per-matrix form with many loads in flight (the default since round
// 2): 128 threads per matrix, four matrices per SM.  A triangular sweep is
// a chain of 32-row block steps whose off-diagonal update streams the
// block's 32 columns of the LU from HBM; with a few rows per thread and one
// column at a time, every step waited out ~32 dependent load latencies.
// Here a thread keeps 4 rows x 4 columns of loads in flight (non-transposed
// sweeps) and every warp stages its own 32-column chunks of the transposed
// panel through a padded shared tile (one coalesced 256-byte load per
// column, 32 in flight).  Same dlacn2 state machine as gecon_step_one.
constexpr int GC_THREADS = 128;
constexpr int GC_WARPS = GC_THREADS / 32;

__device__ __noinline__ void trsv_cta(const double* LU, int lda, int n, double* x, double* tiles, bool upper,
                                      bool trans) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool forward = (!upper && !trans) || (upper && trans);
  const int nblk = (n + 31) / 32;
  double* tile = tiles + wid * (32 * 33);
  double t[32], rd = 1.0;
  if (tid < 32) trsv_load_diag(LU, lda, n, forward ? 0 : nblk - 1, upper, trans, t, rd);
  for (int bb = 0; bb < nblk; ++bb) {
    const int b = forward ? bb : nblk - 1 - bb;
    const int r0 = b * 32, nr = min(32, n - r0);
    if (tid < 32) {
      double v = lane < nr ? x[r0 + lane] : 0.0;
      if (forward) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (lane == j) v *= rd;
          const double xj = __shfl_sync(0xffffffffu, v, j);
          if (lane > j) v -= t[j] * xj;
        }
      } else {
#pragma unroll
        for (int j = 31; j >= 0; --j) {
          if (lane == j) v *= rd;
          const double xj = __shfl_sync(0xffffffffu, v, j);
          if (lane < j) v -= t[j] * xj;
        }
      }
      if (lane < nr) x[r0 + lane] = v;
      if (bb + 1 < nblk) trsv_load_diag(LU, lda, n, forward ? b + 1 : b - 1, upper, trans, t, rd);
    }
    __syncthreads();
    const int lo = forward ? r0 + nr : 0, hi = forward ? n : r0;
    if (!trans) {
      constexpr int RQ = 4, JU = 4;
      for (int base = lo; base < hi; base += GC_THREADS * RQ) {
        double acc[RQ];
#pragma unroll
        for (int q = 0; q < RQ; ++q) {
          const int i = base + tid + GC_THREADS * q;
          acc[q] = i < hi ? x[i] : 0.0;
        }
        for (int j0 = 0; j0 < nr; j0 += JU) {
          double lv[JU][RQ];
#pragma unroll
          for (int jj = 0; jj < JU; ++jj)
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
              const int i = base + tid + GC_THREADS * q;
              lv[jj][q] = (i < hi && j0 + jj < nr) ? LU[i + (size_t)(r0 + j0 + jj) * lda] : 0.0;
            }
#pragma unroll
          for (int jj = 0; jj < JU; ++jj) {
            const double xj = j0 + jj < nr ? x[r0 + j0 + jj] : 0.0;
#pragma unroll
            for (int q = 0; q < RQ; ++q) acc[q] -= lv[jj][q] * xj;
          }
        }
#pragma unroll
        for (int q = 0; q < RQ; ++q) {
          const int i = base + tid + GC_THREADS * q;
          if (i < hi) x[i] = acc[q];
        }
      }
    } else {
      for (int c0 = lo + 32 * wid; c0 < hi; c0 += 32 * GC_WARPS) {
        const int nq = min(32, hi - c0);
        // cp.async: all 32 column loads in flight (a register load + shared
        // store pair per column serialised one DRAM latency per column)
        for (int q = 0; q < 32; ++q) {
          const bool ok = q < nq && lane < nr;
          cp_async8(tile + q * 33 + lane, ok ? LU + r0 + lane + (size_t)(c0 + q) * lda : LU, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        if (lane < nq) {
          double sacc = x[c0 + lane];
#pragma unroll 8
          for (int j = 0; j < nr; ++j) sacc -= tile[lane * 33 + j] * x[r0 + j];
          x[c0 + lane] = sacc;
        }
        __syncwarp();
      }
    }
    __syncthreads();
  }
}

__device__ void gecon_cta_one(const Bases& bases, const LuDesc& L, int m, int stride, int phase, double* x,
                              double* tiles) {
  if (L.rcond == kNull) return;
  const int n = L.n;
  double* st = at<double>(bases, make_ref(kGeconScratchBase, 0)) + (size_t)m * stride;
  double* gx = st;
  double* gsgn = st + n;
  double* sc = st + 2 * (size_t)n;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* rcond = at<double>(bases, L.rcond);
  __shared__ double red_v[8];
  __shared__ int red_i[8];
  __shared__ int s_diff;
  if (phase == 0) {
    int state = GS_A;
    if (n == 0) {
      if (tid == 0) *rcond = 1.0;
      state = GS_DONE;
    } else {
      const double anorm = *at<const double>(bases, L.anorm);
      if (anorm == 0.0 || (L.info != kNull && *at<const int>(bases, L.info) != 0)) {
        if (tid == 0) *rcond = 0.0;
        state = GS_DONE;
      }
    }
    if (state != GS_DONE)
      for (int i = tid; i < n; i += nt) gx[i] = 1.0 / n;
    if (tid == 0) {
      sc[0] = state;
      sc[1] = 1;
      sc[2] = 0;
      sc[3] = 0;
      sc[4] = 0.0;
    }
    return;
  }
  int state = (int)sc[0];
  if (state == GS_DONE) return;
  const double* LUa = at<const double>(bases, L.A);
  const int kase = (int)sc[1];
  int iter = (int)sc[2], j = (int)sc[3];
  double est = sc[4];
  for (int i = tid; i < n; i += nt) x[i] = gx[i];
  __syncthreads();
  if (kase == 1) {
    trsv_cta(LUa, L.lda, n, x, tiles, false, false);
    trsv_cta(LUa, L.lda, n, x, tiles, true, false);
  } else {
    trsv_cta(LUa, L.lda, n, x, tiles, true, true);
    trsv_cta(LUa, L.lda, n, x, tiles, false, true);
  }
  int next_kase = 1;
  auto set_alt = [&]() {
    for (int i = tid; i < n; i += nt) {
      const double sg = (i % 2 == 0) ? 1.0 : -1.0;
      x[i] = sg * (1.0 + (double)i / (double)(n - 1));
    }
    next_kase = 1;
    state = GS_E;
  };
  auto set_unit = [&](int jj) {
    for (int i = tid; i < n; i += nt) x[i] = (i == jj) ? 1.0 : 0.0;
    next_kase = 1;
    state = GS_C;
  };
  if (state == GS_A) {
    if (n == 1) {
      est = fabs(x[0]);
      state = GS_DONE;
    } else {
      est = block_asum(x, n, red_v);
      for (int i = tid; i < n; i += nt) {
        x[i] = x[i] >= 0.0 ? 1.0 : -1.0;
        gsgn[i] = x[i];
      }
      next_kase = 2;
      state = GS_B;
    }
  } else if (state == GS_B) {
    j = block_iamax(x, n, red_v, red_i);
    iter = 2;
    __syncthreads();
    set_unit(j);
  } else if (state == GS_C) {
    const double estold = est;
    est = block_asum(x, n, red_v);
    if (tid == 0) s_diff = 0;
    __syncthreads();
    for (int i = tid; i < n; i += nt) {
      const double xs = x[i] >= 0.0 ? 1.0 : -1.0;
      if (xs != gsgn[i]) s_diff = 1;
    }
    __syncthreads();
    const int diff = s_diff;
    __syncthreads();
    if (!diff || est <= estold) {
      set_alt();
    } else {
      for (int i = tid; i < n; i += nt) {
        x[i] = x[i] >= 0.0 ? 1.0 : -1.0;
        gsgn[i] = x[i];
      }
      next_kase = 2;
      state = GS_D;
    }
  } else if (state == GS_D) {
    const int jlast = j;
    j = block_iamax(x, n, red_v, red_i);
    __syncthreads();
    if (x[jlast] != fabs(x[j]) && iter < 5) {
      ++iter;
      __syncthreads();
      set_unit(j);
    } else {
      __syncthreads();
      set_alt();
    }
  } else {
    const double temp = 2.0 * (block_asum(x, n, red_v) / (double)(3 * n));
    if (temp > est) est = temp;
    state = GS_DONE;
  }
  __syncthreads();
  if (state == GS_DONE) {
    if (tid == 0) {
      const double anorm = *at<const double>(bases, L.anorm);
      *rcond = est != 0.0 ? (1.0 / est) / anorm : 0.0;
    }
  } else {
    for (int i = tid; i < n; i += nt) gx[i] = x[i];
  }
  if (tid == 0) {
    sc[0] = state;
    sc[1] = next_kase;
    sc[2] = iter;
    sc[3] = j;
    sc[4] = est;
  }
}

__global__ void __launch_bounds__(GC_THREADS, 4) gecon_cta_kernel(const Bases* __restrict__ bases_ptr,
                                                                  const LuDesc* __restrict__ descs, int count,
                                                                  int stride, int phase, int xs) {
  extern __shared__ double gcsm[];
  double* x = gcsm;
  double* tiles = gcsm + xs;
  for (int m = blockIdx.x; m < count; m += gridDim.x) {
    gecon_cta_one(*bases_ptr, descs[m], m, stride, phase, x, tiles);
    __syncthreads();
  }
}

// One phase of the estimates of `count` matrices; a CTA walks matrices
// blockIdx.x, + gridDim.x, ...  A grid smaller than the batch leaves SMs
// with no estimate CTA at all, where the factorization's register-heavy
// kernels (the panels) can start at once.
__global__ void __launch_bounds__(GECON_THREADS, 2) gecon_step_kernel(const Bases* __restrict__ bases_ptr,
                                                          const LuDesc* __restrict__ descs, int count,
                                                          int stride, int phase) {
  for (int m = blockIdx.x; m < count; m += gridDim.x) {
    gecon_step_one(*bases_ptr, descs[m], m, stride, phase);
    __syncthreads();  // the next matrix reuses the shared vector
  }
}

}  // namespace

cudaError_t launch_getrf_batched(const Bases* b, const LuDesc* d, int count, int max_n, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int ldp = max_n > 0 ? max_n : 1;
  if (max_n <= 640) {
    const size_t sm = (size_t)ldp * 32 * sizeof(double);
    raise_smem_limit(getrf_kernel<32>, sm);
    getrf_kernel<32><<<count, LU_THREADS, sm, s>>>(b, d, ldp);
  } else if (max_n <= 1280) {
    const size_t sm = (size_t)ldp * 16 * sizeof(double);
    raise_smem_limit(getrf_kernel<16>, sm);
    getrf_kernel<16><<<count, LU_THREADS, sm, s>>>(b, d, ldp);
  } else {
    const size_t sm = (size_t)ldp * 8 * sizeof(double);
    if (sm > 200 * 1024) return cudaErrorInvalidValue;
    raise_smem_limit(getrf_kernel<8>, sm);
    getrf_kernel<8><<<count, LU_THREADS, sm, s>>>(b, d, ldp);
  }
  return cudaGetLastError();
}

cudaError_t launch_getrs_batched(const Bases* b, const LuSolveDesc* d, int count, int max_n, int max_nrhs,
                                 cudaStream_t s) {
  if (count <= 0 || max_n <= 0 || max_nrhs <= 0) return cudaSuccess;
  const int ldx = ((max_n + 15) / 16) * 16 + 4;
  if (max_n <= 640) {
    constexpr int RC = 32;
    const size_t sm = (size_t)ldx * RC * sizeof(double) + (size_t)max_n * sizeof(int);
    raise_smem_limit(getrs_kernel<RC>, sm);
    dim3 grid(count, (max_nrhs + RC - 1) / RC);
    getrs_kernel<RC><<<grid, RS_THREADS, sm, s>>>(b, d, ldx);
  } else {
    constexpr int RC = 16;
    const size_t sm = (size_t)ldx * RC * sizeof(double) + (size_t)max_n * sizeof(int);
    if (sm > 220 * 1024) return cudaErrorInvalidValue;
    raise_smem_limit(getrs_kernel<RC>, sm);
    dim3 grid(count, (max_nrhs + RC - 1) / RC);
    getrs_kernel<RC><<<grid, RS_THREADS, sm, s>>>(b, d, ldx);
  }
  return cudaGetLastError();
}

cudaError_t launch_gecon_batched(const Bases* b, const LuDesc* d, int count, int max_n, cudaStream_t s, int phase) {
  if (count <= 0) return cudaSuccess;
  static const int form = [] {  // 1: warp per matrix (default); 0: 128-thread CTA per matrix; 2: 256-thread CTA
    const char* e = getenv("HKS_GECON_FORM");
    return e ? atoi(e) : 1;
  }();
  if (phase >= 0 && form == 0) {
    const int xs = ((max_n > 0 ? max_n : 1) + 1) / 2 * 2;
    const size_t sm = (size_t)(xs + GC_WARPS * 32 * 33) * sizeof(double);
    raise_smem_limit(gecon_cta_kernel, sm);
    gecon_cta_kernel<<<count, GC_THREADS, sm, s>>>(b, d, count, gecon_stride(max_n), phase, xs);
    return cudaGetLastError();
  }
  if (phase >= 0 && form == 1) {  // one warp per matrix, all matrices in one wave where they fit
    const int xs = ((max_n > 0 ? max_n : 1) + 1) / 2 * 2;
    const size_t sm = (size_t)GW_WARPS * (xs + GW_TILE) * sizeof(double);
    raise_smem_limit(gecon_warp_kernel, sm);
    const int grid = (count + GW_WARPS - 1) / GW_WARPS;
    gecon_warp_kernel<<<grid, 32 * GW_WARPS, sm, s>>>(b, d, count, gecon_stride(max_n), phase, xs);
    return cudaGetLastError();
  }
  if (phase >= 0) {  // split estimate: phase 0 initialises, 1..kGeconSteps apply + advance
    const size_t sm = (size_t)(max_n > 0 ? max_n : 1) * sizeof(double);
    raise_smem_limit(gecon_step_kernel, sm);
    // CTAs per estimate launch: batches up to 4 waves of SMs are walked by
    // at most 112 CTAs, leaving SMs free for the factorization's panels
    // (plan.cu cond_start_level); larger batches get one CTA per matrix so
    // the chain does not outlast the factorization.  HKS_GECON_GRID: the cap
    // (0 = one CTA per matrix).
    static const int cap = [] {
      const char* e = getenv("HKS_GECON_GRID");
      return e ? atoi(e) : 112;
    }();
    const int grid = cap > 0 && count > cap && count <= 4 * 148 ? cap : count;
    gecon_step_kernel<<<grid, GECON_THREADS, sm, s>>>(b, d, count, gecon_stride(max_n), phase);
    return cudaGetLastError();
  }
  const size_t sm = (size_t)(max_n > 0 ? max_n : 1) * (2 * sizeof(double) + sizeof(int));
  raise_smem_limit(gecon_kernel, sm);
  gecon_kernel<<<count, GECON_THREADS, sm, s>>>(b, d);  // a light co-tenant of the factorization
  return cudaGetLastError();
}

}  // namespace hks
