// Kernel-block evaluation and fused kernel summation (FP64, sm_100a).
//
// eval_block (kernels.py:64-105) as a batched tile kernel: squared distances
// in the diff form sum_k (x_k - y_k)^2 accumulated in index order, so
// K(X, Y) == K(Y, X)^T bit for bit and K(x, x) == 1 exactly
// (tests/test_kernels.py:7-9, 69-81); gaussian exp(sq / (-2 h^2)) with a
// true division (kernels.py:95); laplace 1/(4 pi r), r == 0 -> 0
// (kernels.py:96-101); polynomial (x.y + c)^p (kernels.py:102-104).
//
// ksum: U = K(X_rows, X_cols) W (+ lam W) without ever writing K to memory
// -- each 64x64 kernel tile is built in shared memory and consumed at once
// (hmatvec's leaf level, treecode.py:99-101; sampled residual checks).
#include <cstdlib>

#include "common.cuh"
#include "hks_internal.h"

namespace hks {

KernelParams make_kernel_params(const hks_kernel* k) {
  KernelParams p;
  p.family = k->family;
  p.h = k->h;
  p.neg2h2 = -2.0 * (k->h * k->h);
  p.degree = k->degree;
  p.shift = k->shift;
  return p;
}

namespace {

constexpr int TM = 64, TN = 64, DC = 32, XS = DC + 1;

__device__ __forceinline__ double kernel_value(const KernelParams& kp, double acc) {
  if (kp.family == HKS_GAUSSIAN) return exp(acc / kp.neg2h2);
  if (kp.family == HKS_LAPLACE3D) return acc == 0.0 ? 0.0 : 1.0 / ((4.0 * 3.141592653589793) * sqrt(acc));
  const double t = acc + kp.shift;
  if (kp.degree == 1) return t;
  if (kp.degree == 2) return t * t;
  return pow(t, (double)kp.degree);
}

__device__ __forceinline__ int64_t row_id(const int64_t* ids, int64_t base, int i) {
  return ids ? ids[i] : base + i;
}

// 4 x 4 register block of pair terms: rows rb + 16u, columns cb + 16v of the
// staged tiles (u, v < 4), accumulated over k in order with (x_row - x_col)
// -- the diff-form distance of kernels.py:56-61 per pair, 8 shared-memory
// loads per 16 pairs.
template <bool POLY>
__device__ __forceinline__ void accumulate4x4(const double* Xr, const double* Xc, int xs, int dc, int rb, int cb,
                                              double (&acc)[4][4]) {
  for (int k = 0; k < dc; ++k) {
    double a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = Xr[(rb + 16 * u) * xs + k];
#pragma unroll
    for (int v = 0; v < 4; ++v) b[v] = Xc[(cb + 16 * v) * xs + k];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        if (POLY) {
          acc[u][v] = fma(a[u], b[v], acc[u][v]);
        } else {
          const double df = a[u] - b[v];
          acc[u][v] = fma(df, df, acc[u][v]);
        }
      }
  }
}

// Stage rows [r0, r0+TM) of the row set and [c0, c0+TN) of the column set
// for dims [k0, k0+dc) into shared memory.
__device__ __forceinline__ void stage(const double* X, const double* XC, int d, const int64_t* rows, int64_t row0,
                                      int m, int r0, const int64_t* cols, int64_t col0, int n,
                                      int c0, int k0, int dc, double* Xr, double* Xc) {
  // one point per warp iteration, lanes over its (contiguous) coordinates
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = wid; i < TM; i += nw) {
    const bool ok = r0 + i < m;
    const double* src = ok ? X + row_id(rows, row0, r0 + i) * d + k0 : X;
    for (int k = lane; k < dc; k += 32) Xr[i * XS + k] = ok ? src[k] : 0.0;
  }
  for (int j = wid; j < TN; j += nw) {
    const bool ok = c0 + j < n;
    const double* src = ok ? XC + row_id(cols, col0, c0 + j) * d + k0 : XC;
    for (int k = lane; k < dc; k += 32) Xc[j * XS + k] = ok ? src[k] : 0.0;
  }
}

template <bool ROW_MAJOR>
__global__ void __launch_bounds__(256) eval_kernel(const double* __restrict__ X, int d, KernelParams kp,
                                                   const Bases* __restrict__ bases_ptr,
                                                   const EvalDesc* __restrict__ descs, int tiles_n) {
  const Bases& bases = *bases_ptr;
  const EvalDesc e = descs[blockIdx.y];
  const int64_t* erows = e.rows == kNull ? nullptr : at<const int64_t>(bases, e.rows);
  const int64_t* ecols = e.cols == kNull ? nullptr : at<const int64_t>(bases, e.cols);
  double* eout = at<double>(bases, e.out);
  const double ediag = e.diag ? bases.lam : 0.0;
  const int r0 = (blockIdx.x / tiles_n) * TM, c0 = (blockIdx.x % tiles_n) * TN;
  if (r0 >= e.m || c0 >= e.n) return;
  // K(X_a, X_a): the diff-form distance makes the block exactly symmetric,
  // so only tiles on / above the diagonal are computed; each off-diagonal
  // tile also writes its transpose (column-major output only).
  const bool sym = !ROW_MAJOR && e.rows == kNull && e.cols == kNull && e.row0 == e.col0 && e.m == e.n;
  if (sym && r0 > c0) return;
  __shared__ double stage_area[(TM + TN) * XS];
  double* Xr = stage_area;
  double* Xc = stage_area + TM * XS;
  const int t = threadIdx.x;
  // 4 x 4 pairs per thread: rows rb + 16u, columns cb + 16v.  The lanes of a
  // warp run along the stored index (rows for column-major output, columns
  // for row-major), so every store of a (u, v) is one coalesced segment.
  const int rb = ROW_MAJOR ? (t >> 4) : (t & 15), cb = ROW_MAJOR ? (t & 15) : (t >> 4);
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  const bool poly = kp.family == HKS_POLYNOMIAL;
  for (int k0 = 0; k0 < d; k0 += DC) {
    const int dc = min(DC, d - k0);
    stage(X, X, d, erows, e.row0, e.m, r0, ecols, e.col0, e.n, c0, k0, dc, Xr, Xc);
    __syncthreads();
    if (poly)
      accumulate4x4<true>(Xr, Xc, XS, dc, rb, cb, acc);
    else
      accumulate4x4<false>(Xr, Xc, XS, dc, rb, cb, acc);
    __syncthreads();
  }
  const bool mirror = sym && r0 != c0;
  double* Kt = stage_area;  // 64 x 65 tile for the mirrored store (the staging area is free now)
  static_assert(TM * (TN + 1) <= (TM + TN) * XS, "tile must fit the staging area");
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int ii = rb + 16 * u, jj = cb + 16 * v;
      const int i = r0 + ii, j = c0 + jj;
      double val = 0.0;
      if (i < e.m && j < e.n) {
        val = kernel_value(kp, acc[u][v]);
        if (i == j) val += ediag;
        if (ROW_MAJOR)
          eout[(size_t)i * e.ldo + j] = val;
        else
          eout[i + (size_t)j * e.ldo] = val;
      }
      if (mirror) Kt[jj * (TM + 1) + ii] = val;  // Kt[jj][ii]
    }
  if (mirror) {  // K[c0 + jj, r0 + ii] = K[r0 + ii, c0 + jj], stored coalesced along jj
    __syncthreads();
    for (int ii = t >> 6; ii < TM; ii += 4) {
      const int jj = t & 63;
      if (r0 + ii < e.m && c0 + jj < e.n) eout[(c0 + jj) + (size_t)(r0 + ii) * e.ldo] = Kt[jj * (TM + 1) + ii];
    }
  }
}

constexpr int KC = 16;  // right-hand sides per pass

// XC: the column points (X itself except in cross sums, hks_cross_sum).
__global__ void __launch_bounds__(256, 3) ksum_kernel(const double* __restrict__ X, const double* __restrict__ XC,
                                                   int d, KernelParams kp,
                                                   const Bases* __restrict__ bases_ptr,
                                                   const SumDesc* __restrict__ descs) {
  const Bases& bases = *bases_ptr;
  const SumDesc s = descs[blockIdx.y];
  const int64_t* srows = s.rows == kNull ? nullptr : at<const int64_t>(bases, s.rows);
  const int64_t* scols = s.cols == kNull ? nullptr : at<const int64_t>(bases, s.cols);
  const double* sW = at<const double>(bases, s.W);
  double* sU = at<double>(bases, s.U);
  const double sdiag = s.diag ? bases.lam : 0.0;
  const int r0 = blockIdx.x * TM;
  if (r0 >= s.m) return;
  // Kt (the 64x64 kernel tile) reuses the staging area once the d-loop is done
  __shared__ double stage_area[(TM + TN) * XS];
  __shared__ double Ws[TN * KC];
  double* Xr = stage_area;
  double* Xc = stage_area + TM * XS;
  double* Kt = stage_area;
  static_assert(TM * (TN + 1) <= (TM + TN) * XS, "kernel tile must fit the staging area");
  const int t = threadIdx.x;
  const int own = t & 63;  // row of the K W product
  const int kq = (t >> 6) * 4;  // 4 right-hand sides per thread in the product
  const bool poly = kp.family == HKS_POLYNOMIAL;
  for (int kb = 0; kb < s.k; kb += KC) {
    const int kc = min(KC, s.k - kb);
    double out[4] = {0.0, 0.0, 0.0, 0.0};
    for (int c0 = 0; c0 < s.n; c0 += TN) {
      double acc[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
      const int rb = t & 15, cb = t >> 4;
      for (int k0 = 0; k0 < d; k0 += DC) {
        const int dc = min(DC, d - k0);
        stage(X, XC, d, srows, s.row0, s.m, r0, scols, s.col0, s.n, c0, k0, dc, Xr, Xc);
        __syncthreads();
        if (poly)
          accumulate4x4<true>(Xr, Xc, XS, dc, rb, cb, acc);
        else
          accumulate4x4<false>(Xr, Xc, XS, dc, rb, cb, acc);
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int ii = rb + 16 * u, jj = cb + 16 * v;
          Kt[ii * (TN + 1) + jj] = (r0 + ii < s.m && c0 + jj < s.n) ? kernel_value(kp, acc[u][v]) : 0.0;
        }
      for (int e2 = t; e2 < TN * KC; e2 += blockDim.x) {
        const int j = e2 / KC, c = e2 % KC;
        Ws[e2] = (c0 + j < s.n && c < kc) ? sW[(c0 + j) + (size_t)(kb + c) * s.ldw] : 0.0;
      }
      __syncthreads();
      for (int j = 0; j < TN; ++j) {
        const double kv = Kt[own * (TN + 1) + j];
#pragma unroll
        for (int q = 0; q < 4; ++q) out[q] = fma(kv, Ws[j * KC + kq + q], out[q]);
      }
      __syncthreads();
    }
    const int i = r0 + own;
    if (i < s.m) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = kq + q;
        if (c >= kc) continue;
        double* u = sU + i + (size_t)(kb + c) * s.ldu;
        double v = out[q];
        if (s.diag) v += sdiag * sW[i + (size_t)(kb + c) * s.ldw];
        if (s.beta != 0.0) v += s.beta * *u;
        *u = v;
      }
    }
  }
}


// ---------------------------------------------------------------------------
// GEMM-form distances on the FP64 tensor path (d >= kMmaMinDim): the 64 x 64
// dot-product tile X_r X_c^T is a DMMA.884 GEMM over d (4 warps of 32 x 32
// fragments, 16-deep k-slabs staged by cp.async in a 3-stage pipeline, as
// gemm.cu), the squared norms come from the same staged slabs (sequential
// FMA over k), and d^2 = (|x|^2 + |y|^2) - 2 x.y.  The epilogue applies the
// kernel through a shared tile.  Properties kept from the diff form: K(X, Y)
// == K(Y, X)^T bit for bit (the DMMA's per-element k order and the norm
// sums do not depend on which operand is which), K(x, x) == 1 exactly (a
// point against itself gets d^2 = 0), d^2 >= 0.  The values differ from
// the diff form by roundoff of size eps (|x|^2 + |y|^2) in d^2.
constexpr int kMmaMinDim = 64;
constexpr int MBK = 16, MKS = MBK + 4, MST = 3;  // slab depth, smem row stride, pipeline stages
constexpr int MT = 64;                            // tile rows = tile columns
constexpr size_t kMmaStageBytes = (size_t)MST * 2 * MT * MKS * sizeof(double);

struct PointRows {
  const double* X;
  const int64_t* ids;  // nullptr: base + i
  int64_t base;
  int count;           // valid rows
  __device__ __forceinline__ const double* row(int i, int d) const {
    return X + (ids ? ids[i] : base + i) * (int64_t)d;
  }
};

// Stage k-slab [k0, k0 + 16) of 64 rows (from r0) and 64 columns (from c0):
// 16 consecutive threads per point row (128-byte coalesced segments).
__device__ __forceinline__ void mma_stage(const PointRows& R, int r0, const PointRows& C, int c0, int d, int k0,
                                          double* As, double* Bs) {
  const int t = threadIdx.x, kk = t & 15, i0 = t >> 4;
  const int k = k0 + kk;
#pragma unroll
  for (int j = 0; j < MT / 8; ++j) {
    const int i = i0 + 8 * j;
    const bool okr = r0 + i < R.count && k < d;
    cp_async8(As + i * MKS + kk, okr ? R.row(r0 + i, d) + k : R.X, okr);
    const bool okc = c0 + i < C.count && k < d;
    cp_async8(Bs + i * MKS + kk, okc ? C.row(c0 + i, d) + k : C.X, okc);
  }
}

// acc (this warp's 32 x 32 block of the 64 x 64 tile) = X_r X_c^T over all
// d; nr / nc (shared, 64 each) receive the squared norms of the tile's rows
// (when want_rows) and columns.  Ends with every thread past a barrier.
__device__ __forceinline__ void mma_dot_tile(const PointRows& R, int r0, const PointRows& C, int c0, int d,
                                             double* stage_smem, bool want_rows, double* nr, double* nc,
                                             double (&acc)[4][4][2]) {
  double* As = stage_smem;
  double* Bs = stage_smem + MST * MT * MKS;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int wm = (wid >> 1) * 32, wn = (wid & 1) * 32, fr = lane >> 2, fc = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double nrm = 0.0;  // threads 0..63: row t; 64..127: column t - 64
  const bool norm_thread = t >= MT || want_rows;
  const int nk = (d + MBK - 1) / MBK;
#pragma unroll
  for (int st = 0; st < MST - 1; ++st) {
    if (st < nk) mma_stage(R, r0, C, c0, d, st * MBK, As + st * MT * MKS, Bs + st * MT * MKS);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<MST - 2>();
    __syncthreads();
    const int pf = kt + MST - 1;
    if (pf < nk) mma_stage(R, r0, C, c0, d, pf * MBK, As + (pf % MST) * MT * MKS, Bs + (pf % MST) * MT * MKS);
    cp_async_commit();
    const double* as = As + (kt % MST) * MT * MKS;
    const double* bs = Bs + (kt % MST) * MT * MKS;
#pragma unroll
    for (int kk = 0; kk < MBK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = as[(wm + i * 8 + fr) * MKS + kk + fc];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[(wn + j * 8 + fr) * MKS + kk + fc];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    if (norm_thread) {  // squared norm in k order (zero-filled tail adds nothing)
      const double* v = t < MT ? as + t * MKS : bs + (t - MT) * MKS;
#pragma unroll
      for (int kk = 0; kk < MBK; ++kk) nrm = fma(v[kk], v[kk], nrm);
    }
  }
  cp_async_wait<0>();
  if (t < MT) {
    if (want_rows) nr[t] = nrm;
  } else {
    nc[t - MT] = nrm;
  }
  __syncthreads();  // norms visible; the staging area is free
}

__device__ __forceinline__ double mma_kernel_value(const KernelParams& kp, double dot, double sq) {
  if (kp.family == HKS_POLYNOMIAL) {
    const double t = dot + kp.shift;
    if (kp.degree == 1) return t;
    if (kp.degree == 2) return t * t;
    return pow(t, (double)kp.degree);
  }
  return kernel_value(kp, sq);
}

// Writes this warp's fragment of kernel values into Kt (64 x 65, Kt[ii][jj]).
// same_points: rows and columns index the same point array, so equal ids
// are the same point (d^2 = 0).
__device__ __forceinline__ void mma_values_to_smem(const KernelParams& kp, const double (&acc)[4][4][2],
                                                   const double* nr, const double* nc, const PointRows& R, int r0,
                                                   const PointRows& C, int c0, bool same_points, double* Kt) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int wm = (wid >> 1) * 32, wn = (wid & 1) * 32, fr = lane >> 2, fc = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ii = wm + i * 8 + fr, jj = wn + j * 8 + 2 * fc + h;
        double v = 0.0;
        if (r0 + ii < R.count && c0 + jj < C.count) {
          const double dot = acc[i][j][h];
          double sq = fmax((nr[ii] + nc[jj]) - 2.0 * dot, 0.0);
          if (same_points) {
            const int64_t gi = R.ids ? R.ids[r0 + ii] : R.base + r0 + ii;
            const int64_t gj = C.ids ? C.ids[c0 + jj] : C.base + c0 + jj;
            if (gi == gj) sq = 0.0;
          }
          v = mma_kernel_value(kp, dot, sq);
        }
        Kt[ii * (MT + 1) + jj] = v;
      }
}

template <bool ROW_MAJOR>
__global__ void __launch_bounds__(128) eval_mma_kernel(const double* __restrict__ X, int d, KernelParams kp,
                                                       const Bases* __restrict__ bases_ptr,
                                                       const EvalDesc* __restrict__ descs, int tiles_n) {
  const Bases& bases = *bases_ptr;
  const EvalDesc e = descs[blockIdx.y];
  const int r0 = (blockIdx.x / tiles_n) * MT, c0 = (blockIdx.x % tiles_n) * MT;
  if (r0 >= e.m || c0 >= e.n) return;
  const bool sym = !ROW_MAJOR && e.rows == kNull && e.cols == kNull && e.row0 == e.col0 && e.m == e.n;
  if (sym && r0 > c0) return;
  extern __shared__ double msm[];
  __shared__ double nr[MT], nc[MT];
  const PointRows R{X, e.rows == kNull ? nullptr : at<const int64_t>(bases, e.rows), e.row0, e.m};
  const PointRows C{X, e.cols == kNull ? nullptr : at<const int64_t>(bases, e.cols), e.col0, e.n};
  double acc[4][4][2];
  mma_dot_tile(R, r0, C, c0, d, msm, true, nr, nc, acc);
  double* Kt = msm;  // 64 x 65 value tile in the (free) staging area
  mma_values_to_smem(kp, acc, nr, nc, R, r0, C, c0, true, Kt);
  __syncthreads();
  double* eout = at<double>(bases, e.out);
  const double ediag = e.diag ? bases.lam : 0.0;
  const int t = threadIdx.x;
  // coalesced stores: lanes along the stored index
  for (int q = t; q < MT * MT; q += 128) {
    const int a = q & 63, b2 = q >> 6;  // a: fast index
    const int ii = ROW_MAJOR ? b2 : a, jj = ROW_MAJOR ? a : b2;
    const int i = r0 + ii, j = c0 + jj;
    if (i >= e.m || j >= e.n) continue;
    double v = Kt[ii * (MT + 1) + jj];
    if (i == j) v += ediag;
    if (ROW_MAJOR)
      eout[(size_t)i * e.ldo + j] = v;
    else
      eout[i + (size_t)j * e.ldo] = v;
  }
  if (sym && r0 != c0) {  // mirrored tile K[c0 + jj, r0 + ii], coalesced along jj
    for (int q = t; q < MT * MT; q += 128) {
      const int jj = q & 63, ii = q >> 6;
      const int i = r0 + ii, j = c0 + jj;
      if (i < e.m && j < e.n) eout[j + (size_t)i * e.ldo] = Kt[ii * (MT + 1) + jj];
    }
  }
}

constexpr int MKC = 16;  // right-hand sides per pass

__global__ void __launch_bounds__(128, 3) ksum_mma_kernel(const double* __restrict__ X, const double* __restrict__ XC,
                                                       int d, KernelParams kp, const Bases* __restrict__ bases_ptr,
                                                       const SumDesc* __restrict__ descs) {
  const Bases& bases = *bases_ptr;
  const SumDesc s = descs[blockIdx.y];
  const int r0 = blockIdx.x * MT;
  if (r0 >= s.m) return;
  extern __shared__ double msm[];
  __shared__ double nr[MT], nc[MT];
  __shared__ double Ws[MT * MKC];
  const PointRows R{X, s.rows == kNull ? nullptr : at<const int64_t>(bases, s.rows), s.row0, s.m};
  const PointRows C{XC, s.cols == kNull ? nullptr : at<const int64_t>(bases, s.cols), s.col0, s.n};
  const bool same = X == XC;
  const double* sW = at<const double>(bases, s.W);
  double* sU = at<double>(bases, s.U);
  double* Kt = msm;
  const int t = threadIdx.x, own = t & 63, kq = (t >> 6) * (MKC / 2);
  for (int kb = 0; kb < s.k; kb += MKC) {
    const int kc = min(MKC, s.k - kb);
    double out[MKC / 2];
#pragma unroll
    for (int q = 0; q < MKC / 2; ++q) out[q] = 0.0;
    for (int c0 = 0; c0 < s.n; c0 += MT) {
      double acc[4][4][2];
      mma_dot_tile(R, r0, C, c0, d, msm, c0 == 0, nr, nc, acc);
      mma_values_to_smem(kp, acc, nr, nc, R, r0, C, c0, same, Kt);
      for (int e2 = t; e2 < MT * MKC; e2 += 128) {
        const int j = e2 / MKC, c = e2 % MKC;
        Ws[e2] = (c0 + j < s.n && c < kc) ? sW[(c0 + j) + (size_t)(kb + c) * s.ldw] : 0.0;
      }
      __syncthreads();
      for (int j = 0; j < MT; ++j) {  // columns in order: the same sum order as the diff-form kernel
        const double kv = Kt[own * (MT + 1) + j];
#pragma unroll
        for (int q = 0; q < MKC / 2; ++q) out[q] = fma(kv, Ws[j * MKC + kq + q], out[q]);
      }
      __syncthreads();  // Kt / Ws reused by the next tile
    }
    const int i = r0 + own;
    if (i < s.m) {
#pragma unroll
      for (int q = 0; q < MKC / 2; ++q) {
        const int c = kq + q;
        if (c >= kc) continue;
        double* u = sU + i + (size_t)(kb + c) * s.ldu;
        double v = out[q];
        if (s.diag) v += bases.lam * sW[i + (size_t)(kb + c) * s.ldw];
        if (s.beta != 0.0) v += s.beta * *u;
        *u = v;
      }
    }
  }
}

}  // namespace

cudaError_t launch_eval_batched(const double* X, int d, KernelParams kp, const Bases* bases,
                                const EvalDesc* d_descs, int count, int max_m, int max_n, bool row_major,
                                      cudaStream_t stream) {
  if (count <= 0 || max_m <= 0 || max_n <= 0) return cudaSuccess;
  const int tm = (max_m + TM - 1) / TM, tn = (max_n + TN - 1) / TN;
  if (d >= kMmaMinDim && getenv("HKS_DIFF_FORM") == nullptr) {  // tensor-path distances
    static_assert(MT == TM && MT == TN, "tile shapes");
    if (row_major) raise_smem_limit(eval_mma_kernel<true>, kMmaStageBytes);
    else raise_smem_limit(eval_mma_kernel<false>, kMmaStageBytes);
    for (int first = 0; first < count; first += 65535) {
      const int cnt = count - first < 65535 ? count - first : 65535;
      dim3 grid(tm * tn, cnt);
      if (row_major)
        eval_mma_kernel<true><<<grid, 128, kMmaStageBytes, stream>>>(X, d, kp, bases, d_descs + first, tn);
      else
        eval_mma_kernel<false><<<grid, 128, kMmaStageBytes, stream>>>(X, d, kp, bases, d_descs + first, tn);
    }
    return cudaGetLastError();
  }
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    dim3 grid(tm * tn, cnt);
    if (row_major)
      eval_kernel<true><<<grid, 256, 0, stream>>>(X, d, kp, bases, d_descs + first, tn);
    else
      eval_kernel<false><<<grid, 256, 0, stream>>>(X, d, kp, bases, d_descs + first, tn);
  }
  return cudaGetLastError();
}

cudaError_t launch_ksum_batched(const double* X, int d, KernelParams kp, const Bases* bases,
                                const SumDesc* d_descs, int count, int max_m, cudaStream_t stream, const double* XC) {
  if (count <= 0 || max_m <= 0) return cudaSuccess;
  if (d >= kMmaMinDim && getenv("HKS_DIFF_FORM") == nullptr) {  // tensor-path distances
    raise_smem_limit(ksum_mma_kernel, kMmaStageBytes);
    for (int first = 0; first < count; first += 65535) {
      const int cnt = count - first < 65535 ? count - first : 65535;
      ksum_mma_kernel<<<dim3((max_m + MT - 1) / MT, cnt), 128, kMmaStageBytes, stream>>>(X, XC ? XC : X, d, kp,
                                                                                      bases, d_descs + first);
    }
    return cudaGetLastError();
  }
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    dim3 grid((max_m + TM - 1) / TM, cnt);
    ksum_kernel<<<grid, 256, 0, stream>>>(X, XC ? XC : X, d, kp, bases, d_descs + first);
  }
  return cudaGetLastError();
}

}  // namespace hks
