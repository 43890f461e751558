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

}  // namespace

cudaError_t launch_eval_batched(const double* X, int d, KernelParams kp, const Bases* bases,
                                const EvalDesc* d_descs, int count, int max_m, int max_n, bool row_major,
                                      cudaStream_t stream) {
  if (count <= 0 || max_m <= 0 || max_n <= 0) return cudaSuccess;
  const int tm = (max_m + TM - 1) / TM, tn = (max_n + TN - 1) / TN;
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
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    dim3 grid((max_m + TM - 1) / TM, cnt);
    ksum_kernel<<<grid, 256, 0, stream>>>(X, XC ? XC : X, d, kp, bases, d_descs + first);
  }
  return cudaGetLastError();
}

}  // namespace hks
