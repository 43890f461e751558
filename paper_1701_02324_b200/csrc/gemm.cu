// Batched ragged FP64 GEMM on the DMMA tensor path (mma.sync m8n8k4 f64).
//
// One launch runs every GemmDesc of a tree level (or of several independent
// product lists) -- the reference's per-node numpy `@` calls
// (solver.py:136-158, treecode.py:76-127) become one grid whose y index is
// the problem and whose x index is a 64x64 output tile.  Per output element
// the k-reduction order is fixed (k tiles in order, then the DMMA's own
// order) and independent of n, so a column of a multi-RHS product is
// bit-identical to the single-RHS product (solve_multi == solve column-wise,
// tests/test_solver.py:174-185).
#include "common.cuh"
#include "hks_internal.h"

namespace hks {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, KS = BK + 4;  // KS: smem row stride (bank spread)
constexpr int THREADS = 128;

struct GemmOp {
  const double* A;
  const double* B;
  double* C;
  int m, n, k, lda, ldb, ldc, transA, transB;
  double alpha, beta;
};

__device__ __forceinline__ void load_tile_a(const GemmOp& g, int m0, int k0, double (&r)[8]) {
  const int t = threadIdx.x;
  if (!g.transA) {  // A(m,k) = A[m + k*lda], coalesced along m
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int m = m0 + (t & 63), k = k0 + (t >> 6) + 2 * j;
      r[j] = (m < g.m && k < g.k) ? __ldg(g.A + m + (size_t)k * g.lda) : 0.0;
    }
  } else {  // A(m,k) = A[k + m*lda], coalesced along k
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int k = k0 + (t & 15), m = m0 + (t >> 4) + 8 * j;
      r[j] = (m < g.m && k < g.k) ? __ldg(g.A + k + (size_t)m * g.lda) : 0.0;
    }
  }
}

__device__ __forceinline__ void store_tile_a(const GemmOp& g, double* As, const double (&r)[8]) {
  const int t = threadIdx.x;
  if (!g.transA) {
#pragma unroll
    for (int j = 0; j < 8; ++j) As[(t & 63) * KS + (t >> 6) + 2 * j] = r[j];
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) As[((t >> 4) + 8 * j) * KS + (t & 15)] = r[j];
  }
}

__device__ __forceinline__ void load_tile_b(const GemmOp& g, int n0, int k0, double (&r)[8]) {
  const int t = threadIdx.x;
  if (!g.transB) {  // B(k,n) = B[k + n*ldb], coalesced along k
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int k = k0 + (t & 15), n = n0 + (t >> 4) + 8 * j;
      r[j] = (n < g.n && k < g.k) ? __ldg(g.B + k + (size_t)n * g.ldb) : 0.0;
    }
  } else {  // B(k,n) = B[n + k*ldb], coalesced along n
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int n = n0 + (t & 63), k = k0 + (t >> 6) + 2 * j;
      r[j] = (n < g.n && k < g.k) ? __ldg(g.B + n + (size_t)k * g.ldb) : 0.0;
    }
  }
}

__device__ __forceinline__ void store_tile_b(const GemmOp& g, double* Bs, const double (&r)[8]) {
  const int t = threadIdx.x;
  if (!g.transB) {
#pragma unroll
    for (int j = 0; j < 8; ++j) Bs[((t >> 4) + 8 * j) * KS + (t & 15)] = r[j];
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) Bs[(t & 63) * KS + (t >> 6) + 2 * j] = r[j];
  }
}

__global__ void __launch_bounds__(THREADS) gemm_batched_kernel(const Bases bases,
                                                                const GemmDesc* __restrict__ descs,
                                                                int tiles_n) {
  const GemmDesc gd = descs[blockIdx.y];
  const GemmOp g{at<const double>(bases, gd.A), at<const double>(bases, gd.B), at<double>(bases, gd.C),
                 gd.m, gd.n, gd.k, gd.lda, gd.ldb, gd.ldc, gd.transA, gd.transB, gd.alpha, gd.beta};
  const int m0 = (blockIdx.x / tiles_n) * BM, n0 = (blockIdx.x % tiles_n) * BN;
  if (m0 >= g.m || n0 >= g.n) return;

  __shared__ double As[BM * KS];
  __shared__ double Bs[BN * KS];

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wm = (wid >> 1) * 32, wn = (wid & 1) * 32;
  const int fr = lane >> 2, fc = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[8], rb[8];
  if (g.k > 0) {
    load_tile_a(g, m0, 0, ra);
    load_tile_b(g, n0, 0, rb);
  }
  for (int k0 = 0; k0 < g.k; k0 += BK) {
    store_tile_a(g, As, ra);
    store_tile_b(g, Bs, rb);
    __syncthreads();
    if (k0 + BK < g.k) {
      load_tile_a(g, m0, k0 + BK, ra);
      load_tile_b(g, n0, k0 + BK, rb);
    }
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[(wm + i * 8 + fr) * KS + kk + fc];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[(wn + j * 8 + fr) * KS + kk + fc];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }

  const double alpha = g.alpha, beta = g.beta;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + fr;
    if (r >= g.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = n0 + wn + j * 8 + 2 * fc + h;
        if (c >= g.n) continue;
        double* p = g.C + r + (size_t)c * g.ldc;
        double v = alpha * acc[i][j][h];
        if (beta != 0.0) v += beta * *p;
        *p = v;
      }
    }
  }
}

// dst = alpha * op(src) / alpha * I / 0, one descriptor per block row-set.
__global__ void copy_batched_kernel(const Bases bases, const CopyDesc* __restrict__ descs) {
  const CopyDesc c = descs[blockIdx.y];
  const double* src = c.mode == 0 ? at<const double>(bases, c.src) : nullptr;
  double* dst = at<double>(bases, c.dst);
  const int total = c.m * c.n;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int i = e % c.m, j = e / c.m;
    double v;
    if (c.mode == 0) {
      v = c.trans ? src[j + (size_t)i * c.lds] : src[i + (size_t)j * c.lds];
      v *= c.alpha;
    } else {
      v = (c.mode == 1 && i == j) ? c.alpha : 0.0;
    }
    dst[i + (size_t)j * c.ldd] = v;
  }
}

}  // namespace

cudaError_t launch_gemm_batched(const Bases& bases, const GemmDesc* d_descs, int count, int max_m,
                                int max_n, cudaStream_t stream) {
  if (count <= 0 || max_m <= 0 || max_n <= 0) return cudaSuccess;
  const int tm = (max_m + BM - 1) / BM, tn = (max_n + BN - 1) / BN;
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    dim3 grid(tm * tn, cnt);
    gemm_batched_kernel<<<grid, THREADS, 0, stream>>>(bases, d_descs + first, tn);
  }
  return cudaGetLastError();
}

cudaError_t launch_copy_batched(const Bases& bases, const CopyDesc* d_descs, int count, int max_elems,
                                cudaStream_t stream) {
  if (count <= 0 || max_elems <= 0) return cudaSuccess;
  int bx = (max_elems + 255) / 256;
  if (bx > 64) bx = 64;
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    copy_batched_kernel<<<dim3(bx, cnt), 256, 0, stream>>>(bases, d_descs + first);
  }
  return cudaGetLastError();
}

}  // namespace hks
