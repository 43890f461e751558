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
#include <cstdlib>

#include "common.cuh"
#include "hks_internal.h"

namespace hks {
namespace {

// Output tile TBM x 64 (TBM = 64: 4 warps, TBM = 128: 8 warps), each warp a
// 32 x 32 block of 8x8x4 DMMA fragments.
#ifndef HKS_GEMM_BK
#define HKS_GEMM_BK 16
#endif
#ifndef HKS_GEMM_STAGES
#define HKS_GEMM_STAGES 3
#endif
constexpr int BN = 64, BK = HKS_GEMM_BK, KS = BK + 4;  // KS: smem row stride (bank spread)
constexpr int STAGES = HKS_GEMM_STAGES;  // cp.async pipeline depth

// Shared-memory layout of a staged operand follows its global contiguity,
// so every cp.async warp writes consecutive addresses (no bank conflicts on
// the LDGSTS stores -- the transposing [m][k] store of a column-major A was
// 4-way conflicted, 38% of the shared-memory wavefronts):
//   k-contiguous in global (A^T, B):  [row][k], row stride KS = BK + 4
//   row-contiguous in global (A, B^T): [k][row], row stride R + 4
// Both strides are 4 (mod 16) doubles, so the DMMA fragment loads (8 rows x
// 4 k per warp) hit distinct banks in either layout.
template <int R>
struct OperandLayout {
  static constexpr int RS = R + 4;                                     // [k][row] stride
  static constexpr int kElems = (R * KS > BK * RS) ? R * KS : BK * RS;  // per stage
};

struct GemmOp {
  const double* A;
  const double* B;
  double* C;
  int m, n, k, lda, ldb, ldc, transA, transB;
  double alpha, beta;
};


// Stage the A (TBM x TBK) and B (TBK x 64) tiles of k-block k0 into shared
// memory (layouts above); out-of-range elements are zero-filled.
// One operand tile into shared memory in 16-byte pairs along its contiguous
// dimension: CD x OD elements (contiguous x other), smem [o][c] with row
// stride S, global element (c, o) at base[c + o * ld].  `vec`: the base is
// 16-byte aligned and ld is even, so every in-range pair is one cp.async of
// 16 bytes (half the LDGSTS of 8-byte copies); pairs crossing the edge and
// unaligned operands fall back to two zero-filling 8-byte copies.
template <int CD, int OD, int S, int T>
__device__ __forceinline__ void stage_pairs(double* sm, const double* base, int ld, int c0, int climit, int o0,
                                            int olimit, bool vec) {
  constexpr int PC = CD / 2;
  static_assert((PC * OD) % T == 0, "tile / thread mapping");
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < (PC * OD) / T; ++j) {
    const int e = t + j * T;
    const int c = 2 * (e % PC), o = e / PC;
    const int gc = c0 + c, go = o0 + o;
    double* dst = sm + o * S + c;
    const double* src = base + gc + (size_t)go * ld;
    const bool oko = go < olimit;
    if (vec && oko && gc + 1 < climit) {
      cp_async16(dst, src);
    } else {
      const bool ok0 = oko && gc < climit, ok1 = oko && gc + 1 < climit;
      cp_async8(dst, ok0 ? src : base, ok0);
      cp_async8(dst + 1, ok1 ? src + 1 : base, ok1);
    }
  }
}

// Stage the A (TBM x TBK) and B (TBK x 64) tiles of k-block k0 into shared
// memory (layouts above); out-of-range elements are zero-filled.
template <int TBM, int TBK, int TBN>
__device__ __forceinline__ void load_stage(const GemmOp& g, int m0, int n0, int k0, double* As, double* Bs, bool va,
                                           bool vb) {
  constexpr int T = TBM * TBN / 32, KST = TBK + 4;  // threads (one warp per 32 x 32 block), [row][k] stride
  constexpr int AMS = TBM + 4, BNS = TBN + 4;        // [k][row] strides
  if (!g.transA)  // A column-major: m contiguous -> As[k][m]
    stage_pairs<TBM, TBK, AMS, T>(As, g.A, g.lda, m0, g.m, k0, g.k, va);
  else  // A^T stored: k contiguous -> As[m][k]
    stage_pairs<TBK, TBM, KST, T>(As, g.A, g.lda, k0, g.k, m0, g.m, va);
  if (!g.transB)  // B column-major: k contiguous -> Bs[n][k]
    stage_pairs<TBK, TBN, KST, T>(Bs, g.B, g.ldb, k0, g.k, n0, g.n, vb);
  else  // B^T stored: n contiguous -> Bs[k][n]
    stage_pairs<TBN, TBK, BNS, T>(Bs, g.B, g.ldb, n0, g.n, k0, g.k, vb);
}

template <int TBM, int TBK = BK, int TBN = 64>
__global__ void __launch_bounds__(TBM * TBN / 32) gemm_batched_kernel(const Bases* __restrict__ bases_ptr,
                                                                       const GemmDesc* __restrict__ descs,
                                                                       int tiles_n, bool g_vec16) {
  constexpr int BM = TBM, BK = TBK, KS = TBK + 4, BN = TBN, NT = TBM * TBN / 32, WN = TBN / 32;
  const Bases& bases = *bases_ptr;
  const GemmDesc gd = descs[blockIdx.y];
  const GemmOp g{at<const double>(bases, gd.A), at<const double>(bases, gd.B), at<double>(bases, gd.C),
                 gd.m, gd.n, gd.k, gd.lda, gd.ldb, gd.ldc, gd.transA, gd.transB, gd.alpha, gd.beta};
  const int m0 = (blockIdx.x / tiles_n) * BM, n0 = (blockIdx.x % tiles_n) * BN;
  if (m0 >= g.m || n0 >= g.n) return;

  constexpr int AE = OperandLayout<TBM>::kElems, BE = OperandLayout<BN>::kElems;
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                       // STAGES x AE
  double* Bs = gsm + STAGES * AE;         // STAGES x BE

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wm = (wid / WN) * 32, wn = (wid % WN) * 32;
  const int fr = lane >> 2, fc = lane & 3;
  // fragment offsets in either layout: element (row, k) at row * rs + k * ks
  const int ars = g.transA ? KS : 1, aks = g.transA ? 1 : BM + 4;
  const int brs = g.transB ? 1 : KS, bks = g.transB ? BN + 4 : 1;
  int aoff[4], boff[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) aoff[i] = (wm + i * 8 + fr) * ars + fc * aks;
#pragma unroll
  for (int j = 0; j < 4; ++j) boff[j] = (wn + j * 8 + fr) * brs + fc * bks;

  // The DMMA sum starts at 0 (k order fixed by the tiles); the epilogue
  // forms alpha*sum + beta*C.  The C tile is prefetched into L2 at the
  // start (no registers held, no stall at the first DMMA), so the
  // epilogue's loads hit L2 after the k loop.
  if (g.beta != 0.0) {  // one 64-byte line per (column, 8-row group) of the tile
    for (int e = threadIdx.x; e < BN * (BM / 8); e += NT) {
      const int c = n0 + e / (BM / 8), r = m0 + (e % (BM / 8)) * 8;
      if (c < g.n && r < g.m) asm volatile("prefetch.global.L2 [%0];" ::"l"(g.C + r + (size_t)c * g.ldc));
    }
  }
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (g.k + BK - 1) / BK;
  const bool va = g_vec16 && ((reinterpret_cast<uintptr_t>(g.A) & 15) == 0) && (g.lda % 2 == 0);
  const bool vb = g_vec16 && ((reinterpret_cast<uintptr_t>(g.B) & 15) == 0) && (g.ldb % 2 == 0);
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nk) load_stage<TBM, TBK, TBN>(g, m0, n0, st * BK, As + st * AE, Bs + st * BE, va, vb);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int pf = kt + STAGES - 1;
    if (pf < nk)
      load_stage<TBM, TBK, TBN>(g, m0, n0, pf * BK, As + (pf % STAGES) * AE, Bs + (pf % STAGES) * BE, va, vb);
    cp_async_commit();
    const double* as = As + (kt % STAGES) * AE;
    const double* bs = Bs + (kt % STAGES) * BE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = as[aoff[i] + kk * aks];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = bs[boff[j] + kk * bks];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  const double alpha = g.alpha, beta = g.beta;
  if (beta != 0.0) {  // C from L2 (prefetched), all loads first
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = m0 + wm + i * 8 + fr, c = n0 + wn + j * 8 + 2 * fc + h;
          const double cv = (r < g.m && c < g.n) ? g.C[r + (size_t)c * g.ldc] : 0.0;
          acc[i][j][h] = alpha * acc[i][j][h] + beta * cv;
        }
  } else if (alpha != 1.0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[i][j][0] *= alpha;
        acc[i][j][1] *= alpha;
      }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + fr;
    if (r >= g.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = n0 + wn + j * 8 + 2 * fc + h;
        if (c < g.n) g.C[r + (size_t)c * g.ldc] = acc[i][j][h];
      }
    }
  }
}

// Skinny products (n <= 16: the solves' k right-hand sides): 128 x 16
// output tiles, each warp 32 rows x 16 columns, so a CTA streams 128 rows
// of A per k-slab instead of computing a 64 x 64 tile three quarters
// empty.  Same k-slab order and DMMA fragment order per output element as
// gemm_batched_kernel: the results are bit-identical to it.
constexpr int SBM = 128, SBN = 16;
#ifndef HKS_SKINNY_BK
#define HKS_SKINNY_BK 16
#endif
#ifndef HKS_SKINNY_STAGES
#define HKS_SKINNY_STAGES 3
#endif
// 16-deep k-slabs, 3 stages (measured: 8-deep slabs with 4 stages, four
// CTAs per SM instead of three, are slower on the solve)
constexpr int SBK = HKS_SKINNY_BK, SST = HKS_SKINNY_STAGES, SKS = SBK + 4;  // SKS == 4 (mod 8): conflict-free fragments
__global__ void __launch_bounds__(128) gemm_skinny_kernel(const Bases* __restrict__ bases_ptr,
                                                          const GemmDesc* __restrict__ descs) {
  constexpr int BK = SBK, STAGES = SST, KS = SKS;
  const Bases& bases = *bases_ptr;
  const GemmDesc gd = descs[blockIdx.y];
  const GemmOp g{at<const double>(bases, gd.A), at<const double>(bases, gd.B), at<double>(bases, gd.C),
                 gd.m, gd.n, gd.k, gd.lda, gd.ldb, gd.ldc, gd.transA, gd.transB, gd.alpha, gd.beta};
  const int m0 = blockIdx.x * SBM;
  if (m0 >= g.m) return;
  // operand layouts as in gemm_batched_kernel (OperandLayout): [k][row] for
  // row-contiguous global operands, [row][k] for k-contiguous ones
  constexpr int AMS = SBM + 4, BNS = SBN + 4;
  constexpr int AE = (SBM * KS > BK * AMS) ? SBM * KS : BK * AMS;
  constexpr int BE = (SBN * KS > BK * BNS) ? SBN * KS : BK * BNS;
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                        // STAGES x AE
  double* Bs = gsm + STAGES * AE;          // STAGES x BE
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int wm = wid * 32, fr = lane >> 2, fc = lane & 3;
  const int ars = g.transA ? KS : 1, aks = g.transA ? 1 : AMS;
  const int brs = g.transB ? 1 : KS, bks = g.transB ? BNS : 1;
  auto load = [&](int k0, double* as, double* bs) {
    if (!g.transA) {  // m contiguous -> as[k][m]
#pragma unroll
      for (int ki = 0; ki < BK; ++ki) {
        const int m = m0 + t, k = k0 + ki;
        const bool ok = m < g.m && k < g.k;
        cp_async8(as + ki * AMS + t, ok ? g.A + m + (size_t)k * g.lda : g.A, ok);
      }
    } else {
#pragma unroll
      for (int j = 0; j < SBM * BK / 128; ++j) {
        const int ki = t % BK, mi = t / BK + (128 / BK) * j;
        const int m = m0 + mi, k = k0 + ki;
        const bool ok = m < g.m && k < g.k;
        cp_async8(as + mi * KS + ki, ok ? g.A + k + (size_t)m * g.lda : g.A, ok);
      }
    }
#pragma unroll
    for (int j = 0; j < SBN * BK / 128; ++j) {
      const int e = t + 128 * j;  // !transB: along k then n -> bs[n][k]; transB: along n then k -> bs[k][n]
      const int ki = g.transB ? e / SBN : e % BK, ni = g.transB ? e % SBN : e / BK;
      const int k = k0 + ki;
      const bool ok = ni < g.n && k < g.k;
      cp_async8(bs + ni * brs + ki * bks,
                ok ? (g.transB ? g.B + ni + (size_t)k * g.ldb : g.B + k + (size_t)ni * g.ldb) : g.B, ok);
    }
  };
  if (g.beta != 0.0)
    for (int e = t; e < SBN * (SBM / 8); e += 128) {
      const int c = e / (SBM / 8), r = m0 + (e % (SBM / 8)) * 8;
      if (c < g.n && r < g.m) asm volatile("prefetch.global.L2 [%0];" ::"l"(g.C + r + (size_t)c * g.ldc));
    }
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nk = (g.k + BK - 1) / BK;
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nk) load(st * BK, As + st * AE, Bs + st * BE);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int pf = kt + STAGES - 1;
    if (pf < nk) load(pf * BK, As + (pf % STAGES) * AE, Bs + (pf % STAGES) * BE);
    cp_async_commit();
    const double* as = As + (kt % STAGES) * AE;
    const double* bs = Bs + (kt % STAGES) * BE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = as[(wm + i * 8 + fr) * ars + (kk + fc) * aks];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = bs[(j * 8 + fr) * brs + (kk + fc) * bks];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
  const double alpha = g.alpha, beta = g.beta;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + fr;
    if (r >= g.m) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = j * 8 + 2 * fc + h;
        if (c >= g.n) continue;
        double v = acc[i][j][h];
        if (beta != 0.0) v = alpha * v + beta * g.C[r + (size_t)c * g.ldc];
        else if (alpha != 1.0) v *= alpha;
        g.C[r + (size_t)c * g.ldc] = v;
      }
  }
}

// dst = alpha * op(src) / alpha * I / 0 / dst + alpha * op(src), one descriptor per block.
// 32 x 32 output tiles, 256 threads (8 rows of 32 lanes); a transposed
// copy goes through a shared tile so both its reads and its writes are
// coalesced (the leaf level's phi = P^T and the pushes' P^T).
__global__ void __launch_bounds__(256) copy_batched_kernel(const Bases* __restrict__ bases_ptr,
                                                           const CopyDesc* __restrict__ descs) {
  const Bases& bases = *bases_ptr;
  const CopyDesc c = descs[blockIdx.y];
  const double* src = (c.mode == 0 || c.mode >= 3) ? at<const double>(bases, c.src) : nullptr;
  double* dst = at<double>(bases, c.dst);
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int tm = (c.m + 31) / 32, tn = (c.n + 31) / 32;
  for (int tix = blockIdx.x; tix < tm * tn; tix += gridDim.x) {
    const int i0 = (tix % tm) * 32, j0 = (tix / tm) * 32;
    if ((c.mode == 0 || c.mode == 4) && c.trans) {  // dst(i, j) = alpha src(j, i): read along j, write along i
      __syncthreads();
      for (int ii = ty; ii < 32; ii += 8) {
        const int i = i0 + ii, j = j0 + tx;
        tile[ii][tx] = (i < c.m && j < c.n) ? src[j + (size_t)i * c.lds] : 0.0;
      }
      __syncthreads();
      if (c.mode == 4) {  // dst = src^T + alpha src2 (src2 read along i: coalesced)
        const double* src2 = at<const double>(bases, c.src2);
        for (int jj = ty; jj < 32; jj += 8) {
          const int i = i0 + tx, j = j0 + jj;
          if (i < c.m && j < c.n) dst[i + (size_t)j * c.ldd] = src2[i + (size_t)j * c.lds2] * c.alpha + tile[tx][jj];
        }
        continue;
      }
      for (int jj = ty; jj < 32; jj += 8) {
        const int i = i0 + tx, j = j0 + jj;
        if (i < c.m && j < c.n) dst[i + (size_t)j * c.ldd] = tile[tx][jj] * c.alpha;
      }
      continue;
    }
    for (int jj = ty; jj < 32; jj += 8) {
      const int i = i0 + tx, j = j0 + jj;
      if (i >= c.m || j >= c.n) continue;
      double v;
      if (c.mode == 0 || c.mode == 3) {
        v = (c.trans ? src[j + (size_t)i * c.lds] : src[i + (size_t)j * c.lds]) * c.alpha;
        if (c.mode == 3) v += dst[i + (size_t)j * c.ldd];
      } else if (c.mode == 5) {
        v = bases.lam * src[i + (size_t)j * c.lds];
      } else if (c.mode == 6) {
        v = src[i + (size_t)j * c.lds];
        if (i == j) v += bases.lam;
      } else {
        v = (c.mode == 1 && i == j) ? c.alpha : 0.0;
      }
      dst[i + (size_t)j * c.ldd] = v;
    }
  }
}

}  // namespace

cudaError_t launch_gemm_batched(const Bases* bases, const GemmDesc* d_descs, int count, int max_m,
                                int max_n, cudaStream_t stream) {
  if (count <= 0 || max_m <= 0 || max_n <= 0) return cudaSuccess;
  static const int forced = [] {  // development knob: HKS_GEMM_BM = 64 / 128
    const char* e = getenv("HKS_GEMM_BM");
    return e ? atoi(e) : 0;
  }();
  // 128-row tiles (8 warps) once the products are tall and the grid is
  // large: more warps per SM and half the B-operand staging per flop
  static const bool skinny_ok = getenv("HKS_GEMM_SKINNY") == nullptr || atoi(getenv("HKS_GEMM_SKINNY")) != 0;
  if (skinny_ok && max_n <= SBN) {  // the solves' right-hand-side blocks
    constexpr int sae = (SBM * SKS > SBK * (SBM + 4)) ? SBM * SKS : SBK * (SBM + 4);
    constexpr int sbe = (SBN * SKS > SBK * (SBN + 4)) ? SBN * SKS : SBK * (SBN + 4);
    const size_t sm = (size_t)SST * (sae + sbe) * sizeof(double);
    raise_smem_limit(gemm_skinny_kernel, sm);
    for (int first = 0; first < count; first += 65535) {
      const int cnt = count - first < 65535 ? count - first : 65535;
      gemm_skinny_kernel<<<dim3((max_m + SBM - 1) / SBM, cnt), 128, sm, stream>>>(bases, d_descs + first);
    }
    return cudaGetLastError();
  }
  // narrow products (n <= 32: the LU program's in-group panel updates):
  // 128 x 32 tiles, four warps stacked along m -- a 64 x 64 tile would
  // compute and stage a half-empty B operand
  static const bool narrow_ok = getenv("HKS_GEMM_NARROW") == nullptr || atoi(getenv("HKS_GEMM_NARROW")) != 0;
  if (narrow_ok && max_n <= 32 && max_m >= 96) {
    static const bool vec16n = getenv("HKS_GEMM_VEC16") == nullptr || atoi(getenv("HKS_GEMM_VEC16")) != 0;
    const int tmn = (max_m + 127) / 128;
    const size_t smn = (size_t)STAGES * (OperandLayout<128>::kElems + OperandLayout<32>::kElems) * sizeof(double);
    raise_smem_limit(gemm_batched_kernel<128, BK, 32>, smn);
    for (int first = 0; first < count; first += 65535) {
      const int cnt = count - first < 65535 ? count - first : 65535;
      gemm_batched_kernel<128, BK, 32><<<dim3(tmn, cnt), 128, smn, stream>>>(bases, d_descs + first, 1, vec16n);
    }
    return cudaGetLastError();
  }
  const bool tall = forced == 128;  // measured: no gain over 64-row tiles on the plans' products
  static const bool vec16 = getenv("HKS_GEMM_VEC16") == nullptr || atoi(getenv("HKS_GEMM_VEC16")) != 0;
  const int BM = tall ? 128 : 64;
  const int tm = (max_m + BM - 1) / BM, tn = (max_n + BN - 1) / BN;
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    dim3 grid(tm * tn, cnt);
    const size_t sm = (size_t)STAGES *
                      ((tall ? OperandLayout<128>::kElems : OperandLayout<64>::kElems) + OperandLayout<BN>::kElems) *
                      sizeof(double);
    if (tall) {
      raise_smem_limit(gemm_batched_kernel<128>, sm);
      gemm_batched_kernel<128><<<grid, 256, sm, stream>>>(bases, d_descs + first, tn, vec16);
    } else {
      raise_smem_limit(gemm_batched_kernel<64>, sm);
      gemm_batched_kernel<64><<<grid, 128, sm, stream>>>(bases, d_descs + first, tn, vec16);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_copy_batched(const Bases* bases, const CopyDesc* d_descs, int count, int max_elems,
                                cudaStream_t stream) {
  if (count <= 0 || max_elems <= 0) return cudaSuccess;
  int bx = (max_elems + 1023) / 1024;  // ~ one 32 x 32 tile per CTA
  if (bx > 64) bx = 64;
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    copy_batched_kernel<<<dim3(bx, cnt), 256, 0, stream>>>(bases, d_descs + first);
  }
  return cudaGetLastError();
}

}  // namespace hks
