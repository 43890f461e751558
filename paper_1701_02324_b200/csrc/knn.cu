// Exact brute-force kNN (tree.py:163-188) on the FP64 DMMA path.
//
// d^2 = (|x|^2 + |y|^2) - 2 x.y in the reference's GEMM form, self excluded,
// neighbours ordered by (d^2, index) -- the lexsort of tree.py:181-187.  A
// CTA owns 64 queries and streams all points in 64-wide tiles; the dot
// products of a tile are 8x8x4 DMMA fragments staged through shared memory,
// and each warp keeps the running top-k of 16 queries in registers (lane j =
// j-th best), inserting with a ballot when a candidate beats the k-th.
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <vector>

#include "hks_internal.h"

namespace hks {
namespace {

constexpr int QB = 64, CB = 64, DCH = 32, DS = DCH + 4;  // DS: smem row stride
constexpr int KT = 128;

__global__ void sqnorm_kernel(const double* __restrict__ X, int64_t n, int d, double* __restrict__ sq) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const double* x = X + (size_t)p * d;
    double s = 0.0;
    for (int k = 0; k < d; ++k) s = fma(x[k], x[k], s);
    sq[p] = s;
  }
}

__device__ __forceinline__ bool lex_less(double a, int ia, double b, int ib) {
  return a < b || (a == b && ia < ib);
}

// One CTA's 64 queries [q0, qend) against the candidates [clo, chi).
// SEG: per-CTA ranges from `segs` (segmented / approximate kNN: queries of a
// leaf of a random-projection tree against that leaf), ids mapped through
// `perm` and d^2 written beside them; else queries [qlo + 64 b, qhi) against
// all n points (exact kNN).
struct KnnSeg {
  int q0, qhi, clo, chi;
};

template <bool SEG>
__global__ void __launch_bounds__(KT) knn_kernel(const double* __restrict__ X, const double* __restrict__ sq,
                                                 int n, int d, int kk, int qlo, int qhi,
                                                 int64_t* __restrict__ out, const KnnSeg* __restrict__ segs,
                                                 const int64_t* __restrict__ perm, double* __restrict__ out_d2) {
  extern __shared__ double smem[];
  double* Qs = smem;                 // QB x DS
  double* Cs = smem + QB * DS;       // CB x DS
  double* Dt = smem + 2 * QB * DS;   // QB x (CB + 1)
  int q0, qend, clo, chi;
  if (SEG) {
    const KnnSeg g = segs[blockIdx.x];
    q0 = g.q0, qend = g.qhi, clo = g.clo, chi = g.chi;
  } else {
    q0 = qlo + blockIdx.x * QB, qend = qhi, clo = 0, chi = n;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  const int wm = (wid >> 1) * 32, wn = (wid & 1) * 32;
  const bool q_resident = d <= DCH;

  double lv[16];
  int li[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    lv[i] = DBL_MAX;
    li[i] = 0x7fffffff;
  }
  auto stage = [&](double* S, int base, int lim, int k0, int dc) {
    for (int e = threadIdx.x; e < 64 * DS; e += KT) {
      const int r = e / DS, k = e % DS;
      const int p = base + r;
      S[e] = (p < lim && k < dc) ? X[(size_t)p * d + k0 + k] : 0.0;
    }
  };
  if (q_resident) stage(Qs, q0, n, 0, d);

  for (int c0 = clo; c0 < chi; c0 += CB) {
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int k0 = 0; k0 < d; k0 += DCH) {
      const int dc = min(DCH, d - k0);
      __syncthreads();
      if (!q_resident) stage(Qs, q0, n, k0, dc);
      stage(Cs, c0, chi, k0, dc);
      __syncthreads();
      for (int kk4 = 0; kk4 < dc; kk4 += 4) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = Qs[(wm + i * 8 + fr) * DS + kk4 + fc];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Cs[(wn + j * 8 + fr) * DS + kk4 + fc];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    }
    // distance tile (tree.py:179): (|x|^2 + |y|^2) - 2 x.y
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = wm + i * 8 + fr;
      const double sqq = (q0 + r < n) ? sq[q0 + r] : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = wn + j * 8 + 2 * fc + h;
          const double sqc = (c0 + c < chi) ? sq[c0 + c] : 0.0;
          Dt[r * (CB + 1) + c] = (sqq + sqc) - 2.0 * acc[i][j][h];
        }
    }
    __syncthreads();
    // merge: warp wid owns queries wid*16 .. wid*16+15
#pragma unroll
    for (int qi = 0; qi < 16; ++qi) {
      const int ql = wid * 16 + qi, q = q0 + ql;
      if (q >= qend) continue;
      double tv = __shfl_sync(0xffffffffu, lv[qi], kk - 1);
      int ti = __shfl_sync(0xffffffffu, li[qi], kk - 1);
      double cv[2];
      int ci[2];
      unsigned m[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = lane + 32 * h;
        ci[h] = c0 + c;
        cv[h] = Dt[ql * (CB + 1) + c];
        const bool ok = ci[h] < chi && ci[h] != q && lex_less(cv[h], ci[h], tv, ti);
        m[h] = __ballot_sync(0xffffffffu, ok);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        while (m[h]) {
          const int src = __ffs(m[h]) - 1;
          m[h] &= m[h] - 1;
          const double v = __shfl_sync(0xffffffffu, cv[h], src);
          const int vi = __shfl_sync(0xffffffffu, ci[h], src);
          if (!lex_less(v, vi, tv, ti)) continue;  // the k-th moved since the ballot
          const bool gt = lane < kk && lex_less(v, vi, lv[qi], li[qi]);
          const unsigned gm = __ballot_sync(0xffffffffu, gt);
          const int pos = __ffs(gm) - 1;
          const double up_v = __shfl_up_sync(0xffffffffu, lv[qi], 1);
          const int up_i = __shfl_up_sync(0xffffffffu, li[qi], 1);
          if (lane == pos) {
            lv[qi] = v;
            li[qi] = vi;
          } else if (lane > pos) {
            lv[qi] = up_v;
            li[qi] = up_i;
          }
          tv = __shfl_sync(0xffffffffu, lv[qi], kk - 1);
          ti = __shfl_sync(0xffffffffu, li[qi], kk - 1);
        }
      }
    }
  }
#pragma unroll
  for (int qi = 0; qi < 16; ++qi) {
    const int q = q0 + wid * 16 + qi;
    if (q < qend && lane < kk) {
      if (SEG) {  // rows by position, ids through perm, distances beside them
        out[(size_t)q * kk + lane] = perm[li[qi]];
        out_d2[(size_t)q * kk + lane] = lv[qi];
      } else {
        out[(size_t)(q - qlo) * kk + lane] = li[qi];
      }
    }
  }
}

// Exact kNN for d <= 32 (the whole feature vector in one staged slab).  Same
// distances, same (d^2, index) order as knn_kernel, restructured so that the
// common case -- no candidate of a tile beats any query's k-th best -- costs
// the DMMA products and one register-level test:
//   * a warp owns 16 queries and ALL 64 candidates of the tile (2 x 8
//     fragments), so a query's candidates never leave its warp: no distance
//     tile in shared memory, no barrier between the products and the merge;
//   * every lane keeps the k-th best (value, index) of its two query rows in
//     registers and tests its 32 accumulators against them; only when some
//     lane has a hit does the warp insert, into (d^2, index)-sorted lists in
//     shared memory (lane j = j-th best, ballot for the position);
//   * candidate tiles (points and their squared norms) are double-buffered
//     with cp.async behind the previous tile's products: one barrier a tile.
// The sum x.y of a pair runs over k in the same DMMA order wherever the pair
// sits in a tile, so the lists equal knn_kernel's bit for bit.
constexpr int SQB = 64, SCB = 64, SKT = 128;

// Row stride of the staged points: the smallest value >= dpad that keeps the
// DMMA fragment loads conflict-free (stride == 4 or 12 mod 16).
__host__ __device__ inline int knn_stream_stride(int d) {
  int v = (d + 3) & ~3;
  while ((v & 15) != 4 && (v & 15) != 12) v += 4;
  return v;
}
inline size_t knn_stream_smem(int d) {
  return (size_t)(3 * SQB * knn_stream_stride(d) + 2 * SCB + SQB * 32) * sizeof(double) + SQB * 32 * sizeof(int) +
         4 * sizeof(uint64_t);  // + the bulk-copy mbarriers
}

// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier: a
// candidate tile of 64 points is one contiguous 64 d doubles in X, so when
// the staged stride equals d (d = 28: C3) one elected thread moves the whole
// tile with one instruction instead of 7 LDGSTS per thread.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

struct KnnStreamSmem {  // carved from dynamic shared memory (SDS is a run-time stride)
  double* Qs;
  double* Cs[2];
  double* sqc[2];
  double* Lv;
  int* Li;
};

// Epilogue of one candidate tile for a warp's 16 queries x 64 candidates:
// accumulators -> distances, register test against the rows' k-th best, and
// the (rare) insertion into the sorted lists in shared memory.
__device__ __forceinline__ void knn_tile_merge(double (&acc)[2][8][2], const double (&sqq)[2], const double* sqc,
                                               int c0, int n, const int (&qid)[2], const int (&qrow)[2], int qhi,
                                               double (&tv)[2], int (&ti)[2], double* Lv, int* Li, int kk, int wid,
                                               int lane, int fc) {
    // d^2 = (|x|^2 + |y|^2) - 2 x.y (tree.py:179), tested against the rows' k-th best.
    // The test is conservative (d^2 <= k-th: ties, the row's own point and
    // padding included): one FP64 compare per candidate; the insertion path
    // below re-checks every candidate exactly.
    bool hit = false;
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double sc = sqc[8 * j + 2 * fc + h];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double dv = (sqq[i] + sc) - 2.0 * acc[i][j][h];
          acc[i][j][h] = dv;
          hit |= dv <= tv[i];
        }
      }
    if (!__any_sync(0xffffffffu, hit)) return;
    // insertion path: slot by slot (static registers), lanes with a hit one at a time
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int ci = c0 + 8 * j + 2 * fc + h;
          const double dv = acc[i][j][h];
          const bool ok = ci < n && ci != qid[i] && qid[i] < qhi && lex_less(dv, ci, tv[i], ti[i]);
          unsigned m = __ballot_sync(0xffffffffu, ok);
          while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const double v = __shfl_sync(0xffffffffu, dv, src);
            const int vi = __shfl_sync(0xffffffffu, ci, src);
            const int row = wid * 16 + 8 * i + (src >> 2);
            const double lv = Lv[row * 32 + lane];
            const int li = Li[row * 32 + lane];
            const unsigned gm = __ballot_sync(0xffffffffu, lane < kk && lex_less(v, vi, lv, li));
            if (gm == 0) continue;  // the row's k-th moved since the test
            const int pos = __ffs(gm) - 1;
            const double up_v = __shfl_up_sync(0xffffffffu, lv, 1);
            const int up_i = __shfl_up_sync(0xffffffffu, li, 1);
            if (lane == pos) {
              Lv[row * 32 + lane] = v;
              Li[row * 32 + lane] = vi;
            } else if (lane > pos && lane < kk) {
              Lv[row * 32 + lane] = up_v;
              Li[row * 32 + lane] = up_i;
            }
            __syncwarp();
          }
        }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      // rows past the query range never insert: their threshold stays below every distance
      tv[i] = qid[i] < qhi ? Lv[qrow[i] * 32 + kk - 1] : -DBL_MAX;
      ti[i] = Li[qrow[i] * 32 + kk - 1];
    }
  }

template <bool BULK>
__global__ void __launch_bounds__(SKT) knn_stream_kernel(const double* __restrict__ X, const double* __restrict__ sq,
                                                        int n, int d, int kk, int qlo, int qhi,
                                                        int64_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char knn_raw[];
  const int SDS = knn_stream_stride(d);
  KnnStreamSmem sm;
  {
    double* base = reinterpret_cast<double*>(knn_raw);
    sm.Qs = base;
    sm.Cs[0] = base + SQB * SDS;
    sm.Cs[1] = base + 2 * SQB * SDS;
    sm.sqc[0] = base + 3 * SQB * SDS;
    sm.sqc[1] = sm.sqc[0] + SCB;
    sm.Lv = sm.sqc[1] + SCB;
    sm.Li = reinterpret_cast<int*>(sm.Lv + SQB * 32);
  }
  // BULK: bars[0], bars[1] = tile buffers full, bars[2] = queries
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm.Li + SQB * 32);
  const unsigned tile_bytes = (unsigned)(SCB * d * sizeof(double)), sq_bytes = (unsigned)(SCB * sizeof(double));
  const int q0 = qlo + blockIdx.x * SQB;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  const int dpad = (d + 3) & ~3;
  const bool vec16 = (d & 1) == 0;  // rows of X start 16-byte aligned
  auto stage = [&](double* S, int base) {  // 64 points x dpad, zero-filled past n and past d
    if (vec16) {
      const int pr = dpad / 2;  // 16-byte pairs per row (d even: a pair never straddles d)
      for (int e = tid; e < 64 * pr; e += SKT) {
        const int r = e / pr, k = 2 * (e % pr);
        const int pt = base + r;
        if (pt < n && k < d) cp_async16(S + r * SDS + k, X + (size_t)pt * d + k);
        else S[r * SDS + k] = S[r * SDS + k + 1] = 0.0;
      }
    } else {
      for (int e = tid; e < 64 * dpad; e += SKT) {
        const int r = e / dpad, k = e % dpad;
        const int pt = base + r;
        const bool ok = pt < n && k < d;
        cp_async8(S + r * SDS + k, ok ? X + (size_t)pt * d + k : X, ok);
      }
    }
  };
  // BULK: 64 points are one dense block of X and of the staged layout
  // (stride == d): one copy by one thread.  (One copy per row for padded
  // strides was measured 2x slower than the LDGSTS path at d = 18.)
  auto bulk_tile = [&](double* S, int base, uint64_t* bar) {
    if (tid == 0) bulk_g2s(S, X + (size_t)base * d, tile_bytes, bar);
  };
  auto stage_sq = [&](double* S, int base) {
    if (tid < SCB) {
      const bool ok = base + tid < n;
      cp_async8(S + tid, ok ? sq + base + tid : sq, ok);
    }
  };
  {
    const int ntile0 = (n + SCB - 1) / SCB;
    const int c_first = min(q0 / SCB, ntile0 - 1) * SCB;
    if (BULK) {
      if (tid == 0) {
        mbar_init(bars + 0, 1);
        mbar_init(bars + 1, 1);
        mbar_init(bars + 2, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      }
      __syncthreads();
      if (tid == 0) {
        mbar_expect_tx(bars + 2, tile_bytes);
        mbar_expect_tx(bars + 0, tile_bytes + sq_bytes);
        bulk_g2s(sm.sqc[0], sq + c_first, sq_bytes, bars + 0);
      }
      bulk_tile(sm.Qs, q0, bars + 2);
      bulk_tile(sm.Cs[0], c_first, bars + 0);
    } else {
      stage(sm.Qs, q0);
      stage(sm.Cs[0], c_first);
      stage_sq(sm.sqc[0], c_first);
      cp_async_commit();
    }
  }
  for (int e = tid; e < SQB * 32; e += SKT) {
    sm.Lv[e] = DBL_MAX;
    sm.Li[e] = 0x7fffffff;
  }
  // this lane's two query rows: 16 wid + fr and + 8
  int qrow[2], qid[2];
  double sqq[2], tv[2];
  int ti[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    qrow[i] = wid * 16 + 8 * i + fr;
    qid[i] = q0 + qrow[i];
    sqq[i] = qid[i] < n ? sq[qid[i]] : 0.0;
    tv[i] = qid[i] < qhi ? DBL_MAX : -DBL_MAX;  // see knn_tile_merge
    ti[i] = 0x7fffffff;
  }
  // Tiles are visited outwards from the queries' own position: the points
  // are in tree order, so the first tiles hold the spatially nearest
  // candidates, the k-th best distances are tight from the start and almost
  // every later tile takes the no-insertion path.  (The result does not
  // depend on the order: it is the k smallest (d^2, index) pairs.)
  const int ntile = (n + SCB - 1) / SCB;
  const int own = min(q0 / SCB, ntile - 1);
  auto tile_at = [&](int sidx) {  // offsets 0, +1, -1, +2, -2, ... modulo ntile
    const int off = (sidx & 1) ? (sidx + 1) / 2 : ntile - sidx / 2;
    return (own + off) % ntile;
  };
  for (int t = 0; t < ntile; ++t) {
    const int c0 = tile_at(t) * SCB;
    const double* Cs = sm.Cs[t & 1];
    const double* sqc = sm.sqc[t & 1];
    if (BULK) {
      if (t == 0) mbar_wait(bars + 2, 0);
      mbar_wait(bars + (t & 1), (t >> 1) & 1);
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // tile t landed; everyone is done reading tile t - 1's buffer
    if (t + 1 < ntile) {
      const int c1 = tile_at(t + 1) * SCB;
      if (BULK) {
        uint64_t* bar = bars + ((t + 1) & 1);
        if (tid == 0) {
          mbar_expect_tx(bar, tile_bytes + sq_bytes);
          bulk_g2s(sm.sqc[(t + 1) & 1], sq + c1, sq_bytes, bar);
        }
        bulk_tile(sm.Cs[(t + 1) & 1], c1, bar);
      } else {
        stage(sm.Cs[(t + 1) & 1], c1);
        stage_sq(sm.sqc[(t + 1) & 1], c1);
      }
    }
    if (!BULK) cp_async_commit();
    double acc[2][8][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int k4 = 0; k4 < dpad; k4 += 4) {
      double a[2], b[8];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = sm.Qs[qrow[i] * SDS + k4 + fc];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Cs[(8 * j + fr) * SDS + k4 + fc];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    knn_tile_merge(acc, sqq, sqc, c0, n, qid, qrow, qhi, tv, ti, sm.Lv, sm.Li, kk, wid, lane, fc);
  }
  __syncwarp();
  for (int r = 0; r < 16; ++r) {
    const int row = wid * 16 + r, q = q0 + row;
    if (q < qhi && lane < kk) out[(size_t)(q - qlo) * kk + lane] = sm.Li[row * 32 + lane];
  }
}

// d > 32 (C5: d = 784): the same warp-owned merge, with the feature
// dimension walked in 32-wide chunks.  Every (candidate tile, chunk) step
// stages the chunk of the 64 queries and of the 64 candidates (cp.async,
// double-buffered: the next step's 32 KB land behind this step's 512 DMMA),
// the accumulators live across a tile's chunks, and the epilogue runs once
// per tile.  knn_kernel staged each chunk synchronously between two
// barriers and merged through a distance tile in shared memory.
constexpr int CDS = 36;  // staged row stride of a 32-wide chunk
struct KnnChunkSmem {
  double Qs[2][SQB * CDS];
  double Cs[2][SCB * CDS];
  double sqc[2][SCB];
  double Lv[SQB * 32];
  int Li[SQB * 32];
};

__global__ void __launch_bounds__(SKT) knn_chunk_kernel(const double* __restrict__ X, const double* __restrict__ sq,
                                                       int n, int d, int kk, int qlo, int qhi,
                                                       int64_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char knn_raw[];
  KnnChunkSmem& sm = *reinterpret_cast<KnnChunkSmem*>(knn_raw);
  const int q0 = qlo + blockIdx.x * SQB;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  const bool vec16 = (d & 1) == 0;  // rows and 32-wide chunks start 16-byte aligned
  const int nch = (d + 31) / 32;
  // 64 points x 32 features [k0, k0 + 32) (zero past n and past d)
  auto stage = [&](double* S, int base, int k0) {
    if (vec16) {
      for (int e = tid; e < 64 * 16; e += SKT) {
        const int r = e >> 4, k = 2 * (e & 15);
        const int pt = base + r;
        if (pt < n && k0 + k < d) cp_async16(S + r * CDS + k, X + (size_t)pt * d + k0 + k);
        else S[r * CDS + k] = S[r * CDS + k + 1] = 0.0;
      }
    } else {
      for (int e = tid; e < 64 * 32; e += SKT) {
        const int r = e >> 5, k = e & 31;
        const int pt = base + r;
        const bool ok = pt < n && k0 + k < d;
        cp_async8(S + r * CDS + k, ok ? X + (size_t)pt * d + k0 + k : X, ok);
      }
    }
  };
  auto stage_sq = [&](double* S, int base) {
    if (tid < SCB) {
      const bool ok = base + tid < n;
      cp_async8(S + tid, ok ? sq + base + tid : sq, ok);
    }
  };
  const int ntile = (n + SCB - 1) / SCB;
  const int own = min(q0 / SCB, ntile - 1);
  auto tile_at = [&](int sidx) {  // outwards from the queries' own tree position (see knn_stream_kernel)
    const int off = (sidx & 1) ? (sidx + 1) / 2 : ntile - sidx / 2;
    return (own + off) % ntile;
  };
  stage(sm.Qs[0], q0, 0);
  stage(sm.Cs[0], tile_at(0) * SCB, 0);
  stage_sq(sm.sqc[0], tile_at(0) * SCB);
  cp_async_commit();
  for (int e = tid; e < SQB * 32; e += SKT) {
    sm.Lv[e] = DBL_MAX;
    sm.Li[e] = 0x7fffffff;
  }
  int qrow[2], qid[2];
  double sqq[2], tv[2];
  int ti[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    qrow[i] = wid * 16 + 8 * i + fr;
    qid[i] = q0 + qrow[i];
    sqq[i] = qid[i] < n ? sq[qid[i]] : 0.0;
    tv[i] = qid[i] < qhi ? DBL_MAX : -DBL_MAX;  // see knn_tile_merge
    ti[i] = 0x7fffffff;
  }
  int step = 0;
  for (int t = 0; t < ntile; ++t) {
    const int c0 = tile_at(t) * SCB;
    double acc[2][8][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int ch = 0; ch < nch; ++ch, ++step) {
      const double* Qs = sm.Qs[step & 1];
      const double* Cs = sm.Cs[step & 1];
      cp_async_wait<0>();
      __syncthreads();  // this step's chunks landed; everyone is done with the other buffers
      {                 // next step: next chunk of this tile, or chunk 0 of the next tile
        const int nt = ch + 1 < nch ? t : t + 1, nc = ch + 1 < nch ? ch + 1 : 0;
        if (nt < ntile) {
          const int c1 = tile_at(nt) * SCB;
          stage(sm.Qs[(step + 1) & 1], q0, nc * 32);
          stage(sm.Cs[(step + 1) & 1], c1, nc * 32);
          if (nc == 0) stage_sq(sm.sqc[nt & 1], c1);
        }
      }
      cp_async_commit();
      const int dc = min(32, d - ch * 32);
      for (int k4 = 0; k4 < dc; k4 += 4) {
        double a[2], b[8];
#pragma unroll
        for (int i = 0; i < 2; ++i) a[i] = Qs[qrow[i] * CDS + k4 + fc];
#pragma unroll
        for (int j = 0; j < 8; ++j) b[j] = Cs[(8 * j + fr) * CDS + k4 + fc];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    }
    knn_tile_merge(acc, sqq, sm.sqc[t & 1], c0, n, qid, qrow, qhi, tv, ti, sm.Lv, sm.Li, kk, wid, lane, fc);
  }
  __syncwarp();
  for (int r = 0; r < 16; ++r) {
    const int row = wid * 16 + r, q = q0 + row;
    if (q < qhi && lane < kk) out[(size_t)(q - qlo) * kk + lane] = sm.Li[row * 32 + lane];
  }
}

}  // namespace
}  // namespace hks

using namespace hks;

// knn_bruteforce (tree.py:163-188): out[n x k] int64, k <= 32.
extern "C" int hks_knn_rows(const double* X, int64_t n, int64_t d, int64_t k, int64_t q0, int64_t nq, int64_t* out,
                            void* stream) {
  if (!X || !out || n < 2 || d < 1 || k < 1 || k > n - 1 || q0 < 0 || nq < 0 || q0 + nq > n)
    return set_error(HKS_ERR_INVALID, "need 1 <= k <= n - 1 and a query range inside [0, n)");
  if (k > 32) return set_error(HKS_ERR_NOT_SUPPORTED, "hks_knn: k <= 32 supported (got %lld)", (long long)k);
  if (n > 0x7ffffffe) return set_error(HKS_ERR_NOT_SUPPORTED, "hks_knn: n too large");
  if (nq == 0) return HKS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* sq = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&sq), n * sizeof(double), s);
  if (e == cudaSuccess) {
    sqnorm_kernel<<<592, 256, 0, s>>>(X, n, (int)d, sq);
    static const bool stream_off = getenv("HKS_KNN_STREAM") != nullptr && atoi(getenv("HKS_KNN_STREAM")) == 0;
    if (d <= 32 && !stream_off) {
      // whole tiles as TMA bulk copies when a tile is one dense block of the
      // staged layout: stride == d, every tile and query block full, 16-byte
      // aligned rows (d even)
      static const bool bulk_off = getenv("HKS_KNN_BULK") != nullptr && atoi(getenv("HKS_KNN_BULK")) == 0;
      const bool bulk = !bulk_off && knn_stream_stride((int)d) == d && d % 2 == 0 && n % SCB == 0 &&
                        q0 % SQB == 0 && (q0 + nq) % SQB == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
      const unsigned grid = (unsigned)((nq + SQB - 1) / SQB);
      if (bulk) {
        raise_smem_limit(knn_stream_kernel<true>, knn_stream_smem((int)d));
        knn_stream_kernel<true><<<grid, SKT, knn_stream_smem((int)d), s>>>(X, sq, (int)n, (int)d, (int)k, (int)q0,
                                                                           (int)(q0 + nq), out);
      } else {
        raise_smem_limit(knn_stream_kernel<false>, knn_stream_smem((int)d));
        knn_stream_kernel<false><<<grid, SKT, knn_stream_smem((int)d), s>>>(X, sq, (int)n, (int)d, (int)k, (int)q0,
                                                                            (int)(q0 + nq), out);
      }
    } else if (!stream_off) {
      raise_smem_limit(knn_chunk_kernel, sizeof(KnnChunkSmem));
      knn_chunk_kernel<<<(unsigned)((nq + SQB - 1) / SQB), SKT, sizeof(KnnChunkSmem), s>>>(
          X, sq, (int)n, (int)d, (int)k, (int)q0, (int)(q0 + nq), out);
    } else {
      const size_t sm = (size_t)(2 * QB * DS + QB * (CB + 1)) * sizeof(double);
      raise_smem_limit(knn_kernel<false>, sm);
      knn_kernel<false><<<(unsigned)((nq + QB - 1) / QB), KT, sm, s>>>(X, sq, (int)n, (int)d, (int)k, (int)q0,
                                                                      (int)(q0 + nq), out, nullptr, nullptr, nullptr);
    }
    e = cudaGetLastError();
    cudaFreeAsync(sq, s);
  }
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_knn: %s", cudaGetErrorString(e));
  return HKS_OK;
}

extern "C" int hks_knn(const double* X, int64_t n, int64_t d, int64_t k, int64_t* out, void* stream) {
  return hks_knn_rows(X, n, d, k, 0, n, out, stream);
}

// Segmented kNN: every point of segment [seg_off[i], seg_off[i+1]) against
// the points of its own segment (a leaf of a random-projection tree).
// Rows of out_idx / out_d2 follow positions in X; ids are perm[position].
extern "C" int hks_knn_segments(const double* X, int64_t n, int64_t d, int64_t k, const int64_t* seg_off_host,
                                int64_t nseg, const int64_t* perm, int64_t* out_idx, double* out_d2, void* stream) {
  if (!X || !seg_off_host || !perm || !out_idx || !out_d2 || n < 2 || d < 1 || k < 1 || nseg < 1 ||
      seg_off_host[0] != 0 || seg_off_host[nseg] != n)
    return set_error(HKS_ERR_INVALID, "hks_knn_segments: bad arguments");
  if (k > 32) return set_error(HKS_ERR_NOT_SUPPORTED, "hks_knn_segments: k <= 32 supported (got %lld)", (long long)k);
  std::vector<KnnSeg> segs;
  for (int64_t i = 0; i < nseg; ++i) {
    const int64_t b = seg_off_host[i], e = seg_off_host[i + 1];
    if (e - b < k + 1) return set_error(HKS_ERR_INVALID, "hks_knn_segments: segment %lld smaller than k + 1", (long long)i);
    for (int64_t q = b; q < e; q += QB) segs.push_back(KnnSeg{(int)q, (int)e, (int)b, (int)e});
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* sq = nullptr;
  KnnSeg* dsegs = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&sq), n * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dsegs), segs.size() * sizeof(KnnSeg), s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dsegs, segs.data(), segs.size() * sizeof(KnnSeg), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    sqnorm_kernel<<<592, 256, 0, s>>>(X, n, (int)d, sq);
    const size_t sm = (size_t)(2 * QB * DS + QB * (CB + 1)) * sizeof(double);
    raise_smem_limit(knn_kernel<true>, sm);
    knn_kernel<true><<<(unsigned)segs.size(), KT, sm, s>>>(X, sq, (int)n, (int)d, (int)k, 0, 0, out_idx, dsegs, perm,
                                                           out_d2);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the host descriptors die with this call
  if (dsegs) cudaFreeAsync(dsegs, s);
  if (sq) cudaFreeAsync(sq, s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_knn_segments: %s", cudaGetErrorString(e));
  return HKS_OK;
}

namespace hks {
namespace {
// Per query: the union of two (d^2, id)-sorted candidate lists, duplicates
// dropped, first k kept.
__global__ void knn_merge_kernel(const int64_t* __restrict__ ai, const double* __restrict__ ad,
                                 const int64_t* __restrict__ bi, const double* __restrict__ bd, int64_t n, int k,
                                 int64_t* __restrict__ oi, double* __restrict__ od) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t* a = ai + q * k;
    const int64_t* b = bi + q * k;
    const double* da = ad + q * k;
    const double* db = bd + q * k;
    int x = 0, y = 0, o = 0;
    int64_t last = -1;
    double lastd = -1.0;
    while (o < k && (x < k || y < k)) {
      bool take_a;
      if (x >= k) take_a = false;
      else if (y >= k) take_a = true;
      else take_a = da[x] < db[y] || (da[x] == db[y] && a[x] <= b[y]);
      const int64_t id = take_a ? a[x] : b[y];
      const double dv = take_a ? da[x] : db[y];
      if (take_a) ++x; else ++y;
      if (id == last && dv == lastd) continue;  // the same neighbour found by both lists
      oi[q * k + o] = id;
      od[q * k + o] = dv;
      last = id;
      lastd = dv;
      ++o;
    }
    for (; o < k; ++o) {  // cannot happen with two full lists of distinct ids; defensive
      oi[q * k + o] = last;
      od[q * k + o] = lastd;
    }
  }
}
}  // namespace
}  // namespace hks

extern "C" int hks_knn_merge(const int64_t* a_idx, const double* a_d2, const int64_t* b_idx, const double* b_d2,
                             int64_t n, int64_t k, int64_t* out_idx, double* out_d2, void* stream) {
  if (!a_idx || !a_d2 || !b_idx || !b_d2 || !out_idx || !out_d2 || n < 1 || k < 1)
    return set_error(HKS_ERR_INVALID, "hks_knn_merge: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  knn_merge_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(a_idx, a_d2, b_idx, b_d2, n,
                                                                                      (int)k, out_idx, out_d2);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_knn_merge: %s", cudaGetErrorString(e));
  return HKS_OK;
}
