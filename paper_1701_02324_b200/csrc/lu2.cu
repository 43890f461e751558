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
#include <cstdlib>

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
  for (int c = 0; c < pb; ++c) {  // coalesced column loads (LDGSTS: all in flight at once)
    const double* src = A + p0 + (size_t)(p0 + c) * lda;
    for (int i = tid; i < mr; i += PT) cp_async8(P + i + c * ldp, src + i, true);
  }
  cp_async_commit();
  cp_async_wait<0>();
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

// Panel factorization as a loop over blocks of U columns (fully unrolled
// 32-column variants are instruction-cache bound: the straight-line code
// does not fit and every column refetches it).  Row interchanges are
// relabellings: each thread keeps its physical rows and the logical row
// number (label) each one currently holds, so an interchange of rows jj and
// p is two label updates, never a data movement.  The working columns live
// in registers, shifted by U after every block so the block's columns sit at
// compile-time indices; finished columns are parked in shared memory by
// physical row and written to their final (label) rows at the end.  Pivot
// search: |x| as a 64-bit key (IEEE order of a non-negative double is its
// unsigned bit order; bit 63 marks a live row) reduced with three 32-bit
// warp reductions (max high word, max low word among the high-word winners,
// min row label among the key winners -- the lowest current row wins ties,
// as idamax); per-warp winners publish their keys, every thread reduces
// them after a barrier, and only the thread holding the pivot row publishes
// it (a second barrier) -- one row store per column instead of one per warp.
template <int PB, int RPT, int NT, int U>
__global__ void __launch_bounds__(NT) panel_loop_kernel(const Bases* __restrict__ bases_ptr,
                                                        const PanelDesc* __restrict__ descs) {
  constexpr int NW = NT / 32, NR = NT * RPT;
  const Bases& bases = *bases_ptr;
  const PanelDesc D = descs[blockIdx.x];
  double* A = at<double>(bases, D.A);
  int* piv = at<int>(bases, D.piv);
  const int lda = D.lda, p0 = D.p0, pb = D.pb, mr = D.n - D.p0;
  extern __shared__ __align__(16) double psm[];
  double* done = psm;               // [PB][NR] finished columns by physical row
  double* cand = psm + (PB + U) * NR;  // [2][NW][PB] per-warp candidate working rows
  __shared__ unsigned khi[2][NW], klo[2][NW], kid[2][NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double w[RPT][PB];
  int lab[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) lab[q] = tid + q * NT < mr ? tid + q * NT : 0x7fffffff;
#pragma unroll
  for (int c = 0; c < PB; ++c)
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int i = tid + q * NT;
      w[q][c] = (i < mr && c < pb) ? A[p0 + i + (size_t)(p0 + c) * lda] : 0.0;
    }
  // incoming permutations of this CTA's physical rows (identity where they start)
  int tp[RPT], gp[RPT];
  const int* tperm = D.tperm != kNull ? at<const int>(bases, D.tperm) : nullptr;
  const int* gperm = D.gperm != kNull ? at<const int>(bases, D.gperm) : nullptr;
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = p0 + tid + q * NT;
    tp[q] = (tperm && p0 > 0 && i < D.n) ? tperm[i] : i;
    gp[q] = (gperm && p0 > D.g0 && i < D.n) ? gperm[i] : i;
  }
  int info = 0;
#pragma unroll 1
  for (int j0 = 0; j0 < pb; j0 += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int jj = j0 + u;
      if (jj < pb) {
        const int par = jj & 1;
        unsigned long long key = 0;
        int ai = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          if (lab[q] >= jj && lab[q] < mr) {
            const unsigned long long k = (unsigned long long)__double_as_longlong(fabs(w[q][u])) | (1ull << 63);
            if (k > key || (k == key && lab[q] < ai)) {
              key = k;
              ai = lab[q];
            }
          }
        }
        const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
        const unsigned m1 = __reduce_max_sync(0xffffffffu, hi);
        const unsigned m2 = __reduce_max_sync(0xffffffffu, hi == m1 ? lo : 0u);
        const unsigned id = __reduce_min_sync(0xffffffffu, (hi == m1 && lo == m2) ? (unsigned)ai : 0xffffffffu);
        if (lane == 0) {
          khi[par][wid] = m1;
          klo[par][wid] = m2;
          kid[par][wid] = id;
        }
        __syncthreads();
        const unsigned h2 = lane < NW ? khi[par][lane] : 0u, l2 = lane < NW ? klo[par][lane] : 0u;
        const unsigned i2 = lane < NW ? kid[par][lane] : 0xffffffffu;
        const unsigned g1 = __reduce_max_sync(0xffffffffu, h2);
        const unsigned g2 = __reduce_max_sync(0xffffffffu, h2 == g1 ? l2 : 0u);
        const unsigned gi = __reduce_min_sync(0xffffffffu, (h2 == g1 && l2 == g2) ? i2 : 0xffffffffu);
        const int p = g1 != 0u ? (int)gi : jj;
        // only the pivot row is published (one thread), then a second barrier
        double* pr_w = cand + par * PB;
#pragma unroll
        for (int q = 0; q < RPT; ++q)
          if (lab[q] == p)
#pragma unroll
            for (int c = (u & ~1); c < PB; c += 2)
              *reinterpret_cast<double2*>(pr_w + c) = make_double2(w[q][c], w[q][c + 1]);
        __syncthreads();
        const double* pr = pr_w;
        const double pv = pr[u];
        if (tid == 0) {
          piv[p0 + jj] = p0 + p;
          if (pv == 0.0 && info == 0) info = p0 + jj + 1;
        }
        const bool recip = fabs(pv) >= DBL_MIN;
        const double inv = 1.0 / pv;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          if (lab[q] == p)  // interchange rows jj and p: relabel
            lab[q] = jj;
          else if (lab[q] == jj)
            lab[q] = p;
          if (lab[q] > jj && lab[q] < mr) {  // scale (dgetf2: reciprocal when safe), rank-1 update
            double l = w[q][u];
            if (pv != 0.0) {
              l = recip ? l * inv : l / pv;
              w[q][u] = l;
            }
#pragma unroll
            for (int c = u + 1; c < PB; ++c) w[q][c] -= l * pr[c];
          }
        }
      }
    }
    // columns j0 .. j0+U-1 are final for every row: park them, shift the rest down
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
#pragma unroll
      for (int u = 0; u < U; ++u) done[(j0 + u) * NR + tid + q * NT] = w[q][u];
#pragma unroll
      for (int c = 0; c + U < PB; ++c) w[q][c] = w[q][c + U];
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < RPT; ++q)
    if (lab[q] < mr) {
      for (int c = 0; c < pb; ++c) A[p0 + lab[q] + (size_t)(p0 + c) * lda] = done[c * NR + tid + q * NT];
      const int pos = p0 + lab[q];
      if (D.sig != kNull) at<int>(bases, D.sig)[pos] = p0 + tid + q * NT;
      if (tperm) at<int>(bases, D.tperm)[pos] = tp[q];
      if (gperm) at<int>(bases, D.gperm)[pos] = gp[q];
    }
  if (tid == 0 && info && D.info != kNull) {
    int* g = at<int>(bases, D.info);
    if (*g == 0) *g = info;  // panels run in order: keep the first zero pivot
  }
}

template <int PB, int RPT, int NT, int U>
cudaError_t launch_panel_loop(const Bases* b, const PanelDesc* d, int count, cudaStream_t s) {
  // done[] is PB + U rows deep: the last block may run past pb
  const size_t sm = (size_t)((PB + U) * NT * RPT + 2 * (NT / 32) * PB) * sizeof(double);
  raise_smem_limit(panel_loop_kernel<PB, RPT, NT, U>, sm);
  panel_loop_kernel<PB, RPT, NT, U><<<count, NT, sm, s>>>(b, d);
  return cudaGetLastError();
}

// A[i, c] := A[perm[i], c], rows [r0, r1), for a block of cb columns per
// CTA.  The rows the permutation moves are compacted first (a matrix that
// pivots little costs one scan of perm), then staged GS columns at a time
// through shared memory (all reads of a column chunk before any write).
constexpr int GS = 8;  // columns per staged chunk
__global__ void __launch_bounds__(256) gather_rows_kernel(const Bases* __restrict__ bases_ptr,
                                                          const GatherDesc* __restrict__ descs, int cb) {
  const Bases& bases = *bases_ptr;
  const GatherDesc D = descs[blockIdx.y];
  const int c0 = D.c0 + blockIdx.x * cb;
  if (c0 >= D.c1) return;
  const int nc = min(cb, D.c1 - c0), nr = D.r1 - D.r0;
  double* A = at<double>(bases, D.A) + D.r0 + (size_t)c0 * D.lda;
  const int* perm = at<const int>(bases, D.perm) + D.r0;
  extern __shared__ double gsm[];
  int* dst = reinterpret_cast<int*>(gsm + (size_t)nr * GS);  // moved rows: destination, source
  int* src = dst + nr;
  __shared__ int moved;
  if (threadIdx.x == 0) moved = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int i0 = 0; i0 < nr; i0 += blockDim.x) {  // warp-aggregated compaction
    const int i = i0 + threadIdx.x;
    const int sidx = i < nr ? perm[i] - D.r0 : i;
    const bool mv = i < nr && sidx != i;
    const unsigned bal = __ballot_sync(0xffffffffu, mv);
    int base = 0;
    if (lane == 0 && bal) base = atomicAdd(&moved, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (mv) {
      const int k = base + __popc(bal & ((1u << lane) - 1u));
      dst[k] = i;
      src[k] = sidx;
    }
  }
  __syncthreads();
  const int M = moved;
  if (M == 0) return;
  for (int cc = 0; cc < nc; cc += GS) {
    const int ncc = min(GS, nc - cc);
    for (int e = threadIdx.x; e < M * ncc; e += blockDim.x) {
      const int k = e % M, c = e / M;
      gsm[c * M + k] = A[src[k] + (size_t)(cc + c) * D.lda];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < M * ncc; e += blockDim.x) {
      const int k = e % M, c = e / M;
      A[dst[k] + (size_t)(cc + c) * D.lda] = gsm[c * M + k];
    }
    __syncthreads();
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
// upper), k <= 128, B k x ncols.  A CTA owns NC columns (one per thread,
// NC = 32/64/128 by the step's widest descriptor) held in shared memory.
// Per 32-row block: the contribution of the already-solved rows is one DMMA
// product (each warp a 32 x 32 tile), then every thread solves its column
// against the 32 x 32 diagonal block in registers, column-oriented (axpy)
// order so the 31 updates of each step are independent.  All global reads
// are LDGSTS (cp.async): the block of B and the first 32 rows of T are in
// flight together, and the next block's rows of T are prefetched into the
// second buffer while the current block computes.  Shared memory is sized
// by the step's largest k, so narrow / shallow solves pack several CTAs per
// SM.
template <bool UPPER, int NW>
__device__ __forceinline__ void trsm_stage_rows(double* Ts, int tts, const double* T, int ldt, int k, int b,
                                                int wid, int lane) {
  const int r0 = b * 32, nr = min(32, k - r0);
  const int klo = UPPER ? r0 : 0, khi = UPPER ? k : r0 + nr;
  const bool ok = lane < nr;
  for (int cc = klo + wid; cc < khi; cc += NW)
    cp_async8(Ts + lane * tts + cc, ok ? T + (r0 + lane) + (size_t)cc * ldt : T, ok);
}

// a / b, correctly rounded (bit-identical to the IEEE division), from the
// correctly rounded reciprocal y = 1 / b computed off the caller's
// dependency chain: q = a y, one FMA residual, one FMA correction
// (Markstein).  Three dependent operations instead of the division
// sequence; operands near the exponent limits branch to the division.
__device__ __noinline__ double div_slow(double a, double b) { return a / b; }
__device__ __forceinline__ double div_rn(double a, double b, double y) {
  const double aa = fabs(a), ab = fabs(b);
  const bool safe = (aa == 0.0 || (aa > 0x1p-900 && aa < 0x1p900)) && ab > 0x1p-900 && ab < 0x1p900;
  if (__builtin_expect(!safe, 0)) return div_slow(a, b);
  const double q = a * y;
  return fma(fma(-q, b, a), y, q);
}

// One triangular sweep X := T^-1 X over a k x NC block of right-hand sides
// already in shared memory (X row-major, ld NC + 4); T is read through the
// double-buffered 32-row staging area Tbuf (ld tts).  Ends with a barrier.
// Bin / Bout (optional, ld ldb): X comes from / goes back to global memory
// block by block -- each 32-row block of X is loaded (rows through `perm`
// when given) with the T rows of its step (one cp.async group, prefetched
// while the previous block computes) and stored as soon as it is final,
// instead of whole-X load / store phases.
template <bool UPPER, int NC, int NT = NC, bool SINGLE_T = false>
__device__ __forceinline__ void trsm_sweep(double* X, double* Tbuf, int tts, const double* T, int ldt, int k,
                                           int nc, const double* Bin = nullptr, double* Bout = nullptr,
                                           int ldb = 0, const int* perm = nullptr) {
  static_assert(NT == NC || (NC == 32 && (NT == 128 || NT == 256)) || NT == 2 * NC, "warp <-> tile mapping");
  constexpr int NW = NT / 32;
  constexpr int TXS = NC + 4;  // X row stride: == 4 (mod 16), conflict-free DMMA B fragments
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nblk = (k + 31) / 32;
  __shared__ double rdiag[32];
  auto stage_x = [&](int blk) {  // rows of X block blk, lanes along a column's rows
    const int xr0 = blk * 32, xnr = min(32, k - xr0);
    if (lane < xnr) {
      const int src = perm ? perm[xr0 + lane] : xr0 + lane;
      for (int c = wid; c < nc; c += NW) cp_async8(X + (xr0 + lane) * TXS + c, Bin + src + (size_t)c * ldb, true);
    }
  };
  auto store_x = [&](int blk) {
    const int xr0 = blk * 32, xnr = min(32, k - xr0);
    for (int c = wid; c < nc; c += NW)
      if (lane < xnr) Bout[xr0 + lane + (size_t)c * ldb] = X[(xr0 + lane) * TXS + c];
  };
  if (Bin) stage_x(UPPER ? nblk - 1 : 0);
  trsm_stage_rows<UPPER, NW>(Tbuf, tts, T, ldt, k, UPPER ? nblk - 1 : 0, wid, lane);
  cp_async_commit();
  const int fr = lane >> 2, fc = lane & 3;
  for (int bb = 0; bb < nblk; ++bb) {
    const int b = UPPER ? nblk - 1 - bb : bb;
    const int r0 = b * 32, nr = min(32, k - r0);
    double* Ts = SINGLE_T ? Tbuf : Tbuf + (bb & 1) * 32 * tts;
    cp_async_wait<0>();
    __syncthreads();  // X / this block's rows of T landed; the previous block's solve is complete
    if (Bout && bb > 0) store_x(UPPER ? b + 1 : b - 1);  // the previous block is final
    if (bb + 1 < nblk) {
      if (Bin) stage_x(UPPER ? b - 1 : b + 1);
      if (!SINGLE_T)  // next block's rows of T into the other buffer, behind this block's work
        trsm_stage_rows<UPPER, NW>(Tbuf + ((bb + 1) & 1) * 32 * tts, tts, T, ldt, k, UPPER ? b - 1 : b + 1, wid,
                                   lane);
      cp_async_commit();
    }
    // reciprocals of this block's diagonal, off the solve's dependency chain
    if (UPPER && tid < nr) rdiag[tid] = 1.0 / Ts[tid * tts + r0 + tid];
    // X[r0:r0+nr, :] -= T[r0:r0+nr, u] X[u, :] over the solved rows u (DMMA)
    const int ulo = UPPER ? r0 + nr : 0, uhi = UPPER ? k : r0;
    if (NT == 2 * NC && NC >= 64) {  // two warps per 32-column tile, 16 rows each
      const int tile = wid >> 1, rb = (wid & 1) * 16, cb = tile * 32;
      if (uhi > ulo && cb < nc) {
        double acc[2][4][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int kk = ulo; kk < uhi; kk += 4) {
          const int kq = kk + fc;
          const bool kin = kq < uhi;
          double a[2], bv[4];
#pragma unroll
          for (int i = 0; i < 2; ++i) a[i] = kin ? Ts[(rb + i * 8 + fr) * tts + kq] : 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) bv[j] = kin ? X[kq * TXS + cb + j * 8 + fr] : 0.0;
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], bv[j]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int rr = rb + i * 8 + fr, c = cb + j * 8 + 2 * fc + h;
              if (rr < nr) X[(r0 + rr) * TXS + c] -= acc[i][j][h];
            }
      }
    } else if (NT != NC) {  // 4 warps on one 32-column tile: warp w owns rows 8w .. 8w+7
      // (8 warps: warps 4..7 take the second half of the solved rows u and
      // subtract their partial sums after warps 0..3, a fixed order)
      constexpr int KSPLIT = NW / 4;
      const int part = wid / 4, rw = wid % 4;
      const int kh = KSPLIT == 1 ? uhi : ulo + ((uhi - ulo) / 8) * 4;
      const int klo2 = part == 0 ? ulo : kh, khi2 = part == 0 ? kh : uhi;
      double acc[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
      for (int kk = klo2; kk < khi2; kk += 4) {
        const int kq = kk + fc;
        const bool kin = kq < khi2;
        const double a = kin ? Ts[(rw * 8 + fr) * tts + kq] : 0.0;
        double bv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = kin ? X[kq * TXS + j * 8 + fr] : 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[j][0], acc[j][1], a, bv[j]);
      }
      const int rr = rw * 8 + fr;
#pragma unroll
      for (int p = 0; p < KSPLIT; ++p) {
        if (p > 0) __syncthreads();  // uniform: KSPLIT is a compile-time constant
        if (part == p && khi2 > klo2)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (rr < nr) X[(r0 + rr) * TXS + j * 8 + 2 * fc + h] -= acc[j][h];
      }
    } else if (uhi > ulo && wid * 32 < nc) {
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
        for (int i = 0; i < 4; ++i) a[i] = kin ? Ts[(i * 8 + fr) * tts + kq] : 0.0;
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
    }
    __syncthreads();
    // diagonal block: thread = column, values in registers
    if (tid < nc) {
      double x[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = i < nr ? X[(r0 + i) * TXS + tid] : 0.0;
      if (!UPPER) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
#pragma unroll
          for (int i = j + 1; i < 32; ++i) x[i] -= Ts[i * tts + r0 + j] * x[j];
        }
      } else {
#pragma unroll
        for (int j = 31; j >= 0; --j) {
          if (j < nr) {
            x[j] = div_rn(x[j], Ts[j * tts + r0 + j], rdiag[j]);  // == x[j] / T(j, j), as dtrsm (c5 is sensitive to it)
#pragma unroll
            for (int i = 0; i < j; ++i) x[i] -= Ts[i * tts + r0 + j] * x[j];
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < nr) X[(r0 + i) * TXS + tid] = x[i];
    }
    if (SINGLE_T && bb + 1 < nblk) {  // one T buffer (half the staging smem): refill once it is read
      __syncthreads();
      trsm_stage_rows<UPPER, NW>(Tbuf, tts, T, ldt, k, UPPER ? b - 1 : b + 1, wid, lane);
      cp_async_commit();
    }
  }
  __syncthreads();
  if (Bout) store_x(UPPER ? 0 : nblk - 1);
}

template <bool UPPER, int NC, int NT, bool SINGLE_T = false>
__global__ void __launch_bounds__(NT) trsm_kernel(const Bases* __restrict__ bases_ptr,
                                                  const TrsmDesc* __restrict__ descs, int kcap, int tts) {
  constexpr int TXS = NC + 4;
  const Bases& bases = *bases_ptr;
  const TrsmDesc D = descs[blockIdx.y];
  const int c0 = blockIdx.x * NC;
  if (c0 >= D.ncols) return;
  const int nc = min(NC, D.ncols - c0), k = D.k;
  const double* T = at<const double>(bases, D.T);
  double* B = at<double>(bases, D.B) + (size_t)c0 * D.ldb;
  extern __shared__ double tsm[];
  double* X = tsm;                    // k x NC, row-major (ld TXS)
  double* Tbuf = tsm + kcap * TXS;    // 2 x 32 rows of T, row-major (ld tts)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  (void)lane;
  (void)wid;
  // X streams in and out block by block inside the sweep (256-byte coalesced
  // LDGSTS along each column's rows)
  trsm_sweep<UPPER, NC, NT, SINGLE_T>(X, Tbuf, tts, T, D.ldt, k, nc, B, B, D.ldb);
}

// Whole getrs of a small matrix (n <= kGetrsFusedMax) in one CTA per block of
// NC right-hand-side columns: the recorded total row permutation is applied
// while B is gathered into shared memory, then the unit-lower and upper
// sweeps run back to back, one store at the end.  Replaces 2 + 4 n/128
// level-wide launches of the solve program.
template <int NC, int NT>
__global__ void __launch_bounds__(NT) getrs_fused_kernel(const Bases* __restrict__ bases_ptr,
                                                         const GetrsDesc* __restrict__ descs, int kcap, int tts) {
  constexpr int TXS = NC + 4;
  const Bases& bases = *bases_ptr;
  const GetrsDesc D = descs[blockIdx.y];
  const int c0 = blockIdx.x * NC;
  if (c0 >= D.ncols) return;
  const int nc = min(NC, D.ncols - c0), n = D.n;
  const double* LU = at<const double>(bases, D.LU);
  const int* perm = at<const int>(bases, D.perm);
  double* B = at<double>(bases, D.B) + (size_t)c0 * D.ldb;
  const double* Bin = D.Bin != kNull ? at<const double>(bases, D.Bin) + (size_t)c0 * D.ldb : B;
  extern __shared__ double tsm[];
  double* X = tsm;
  double* Tbuf = tsm + kcap * TXS;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // the whole gathered B in flight at once (measured: better than streaming
  // it block by block into the latency-bound sweeps)
  for (int i = lane; i < n; i += 32) {
    const int src = perm[i];
    for (int c = wid; c < nc; c += NT / 32) cp_async8(X + i * TXS + c, Bin + src + (size_t)c * D.ldb, true);
  }
  if (D.lower) trsm_sweep<false, NC, NT>(X, Tbuf, tts, LU, D.lda, n, nc);
  trsm_sweep<true, NC, NT>(X, Tbuf, tts, LU, D.lda, n, nc, nullptr, B, D.ldb);  // stores streamed out
}

// ||A||_1 (max column abs sum) of each n x n matrix, before factoring.
// One warp per column, lanes along the rows (coalesced).
__global__ void norm1_kernel(const Bases* __restrict__ bases_ptr, const LuDesc* __restrict__ descs) {
  const Bases& bases = *bases_ptr;
  const LuDesc L = descs[blockIdx.x];
  __shared__ double rv[32];
  __shared__ int ri[32];
  const double* A = at<const double>(bases, L.A);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double best = 0.0;
  for (int c = wid; c < L.n; c += nw) {
    const double* col = A + (size_t)c * L.lda;
    double s = 0.0;
    for (int r = lane; r < L.n; r += 32) s += fabs(col[r]);
    best = fmax(best, warp_sum(s));
  }
  ArgMax m = block_argmax(ArgMax{best, (int)threadIdx.x}, rv, ri);
  if (threadIdx.x == 0 && L.anorm != kNull) *at<double>(bases, L.anorm) = m.v;
  if (threadIdx.x == 0 && L.info != kNull) *at<int>(bases, L.info) = 0;
}

}  // namespace

cudaError_t launch_panel_batched(const Bases* b, const PanelDesc* d, int count, int max_rows, int pb,
                                 cudaStream_t s) {
  if (count <= 0 || max_rows <= 0) return cudaSuccess;
  // 256 threads, one to four rows each; PB x RPT doubles stay in registers.
  // plan.cu uses pb = 32 only for rows <= 256 (panel32_max_rows).
  const int rpt = (max_rows + 255) / 256;
  // 257..512 rows (leaf blocks): 512 threads, one row each -- twice the
  // warps of the 256 x 2 layout hide more of the per-column latency chain
  if (max_rows > 256 && max_rows <= 512 && pb > 16 && pb <= 32)
    return launch_panel_loop<32, 1, 512, 8>(b, d, count, s);
  static const bool narrow1024 = getenv("HKS_PANEL_NARROW") != nullptr;  // development knob
  if (!narrow1024 && max_rows > 512 && max_rows <= 1024 && pb <= 16)
    return launch_panel_loop<16, 2, 512, 8>(b, d, count, s);
  if (pb > 32) {
    if (rpt == 1) return launch_panel_loop<64, 1, 256, 16>(b, d, count, s);
  } else if (pb > 16) {
    if (rpt == 1) return launch_panel_loop<32, 1, 256, 8>(b, d, count, s);
    if (rpt == 2) return launch_panel_loop<32, 2, 256, 8>(b, d, count, s);
  } else {
    switch (rpt) {
      case 1: return launch_panel_loop<16, 1, 256, 8>(b, d, count, s);
      case 2: return launch_panel_loop<16, 2, 256, 8>(b, d, count, s);
      case 3: return launch_panel_loop<16, 3, 256, 8>(b, d, count, s);
      case 4: return launch_panel_loop<16, 4, 256, 8>(b, d, count, s);
      default: break;
    }
  }
  // taller panels: shared-memory panel (no permutation tracking: plan.cu
  // falls back to interchange sweeps for matrices above kPermMaxRows)
  const int ldp = max_rows;
  if (pb <= 16) {
    const size_t sm = (size_t)ldp * 16 * sizeof(double);
    raise_smem_limit(panel_kernel<16>, sm);
    panel_kernel<16><<<count, PT, sm, s>>>(b, d, ldp);
  } else {
    const size_t sm = (size_t)ldp * 32 * sizeof(double);
    raise_smem_limit(panel_kernel<32>, sm);
    panel_kernel<32><<<count, PT, sm, s>>>(b, d, ldp);
  }
  return cudaGetLastError();
}

cudaError_t launch_gather_batched(const Bases* b, const GatherDesc* d, int count, int max_rows, int max_cols,
                                  cudaStream_t s) {
  if (count <= 0 || max_rows <= 0 || max_cols <= 0) return cudaSuccess;
  // columns per CTA: one perm scan per 64 columns; narrow batches (the top
  // levels) take one staged chunk per CTA instead of a chain of 8
  const int cb = (long long)count * ((max_cols + 63) / 64) < 148 ? GS : 64;
  const size_t sm = (size_t)max_rows * GS * sizeof(double) + 2 * (size_t)max_rows * sizeof(int);
  raise_smem_limit(gather_rows_kernel, sm);
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    gather_rows_kernel<<<dim3((max_cols + cb - 1) / cb, cnt), 256, sm, s>>>(b, d + first, cb);
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

template <bool UPPER, int NC, int NT = NC, bool SINGLE_T = false>
static cudaError_t launch_trsm_nc(const Bases* b, const TrsmDesc* d, int count, int max_cols, int max_k,
                                  cudaStream_t s) {
  // tts == 4 (mod 16), and > every column r0 + 31 the register diagonal solve touches
  const int kcap = (max_k + 31) / 32 * 32, tts = kcap + 4;
  const size_t sm = (size_t)(kcap * (NC + 4) + (SINGLE_T ? 1 : 2) * 32 * tts) * sizeof(double);
  raise_smem_limit(trsm_kernel<UPPER, NC, NT, SINGLE_T>, sm);
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    trsm_kernel<UPPER, NC, NT, SINGLE_T><<<dim3((max_cols + NC - 1) / NC, cnt), NT, sm, s>>>(b, d + first, kcap,
                                                                                          tts);
  }
  return cudaGetLastError();
}

template <bool UPPER>
static cudaError_t launch_trsm_t(const Bases* b, const TrsmDesc* d, int count, int max_cols, int max_k,
                                 cudaStream_t s) {
  static const int cap = [] {  // development knob: widest column block per CTA
    const char* e = getenv("HKS_TRSM_NC");
    return e ? atoi(e) : 128;
  }();
  // experiment knob: 64-column blocks with 4 warps and one T staging buffer
  // (103 KB of shared memory at k = 128: two CTAs per SM instead of one)
  static const int single_t = [] {
    const char* e = getenv("HKS_TRSM_SINGLE_T");
    return e ? atoi(e) : 0;
  }();
  if (single_t && max_cols > 32) return launch_trsm_nc<UPPER, 64, 128, true>(b, d, count, max_cols, max_k, s);
  // few matrices (the narrow top levels): 32-column blocks, 4x the CTAs for
  // the latency-bound sweeps; wide batches keep 128 (more reuse of T)
  const bool narrow_batch = (long long)count * ((max_cols + 127) / 128) < 96;
  if (max_cols <= 32 || cap == 32 || (narrow_batch && cap == 128))
    return launch_trsm_nc<UPPER, 32, 128>(b, d, count, max_cols, max_k, s);
  // wide upper solves (the leaf backward sweep): 8 warps per 128 columns --
  // the CTA is alone on its SM (202 KB of staging), so more warps hide the
  // division chain and the loads (measured -23%); lower solves gain nothing
  if (cap == 256 || (UPPER && cap == 128 && max_cols > 64))
    return launch_trsm_nc<UPPER, 128, 256>(b, d, count, max_cols, max_k, s);
  if (cap == 64) return launch_trsm_nc<UPPER, 64>(b, d, count, max_cols, max_k, s);
  if (max_cols <= 64) return launch_trsm_nc<UPPER, 64>(b, d, count, max_cols, max_k, s);
  return launch_trsm_nc<UPPER, 128>(b, d, count, max_cols, max_k, s);
}

cudaError_t launch_trsm_batched(const Bases* b, const TrsmDesc* d, int count, int max_cols, int max_k, bool upper,
                                cudaStream_t s) {
  if (count <= 0 || max_cols <= 0 || max_k <= 0) return cudaSuccess;
  if (max_k > 128) return cudaErrorInvalidValue;
  return upper ? launch_trsm_t<true>(b, d, count, max_cols, max_k, s)
               : launch_trsm_t<false>(b, d, count, max_cols, max_k, s);
}

cudaError_t launch_getrs_fused(const Bases* b, const GetrsDesc* d, int count, int max_n, int max_cols,
                               cudaStream_t s) {
  if (count <= 0 || max_n <= 0 || max_cols <= 0) return cudaSuccess;
  if (max_n > kGetrsFusedMax) return cudaErrorInvalidValue;
  constexpr int NC = 32;
  const int kcap = (max_n + 31) / 32 * 32, tts = kcap + 4;
  const size_t sm = (size_t)(kcap * (NC + 4) + 2 * 32 * tts) * sizeof(double);
  // few matrices (the solve's top levels): 8 warps, the sweeps' updates
  // split over the solved rows
  const bool wide = (long long)count * ((max_cols + NC - 1) / NC) < 96 && getenv("HKS_GETRS_NT128") == nullptr;
  if (wide) raise_smem_limit(getrs_fused_kernel<NC, 256>, sm);
  else raise_smem_limit(getrs_fused_kernel<NC, 128>, sm);
  for (int first = 0; first < count; first += 65535) {
    const int cnt = count - first < 65535 ? count - first : 65535;
    if (wide)
      getrs_fused_kernel<NC, 256><<<dim3((max_cols + NC - 1) / NC, cnt), 256, sm, s>>>(b, d + first, kcap, tts);
    else
      getrs_fused_kernel<NC, 128><<<dim3((max_cols + NC - 1) / NC, cnt), 128, sm, s>>>(b, d + first, kcap, tts);
  }
  return cudaGetLastError();
}

cudaError_t launch_norm1_batched(const Bases* b, const LuDesc* d, int count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  // few matrices (the top levels, where the norm gates the level's LU):
  // 32 warps per matrix; the column sums and their max do not depend on it
  norm1_kernel<<<count, count < 148 ? 1024 : 256, 0, s>>>(b, d);
  return cudaGetLastError();
}

}  // namespace hks
