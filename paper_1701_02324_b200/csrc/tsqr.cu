// Tall-skinny Householder QR pre-reduction for the skeletonization blocks.
//
// knn_augmented sampling returns every outside neighbour of a node
// (skeleton.py:111-114): the sampled block K(X[rows], X[cands]) of a C3 node
// has 3.5 k (leaves) to 150 k (level 1) rows for at most 512 candidate
// columns, and the reference's pivoted QR (linalg.py:75-102) streams that
// whole block at every one of its <= max_rank steps.  Column norms of the
// trailing matrix are invariant under orthogonal row transformations, so the
// pivots, the stopping step and R11^-1 R12 (the interpolation coefficients)
// of the QRCP of A equal those of the QRCP of the c x c triangular factor R
// of A = Q R.  This file computes R, one pass over A on the tensor pipe; the
// QRCP kernels (qrcp.cu) then run on R.
//
// R (c x c, row-major, upper triangular) absorbs the rows of A slab by slab:
// for a slab S of B rows the stacked matrix [R; S] is re-triangularised by
// Householder reflectors that each touch one row of R and the rows of S
// (the structured QR update).  Per 32-column panel: the panel of S and the
// diagonal block of R are factored in shared memory (dlarfg reflectors,
// v = [e_k; v_s]), the block reflector I - V T V^T is formed (dlarft; the
// top of V is the identity so V^T V = I + Vs^T Vs), and the trailing columns
// are updated 16 at a time, streamed through three cp.async buffers in shared
// memory (two tiles in flight), with DMMA products per tile: W = R_rows +
// Vs^T S_t, W2 = T^T W, R_rows -= W2, S_t -= Vs W2 (stored straight from the
// accumulators; a panel's own columns of S are dead once factored and are
// never written back).  "One pass over A" above means one read and one
// write of the slab's trailing columns per 32-column panel; 2 c^2 flops per
// absorbed row, the cost of an unpivoted QR.
// One CTA per (node, row chunk) job; the chunks' triangles are merged
// pairwise by the same kernel (a triangular source skips its zero panels).
// Every reduction has a fixed order: results are deterministic.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "hks_internal.h"

namespace hks {
namespace {

constexpr int TNT = 256;  // threads
constexpr int TNW = TNT / 32;
constexpr int TPB = 32;   // panel width
constexpr int TTW = 16;   // trailing tile width

constexpr int TWLD = 20;  // ld of W / W2 (== 4 mod 16: conflict-free DMMA B fragments)
constexpr int TTLD = 36;  // ld of T^T
constexpr int TNB = 3;    // trailing tile buffers (two tiles in flight)

template <int B>
struct TsqrSmem {
  static constexpr int LD = B + 4;  // == 4 (mod 16)
  double Vs[TPB * LD];              // panel of S, column-major (v_s after the panel is factored)
  double St[TNB][TTW * LD];         // trailing tiles, column-major
  double Tt[TPB * TTLD];            // T^T of the block reflector (Tt[k][i] = T[i][k])
  // one scratch region, three lives: the diagonal block of R (row-major ld
  // 33) while the panel is factored, the Gram matrix Vs^T Vs (ld 32) while T
  // is built, then W and W2 (ld 20) in the trailing loop
  double X[2 * TPB * TWLD > TPB * 33 ? 2 * TPB * TWLD : TPB * 33];
  double tau[TPB];
};

template <int B>
__device__ __forceinline__ void tsqr_load_tile(double* St, const double* S, int lds, int s0, int nb, int col0, int c,
                                               int wid, int lane) {
  constexpr int LD = TsqrSmem<B>::LD;
  // a warp instruction covers 4 rows x 8 columns: 64-byte row segments in
  // global memory, 16 distinct shared-memory banks per half warp
  const int rr = lane & 3, cc = lane >> 2;
#pragma unroll
  for (int it = 0; it < B / 32; ++it) {
    const int row = 4 * (wid + TNW * it) + rr;
#pragma unroll
    for (int h = 0; h < TTW / 8; ++h) {
      const int col = 8 * h + cc;
      const bool ok = row < nb && col0 + col < c;
      cp_async8(St + col * LD + row, ok ? S + (size_t)(s0 + row) * lds + col0 + col : S, ok);
    }
  }
}

// dlarfg on [R_kk; x]: x (this lane's rows of column k, in registers) becomes
// v_s in shared memory, R_kk becomes beta, tau[k] is published (one warp).
template <int B>
__device__ __forceinline__ void tsqr_reflector(TsqrSmem<B>& sm, double* Rd, int k, const double (&x)[B / 32],
                                               int lane) {
  constexpr int LD = TsqrSmem<B>::LD;
  double ss = 0.0;
#pragma unroll
  for (int q = 0; q < B / 32; ++q) ss = fma(x[q], x[q], ss);
  ss = warp_sum(ss);
  const double x0 = Rd[k * 33 + k];
  double tau = 0.0;
  if (ss > 0.0) {
    // beta = -sign(x0) ||[x0; x]||, tau = (beta - x0) / beta, v_s = x / (x0 - beta):
    // one division for both quotients (the reflector is orthogonal to roundoff either way)
    const double beta = -copysign(sqrt(fma(x0, x0, ss)), x0);
    const double d = x0 - beta, bd = beta * d;
    double scale;
    if (fabs(bd) >= 1e-290 && fabs(bd) <= 1e290) {
      const double rcp = 1.0 / bd;
      scale = beta * rcp;
      tau = -(d * d) * rcp;
    } else {
      scale = 1.0 / d;
      tau = (beta - x0) / beta;
    }
#pragma unroll
    for (int q = 0; q < B / 32; ++q) sm.Vs[k * LD + lane + 32 * q] = x[q] * scale;
    if (lane == 0) Rd[k * 33 + k] = beta;
  }
  if (lane == 0) sm.tau[k] = tau;
}

template <int B>
__global__ void __launch_bounds__(TNT, B <= 128 ? 2 : 1) tsqr_absorb_kernel(const TsqrJob* __restrict__ jobs) {
  constexpr int LD = TsqrSmem<B>::LD;
  constexpr int RQ = B / 32;  // rows per lane in the panel factorization
  constexpr int CW = TPB / TNW;  // panel columns per warp
  extern __shared__ __align__(16) unsigned char tsqr_raw[];
  TsqrSmem<B>& sm = *reinterpret_cast<TsqrSmem<B>*>(tsqr_raw);
  const TsqrJob J = jobs[blockIdx.x];
  const int c = J.c, lds = J.lds;
  double* __restrict__ R = J.R;
  double* __restrict__ S = J.S;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  double* Rd = sm.X;
  double* G = sm.X;
  double* Wm = sm.X;
  double* W2 = sm.X + TPB * TWLD;

  for (int s0 = 0; s0 < J.nrows; s0 += B) {
    const int nb = min(B, J.nrows - s0);
    // a triangular source (another chunk's R) has zeros left of its diagonal
    const int pstart = J.tri ? s0 / TPB : 0;
    for (int j0 = pstart * TPB; j0 < c; j0 += TPB) {
      const int ntile = (c - j0 - TPB + TTW - 1) / TTW;  // trailing tiles (<= 0: none)
      // ---- stage the panel of S, the diagonal block of R and the first two trailing tiles
      __syncthreads();  // the previous panel's trailing loop is complete
      {
        const int rr = lane & 3, cc = lane >> 2;
#pragma unroll
        for (int it = 0; it < B / 32; ++it) {
          const int row = 4 * (wid + TNW * it) + rr;
#pragma unroll
          for (int h = 0; h < TPB / 8; ++h) {
            const int col = 8 * h + cc;
            const bool ok = row < nb && j0 + col < c;
            cp_async8(sm.Vs + col * LD + row, ok ? S + (size_t)(s0 + row) * lds + j0 + col : S, ok);
          }
        }
      }
      cp_async_commit();
      if (ntile > 0) tsqr_load_tile<B>(sm.St[0], S, lds, s0, nb, j0 + TPB, c, wid, lane);
      cp_async_commit();
      if (ntile > 1) tsqr_load_tile<B>(sm.St[1], S, lds, s0, nb, j0 + TPB + TTW, c, wid, lane);
      cp_async_commit();
      for (int e = tid; e < TPB * TPB; e += TNT) {
        const int i = e >> 5, k = e & 31;
        Rd[i * 33 + k] = (j0 + i < c && j0 + k < c && k >= i) ? R[(size_t)(j0 + i) * c + j0 + k] : 0.0;
      }
      cp_async_wait<2>();
      __syncthreads();
      // ---- panel factorization: warp w owns columns w, w + 8, w + 16, w + 24.
      // Step k: every warp applies reflector k to its columns j > k (the four
      // dot products reduced together); the owner of column k + 1 then forms
      // reflector k + 1 from the registers it just updated, ahead of the barrier.
      if (wid == 0) {
        double x[RQ];
#pragma unroll
        for (int q = 0; q < RQ; ++q) x[q] = sm.Vs[lane + 32 * q];
        tsqr_reflector<B>(sm, Rd, 0, x, lane);
      }
      __syncthreads();
      for (int k = 0; k < TPB; ++k) {
        const double tau = sm.tau[k];
        double v[RQ], a[CW][RQ], dot[CW], rk[CW];
#pragma unroll
        for (int q = 0; q < RQ; ++q) v[q] = sm.Vs[k * LD + lane + 32 * q];
#pragma unroll
        for (int t = 0; t < CW; ++t) {
          const int j = wid + TNW * t;
          dot[t] = 0.0;
          rk[t] = j > k ? Rd[k * 33 + j] : 0.0;
#pragma unroll
          for (int q = 0; q < RQ; ++q) {
            a[t][q] = j > k ? sm.Vs[j * LD + lane + 32 * q] : 0.0;
            dot[t] = fma(v[q], a[t][q], dot[t]);
          }
        }
        {
          // four sums over the warp in 6 + 4 shuffles instead of 20: the first
          // two butterfly rounds also hand each lane ONE of the four columns
          // (lanes 16..31 keep columns 2, 3; odd 8-lane groups keep the odd
          // one), three rounds finish it inside the 8-lane group, and the
          // totals are broadcast from lanes 0, 8, 16, 24.  Fixed order.
          static_assert(CW == 4, "butterfly reduction is written for four columns per warp");
          const bool b4 = (lane & 16) != 0, b3 = (lane & 8) != 0;
          const double s0 = b4 ? dot[0] : dot[2], s1 = b4 ? dot[1] : dot[3];
          double k0 = b4 ? dot[2] : dot[0], k1 = b4 ? dot[3] : dot[1];
          k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
          k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
          double kq = b3 ? k1 : k0;
          kq += __shfl_xor_sync(0xffffffffu, b3 ? k0 : k1, 8);
          kq += __shfl_xor_sync(0xffffffffu, kq, 4);
          kq += __shfl_xor_sync(0xffffffffu, kq, 2);
          kq += __shfl_xor_sync(0xffffffffu, kq, 1);
#pragma unroll
          for (int t = 0; t < CW; ++t) dot[t] = __shfl_sync(0xffffffffu, kq, 8 * t);
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < CW; ++t) {
          const int j = wid + TNW * t;
          if (j > k) {
            const double tw = tau * (rk[t] + dot[t]);
            if (lane == 0) Rd[k * 33 + j] = rk[t] - tw;
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
              a[t][q] = fma(-tw, v[q], a[t][q]);
              sm.Vs[j * LD + lane + 32 * q] = a[t][q];
            }
          }
        }
        if (k + 1 < TPB && ((k + 1) & (TNW - 1)) == wid) {
          double x[RQ];
          const int ts = (k + 1) >> 3;
#pragma unroll
          for (int q = 0; q < RQ; ++q) {
            x[q] = a[0][q];
#pragma unroll
            for (int t = 1; t < CW; ++t) x[q] = t == ts ? a[t][q] : x[q];
          }
          tsqr_reflector<B>(sm, Rd, k + 1, x, lane);
        }
        __syncthreads();
      }
      // ---- R's diagonal block back; Gram matrix G = Vs^T Vs
      for (int e = tid; e < TPB * TPB; e += TNT) {
        const int i = e >> 5, k = e & 31;
        if (k >= i && j0 + k < c) R[(size_t)(j0 + i) * c + j0 + k] = Rd[i * 33 + k];
      }
      if (ntile <= 0) continue;  // last panel: nothing to update (uniform)
      __syncthreads();           // Rd is read; G takes its place
      {
        const int mf = wid >> 1, nf0 = (wid & 1) * 2;
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        for (int kk = 0; kk < B; kk += 4) {
          const double av = sm.Vs[(8 * mf + fr) * LD + kk + fc];
#pragma unroll
          for (int n = 0; n < 2; ++n) {
            const double bv = sm.Vs[(8 * (nf0 + n) + fr) * LD + kk + fc];
            dmma884(acc[n][0], acc[n][1], av, bv);
          }
        }
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int h = 0; h < 2; ++h) G[(8 * mf + fr) * 32 + 8 * (nf0 + n) + 2 * fc + h] = acc[n][h];
      }
      __syncthreads();
      // ---- T (dlarft, forward columnwise): T[k,k] = tau_k, T[0:k,k] = -tau_k T[0:k,0:k] G[0:k,k];
      // stored transposed (lane = row i of T)
      if (wid == 0) {
        for (int k = 0; k < TPB; ++k) {
          const double tk = sm.tau[k];
          double sacc = 0.0;
          if (lane < k)
            for (int l = lane; l < k; ++l) sacc = fma(sm.Tt[l * TTLD + lane], G[l * 32 + k], sacc);
          __syncwarp();
          sm.Tt[k * TTLD + lane] = lane < k ? -tk * sacc : (lane == k ? tk : 0.0);
          __syncwarp();
        }
      }
      // ---- trailing tiles: warp = fragment (mf, nf) of the 32 x 16 W / W2, rows [wid B/8, +B/8) of S_t
      const int mf = wid >> 1, nf = wid & 1;
      for (int t = 0; t < ntile; ++t) {
        const int col0 = j0 + TPB + t * TTW;
        const double* St = sm.St[t % TNB];
        // this lane's two entries of R_rows (consumed after the first product)
        double rold[2];
        bool rok[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          rok[h] = j0 + 8 * mf + fr < c && col0 + 8 * nf + 2 * fc + h < c;
          rold[h] = rok[h] ? R[(size_t)(j0 + 8 * mf + fr) * c + col0 + 8 * nf + 2 * fc + h] : 0.0;
        }
        cp_async_wait<1>();
        __syncthreads();  // tile t landed; everyone is done with tile t-1, W, W2 (and T is built)
        if (t + 2 < ntile)
          tsqr_load_tile<B>(sm.St[(t + 2) % TNB], S, lds, s0, nb, col0 + 2 * TTW, c, wid, lane);
        cp_async_commit();
        // W = R_rows + Vs^T S_t, one 8 x 8 fragment per warp over all B rows
        {
          double acc[4][2];  // four independent chains over interleaved k steps, summed in a fixed order
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[u][0] = acc[u][1] = 0.0;
          const double* ap = sm.Vs + (8 * mf + fr) * LD + fc;
          const double* bp = St + (8 * nf + fr) * LD + fc;
#pragma unroll 2
          for (int kk = 0; kk < B; kk += 16) {
            double av[4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              av[u] = ap[kk + 4 * u];
              bv[u] = bp[kk + 4 * u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) dmma884(acc[u][0], acc[u][1], av[u], bv[u]);
          }
          Wm[(8 * mf + fr) * TWLD + 8 * nf + 2 * fc] = rold[0] + ((acc[0][0] + acc[1][0]) + (acc[2][0] + acc[3][0]));
          Wm[(8 * mf + fr) * TWLD + 8 * nf + 2 * fc + 1] = rold[1] + ((acc[0][1] + acc[1][1]) + (acc[2][1] + acc[3][1]));
        }
        __syncthreads();
        // W2 = T^T W (T upper triangular: rows 0 .. 8 mf + 7 of W), R_rows -= W2
        {
          double a0 = 0.0, a1 = 0.0;
          for (int kk = 0; kk < 8 * (mf + 1); kk += 4) {
            const double av = sm.Tt[(8 * mf + fr) * TTLD + kk + fc];
            const double bv = Wm[(kk + fc) * TWLD + 8 * nf + fr];
            dmma884(a0, a1, av, bv);
          }
          W2[(8 * mf + fr) * TWLD + 8 * nf + 2 * fc] = a0;
          W2[(8 * mf + fr) * TWLD + 8 * nf + 2 * fc + 1] = a1;
          if (rok[0]) R[(size_t)(j0 + 8 * mf + fr) * c + col0 + 8 * nf + 2 * fc] = rold[0] - a0;
          if (rok[1]) R[(size_t)(j0 + 8 * mf + fr) * c + col0 + 8 * nf + 2 * fc + 1] = rold[1] - a1;
        }
        __syncthreads();
        // S_t -= Vs W2, straight from the accumulators to global memory
        {
          constexpr int MF = B / 64;
          const int r0 = wid * (B / 8);
          double acc[MF][2][2];
#pragma unroll
          for (int m = 0; m < MF; ++m)
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
              for (int h = 0; h < 2; ++h) acc[m][n][h] = St[(8 * n + 2 * fc + h) * LD + r0 + 8 * m + fr];
#pragma unroll
          for (int kk = 0; kk < TPB; kk += 4) {
            double av[MF], bv[2];
#pragma unroll
            for (int m = 0; m < MF; ++m) av[m] = -sm.Vs[(kk + fc) * LD + r0 + 8 * m + fr];
#pragma unroll
            for (int n = 0; n < 2; ++n) bv[n] = W2[(kk + fc) * TWLD + 8 * n + fr];
#pragma unroll
            for (int m = 0; m < MF; ++m)
#pragma unroll
              for (int n = 0; n < 2; ++n) dmma884(acc[m][n][0], acc[m][n][1], av[m], bv[n]);
          }
#pragma unroll
          for (int m = 0; m < MF; ++m) {
            const int row = r0 + 8 * m + fr;
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int col = col0 + 8 * n + 2 * fc + h;
                if (row < nb && col < c) S[(size_t)(s0 + row) * lds + col] = acc[m][n][h];
              }
          }
        }
      }
    }
  }
}

template <int B>
cudaError_t launch_tsqr(const TsqrJob* d_jobs, int count, cudaStream_t s) {
  const size_t sm = sizeof(TsqrSmem<B>);
  cudaError_t e = raise_smem_limit(tsqr_absorb_kernel<B>, sm);
  if (e != cudaSuccess) return e;
  tsqr_absorb_kernel<B><<<count, TNT, sm, s>>>(d_jobs);
  return cudaGetLastError();
}

}  // namespace

int tsqr_slab_rows() {
  static const int v = [] {
    const char* e = getenv("HKS_TSQR_SLAB");
    return e && atoi(e) == 256 ? 256 : 128;
  }();
  return v;
}

cudaError_t launch_tsqr_absorb(const TsqrJob* d_jobs, int count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  return tsqr_slab_rows() == 256 ? launch_tsqr<256>(d_jobs, count, s) : launch_tsqr<128>(d_jobs, count, s);
}

}  // namespace hks
