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
// are updated 16 at a time, double-buffered through shared memory, with two
// DMMA products per tile: W = R_rows + Vs^T S_t, W2 = T^T W, R_rows -= W2,
// S_t -= Vs W2.  2 c^2 flops per absorbed row, the cost of an unpivoted QR.
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
constexpr int TW2LD = 20; // ld of W2 (== 4 mod 16: conflict-free DMMA B fragments)

template <int B>
struct TsqrSmem {
  static constexpr int LD = B + 4;  // == 4 (mod 16)
  double Vs[TPB * LD];              // panel of S, column-major (v_s after the panel is factored)
  double St[2][TTW * LD];           // trailing tiles, column-major
  double Wp[4][TPB * TTW];          // split-K partials of Vs^T S_t; Wp[0] then holds W; also the Gram matrix
  double T[TPB * 33];               // block reflector factor, row-major ld 33
  double Rd[TPB * 33];              // diagonal block of R, row-major ld 33
  double W2[TPB * TW2LD];           // T^T W
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

template <int B>
__global__ void __launch_bounds__(TNT, B <= 128 ? 2 : 1) tsqr_absorb_kernel(const TsqrJob* __restrict__ jobs) {
  constexpr int LD = TsqrSmem<B>::LD;
  constexpr int RQ = B / 32;  // rows per lane in the panel factorization
  extern __shared__ __align__(16) unsigned char tsqr_raw[];
  TsqrSmem<B>& sm = *reinterpret_cast<TsqrSmem<B>*>(tsqr_raw);
  const TsqrJob J = jobs[blockIdx.x];
  const int c = J.c, lds = J.lds;
  double* __restrict__ R = J.R;
  double* __restrict__ S = J.S;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int fr = lane >> 2, fc = lane & 3;

  for (int s0 = 0; s0 < J.nrows; s0 += B) {
    const int nb = min(B, J.nrows - s0);
    // a triangular source (another chunk's R) has zeros left of its diagonal
    const int pstart = J.tri ? s0 / TPB : 0;
    for (int j0 = pstart * TPB; j0 < c; j0 += TPB) {
      const int ntile = (c - j0 - TPB + TTW - 1) / TTW;  // trailing tiles (<= 0: none)
      // ---- stage the panel of S, the diagonal block of R and the first trailing tile
      __syncthreads();  // the previous panel's last tile is written out
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
      for (int e = tid; e < TPB * TPB; e += TNT) {
        const int i = e >> 5, k = e & 31;
        sm.Rd[i * 33 + k] = (j0 + i < c && j0 + k < c && k >= i) ? R[(size_t)(j0 + i) * c + j0 + k] : 0.0;
      }
      cp_async_wait<1>();
      __syncthreads();
      // ---- panel factorization: warp w owns columns w, w + 8, w + 16, w + 24
      for (int k = 0; k < TPB; ++k) {
        if ((k & (TNW - 1)) == wid) {  // dlarfg on [R_kk; S[:, k]]
          double xv[RQ], ss = 0.0;
#pragma unroll
          for (int q = 0; q < RQ; ++q) {
            xv[q] = sm.Vs[k * LD + lane + 32 * q];
            ss = fma(xv[q], xv[q], ss);
          }
          ss = warp_sum(ss);
          const double x0 = sm.Rd[k * 33 + k];
          double tau = 0.0;
          if (ss > 0.0) {
            const double beta = -copysign(sqrt(fma(x0, x0, ss)), x0);
            tau = (beta - x0) / beta;
            const double scale = 1.0 / (x0 - beta);
#pragma unroll
            for (int q = 0; q < RQ; ++q) sm.Vs[k * LD + lane + 32 * q] = xv[q] * scale;
            if (lane == 0) sm.Rd[k * 33 + k] = beta;
          }
          if (lane == 0) sm.tau[k] = tau;
        }
        __syncthreads();
        const double tau = sm.tau[k];
        if (tau != 0.0) {
          double v[RQ];
#pragma unroll
          for (int q = 0; q < RQ; ++q) v[q] = sm.Vs[k * LD + lane + 32 * q];
#pragma unroll
          for (int t = 0; t < TPB / TNW; ++t) {
            const int j = wid + TNW * t;
            if (j > k) {
              double a[RQ], dot = 0.0;
#pragma unroll
              for (int q = 0; q < RQ; ++q) {
                a[q] = sm.Vs[j * LD + lane + 32 * q];
                dot = fma(v[q], a[q], dot);
              }
              dot = warp_sum(dot);
              const double tw = tau * (sm.Rd[k * 33 + j] + dot);
              __syncwarp();
              if (lane == 0) sm.Rd[k * 33 + j] -= tw;
#pragma unroll
              for (int q = 0; q < RQ; ++q) sm.Vs[j * LD + lane + 32 * q] = fma(-tw, v[q], a[q]);
            }
          }
        }
      }
      __syncthreads();
      // ---- R's diagonal block back; Gram matrix G = Vs^T Vs (into Wp)
      for (int e = tid; e < TPB * TPB; e += TNT) {
        const int i = e >> 5, k = e & 31;
        if (k >= i && j0 + k < c) R[(size_t)(j0 + i) * c + j0 + k] = sm.Rd[i * 33 + k];
      }
      if (ntile <= 0) continue;  // last panel: nothing to update (uniform)
      double* G = &sm.Wp[0][0];  // 32 x 32, row-major ld 32
      {
        const int mf = wid >> 1, nf0 = (wid & 1) * 2;
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        for (int kk = 0; kk < B; kk += 4) {
          const double a = sm.Vs[(8 * mf + fr) * LD + kk + fc];
#pragma unroll
          for (int n = 0; n < 2; ++n) {
            const double b = sm.Vs[(8 * (nf0 + n) + fr) * LD + kk + fc];
            dmma884(acc[n][0], acc[n][1], a, b);
          }
        }
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int h = 0; h < 2; ++h) G[(8 * mf + fr) * 32 + 8 * (nf0 + n) + 2 * fc + h] = acc[n][h];
      }
      __syncthreads();
      // ---- T (dlarft, forward columnwise): T[k,k] = tau_k, T[0:k,k] = -tau_k T[0:k,0:k] G[0:k,k]
      if (wid == 0) {
        for (int k = 0; k < TPB; ++k) {
          const double tk = sm.tau[k];
          double s = 0.0;
          if (lane < k)
            for (int l = lane; l < k; ++l) s = fma(sm.T[lane * 33 + l], G[l * 32 + k], s);
          __syncwarp();
          sm.T[lane * 33 + k] = lane < k ? -tk * s : (lane == k ? tk : 0.0);
          __syncwarp();
        }
      }
      // ---- trailing tiles
      for (int t = 0; t < ntile; ++t) {
        const int col0 = j0 + TPB + t * TTW;
        double* St = sm.St[t & 1];
        cp_async_wait<0>();
        __syncthreads();  // tile t landed; tile t-1 is written out; T is built
        if (t + 1 < ntile) tsqr_load_tile<B>(sm.St[(t + 1) & 1], S, lds, s0, nb, col0 + TTW, c, wid, lane);
        cp_async_commit();
        // W partials: warp = (K quarter, n fragment), 4 m fragments each
        {
          const int kq = wid & 3, nf = wid >> 2;
          double acc[4][2];
#pragma unroll
          for (int m = 0; m < 4; ++m) acc[m][0] = acc[m][1] = 0.0;
          for (int kk = kq * (B / 4); kk < (kq + 1) * (B / 4); kk += 4) {
            const double b = St[(8 * nf + fr) * LD + kk + fc];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const double a = sm.Vs[(8 * m + fr) * LD + kk + fc];
              dmma884(acc[m][0], acc[m][1], a, b);
            }
          }
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int h = 0; h < 2; ++h) sm.Wp[kq][(8 * m + fr) * TTW + 8 * nf + 2 * fc + h] = acc[m][h];
        }
        __syncthreads();
        // W = R_rows + sum of partials (fixed order); thread owns elements tid, tid + 256
        double rold[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int o = tid + TNT * u, i = o / TTW, jj = o % TTW;
          const bool ok = j0 + i < c && col0 + jj < c;
          rold[u] = ok ? R[(size_t)(j0 + i) * c + col0 + jj] : 0.0;
          sm.Wp[0][o] = rold[u] + (((sm.Wp[0][o] + sm.Wp[1][o]) + sm.Wp[2][o]) + sm.Wp[3][o]);
        }
        __syncthreads();
        // W2 = T^T W (T upper triangular), R_rows -= W2
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int o = tid + TNT * u, k = o / TTW, jj = o % TTW;
          double s = 0.0;
          for (int i = 0; i <= k; ++i) s = fma(sm.T[i * 33 + k], sm.Wp[0][i * TTW + jj], s);
          sm.W2[k * TW2LD + jj] = s;
          if (j0 + k < c && col0 + jj < c) R[(size_t)(j0 + k) * c + col0 + jj] = rold[u] - s;
        }
        __syncthreads();
        // S_t -= Vs W2: warp owns rows [wid * B/8, +B/8)
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
            double a[MF], b[2];
#pragma unroll
            for (int m = 0; m < MF; ++m) a[m] = -sm.Vs[(kk + fc) * LD + r0 + 8 * m + fr];
#pragma unroll
            for (int n = 0; n < 2; ++n) b[n] = sm.W2[(kk + fc) * TW2LD + 8 * n + fr];
#pragma unroll
            for (int m = 0; m < MF; ++m)
#pragma unroll
              for (int n = 0; n < 2; ++n) dmma884(acc[m][n][0], acc[m][n][1], a[m], b[n]);
          }
#pragma unroll
          for (int m = 0; m < MF; ++m)
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
              for (int h = 0; h < 2; ++h) St[(8 * n + 2 * fc + h) * LD + r0 + 8 * m + fr] = acc[m][n][h];
        }
        __syncthreads();
        // tile back to S (row-major: 64-byte row segments per warp instruction)
        {
          const int rr = lane & 3, cc = lane >> 2;
#pragma unroll
          for (int it = 0; it < B / 32; ++it) {
            const int row = 4 * (wid + TNW * it) + rr;
#pragma unroll
            for (int h = 0; h < TTW / 8; ++h) {
              const int col = 8 * h + cc;
              if (row < nb && col0 + col < c) S[(size_t)(s0 + row) * lds + col0 + col] = St[col * LD + row];
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
