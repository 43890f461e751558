// Shared device helpers for libhks (sm_100a, FP64 throughout).
//
// Matrices are column-major with an explicit leading dimension unless a
// kernel says otherwise (LAPACK convention, so the host views reproduce
// scipy's lu_factor / lu_solve layout).  Every batched kernel takes a
// descriptor table in device memory -- one entry per independent problem --
// so ragged (adaptive-rank) levels and sub-block writes (Z's off-diagonal
// blocks, stacked sibling vectors) need no padding or copies.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hks {

constexpr int kWarp = 32;

// D = A*B + D for one 8x8x4 FP64 tile (SASS: DMMA.884).  Fragment layout
// (PTX ISA m8n8k4 .f64): lane t holds A[t/4][t%4], B[t%4][t/4] and
// D[t/4][2*(t%4) + {0,1}].
// 8-byte asynchronous global->shared copy (LDGSTS); pred false zero-fills.
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(pred ? 8 : 0));
}
// 16-byte asynchronous copy (both addresses 16-byte aligned), L1 bypass.
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// (value, index) argmax with the lowest index winning ties -- the rule of
// numpy.argmax (linalg.py:81) and LAPACK idamax.
struct ArgMax {
  double v;
  int i;
};

__device__ __forceinline__ ArgMax argmax_pick(ArgMax a, ArgMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__device__ __forceinline__ ArgMax warp_argmax(ArgMax a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
    a = argmax_pick(a, b);
  }
  return a;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide argmax; `scratch` needs 2 * (blockDim.x / 32) slots.
__device__ inline ArgMax block_argmax(ArgMax a, double* sv, int* si) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  a = warp_argmax(a);
  if (lane == 0) { sv[wid] = a.v; si[wid] = a.i; }
  __syncthreads();
  if (wid == 0) {
    ArgMax b = lane < nw ? ArgMax{sv[lane], si[lane]} : ArgMax{-1.0, 0x7fffffff};
    b = warp_argmax(b);
    if (lane == 0) { sv[0] = b.v; si[0] = b.i; }
  }
  __syncthreads();
  ArgMax r{sv[0], si[0]};
  __syncthreads();
  return r;
}

// Block-wide sum in a fixed order (deterministic); `sv` needs blockDim/32.
__device__ inline double block_sum(double v, double* sv) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sv[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double b = lane < nw ? sv[lane] : 0.0;
    b = warp_sum(b);
    if (lane == 0) sv[0] = b;
  }
  __syncthreads();
  double r = sv[0];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------- descriptors
//
// Operands are relocatable references: the top 8 bits select a base pointer
// from a small table (Bases, passed by value as a kernel parameter), the low
// 56 bits are a byte offset.  One uploaded descriptor program therefore
// serves every factorization of an operator and every right-hand-side
// buffer; a call only supplies its base pointers.
// Buffer id kAbs (= 17) has base 0, i.e. the offset is a raw address.
using Ref = uint64_t;
constexpr int kNumBases = 18;
constexpr int kAbs = 17;
constexpr uint64_t kOffMask = (uint64_t(1) << 56) - 1;
constexpr uint64_t kNull = ~uint64_t(0);  // "no operand"

struct Bases {
  char* p[kNumBases];
  double lam;  // regularization for eval/ksum descriptors flagged `diag`
  double pad[1];
};

__host__ __device__ inline Ref make_ref(int buf, uint64_t byte_off) {
  return (uint64_t(buf) << 56) | (byte_off & kOffMask);
}
__host__ inline Ref abs_ref(const void* p) { return make_ref(kAbs, reinterpret_cast<uint64_t>(p)); }

// Integer arithmetic on purpose: for kAbs the base is null, and pointer
// arithmetic on a null base is undefined behaviour the optimiser exploits.
template <class T>
__device__ __forceinline__ T* at(const Bases& b, Ref r) {
  return reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(b.p[r >> 56]) + (uintptr_t)(r & kOffMask));
}

// C = alpha * op(A) * op(B) + beta * C, op(X) = X or X^T (column-major).
struct GemmDesc {
  Ref A, B, C;
  int m, n, k;
  int lda, ldb, ldc;
  int transA, transB;
  double alpha, beta;
};

// dst = alpha * op(src) (m x n result); mode 0: copy, 1: alpha * I, 2: zero,
// 3: accumulate (dst += alpha * op(src)).
// mode 0: dst = alpha op(src); 1: identity * alpha; 2: zeros; 3: dst += alpha src;
// 4: dst = src^T + alpha src2 (trans must be 1; e.g. push = P^T - F);
// 5: dst = Bases::lam * src; 6: dst = src + Bases::lam I (trans 0 for 5, 6)
struct CopyDesc {
  Ref src, dst;
  int m, n;
  int lds, ldd;
  int trans;
  int mode;
  double alpha;
  Ref src2 = 0;
  int lds2 = 0;
  int pad_ = 0;
};

// In-place LU with partial pivoting of an n x n matrix.
struct LuDesc {
  Ref A;
  Ref piv;    // int32, 0-based row interchanges (scipy lu_factor convention)
  Ref info;   // int32: 0 or 1-based step of the first exactly-zero pivot
  Ref anorm;  // double: ||A||_1 before factoring (for gecon); kNull = skip
  Ref rcond;  // double: LAPACK dgecon reciprocal condition; kNull = skip
  int n, lda;
};

// Solve A X = B in place for nrhs columns with an LU from LuDesc.
struct LuSolveDesc {
  Ref LU, piv, B;
  int n, nrhs;
  int lda, ldb;
};

// Factor rows p0..n-1 of panel columns [p0, p0 + pb) (partial pivoting).
// Optional int32 row permutations over absolute positions (kNull: skip):
// after the panel, position i holds the original row tperm[i] (total, since
// column 0), the row that was at position gperm[i] when the 128-column group
// starting at g0 began, and the row that was at sig[i] when this panel began.
struct PanelDesc {
  Ref A, piv, info;
  int lda, n, p0, pb;
  Ref tperm, sig, gperm;
  int g0, pad;
};

// B := A^-1 B for an LU (getrf storage, n <= kGetrsFusedMax) and its recorded
// total row permutation (perm[i] = row of B that lands at i); lower = 0
// skips the forward sweep (B already forward-substituted).
constexpr int kGetrsFusedMax = 256;
struct GetrsDesc {
  Ref LU, perm, B;
  int n, lda, ldb, ncols, lower, pad;
  Ref Bin;  // right-hand sides read from here (ld ldb) when not kNull, else from B
};

// Row gather A[i, c] := A[perm[i], c] for rows [r0, r1) and columns [c0, c1)
// (perm maps [r0, r1) onto itself): the interchanges of a pivot sequence
// applied in one parallel pass.
struct GatherDesc {
  Ref A, perm;
  int lda, r0, r1, c0, c1, pad;
};

// Row interchanges piv[r0..r1) applied to columns [c0, c1) of A.
struct SwapDesc {
  Ref A, piv;
  int lda, r0, r1, c0, c1;
  int pad;
};

// B := T^-1 B, T the k x k unit-lower (or non-unit upper) block at T.
struct TrsmDesc {
  Ref T, B;
  int ldt, ldb, k, ncols;
};

// Whole LU (+ carried right-hand sides B, n x r, and backward solve) of one
// matrix in one CTA (lu_fused.cu).
struct LuFusedDesc {
  Ref A, piv, info, B;
  int n, lda, r, ldb;
};

}  // namespace hks

#define HKS_CUDA_CHECK(expr)                                                 \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) return ::hks::set_error(HKS_ERR_CUDA, "%s: %s (%s:%d)", #expr, \
                                                   cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)
