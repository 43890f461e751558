// Device BLAS-1 for the GMRES driver (krylov.py:82-130): deterministic
// dot products (fixed grid, fixed-order second stage), axpy with a
// device-resident scalar, and the multi-vector dot / update of the
// modified-Gram-Schmidt re-orthogonalisation pass.
#include "hks_internal.h"

namespace hks {
namespace {

constexpr int VB = 256;
constexpr int VG = 296;  // 2 blocks per SM, fixed so results do not depend on n

__global__ void dot_partial(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                            int64_t ldv, int m, double* __restrict__ part) {
  // part[v * VG + blockIdx.x] = partial dot of vector v of x (ldv stride) with y
  __shared__ double red[VB / 32];
  for (int v = blockIdx.y; v < m; v += gridDim.y) {
    const double* xv = x + (size_t)v * ldv;
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)VB + threadIdx.x; i < n; i += (int64_t)VG * VB) s = fma(xv[i], y[i], s);
    s = block_sum(s, red);
    if (threadIdx.x == 0) part[(size_t)v * VG + blockIdx.x] = s;
  }
}

__global__ void dot_final(const double* __restrict__ part, int m, double* __restrict__ out, double scale,
                          int accumulate) {
  __shared__ double red[VB / 32];
  for (int v = blockIdx.x; v < m; v += gridDim.x) {
    double s = 0.0;
    for (int i = threadIdx.x; i < VG; i += VB) s += part[(size_t)v * VG + i];
    s = block_sum(s, red);
    if (threadIdx.x == 0) out[v] = accumulate ? out[v] + scale * s : scale * s;
  }
}

// y[i] += scale * sum_v coef[v] * X[v][i]  (coef on the device)
__global__ void multi_axpy(const double* __restrict__ X, int64_t ldv, int m, const double* __restrict__ coef,
                           double scale, double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = y[i];
    for (int v = 0; v < m; ++v) acc -= (-scale * coef[v]) * X[(size_t)v * ldv + i];
    y[i] = acc;
  }
}

}  // namespace
}  // namespace hks

using namespace hks;

// out[v] = scale * <X[v], y> for v < m (X rows at stride ldv); accumulate adds.
// `part` is caller scratch of m * 296 doubles.
extern "C" int hks_vdots(const double* X, int64_t ldv, int64_t m, const double* y, int64_t n, double* out,
                         double scale, int32_t accumulate, double* part, void* stream) {
  if (m <= 0) return HKS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  dim3 g1(VG, m < 64 ? (unsigned)m : 64u);
  dot_partial<<<g1, VB, 0, s>>>(X, y, n, ldv, (int)m, part);
  dot_final<<<(unsigned)(m < 1024 ? m : 1024), VB, 0, s>>>(part, (int)m, out, scale, accumulate);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HKS_OK : set_error(HKS_ERR_CUDA, "hks_vdots: %s", cudaGetErrorString(e));
}

// y += scale * sum_v coef[v] X[v]; with m = 1 this is the MGS update
// w -= h * v (krylov.py:84-86) with scale = -1.
extern "C" int hks_vaxpys(const double* X, int64_t ldv, int64_t m, const double* coef, double scale, double* y,
                          int64_t n, void* stream) {
  if (m <= 0 || n <= 0) return HKS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  multi_axpy<<<592, 256, 0, s>>>(X, ldv, (int)m, coef, scale, y, n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HKS_OK : set_error(HKS_ERR_CUDA, "hks_vaxpys: %s", cudaGetErrorString(e));
}
