// Microbenchmark: FP64 DFMA vs DMMA (mma.sync m8n8k4 f64) throughput on one GPU.
// Used once to establish the FP64 roofline denominators (MEASURED_PEAKS has only bf16/HBM).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = threadIdx.x; acc[i][1] = i; }
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < NACC; ++u) dmma(acc[u][0], acc[u][1], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int bpsm : {4, 8}) {
    int blocks = sms * bpsm, threads = 256, iters = 4096;
    dfma_kernel<<<blocks, threads>>>(out, 16, 0.999, 1e-3);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)blocks * threads;
    printf("{\"kind\":\"dfma\",\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", bpsm, flops / ms / 1e9);
  }
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm, threads = 256, iters = 4096;
    dmma_kernel<4><<<blocks, threads>>>(out, 16, 0.999, 1e-3);
    cudaEventRecord(e0);
    dmma_kernel<4><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 512.0 * 4 * iters * (double)blocks * (threads / 32);
    printf("{\"kind\":\"dmma_acc4\",\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", bpsm, flops / ms / 1e9);
    dmma_kernel<8><<<blocks, threads>>>(out, 16, 0.999, 1e-3);
    cudaEventRecord(e0);
    dmma_kernel<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    flops = 512.0 * 8 * iters * (double)blocks * (threads / 32);
    printf("{\"kind\":\"dmma_acc8\",\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", bpsm, flops / ms / 1e9);
  }
  size_t n = (size_t)1 << 27;  // 2 GiB of double2 per buffer
  double2 *a, *b; cudaMalloc(&a, n * sizeof(double2)); cudaMalloc(&b, n * sizeof(double2));
  cudaMemset(a, 0, n * sizeof(double2));
  copy_kernel<<<sms * 8, 512>>>(a, b, n);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("{\"kind\":\"copy\",\"gbs\":%.1f}\n", 2.0 * n * sizeof(double2) / best / 1e6);
  cudaError_t err = cudaGetLastError();
  printf("{\"err\":\"%s\",\"sms\":%d}\n", cudaGetErrorString(err), sms);
  return 0;
}
