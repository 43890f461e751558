// Dependent-chain latencies of a few SASS ops on this GPU (development tool).
#include <cstdio>
__global__ void lat(double* out, long long* cyc, int n) {
  __shared__ double sm[64];
  __shared__ unsigned su[64];
  const int t = threadIdx.x;
  sm[t] = t * 0.5;
  su[t] = t;
  __syncthreads();
  double x = out[t];
  unsigned u = t;
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 1.0000001, 0.5);
  long long c1 = clock64();
  int idx = t & 63;
  for (int i = 0; i < n; ++i) idx = (int)sm[idx] & 63;
  long long c2 = clock64();
  for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u + i);
  long long c3 = clock64();
  double y = x;
  for (int i = 0; i < n; ++i) y = __shfl_xor_sync(0xffffffffu, y, 1) + 1.0;
  long long c4 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long c5 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) z = 1.0 / z + 0.5;
  long long c6 = clock64();
  for (int i = 0; i < n; ++i) idx = su[idx] & 63;
  long long c7 = clock64();
  out[t] = x + idx + u + y + z;
  if (t == 0) {
    cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; cyc[3] = c4 - c3; cyc[4] = c5 - c4; cyc[5] = c6 - c5; cyc[6] = c7 - c6;
  }
}
int main() {
  double* o; long long* c; long long h[7];
  cudaMalloc(&o, 1024 * 8); cudaMemset(o, 0, 1024 * 8); cudaMalloc(&c, 64);
  const char* names[7] = {"DFMA chain", "LDS.64->int chain", "CREDUX chain", "SHFL+DADD chain", "bar.sync (256 thr)", "DP divide chain", "LDS.32 chain"};
  for (int threads : {32, 256}) {
    lat<<<1, threads>>>(o, c, 1000);
    lat<<<1, threads>>>(o, c, 1000);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %d\n", threads);
    for (int i = 0; i < 7; ++i) printf("  %-20s %.1f cycles/op\n", names[i], h[i] / 1000.0);
  }
  return 0;
}
