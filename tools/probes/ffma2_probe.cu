// Probe: dependent-chain latency and independent throughput of FFMA vs FFMA2 on one SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS, bool PACKED>
__global__ void k(float* out, int iters, long long* cyc) {
  float2 a[CHAINS];
  for (int c = 0; c < CHAINS; ++c) a[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  const float2 m = make_float2(0.999f, 0.998f), s = make_float2(1e-3f, 2e-3f);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (PACKED) {
        a[c] = __ffma2_rn(a[c], m, s);
      } else {
        a[c].x = fmaf(a[c].x, m.x, s.x);
        a[c].y = fmaf(a[c].y, m.y, s.y);
      }
    }
  }
  long long t1 = clock64();
  float acc = 0;
  for (int c = 0; c < CHAINS; ++c) acc += a[c].x + a[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CHAINS, bool PACKED>
void run(int warps) {
  float* out; long long* cyc; long long h;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
  const int iters = 4096;
  k<CHAINS, PACKED><<<1, 32 * warps>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  k<CHAINS, PACKED><<<1, 32 * warps>>>(out, iters, cyc);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (iters * CHAINS);
  printf("%s chains=%d warps/SM=%d: %.2f cycles per (pair-)FMA instr per warp; SM pair-FMA/clk=%.2f\n",
         PACKED ? "FFMA2" : "2xFFMA", CHAINS, warps, per, warps / per);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  run<1, true>(1); run<1, false>(1);
  run<4, true>(1); run<8, true>(1); run<8, false>(1);
  run<8, true>(4); run<8, true>(8); run<8, true>(16); run<8, false>(16);
  run<2, true>(16); run<1, true>(16);
  return 0;
}
