// FP64 peak microbenchmark for the roofline denominator (SURVEY.md §8(d) "P_peak measured").
// Register-resident back-to-back mma.sync .f64 chains (lowers to DMMA on sm_100a) and DFMA chains,
// on all SMs; CUDA-event timed. Not part of the product path.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int NCH>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NCH][2];
#pragma unroll
  for (int i = 0; i < NCH; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NCH>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[NCH][4];
#pragma unroll
  for (int i = 0; i < NCH; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NCH>
__global__ void dfma_chain(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
double run(K kern, int blocks, int threads, int iters, double flop_per_warp_iter, const char* name, double* out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int w = 0; w < 3; ++w) kern<<<blocks, threads>>>(out, iters);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<blocks, threads>>>(out, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  double warps = (double)blocks * threads / 32;
  double tf = warps * iters * flop_per_warp_iter / (best * 1e-3) / 1e12;
  printf("{\"kernel\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", name, blocks, threads, best, tf);
  return tf;
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %d}\n", prop.name, sms, clk_khz / 1000);
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 16 * 1024));
  int iters = argc > 1 ? atoi(argv[1]) : 20000;
  for (int tpb : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      run(dmma_m8n8k4<8>, sms * bps, tpb, iters, 8 * 512.0, "dmma_m8n8k4_x8", out);
    }
  }
  run(dmma_m8n8k4<4>, sms * 2, 256, iters, 4 * 512.0, "dmma_m8n8k4_x4", out);
  run(dmma_m8n8k4<16>, sms * 2, 256, iters, 16 * 512.0, "dmma_m8n8k4_x16", out);
  run(dmma_m16n8k16<4>, sms * 2, 256, iters / 4, 4 * 4096.0, "dmma_m16n8k16_x4", out);
  run(dmma_m16n8k16<8>, sms * 2, 256, iters / 4, 8 * 4096.0, "dmma_m16n8k16_x8", out);
  for (int bps : {1, 2, 4, 8})
    run(dfma_chain<8>, sms * bps, 256, iters * 4, 8 * 64.0, "dfma_x8", out);
  run(dfma_chain<16>, sms * 4, 256, iters * 2, 16 * 64.0, "dfma_x16", out);
  CK(cudaFree(out));
  return 0;
}
