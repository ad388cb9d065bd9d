// Microbenchmark: tcgen05.mma.cta_group::2 kind::i8 (M = 256 over a CTA pair, N = 256) with operands resident in
// shared memory: each CTA holds its 128 A rows and half of the B rows (N split across the pair), so every MMA reads
// the peer's B half through the cluster.  Compared with the 1-SM rate of tools/umma_i8_peak.cu, it tells whether a
// 2-SM int8 mainloop can beat the 1-SM one.  Not product code.
#include <cstdio>
#include <cstdlib>
#include "../paper_1207_2169_b200/csrc/gemm_i8.cuh"
using namespace gw;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int NCHUNK>
__global__ void __launch_bounds__(128, 1) umma2_loop(int iters, int* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                         // 128 rows x 64 B (this CTA's half of M)
  uint8_t* sB = smem + 128 * 64;              // NCHUNK x 128 rows x 64 B (this CTA's half of each N = 256 chunk)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + NCHUNK * 128 * 64);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (128 + NCHUNK * 128) * 64 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 3);
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0 && rank == 0) {
    constexpr uint32_t idesc = idesc_i8_m256(256);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
#pragma unroll
        for (int c = 0; c < NCHUNK; ++c)
          umma_i8_2sm(tmem + c * 256, umma_desc_sw64(a0 + kk * 32), umma_desc_sw64(b0 + c * 128 * 64 + kk * 32), idesc, 1u);
    }
    umma_commit_2sm(bar);
  }
  if (threadIdx.x == 0) mbar_wait(bar, 0);
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x < 32) {
    int32_t v[16];
    tmem_ld16(tmem, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (threadIdx.x == 0) out[blockIdx.x] = v[0];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

template <int NCHUNK>
void run(int sms, int iters, const char* name) {
  int* out; CK(cudaMalloc(&out, sizeof(int) * sms * 4));
  size_t smem = 1024 + (128 + NCHUNK * 128) * 64 + 64;
  CK(cudaFuncSetAttribute(umma2_loop<NCHUNK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, umma2_loop<NCHUNK>, 10, out));
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  CK(cudaLaunchKernelEx(&cfg, umma2_loop<NCHUNK>, iters, out));
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 2.0 * 256 * (NCHUNK * 256) * 64.0 * iters * (sms / 2);
  printf("{\"case\": \"%s\", \"ms\": %.3f, \"tops\": %.1f}\n", name, ms, ops / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  run<2>(148, 20000, "2SM M256 N256 x2 (512 cols), K=32 x2 per iter");
  run<1>(148, 40000, "2SM M256 N256 x1");
  return 0;
}
