// Microbenchmark: tcgen05.mma kind::i8 throughput with operands resident in shared memory (no TMA), to bound
// what the int8-sliced K1i kernel can reach.  Not product code.
#include <cstdio>
#include <cstdlib>
#include "../paper_1207_2169_b200/csrc/gemm_i8.cuh"
using namespace gw;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int N_PER_MMA, int BROWS>
__global__ void __launch_bounds__(128, 1) umma_loop(int iters, int* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                   // 128 rows x 64 B
  uint8_t* sB = smem + 128 * 64;        // BROWS rows x 64 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + BROWS * 64);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (128 + BROWS) * 64 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_i8(N_PER_MMA);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
        for (int c = 0; c < BROWS / N_PER_MMA; ++c)
          umma_i8(tmem + c * N_PER_MMA, umma_desc_sw64(a0 + kk * 32), umma_desc_sw64(b0 + c * N_PER_MMA * 64 + kk * 32), idesc, 1u);
      }
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    int32_t v[16];
    tmem_ld16(tmem + ((uint32_t)0 << 16), v);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (threadIdx.x == 0) out[blockIdx.x] = v[0];
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

template <int NPM, int BR>
void run(int sms, int iters, const char* name) {
  int* out; CK(cudaMalloc(&out, sizeof(int) * sms * 4));
  size_t smem = 1024 + (128 + BR) * 64 + 64;
  CK(cudaFuncSetAttribute(umma_loop<NPM, BR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  umma_loop<NPM, BR><<<sms, 128, smem>>>(10, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  umma_loop<NPM, BR><<<sms, 128, smem>>>(iters, out);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 2.0 * 128 * BR * 64.0 * iters * sms;   // per iter: K = 64 bytes over BR columns
  printf("{\"case\": \"%s\", \"ms\": %.3f, \"tops\": %.1f}\n", name, ms, ops / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  int sms = 148;
  run<256, 512>(sms, 20000, "M128 N256 x2 (512 cols), K=32 x2 per iter");
  run<128, 512>(sms, 20000, "M128 N128 x4");
  run<256, 256>(sms, 40000, "M128 N256 x1");
  run<64, 512>(sms, 20000, "M128 N64 x8");
  return 0;
}
