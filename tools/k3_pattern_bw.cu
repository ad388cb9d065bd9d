// Roofline probe for K3 (schur_solve): the HBM bandwidth its access pattern can reach on this B200, without its
// arithmetic.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/k3_pattern_bw tools/k3_pattern_bw.cu && tools/k3_pattern_bw
// A: K3's exact pattern (one thread per trait j, 16 SNP rows per thread, P + 2 = 7 fields of row i read at
//    C[i * ldc + f * t + j], b / var / status written at [i * t + j]) with the solve replaced by a sum.
// B: the same bytes read and written as flat contiguous streams (16-byte vector loads, grid-stride).
// C: a plain device-to-device copy of the same total bytes (cudaMemcpyAsync) for reference.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void pattern_k3(const double* __restrict__ C, long long ldc, int t, int nsq, int cols, double* b,
                           double* var, signed char* st) {
  const int j = blockIdx.x * 128 + threadIdx.x;
  if (j >= t) return;
  const int i0 = blockIdx.y * 16, i1 = min(cols, i0 + 16);
  for (int i = i0; i < i1; ++i) {
    const double* row = C + (long long)i * ldc;
    double acc = 0.0;
#pragma unroll
    for (int f = 0; f < 6; ++f) acc += __ldg(row + f * t + j);
    acc += __ldg(row + nsq + j);
    const long long idx = (long long)i * t + j;
    b[idx] = acc;
    var[idx] = acc * 0.5;
    st[idx] = (signed char)(acc > 0);
  }
}

// D: K3 with C stored trait-block-major, [i][jb][f][128] (each (row, 128-trait block) one contiguous 7 KB chunk)
__global__ void pattern_tiled(const double* __restrict__ C, long long ldc, int t, int cols, double* b, double* var,
                              signed char* st, int mode) {
  const int j = blockIdx.x * 128 + threadIdx.x;
  if (j >= t) return;
  const int i0 = blockIdx.y * 16, i1 = min(cols, i0 + 16);
  for (int i = i0; i < i1; ++i) {
    const double* chunk = C + (long long)i * ldc + (long long)blockIdx.x * 7 * 128 + threadIdx.x;
    double acc = 0.0;
    if (mode != 2) {
#pragma unroll
      for (int f = 0; f < 7; ++f) acc += __ldg(chunk + f * 128);
    }
    const long long idx = (long long)i * t + j;
    if (mode != 1) {
      b[idx] = acc;
      var[idx] = acc * 0.5;
      st[idx] = (signed char)(acc > 0);
    } else if (acc == 12345.0) {
      b[idx] = acc;
    }
  }
}

__global__ void flat_stream(const double2* __restrict__ in, long long n_in, double2* out, long long n_out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  double s = 0.0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n_in; k += stride) {
    const double2 v = __ldg(in + k);
    s += v.x + v.y;
    if (k < n_out) out[k] = make_double2(s, v.y);
  }
}

int main() {
  const int t = 1000, cols = 15104;
  const int nsq = 6016, n2 = nsq + t;
  const long long ldc = n2 + (n2 & 1);
  double *C, *b, *v, *o;
  signed char* st;
  cudaMalloc(&C, sizeof(double) * ldc * cols);
  cudaMalloc(&b, sizeof(double) * (long long)t * cols);
  cudaMalloc(&v, sizeof(double) * (long long)t * cols);
  cudaMalloc(&st, (long long)t * cols);
  cudaMemset(C, 0, sizeof(double) * ldc * cols);
  const double rd = 7.0 * 8 * t * cols, wr = 17.0 * t * cols;
  cudaMalloc(&o, (size_t)(rd + wr) + 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0.f, best = 1e9f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(e0);
    pattern_k3<<<dim3((t + 127) / 128, (cols + 15) / 16), 128>>>(C, ldc, t, nsq, cols, b, v, st);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  printf("{\"case\": \"A: K3 access pattern, no arithmetic\", \"ms\": %.4f, \"gbs\": %.1f}\n", best, (rd + wr) / best / 1e6);
  const char* names[3] = {"D: C trait-block-major [i][jb][f][128], reads + writes", "E: D reads only",
                          "F: D writes only"};
  for (int mode = 0; mode < 3; ++mode) {
    best = 1e9f;
    for (int rep = 0; rep < 10; ++rep) {
      cudaEventRecord(e0);
      pattern_tiled<<<dim3((t + 127) / 128, (cols + 15) / 16), 128>>>(C, ldc, t, cols, b, v, st, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double by = mode == 0 ? rd + wr : mode == 1 ? rd : wr;
    printf("{\"case\": \"%s\", \"ms\": %.4f, \"gbs\": %.1f}\n", names[mode], best, by / best / 1e6);
  }
  best = 1e9f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(e0);
    flat_stream<<<148 * 16, 256>>>(reinterpret_cast<const double2*>(C), (long long)(rd / 16),
                                   reinterpret_cast<double2*>(o), (long long)(wr / 16));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  printf("{\"case\": \"B: same bytes, flat contiguous streams\", \"ms\": %.4f, \"gbs\": %.1f}\n", best, (rd + wr) / best / 1e6);
  best = 1e9f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(e0);
    cudaMemcpyAsync(o, C, (size_t)((rd + wr) / 2) / 16 * 16, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  printf("{\"case\": \"C: cudaMemcpy D2D of (read + write) / 2 bytes\", \"ms\": %.4f, \"gbs\": %.1f}\n", best,
         (rd + wr) / best / 1e6);
  return 0;
}
