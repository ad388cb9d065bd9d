// Host-side launch of the estimation kernels (estimate.cuh) for a compile-time p; instantiated for p = 1..12 in
// est_p1_3.cu .. est_p10_12.cu (separate translation units, compiled in parallel by build.py).
#pragma once
#include <cuda_runtime.h>

#include "estimate.cuh"

namespace gw {

template <int P>
cudaError_t est_launch(const double* W, const double* xlp, const double* yp, int n, int kpad, int t, int method,
                       double eps_spd, double* rec, EstOut eo, cudaStream_t st) {
  est_grid_shared<P><<<EST_GRID + 1, EST_THREADS, 0, st>>>(W, xlp, n, kpad, eps_spd, rec);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  est_traits<P><<<(unsigned)t, EST_THREADS, 0, st>>>(W, xlp, yp, n, kpad, t, method, rec, eo);
  return cudaGetLastError();
}

// Defined in est_p1_3.cu .. est_p10_12.cu: cudaErrorInvalidValue for p outside the file's range.
cudaError_t est_launch_p1_3(int p, const double* W, const double* xlp, const double* yp, int n, int kpad, int t,
                            int method, double eps_spd, double* rec, EstOut eo, cudaStream_t st);
cudaError_t est_launch_p4_6(int p, const double* W, const double* xlp, const double* yp, int n, int kpad, int t,
                            int method, double eps_spd, double* rec, EstOut eo, cudaStream_t st);
cudaError_t est_launch_p7_9(int p, const double* W, const double* xlp, const double* yp, int n, int kpad, int t,
                            int method, double eps_spd, double* rec, EstOut eo, cudaStream_t st);
cudaError_t est_launch_p10_12(int p, const double* W, const double* xlp, const double* yp, int n, int kpad, int t,
                            int method, double eps_spd, double* rec, EstOut eo, cudaStream_t st);

}  // namespace gw
