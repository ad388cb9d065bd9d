// Estimation kernels (estimate.cuh) instantiated for p = 1..3 -- a separate translation unit so build.py
// compiles the estimation variants in parallel with the rest of libgwas.so.
#include "estimate_launch.cuh"

namespace gw {

cudaError_t est_launch_p1_3(int p, const double* W, const double* xlp, const double* yp, int n, int kpad, int t,
                            int method, double eps_spd, double* rec, EstOut eo, cudaStream_t st) {
  switch (p) {
    case 1: return est_launch<1>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    case 2: return est_launch<2>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    case 3: return est_launch<3>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gw
