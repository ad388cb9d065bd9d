// Estimation kernels (estimate.cuh) instantiated for p = 7..9 -- a separate translation unit so build.py
// compiles the estimation variants in parallel with the rest of libgwas.so.
#include "estimate_launch.cuh"

namespace gw {

cudaError_t est_launch_p7_9(int p, const double* W, const double* xlp, const double* yp, int n, int kpad, int t,
                            int method, double eps_spd, double* rec, EstOut eo, cudaStream_t st) {
  switch (p) {
    case 7: return est_launch<7>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    case 8: return est_launch<8>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    case 9: return est_launch<9>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gw
