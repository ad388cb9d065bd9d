// Estimation kernels (estimate.cuh) instantiated for p = 4..6 -- a separate translation unit so build.py
// compiles the estimation variants in parallel with the rest of libgwas.so.
#include "estimate_launch.cuh"

namespace gw {

cudaError_t est_launch_p4_6(int p, const double* W, const double* xlp, const double* yp, int n, int kpad, int t,
                            int method, double eps_spd, double* rec, EstOut eo, cudaStream_t st) {
  switch (p) {
    case 4: return est_launch<4>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    case 5: return est_launch<5>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    case 6: return est_launch<6>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gw
