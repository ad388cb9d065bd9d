// Estimation kernels (estimate.cuh) instantiated for p = 10..12 -- a separate translation unit so build.py
// compiles the estimation variants in parallel with the rest of libgwas.so.
#include "estimate_launch.cuh"

namespace gw {

cudaError_t est_launch_p10_12(int p, const double* W, const double* xlp, const double* yp, int n, int kpad, int t,
                            int method, double eps_spd, double* rec, EstOut eo, cudaStream_t st) {
  switch (p) {
    case 10: return est_launch<10>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    case 11: return est_launch<11>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    case 12: return est_launch<12>(W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace gw
