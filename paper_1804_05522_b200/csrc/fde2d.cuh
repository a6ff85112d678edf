// fde2d.cuh -- 2D Sylvester time step (Eq. 4.3) -- placeholder until the
// extended Krylov driver lands; returns FDE_EDOMAIN so callers fail loudly.
extern "C" int fde2d_step(int nx, int ny, double alpha1, double alpha2, double hx, double hy, double dt,
                          const double* d1p, const double* d1m, const double* d2p, const double* d2m,
                          const double* Fu, const double* Fv, int rf, const double* Uu, const double* Uv,
                          int ru, double* Xu, double* Xv, int rmax, int* rx, double tol, double ek_tol,
                          int ek_maxit, int leaf, fde_hodlr_t* cache, double* resid_out, int* iters_out,
                          unsigned flags, void* stream) {
  return set_err(FDE_EDOMAIN, "fde2d_step: not available in this build yet");
}
