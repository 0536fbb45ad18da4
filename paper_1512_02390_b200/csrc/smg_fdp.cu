// Paired-line Schwarz kernel: instantiations and the (p, n_o, mesh) -> launcher table.
#include "smg_fdp.cuh"
namespace smg {
namespace {
struct Cfg { int p, n_o, tx, ty; FDTLaunchFn fn; };
const Cfg kCfgs[] = {
  {16, 1, 4, 4, &fdp_launch_k<16, 1, 4, 4>},
  {16, 1, 4, 2, &fdp_launch_k<16, 1, 4, 2>},
};
}  // namespace
FDTLaunchFn fdp_dispatch(int p, int n_o, int n_x, int n_y, int* TX, int* TY) {
  static const int force_all = env_int("SMG_FDP_TILE", 0);  // TX*10+TY (tuning aid)
  for (const Cfg& c : kCfgs) {
    if (c.p != p || c.n_o != n_o || n_x % c.tx || n_y % c.ty) continue;
    if (force_all && c.tx * 10 + c.ty != force_all) continue;
    *TX = c.tx;
    *TY = c.ty;
    return c.fn;
  }
  return nullptr;
}
}  // namespace smg
