// Paired-line Schwarz kernel: instantiations and the (p, n_o, mesh) -> launcher table.
#include "smg_fdp.cuh"
namespace smg {
namespace {
struct Cfg { int p, n_o, tx, ty; FDTLaunchFn fn; };
// per order: largest tile first (B200, 256^2 elements, us per correction: p = 16 4x4 175.0 /
// 4x2 205.7; p = 24 4x4 429 / 4x2 437 / 2x2 509 (512^2: 1624 / 1693); p = 32 4x2 871.3 / 2x2 1055.8)
const Cfg kCfgs[] = {
  {2, 1, 8, 8, &fdp_launch_k<2, 1, 8, 8>},
  {4, 1, 8, 4, &fdp_launch_k<4, 1, 8, 4>},
  {4, 1, 4, 4, &fdp_launch_k<4, 1, 4, 4>},
  {6, 1, 4, 4, &fdp_launch_k<6, 1, 4, 4>},
  {8, 1, 4, 4, &fdp_launch_k<8, 1, 4, 4>},
  {12, 1, 4, 4, &fdp_launch_k<12, 1, 4, 4>},
  {12, 2, 4, 4, &fdp_launch_k<12, 2, 4, 4>},
  {16, 1, 4, 4, &fdp_launch_k<16, 1, 4, 4>},
  {16, 1, 4, 2, &fdp_launch_k<16, 1, 4, 2>},
  {16, 1, 2, 2, &fdp_launch_k<16, 1, 2, 2>},
  {16, 2, 4, 4, &fdp_launch_k<16, 2, 4, 4>},
  {16, 2, 4, 2, &fdp_launch_k<16, 2, 4, 2>},
  {24, 1, 4, 4, &fdp_launch_k<24, 1, 4, 4>},
  {24, 1, 4, 2, &fdp_launch_k<24, 1, 4, 2>},
  {24, 1, 2, 2, &fdp_launch_k<24, 1, 2, 2>},
  {24, 3, 4, 2, &fdp_launch_k<24, 3, 4, 2>},
  {24, 3, 2, 2, &fdp_launch_k<24, 3, 2, 2>},
  {32, 1, 4, 2, &fdp_launch_k<32, 1, 4, 2>},
  {32, 1, 2, 2, &fdp_launch_k<32, 1, 2, 2>},
  {32, 4, 2, 2, &fdp_launch_k<32, 4, 2, 2>},
};
}  // namespace
FDTLaunchFn fdp_dispatch(int p, int n_o, int n_x, int n_y, int* TX, int* TY) {
  // the first (largest) tile that divides the mesh and still gives every SM a
  // tile, else the divisible one with most tiles
  static const int min_tiles = env_int("SMG_FDT_MIN_TILES", 148);
  static const int force_all = env_int("SMG_FDP_TILE", 0);  // TX*10+TY (tuning aid)
  const Cfg* best = nullptr;
  long best_tiles = -1;
  for (const Cfg& c : kCfgs) {
    if (c.p != p || c.n_o != n_o || n_x % c.tx || n_y % c.ty) continue;
    if (force_all && c.tx * 10 + c.ty != force_all) continue;
    const long tiles = (long)(n_x / c.tx) * (n_y / c.ty);
    if (tiles >= min_tiles) { best = &c; break; }
    if (tiles > best_tiles) { best = &c; best_tiles = tiles; }
  }
  if (!best) return nullptr;
  // p <= 4 (measured: 256^2 elements p = 4 38.0 -> 31.7 us, p = 2 25.8 -> 23.6; equal on
  // small meshes): only where every SM gets a tile, else fdt_kernel's smaller tiles
  if (p <= 4 && (long)(n_x / best->tx) * (n_y / best->ty) < min_tiles) return nullptr;
  *TX = best->tx;
  *TY = best->ty;
  return best->fn;
}
}  // namespace smg
