// Explicit instantiations of the operator kernel and the p -> launcher table.
#include "smg_op.cuh"
namespace smg {
OpLaunchFn op_dispatch(int p) {
  switch (p) {
#define SMG_OPP(P) case P: return &op_launch<P>;
    SMG_OPP(1) SMG_OPP(2) SMG_OPP(3) SMG_OPP(4) SMG_OPP(5) SMG_OPP(6) SMG_OPP(8)
    SMG_OPP(12) SMG_OPP(16) SMG_OPP(24) SMG_OPP(32)
#undef SMG_OPP
    default: return nullptr;
  }
}
}  // namespace smg
