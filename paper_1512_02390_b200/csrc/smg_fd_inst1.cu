// Generated: explicit instantiations of the FD Schwarz kernel.
#include "smg_fd.cuh"
namespace smg {
template int fd_launch<4>(const FDLaunch&, cudaStream_t);
template int fd_launch<8>(const FDLaunch&, cudaStream_t);
template int fd_launch<12>(const FDLaunch&, cudaStream_t);
template int fd_launch<16>(const FDLaunch&, cudaStream_t);
template int fd_launch<20>(const FDLaunch&, cudaStream_t);
template int fd_launch<24>(const FDLaunch&, cudaStream_t);
template int fd_launch<28>(const FDLaunch&, cudaStream_t);
template int fd_launch<32>(const FDLaunch&, cudaStream_t);
template int fd_launch<36>(const FDLaunch&, cudaStream_t);
template int fd_launch<40>(const FDLaunch&, cudaStream_t);
}  // namespace smg
