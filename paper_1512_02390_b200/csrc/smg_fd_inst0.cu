// Generated: explicit instantiations of the FD Schwarz kernel.
#include "smg_fd.cuh"
namespace smg {
template int fd_launch<3>(const FDLaunch&, cudaStream_t);
template int fd_launch<7>(const FDLaunch&, cudaStream_t);
template int fd_launch<11>(const FDLaunch&, cudaStream_t);
template int fd_launch<15>(const FDLaunch&, cudaStream_t);
template int fd_launch<19>(const FDLaunch&, cudaStream_t);
template int fd_launch<23>(const FDLaunch&, cudaStream_t);
template int fd_launch<27>(const FDLaunch&, cudaStream_t);
template int fd_launch<31>(const FDLaunch&, cudaStream_t);
template int fd_launch<35>(const FDLaunch&, cudaStream_t);
template int fd_launch<39>(const FDLaunch&, cudaStream_t);
}  // namespace smg
