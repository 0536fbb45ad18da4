// Generated: explicit instantiations of the FD Schwarz kernel.
#include "smg_fd.cuh"
namespace smg {
template int fd_launch<5>(const FDLaunch&, cudaStream_t);
template int fd_launch<9>(const FDLaunch&, cudaStream_t);
template int fd_launch<13>(const FDLaunch&, cudaStream_t);
template int fd_launch<17>(const FDLaunch&, cudaStream_t);
template int fd_launch<21>(const FDLaunch&, cudaStream_t);
template int fd_launch<25>(const FDLaunch&, cudaStream_t);
template int fd_launch<29>(const FDLaunch&, cudaStream_t);
template int fd_launch<33>(const FDLaunch&, cudaStream_t);
template int fd_launch<37>(const FDLaunch&, cudaStream_t);
template int fd_launch<41>(const FDLaunch&, cudaStream_t);
}  // namespace smg
