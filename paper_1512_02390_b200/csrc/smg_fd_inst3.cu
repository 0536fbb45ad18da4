// Generated: explicit instantiations of the FD Schwarz kernel.
#include "smg_fd.cuh"
namespace smg {
template int fd_launch<6>(const FDLaunch&, cudaStream_t);
template int fd_launch<10>(const FDLaunch&, cudaStream_t);
template int fd_launch<14>(const FDLaunch&, cudaStream_t);
template int fd_launch<18>(const FDLaunch&, cudaStream_t);
template int fd_launch<22>(const FDLaunch&, cudaStream_t);
template int fd_launch<26>(const FDLaunch&, cudaStream_t);
template int fd_launch<30>(const FDLaunch&, cudaStream_t);
template int fd_launch<34>(const FDLaunch&, cudaStream_t);
template int fd_launch<38>(const FDLaunch&, cudaStream_t);
}  // namespace smg
