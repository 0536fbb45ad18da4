// Generated: m -> coloured dense FD launcher table.
#include "smg_fd.cuh"
namespace smg {
extern template int fd_launch<3>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<4>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<5>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<6>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<7>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<8>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<9>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<10>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<11>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<12>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<13>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<14>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<15>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<16>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<17>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<18>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<19>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<20>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<21>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<22>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<23>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<24>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<25>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<26>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<27>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<28>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<29>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<30>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<31>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<32>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<33>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<34>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<35>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<36>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<37>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<38>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<39>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<40>(const FDLaunch&, cudaStream_t);
extern template int fd_launch<41>(const FDLaunch&, cudaStream_t);
FDLaunchFn fd_dispatch(int m) {
  switch (m) {
    case 3: return &fd_launch<3>;
    case 4: return &fd_launch<4>;
    case 5: return &fd_launch<5>;
    case 6: return &fd_launch<6>;
    case 7: return &fd_launch<7>;
    case 8: return &fd_launch<8>;
    case 9: return &fd_launch<9>;
    case 10: return &fd_launch<10>;
    case 11: return &fd_launch<11>;
    case 12: return &fd_launch<12>;
    case 13: return &fd_launch<13>;
    case 14: return &fd_launch<14>;
    case 15: return &fd_launch<15>;
    case 16: return &fd_launch<16>;
    case 17: return &fd_launch<17>;
    case 18: return &fd_launch<18>;
    case 19: return &fd_launch<19>;
    case 20: return &fd_launch<20>;
    case 21: return &fd_launch<21>;
    case 22: return &fd_launch<22>;
    case 23: return &fd_launch<23>;
    case 24: return &fd_launch<24>;
    case 25: return &fd_launch<25>;
    case 26: return &fd_launch<26>;
    case 27: return &fd_launch<27>;
    case 28: return &fd_launch<28>;
    case 29: return &fd_launch<29>;
    case 30: return &fd_launch<30>;
    case 31: return &fd_launch<31>;
    case 32: return &fd_launch<32>;
    case 33: return &fd_launch<33>;
    case 34: return &fd_launch<34>;
    case 35: return &fd_launch<35>;
    case 36: return &fd_launch<36>;
    case 37: return &fd_launch<37>;
    case 38: return &fd_launch<38>;
    case 39: return &fd_launch<39>;
    case 40: return &fd_launch<40>;
    case 41: return &fd_launch<41>;
    default: return nullptr;
  }
}
}  // namespace smg
