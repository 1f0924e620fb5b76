// Kernel instantiations for c == 32 (17 <= c <= 32 runs here with runtime c:
// register-staged pass kernel, prologue and epilogue only).
#include "fcm_kernels.cuh"
namespace fcm {
FCM_INSTANTIATE(32)
}
