// Kernel instantiations for c == 16 (9 <= c <= 16 runs here with runtime c).
#include "fcm_kernels.cuh"
namespace fcm {
FCM_INSTANTIATE(16)
}
