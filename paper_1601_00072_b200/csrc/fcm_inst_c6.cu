// Kernel instantiations for c == 6.
#include "fcm_kernels.cuh"
namespace fcm {
FCM_INSTANTIATE(6)
}
