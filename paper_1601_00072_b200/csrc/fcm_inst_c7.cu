// Kernel instantiations for c == 7.
#include "fcm_kernels.cuh"
namespace fcm {
FCM_INSTANTIATE(7)
}
