// Kernel instantiations for c == 4.
#include "fcm_kernels.cuh"
namespace fcm {
FCM_INSTANTIATE(4)
}
