// Kernel instantiations for c == 2.
#include "fcm_kernels.cuh"
namespace fcm {
FCM_INSTANTIATE(2)
}
