// Kernel instantiations for c == 8.
#include "fcm_kernels.cuh"
namespace fcm {
FCM_INSTANTIATE(8)
}
