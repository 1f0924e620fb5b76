// Kernel instantiations for c == 3.
#include "fcm_kernels.cuh"
namespace fcm {
FCM_INSTANTIATE(3)
}
