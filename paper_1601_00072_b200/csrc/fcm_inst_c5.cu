// Kernel instantiations for c == 5.
#include "fcm_kernels.cuh"
namespace fcm {
FCM_INSTANTIATE(5)
}
