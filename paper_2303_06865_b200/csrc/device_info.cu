// device_info.cu -- per-device launch facts shared by the launchers (SM count), computed once
// per device under a lock: the library's only cached state (include/flexq.h).
#include <cuda_runtime.h>

#include <mutex>

#include "flexq_internal.h"

namespace flexq {

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < kMaxDevices ? dev : 0;
}

int device_sm_count() {
    static int sms[kMaxDevices];
    static std::once_flag once[kMaxDevices];
    const int dev = current_device();
    std::call_once(once[dev], [dev] {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        sms[dev] = n > 0 ? n : 148;
    });
    return sms[dev];
}

}  // namespace flexq
