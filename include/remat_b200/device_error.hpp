// device_error.hpp -- the one exception type the device-backed solver adds to
// the reference's vocabulary (errors.hpp has no device, hence no equivalent).
#pragma once

#include <stdexcept>

namespace remat {

// Raised when the device path cannot run (no sm_100 GPU, CUDA error, device
// OOM).  There is no CPU fallback to hide behind.
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

}  // namespace remat
