// Library-level entry points: error string, ABI version, device check.
#include <cuda_runtime.h>

#include "nif_b200.h"
#include "kernels.h"
#include "status.h"

extern "C" const char* nif_last_error(void) { return nif::last_error().c_str(); }

extern "C" int nif_abi_version(void) { return 1; }

extern "C" int nif_device_check(int device) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    nif::fail(NIF_ERR_CUDA, "no CUDA device %d", device);
    return 0;
  }
  if (prop.major != 10 || prop.minor != 0) {
    nif::fail(NIF_ERR_UNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a", device,
              prop.major, prop.minor);
    return 0;
  }
  return 1;
}

namespace nif {
int sm_count() {
  static thread_local int count = 0;
  if (count == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev);
    if (count <= 0) count = 148;
  }
  return count;
}
}  // namespace nif
