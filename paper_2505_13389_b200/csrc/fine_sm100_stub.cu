// placeholder until the tcgen05 fine kernels land
#include "common.cuh"
#include "launch.h"
namespace vsa_host {
bool sm100_fine_supported(const vsa_layout_t&, int64_t, int32_t) { return false; }
int launch_fine_forward_sm100(const vsa_layout_t&, int64_t, int64_t, const void*, const void*, const void*,
                              const int32_t*, int64_t, void*, float*, float*, const void*, const void*, const float*,
                              int32_t, void*, cudaStream_t) { return VSA_EINVAL; }
int launch_fine_backward_sm100(const vsa_layout_t&, int64_t, int64_t, const void*, const void*, const void*,
                               const void*, const float*, const float*, const int32_t*, int64_t, const int32_t*,
                               const int32_t*, const float*, const float*, const float*, int32_t, void*, void*, void*,
                               cudaStream_t) { return VSA_EINVAL; }
}
