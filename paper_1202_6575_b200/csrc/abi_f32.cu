// abi_f32.cu -- C-ABI entry points of key type f32 (ascending and
// descending order): one translation unit per key type, so the library
// builds in parallel (include/stablemerge.h; drivers in sm_host.cuh).
#include "sm_host.cuh"

extern "C" {
SM_DEFINE_ABI(f32, float, float)
SM_DEFINE_ABI(desc_f32, sm::Desc<float>, float)
}  // extern "C"
