// abi_i32.cu -- C-ABI entry points of key type i32 (ascending and
// descending order): one translation unit per key type, so the library
// builds in parallel (include/stablemerge.h; drivers in sm_host.cuh).
#include "sm_host.cuh"

extern "C" {
SM_DEFINE_ABI(i32, int32_t, int32_t)
SM_DEFINE_ABI(desc_i32, sm::Desc<int32_t>, int32_t)
}  // extern "C"
