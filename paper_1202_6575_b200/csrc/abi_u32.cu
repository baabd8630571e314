// abi_u32.cu -- C-ABI entry points of key type u32 (ascending and
// descending order): one translation unit per key type, so the library
// builds in parallel (include/stablemerge.h; drivers in sm_host.cuh).
#include "sm_host.cuh"

extern "C" {
SM_DEFINE_ABI(u32, uint32_t, uint32_t)
SM_DEFINE_ABI(desc_u32, sm::Desc<uint32_t>, uint32_t)
}  // extern "C"
