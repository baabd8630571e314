// abi_u64.cu -- C-ABI entry points of key type u64 (ascending and
// descending order): one translation unit per key type, so the library
// builds in parallel (include/stablemerge.h; drivers in sm_host.cuh).
#include "sm_host.cuh"

extern "C" {
SM_DEFINE_ABI(u64, uint64_t, uint64_t)
SM_DEFINE_ABI(desc_u64, sm::Desc<uint64_t>, uint64_t)
}  // extern "C"
