// abi_u128.cu -- C-ABI entry points of key type u128 (ascending and
// descending order): one translation unit per key type, so the library
// builds in parallel (include/stablemerge.h; drivers in sm_host.cuh).
#include "sm_host.cuh"

extern "C" {
SM_DEFINE_ABI(u128, sm::u128, sm_u128)
SM_DEFINE_ABI(desc_u128, sm::Desc<sm::u128>, sm_u128)
}  // extern "C"
