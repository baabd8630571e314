// abi_i64.cu -- C-ABI entry points of key type i64 (ascending and
// descending order): one translation unit per key type, so the library
// builds in parallel (include/stablemerge.h; drivers in sm_host.cuh).
#include "sm_host.cuh"

extern "C" {
SM_DEFINE_ABI(i64, int64_t, int64_t)
SM_DEFINE_ABI(desc_i64, sm::Desc<int64_t>, int64_t)
}  // extern "C"
