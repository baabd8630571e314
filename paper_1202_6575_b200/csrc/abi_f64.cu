// abi_f64.cu -- C-ABI entry points of key type f64 (ascending and
// descending order): one translation unit per key type, so the library
// builds in parallel (include/stablemerge.h; drivers in sm_host.cuh).
#include "sm_host.cuh"

extern "C" {
SM_DEFINE_ABI(f64, double, double)
SM_DEFINE_ABI(desc_f64, sm::Desc<double>, double)
}  // extern "C"
