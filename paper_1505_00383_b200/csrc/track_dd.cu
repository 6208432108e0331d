// track_dd.cu -- compiled kernel variants at level dd (see kernels.hpp / track_impl.cuh).
#include "track_impl.cuh"

namespace pp {
namespace dev {

static const Variant kVariants[] = {
    PP_VARIANT(pp::dd_t, 4), PP_VARIANT(pp::dd_t, 8), PP_VARIANT(pp::dd_t, 10), PP_VARIANT(pp::dd_t, 16),
};

// Measured (cyclic-10, 131,072 paths, one B200): the register-resident solvers are slower than the
// shared-memory column in double-double (lsq 7.2 s streaming / 6.5 s holding q_i vs 5.5 s), because
// 128-255 registers per thread leave 8-16 warps per SM for FP64 chains of little ILP; none are built.
const LsqReg* lsq_reg_dd(int* count) {
  *count = 0;
  return nullptr;
}

const Variant* variants_dd(int* count) {
  *count = static_cast<int>(sizeof(kVariants) / sizeof(kVariants[0]));
  return kVariants;
}

}  // namespace dev
}  // namespace pp
