// track_d.cu -- compiled kernel variants at level d (see kernels.hpp / track_impl.cuh).
#include "track_impl.cuh"

namespace pp {
namespace dev {

static const Variant kVariants[] = {
    PP_VARIANT(double, 4), PP_VARIANT(double, 8), PP_VARIANT(double, 10), PP_VARIANT(double, 16),
};

static const LsqReg kLsqReg[] = {
    PP_LSQ_REG(double, 5), PP_LSQ_REG(double, 8), PP_LSQ_REG(double, 10), PP_LSQ_REG(double, 13),
};

const LsqReg* lsq_reg_d(int* count) {
  *count = static_cast<int>(sizeof(kLsqReg) / sizeof(kLsqReg[0]));
  return kLsqReg;
}

const Variant* variants_d(int* count) {
  *count = static_cast<int>(sizeof(kVariants) / sizeof(kVariants[0]));
  return kVariants;
}

}  // namespace dev
}  // namespace pp
