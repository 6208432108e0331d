// track_qd.cu -- compiled kernel variants at level qd (see kernels.hpp / track_impl.cuh).
#include "track_impl.cuh"

namespace pp {
namespace dev {

static const Variant kVariants[] = {
    PP_VARIANT(pp::qd_t, 4), PP_VARIANT(pp::qd_t, 8), PP_VARIANT(pp::qd_t, 10), PP_VARIANT(pp::qd_t, 16),
};

const Variant* variants_qd(int* count) {
  *count = static_cast<int>(sizeof(kVariants) / sizeof(kVariants[0]));
  return kVariants;
}

}  // namespace dev
}  // namespace pp
