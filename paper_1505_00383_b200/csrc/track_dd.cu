// track_dd.cu -- compiled kernel variants at level dd (see kernels.hpp / track_impl.cuh).
#include "track_impl.cuh"

namespace pp {
namespace dev {

static const Variant kVariants[] = {
    PP_VARIANT(pp::dd_t, 4), PP_VARIANT(pp::dd_t, 8), PP_VARIANT(pp::dd_t, 10), PP_VARIANT(pp::dd_t, 16),
};

const Variant* variants_dd(int* count) {
  *count = static_cast<int>(sizeof(kVariants) / sizeof(kVariants[0]));
  return kVariants;
}

}  // namespace dev
}  // namespace pp
