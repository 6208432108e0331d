// track_d.cu -- compiled kernel variants at level d (see kernels.hpp / track_impl.cuh).
#include "track_impl.cuh"

namespace pp {
namespace dev {

static const Variant kVariants[] = {
    PP_VARIANT(double, 4), PP_VARIANT(double, 8), PP_VARIANT(double, 10), PP_VARIANT(double, 16),
};

const Variant* variants_d(int* count) {
  *count = static_cast<int>(sizeof(kVariants) / sizeof(kVariants[0]));
  return kVariants;
}

}  // namespace dev
}  // namespace pp
