// DP variants 14- with the block-end label table in global memory (dp2_plan's last
// pass): tall or wide images whose table does not fit in shared memory (round 1
// failed with image_too_large there). Same shapes as 0, 11 and 13.
#define CARVE_KERNELS_HELPERS_ONLY
#include "carve_kernels.cuh"
#include "dp_variants.h"

namespace carve_dev {
void dp2_variants_d(std::vector<Dp2Variant>& t) {
    t.push_back(dp2_variant<2, 16, 4, 16, 1, true>());  // 14: as 0 (narrow, very tall)
    t.push_back(dp2_variant<4, 16, 5, 16, 1, true>());  // 15: as 11
    t.push_back(dp2_variant<4, 16, 16, 8, 1, true>());  // 16: as 13 (widths above 12288)
}
}  // namespace carve_dev
