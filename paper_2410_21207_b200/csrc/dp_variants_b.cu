// DP variants 4-8 (fallbacks for tall or wide images; small batches)
#define CARVE_KERNELS_HELPERS_ONLY
#include "carve_kernels.cuh"
#include "dp_variants.h"

namespace carve_dev {
void dp2_variants_b(std::vector<Dp2Variant>& t) {
    t.push_back(dp2_variant<2, 8, 16, 8>());   // 4: S=48,  768 cols/CTA
    t.push_back(dp2_variant<4, 16, 4, 8>());   // 5: S=96,  384 cols/CTA (small batches)
    t.push_back(dp2_variant<4, 16, 4, 16>());  // 6: S=96,  384 cols/CTA, 16-row ring
    t.push_back(dp2_variant<4, 32, 4, 8>());   // 7: S=64,  256 cols/CTA
    t.push_back(dp2_variant<2, 16, 4, 8>());   // 8: S=32,  128 cols/CTA, 8-row ring
}
}  // namespace carve_dev
