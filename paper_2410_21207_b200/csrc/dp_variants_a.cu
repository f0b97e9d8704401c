// DP variants 0-3 (single images: latency-bound rows, one C=2 warp per scheduler first)
#define CARVE_KERNELS_HELPERS_ONLY
#include "carve_kernels.cuh"
#include "dp_variants.h"

namespace carve_dev {
void dp2_variants_a(std::vector<Dp2Variant>& t) {
    t.push_back(dp2_variant<2, 16, 4, 16>());  // 0: S=32,  128 cols/CTA, one warp per scheduler (C1/C2/C5-wide rows)
    t.push_back(dp2_variant<2, 16, 8, 16>());  // 1: S=32,  256 cols/CTA (C3, up to 4096 columns)
    t.push_back(dp2_variant<2, 16, 8, 8>());   // 2: S=32,  256 cols/CTA, 8-row ring
    t.push_back(dp2_variant<4, 16, 8, 8>());   // 3: S=96,  768 cols/CTA (C4: 7680 columns in 10 CTAs)
}
}  // namespace carve_dev
