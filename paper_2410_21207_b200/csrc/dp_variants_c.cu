// DP variants 9- (9: large batches: one 10-warp CTA per image up to 1120 columns,
// two CTAs per SM; measured on B200 against K=4 / K=16 / C=8 / 9-warp shapes,
// DESIGN.md §4.3b). Small batches (fewer images than SMs) keep variant 5; the
// 2- and 3-CTA shapes <2,8,8,8> <4,8,5,4> <2,8,12,8> <4,8,4,8> measured slower.
#define CARVE_KERNELS_HELPERS_ONLY
#include "carve_kernels.cuh"
#include "dp_variants.h"

namespace carve_dev {
void dp2_variants_c(std::vector<Dp2Variant>& t) {
    t.push_back(dp2_variant<4, 8, 10, 4, 2>());  // 9: S=112, 1120 cols/CTA, 4-row ring
    // single images wider than 2048 columns (tools/prof_dp_phases.py, B200 forward
    // cycles per row): 2160 wide 153 (v1) -> 137 (v13); 7680 wide 275 (v3) -> 204 (v11)
    t.push_back(dp2_variant<4, 16, 5, 8>());   // 10: S=96, 480 cols/CTA (smem fallback of 11)
    t.push_back(dp2_variant<4, 16, 5, 16>());  // 11: S=96, 480 cols/CTA, 16-row ring (C4: 16 CTAs)
    t.push_back(dp2_variant<2, 16, 5, 16>());  // 12: S=32, 160 cols/CTA (C3 height phase: 14 CTAs)
    // 13: S=96, 1536 cols/CTA: widths above 12288 (up to 24576 in 16 CTAs)
    t.push_back(dp2_variant<4, 16, 16, 8>());
}
}  // namespace carve_dev
