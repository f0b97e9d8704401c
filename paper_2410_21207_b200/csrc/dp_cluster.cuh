// dp_cluster.cuh — K2+K3 v2: cluster-spread trapezoid DP, argmin, backtrack.
//
// Recurrence (solvers.hpp:116-157, 263-289): M[0][j] = e[0][j];
//   M[i][j] = e[i][j] + min(M[i-1][j-1], M[i-1][j], M[i-1][j+1]) scanned
//   left, mid, right with strict < (smallest column wins ties); out-of-range
//   neighbours excluded. Out-of-image columns hold +inf here (e := +inf), which
//   is equivalent because the middle candidate is always finite.
//
// Work decomposition. The row is cut into warp segments of
// S = 32*C - 2*K useful columns. Warp g holds 32*C consecutive columns
// [g*S - K, g*S - K + 32*C) in registers (C per lane): its S useful columns
// plus a K-column halo on each side that overlaps its neighbours. It then
// computes K rows with lane shuffles only; the valid region shrinks by one
// column per row on each side, so after K rows exactly its S useful columns
// are exact. Only then do neighbouring warps swap K halo values through a
// shared-memory mailbox — in the neighbour CTA's shared memory (DSMEM) when
// the neighbour lives in another CTA of the thread-block cluster — followed
// by one barrier. One barrier per K rows instead of one per row; the price is
// 2K/(32C) redundant halo cells.
//
// Backtrack (solvers.hpp:94-111) without an H-step serial chain:
//  * labels: every cell also carries the column, at the row above its
//    32-row block, that its optimal path descends from (selected with the same
//    predicates as M). Each block's last-row labels stay in shared memory as
//    int8 offsets; phase 1 hops block to block (one lookup per 32 rows).
//  * M-boundary rows: M of every 32nd row goes to global memory. Phase 2
//    recomputes each block's 32 rows bit-identically inside a 128-column
//    window around the block's known bottom column (one warp per block, all
//    blocks in parallel), records directions in shared memory and walks them.
// No per-cell direction plane is written in the hot loop.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <type_traits>
#include <cstdio>

namespace carve_dev {

namespace cg = cooperative_groups;

#ifdef CARVE_DEBUG
#define DP2_ALIGN(ptr, n, tag)                                                                                  \
    do {                                                                                                       \
        if ((reinterpret_cast<uintptr_t>(ptr) % (n)) != 0)                                                    \
            printf("misaligned %s: %p blk %d thr %d\n", tag, (const void*)(ptr), int(blockIdx.x), int(threadIdx.x)); \
    } while (0)
#else
#define DP2_ALIGN(ptr, n, tag) \
    do {                       \
    } while (0)
#endif

constexpr int LBLK = 32;      // label / M-boundary block height (rows)
constexpr int P2_COLS = 128;  // phase-2 window: 32 lanes x 4 columns

struct Dp2Params {
    double* e;         // energy plane (pitch epitch), image stride e_istride
    int epitch;
    int W, H;
    int G;             // warps in the cluster (= ncl * NWARP)
    int nblk;          // label blocks: ceil((H-1)/LBLK)
    double* mbound;    // [nblk][mpitch] M rows 0, 32, 64, ... (global scratch), image stride mb_istride
    int mpitch;
    int* seam;         // H ints, image stride s_istride
    double* m_out;     // optional full cost table (pitch W)
    int* b_out;        // optional predecessor table (pitch W)
    unsigned long long* stamps;  // optional per-seam record [energy start, energy end, solve start, solve end, ...]
    const int* stop;             // optional device flag: nonzero = return at once (data-dependent loops)
    long long e_istride, mb_istride, s_istride, st_istride;
    int dbg;           // debugging: bit0 skips phase 2, bit1 skips phase 1, bit2 skips the walk
    long long* prof;   // MODE 2 only: [G][8] per-warp clock64 counters
    // K1 fix-up for the previous seam (nullable): the removal kernel shifted
    // the planes in place; the two new-grid columns per row around the
    // previous seam get their energy recomputed here from the compacted RGBX
    const int* prev_seam;  // image stride s_istride
    const uint32_t* rgb;   // RGBX plane (pitch rpitch), image stride rgb_istride
    int rpitch;
    long long rgb_istride;
    int gather;  // 1: CTA 0 holds a gathered copy of every CTA's block-end labels (phase 1 stays local)
    long long cplane;  // FWD without FUSED: element stride from the cost_left plane (e) to cost_up and
                       // from cost_up to cost_right (three padded planes of the same pitch)
    // label table in global memory ([nblk][G*S] int8 offsets, image stride glab_istride)
    // instead of shared memory: tall or wide images whose table does not fit on chip
    int8_t* glab;
    long long glab_istride;
};

// smem layout (dynamic): labels int8 [nblk][NWARP*S], aliased by the phase-2
// dirs (labels are dead once phase 1 has hopped through them) | mailbox |
// reduce | energy/RGBX ring | gathered label table (optional)
// RE = ring bytes per column: FP64 energies, or RGBX pixels in the fused mode
template <int C, int K, int NWARP, int RE = 8>
struct Dp2Smem {
    static constexpr int S = 32 * C - 2 * K;
    static constexpr int COLS = NWARP * S;  // useful columns per CTA
    __host__ __device__ static size_t labels_bytes(int nblk) { return (size_t(nblk) * COLS + 15) & ~size_t(15); }
    static constexpr size_t mail_bytes = size_t(2) * NWARP * 2 * K * (8 + 4);
    static constexpr size_t p2_bytes = size_t(NWARP) * LBLK * P2_COLS;
    __host__ __device__ static size_t lp2_bytes(int nblk) {
        return labels_bytes(nblk) > p2_bytes ? labels_bytes(nblk) : p2_bytes;
    }
    static constexpr size_t red_bytes = 64 * 16 + NWARP * 2 * 8;  // argmin scratch + halo mbarriers
    __host__ __device__ static constexpr size_t ring_bytes(int D) { return size_t(NWARP) * D * 32 * C * RE; }
    __host__ __device__ static size_t total(int nblk, int D) {
        return lp2_bytes(nblk) + mail_bytes + red_bytes + ring_bytes(D);
    }
};

// the 9-instruction cell update shared by the forward pass and phase 2
// (DSETP, 2xFSEL, DSETP, 2xFSEL, DADD + the selects that carry the label)
__device__ __forceinline__ void dp_cell(double L, double M, double R, int lL, int lM, int lR, double e, double& out,
                                        int& lab, int& d) {
    double best = L;
    int bl = lL;
    d = 0;
    if (M < best) { best = M; bl = lM; d = 1; }
    if (R < best) { best = R; bl = lR; d = 2; }
    out = __dadd_rn(e, best);
    lab = bl;
}

// C consecutive energies starting at col0 (even): unconditional aligned
// 128-bit loads — the padded plane (EPAD_L/EPAD_R, +inf) covers every column a
// warp or a phase-2 window can touch.
// Same result and tie-break as dp_cell, but the left candidate (the one that
// arrives last, by shuffle, for a lane's first column) is combined last:
// t = argmin(M, R) with M winning ties, then L wins if L <= t. The scan order
// L, M, R with strict < selects exactly this cell, so the seam is unchanged,
// while only one compare-select sits between the shuffle and the add.
__device__ __forceinline__ void dp_cell_left_last(double L, double M, double R, int lL, int lM, int lR, double e,
                                                  double& out, int& lab, int& d) {
    double t = M;
    int tl = lM, td = 1;
    if (R < t) { t = R; tl = lR; td = 2; }
    const bool left = L <= t;
    out = __dadd_rn(e, left ? L : t);
    lab = left ? lL : tl;
    d = left ? 0 : td;
}

// Forward-energy cell (dp_seam_forward, solvers.hpp:304-323): the candidates
// are prev + transition cost, compared in the order left, up, right with strict
// < (smallest column on ties). Out-of-image neighbours are +inf (pads), so
// `best = left` first is the reference's `best = +inf` start.
__device__ __forceinline__ void fwd_cell(double L, double M, double R, int lL, int lM, int lR, double cl, double cu,
                                         double cr, double& out, int& lab, int& d) {
    double best = __dadd_rn(L, cl);
    int bl = lL;
    d = 0;
    const double mv = __dadd_rn(M, cu);
    if (mv < best) { best = mv; bl = lM; d = 1; }
    const double rv = __dadd_rn(R, cr);
    if (rv < best) { best = rv; bl = lR; d = 2; }
    out = best;
    lab = bl;
}
// same cell with the shuffled left operand compared last (see dp_cell_left_last)
__device__ __forceinline__ void fwd_cell_left_last(double L, double M, double R, int lL, int lM, int lR, double cl,
                                                   double cu, double cr, double& out, int& lab, int& d) {
    double t = __dadd_rn(M, cu);
    int tl = lM, td = 1;
    const double rv = __dadd_rn(R, cr);
    if (rv < t) { t = rv; tl = lR; td = 2; }
    const double lv = __dadd_rn(L, cl);
    const bool left = lv <= t;
    out = left ? lv : t;
    lab = left ? lL : tl;
    d = left ? 0 : td;
}

// `coherent`: the row may have been written earlier in this same launch (the
// prologue's fix-up), so it is read through L2 (ld.global.cg) rather than the
// read-only path, which is only defined for data constant during the kernel.
template <int C>
__device__ __forceinline__ void load_row(const double* __restrict__ row, int col0, double (&v)[C],
                                         bool coherent = false) {
#pragma unroll
    for (int k = 0; k < C; k += 2) {
        const double2* a = reinterpret_cast<const double2*>(row + col0 + k);
        const double2 x = coherent ? __ldcg(a) : __ldg(a);
        v[k] = x.x;
        v[k + 1] = x.y;
    }
}

// ---- DSMEM point-to-point halo transport (st.async + mbarrier complete_tx) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t a, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(tx) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t a, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void st_async_b64(uint32_t raddr, double v, uint32_t rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rmbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_b32(uint32_t raddr, uint32_t v, uint32_t rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr), "r"(v),
                 "r"(rmbar)
                 : "memory");
}

// predicated vector forms (one role per lane, no branch in the exchange)
__device__ __forceinline__ void st_async_v2_b64_if(bool pr, uint32_t raddr, double a, double b, uint32_t rmbar) {
    asm volatile(
        "{ .reg .pred p; setp.ne.u32 p, %4, 0;\n"
        "@p st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3]; }" ::"r"(raddr),
        "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(rmbar), "r"(uint32_t(pr))
        : "memory");
}
__device__ __forceinline__ int ld_shared_s32(uint32_t a) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_async_v2_b32_if(bool pr, uint32_t raddr, uint32_t a, uint32_t b, uint32_t rmbar) {
    asm volatile(
        "{ .reg .pred p; setp.ne.u32 p, %4, 0;\n"
        "@p st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3]; }" ::"r"(raddr),
        "r"(a), "r"(b), "r"(rmbar), "r"(uint32_t(pr))
        : "memory");
}

// ---- energy-row ring: per-lane cp.async (LDGSTS) into shared memory ----------
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t saddr, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr), "l"(g) : "memory");
}
// predicated form: a lane whose bytes are never used skips the global read
__device__ __forceinline__ void cp_async16_if(bool pred, uint32_t saddr, const void* g) {
    asm volatile("{.reg .pred q; setp.ne.b32 q, %0, 0; @q cp.async.cg.shared.global [%1], [%2], 16;}" ::"r"(int(pred)),
                 "r"(saddr), "l"(g)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// e1 of a lane's C columns from three luma rows (up, cur, down); the columns
// just outside the lane come from the neighbouring lanes (garbage at a warp's
// outermost columns, which the trapezoid treats as invalid anyway); columns
// outside the image are +inf (candidate exclusion).
template <int C>
__device__ __forceinline__ void energy_cols(const double (&Lp)[C], const double (&Lc)[C], const double (&Ln)[C],
                                            uint32_t oob, double (&ev)[C]) {
    const double lL = __shfl_up_sync(FULL, Lc[C - 1], 1);
    const double lR = __shfl_down_sync(FULL, Lc[0], 1);
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const double left = k > 0 ? Lc[k - 1] : lL;
        const double right = k + 1 < C ? Lc[k + 1] : lR;
        ev[k] = e1(left, right, Lp[k], Ln[k]);
    }
    if (oob) {
#pragma unroll
        for (int k = 0; k < C; ++k)
            if (oob >> k & 1) ev[k] = dinf();
    }
}

// forward_costs (energy.hpp:196-216) of a lane's C columns from the luma rows
// above (Lp) and current (Lc): cu = |R - L|, cl = cu + |A - L|, cr = cu + |A - R|,
// horizontal neighbours clamped through the RGBX replica columns; +inf outside.
template <int C>
__device__ __forceinline__ void fwd_cols(const double (&Lp)[C], const double (&Lc)[C], uint32_t oob, double (&cl)[C],
                                         double (&cu)[C], double (&cr)[C]) {
    const double lL = __shfl_up_sync(FULL, Lc[C - 1], 1);
    const double lR = __shfl_down_sync(FULL, Lc[0], 1);
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const double left = k > 0 ? Lc[k - 1] : lL;
        const double right = k + 1 < C ? Lc[k + 1] : lR;
        const double up = fabs(__dsub_rn(right, left));
        cu[k] = up;
        cl[k] = __dadd_rn(up, fabs(__dsub_rn(Lp[k], left)));
        cr[k] = __dadd_rn(up, fabs(__dsub_rn(Lp[k], right)));
    }
    if (oob) {
#pragma unroll
        for (int k = 0; k < C; ++k)
            if (oob >> k & 1) cl[k] = cu[k] = cr[k] = dinf();
    }
}

template <int C>
__device__ __forceinline__ void luma_cols(const uint32_t* px, double (&L)[C]) {
#pragma unroll
    for (int k = 0; k < C; ++k) L[k] = luma(px[k]);
}

__device__ __forceinline__ void argmin_combine(double& v, int& i, double ov, int oi) {
    if (ov < v || (ov == v && oi < i)) { v = ov; i = oi; }
}

// MODE 0: hot kernel; 1: also writes the full cost/predecessor tables (parity
// API); 2: hot kernel + per-warp clock64 phase counters into p.prof (tools only)
// FUSED: no energy plane — e1 is recomputed in registers from RGBX rows
// streamed through the same ring (rolling three luma rows per lane). Used for
// batches, where the energy plane's 16 B/px/seam of traffic bounds throughput.
// FWD: forward energy (CarveConfig::forward, carver.hpp:155-169): the cells take
// dp_seam_forward's transition costs — with FUSED computed in registers from the
// luma of the RGBX rows above and current; without FUSED streamed from three
// caller-given FP64 cost planes (cost_left at e, cost_up at e + cplane,
// cost_right at e + 2*cplane), 24 B per column through the same ring: the
// dp_seam_forward(gray, costs) API with arbitrary costs (solvers.hpp:294-326)
// and the recompute=false forward loop, whose costs are carved, not recomputed
// (carver.hpp:175-184).
// GLAB: the block-end label table lives in global memory (Dp2Params::glab) instead
// of shared memory — separate instances for images whose table does not fit on chip.
template <int C, int K, int NWARP, int D, int MODE, bool FUSED = false, bool FWD = false, int MINB = 1,
          bool GLAB = false>
__global__ void __launch_bounds__(NWARP * 32, MINB) k_dp2(Dp2Params p) {
    constexpr bool TABLES = MODE == 1;
    constexpr bool PROF = MODE == 2;
    long long pf_t0 = 0, pf_wait = 0;
    if constexpr (PROF) pf_t0 = clock64();
    static_assert(K % C == 0 && (32 * C) > 2 * K, "halo must be whole lanes and leave useful columns");
    constexpr int RE = FUSED ? 4 : (FWD ? 24 : 8);  // ring bytes per column
    using SM = Dp2Smem<C, K, NWARP, RE>;
    constexpr int S = SM::S;
    constexpr int KL = K / C;  // lanes per halo
    extern __shared__ __align__(16) unsigned char dsm[];
    cg::cluster_group cluster = cg::this_cluster();
    const int ncl = int(cluster.num_blocks());
    const int cta = int(cluster.block_rank());
    const int img = blockIdx.x / ncl;

    double* __restrict__ e = p.e + img * p.e_istride;
    double* __restrict__ mbound = p.mbound + img * p.mb_istride;
    int* __restrict__ seam = p.seam + img * p.s_istride;
    const int W = p.W, H = p.H, G = p.G, nblk = p.nblk;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = cta * NWARP + warp;
    const int ucol0 = g * S;                   // first useful column of this warp
    const int col0 = ucol0 - K + lane * C;     // first column held by this lane
    const int cta_col0 = cta * SM::COLS;

    int8_t* labels = reinterpret_cast<int8_t*>(dsm);
    uint8_t* p2 = dsm;  // phase-2 dirs alias the labels
    int8_t* glab = GLAB ? p.glab + img * p.glab_istride : nullptr;  // global label table (else shared)
    double* mail_m = reinterpret_cast<double*>(dsm + SM::lp2_bytes(GLAB ? 0 : nblk));  // [2][NWARP][2][K]
    int* mail_l = reinterpret_cast<int*>(mail_m + 2 * NWARP * 2 * K);
    double* red_v = reinterpret_cast<double*>(mail_l + 2 * NWARP * 2 * K);
    int* red_i = reinterpret_cast<int*>(red_v + 32);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(red_v + 64);  // [NWARP][2 parities]: my halos have landed
    unsigned char* ring_b = reinterpret_cast<unsigned char*>(red_v) + SM::red_bytes;
    // this lane's C columns of stage u: ring_b[(((warp * D + u) * 32 + lane) * C) * RE]
    const uint32_t ring_lane = smem_u32(ring_b + (size_t(warp) * D * 32 + lane) * C * RE);

    // the previous seam was written by the DP before the removal this launch depends on
    // (that DP had completed before the removal ran), so its column of my first fix-up
    // row is read before the grid dependency wait, off the prologue's latency chain
    const int fx_nthr = ncl * NWARP * 32, fx_tid = cta * NWARP * 32 + threadIdx.x;
    int fx_sp0 = 0;
    if (p.prev_seam && fx_tid < H) fx_sp0 = __ldcg(p.prev_seam + img * p.s_istride + fx_tid);
    pdl_wait();  // the previous removal has completed (its planes and seam log are visible)
    pdl_launch_dependents();
    // a data-dependent loop (object removal) enqueued past its end: every CTA reads the
    // same flag (set by a kernel that completed before this one), so all return together
    if (p.stop && *p.stop) return;
    // energy = the prologue's incremental fix-up (seams after a phase's first; the first
    // seam's energy is the K1 launch), solve = the rest of this launch
    if (p.stamps && cta == 0 && threadIdx.x == 0)
        p.stamps[img * p.st_istride + (p.prev_seam ? 0 : 2)] = globaltimer();

    // K1 fix-up of the previous removal: rows are
    // spread over every thread of the cluster; made visible by the cluster barrier below
    if (p.prev_seam) {
        const int* ps = p.prev_seam + img * p.s_istride;
        const uint32_t* rgb = p.rgb + img * p.rgb_istride;
        const int nthr = fx_nthr, tid = fx_tid;
        for (int i = tid; i < H; i += nthr) {
            const int sp = i == tid ? fx_sp0 : __ldg(ps + i);
            const uint32_t* row = rgb + (long long)i * p.rpitch;
            const uint32_t* up = rgb + (long long)max(i - 1, 0) * p.rpitch;
            const uint32_t* dn = rgb + (long long)min(i + 1, H - 1) * p.rpitch;
#pragma unroll
            for (int x = sp - 1; x <= sp; ++x)
                if (x >= 0 && x < W)
                    e[(long long)i * p.epitch + x] =
                        e1(luma(row[max(x - 1, 0)]), luma(row[min(x + 1, W - 1)]), luma(up[x]), luma(dn[x]));
        }
        // no gpu-scope fence: every reader of these energies is in this cluster, and the
        // cluster barrier below (arrive.release / wait.acquire) orders global writes at
        // cluster scope (measured: fix-up lap 2.59 -> 2.30 us per seam at C2)
    }

    // which of my C columns are useful (inside my segment and the image)
    uint32_t useful = 0;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const int j = col0 + k;
        if (j >= ucol0 && j < ucol0 + S && j < W) useful |= 1u << k;
    }

    double m[C];
    int lab[C];

    // Halo mailboxes. My left neighbour's right-halo slot (side 1) and my right
    // neighbour's left-halo slot (side 0), as shared::cluster addresses (the
    // neighbour may live in another CTA), plus their "landed" mbarriers.
    const int gl = g - 1, gr = g + 1;
    constexpr int PSTRIDE = NWARP * 2 * K;  // elements per parity
    uint32_t nl_m = 0, nl_l = 0, nl_b = 0, nr_m = 0, nr_l = 0, nr_b = 0;
    if (gl >= 0) {
        const uint32_t rk = uint32_t(gl / NWARP), w = uint32_t(gl % NWARP);
        nl_m = mapa_u32(smem_u32(mail_m + (w * 2 + 1) * K), rk);
        nl_l = mapa_u32(smem_u32(mail_l + (w * 2 + 1) * K), rk);
        nl_b = mapa_u32(smem_u32(mbar + w * 2), rk);
    }
    if (gr < G) {
        const uint32_t rk = uint32_t(gr / NWARP), w = uint32_t(gr % NWARP);
        nr_m = mapa_u32(smem_u32(mail_m + (w * 2 + 0) * K), rk);
        nr_l = mapa_u32(smem_u32(mail_l + (w * 2 + 0) * K), rk);
        nr_b = mapa_u32(smem_u32(mbar + w * 2), rk);
    }
    const double* my_m = mail_m + (warp * 2) * K;  // + side*K, + parity*PSTRIDE
    const int* my_l = mail_l + (warp * 2) * K;
    const uint32_t my_b = smem_u32(mbar + warp * 2);  // + parity*8
    const uint32_t halo_tx = uint32_t(((gl >= 0) + (gr < G)) * K * (8 + 4));
    // phase 1 hand-off (label tables left distributed): a (block, column) token message
    // slot and its mbarrier, after the argmin scratch (red_v[120..122))
    uint64_t* p1bar = reinterpret_cast<uint64_t*>(red_v + 120);
    int* p1msg = reinterpret_cast<int*>(red_v + 121);
    if (lane == 0) {
        mbar_init(my_b, 1);
        mbar_init(my_b + 8, 1);
        if (threadIdx.x == 0) mbar_init(smem_u32(p1bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // every mbarrier of the cluster is initialised before any halo is sent, and
    // every fix-up store is visible before any energy row is read
    if (ncl > 1) cluster.sync();
    else __syncthreads();
    if (p.stamps && p.prev_seam && cta == 0 && threadIdx.x == 0) {
        const unsigned long long t = globaltimer();
        p.stamps[img * p.st_istride + 1] = t;
        p.stamps[img * p.st_istride + 2] = t;
    }

    // fused mode: rolling luma rows (i-1, i, i+1) of my columns; rows clamp at the borders
    double Lp[C], Lc[C], Ln[C];
    uint32_t oob = 0;
    const uint32_t* rgbf = FUSED ? p.rgb + img * p.rgb_istride + col0 : nullptr;
    if constexpr (FUSED) {
#pragma unroll
        for (int k = 0; k < C; ++k)
            if (col0 + k < 0 || col0 + k >= W) oob |= 1u << k;
        uint32_t px[C];
#pragma unroll
        for (int k = 0; k < C; ++k) px[k] = __ldg(rgbf + k);
        luma_cols<C>(px, Lc);
        const uint32_t* r1 = rgbf + (long long)min(1, H - 1) * p.rpitch;
#pragma unroll
        for (int k = 0; k < C; ++k) px[k] = __ldg(r1 + k);
        luma_cols<C>(px, Ln);
#pragma unroll
        for (int k = 0; k < C; ++k) Lp[k] = Lc[k];
        if constexpr (FWD) {  // M[0] = cost_up(0, j) (solvers.hpp:300-302)
            double cl0[C], cr0[C];
            fwd_cols<C>(Lc, Lc, oob, cl0, m, cr0);
        } else {
            energy_cols<C>(Lp, Lc, Ln, oob, m);  // M[0] = e[0]
        }
    } else if constexpr (FWD) {  // cost planes: M[0] = cost_up(0, j); +inf outside the image
#pragma unroll
        for (int k = 0; k < C; ++k)
            if (col0 + k < 0 || col0 + k >= W) oob |= 1u << k;
        load_row<C>(e + p.cplane, col0, m);
#pragma unroll
        for (int k = 0; k < C; ++k)
            if (oob >> k & 1) m[k] = dinf();
    } else {
        load_row<C>(e, col0, m, p.prev_seam != nullptr);
    }
#pragma unroll
    for (int k = 0; k < C; ++k) lab[k] = col0 + k;
    // M-boundary row 0 (block 0 starts from it)
#pragma unroll
    for (int k = 0; k < C; ++k)
        if (useful >> k & 1) mbound[col0 + k] = m[k];
    if constexpr (TABLES) {
#pragma unroll
        for (int k = 0; k < C; ++k)
            if (useful >> k & 1) { p.m_out[col0 + k] = m[k]; p.b_out[col0 + k] = col0 + k; }
    }

    // Forward pass. Rows 1..H-1 run in K-row blocks, each fully unrolled so
    // the ring slot, the halo exchange point and the loop control are
    // compile-time; energy rows i+1..i+D are in flight while row i computes
    // (slot (i-1) % D is consumed, then refilled with row i+D).
    const double* nrow = e + p.epitch + col0;  // my slice of the next row to fetch (spare rows past H-1 are harmless)
    static_assert(C % 2 == 0, "cp.async moves 16-byte pairs of doubles");
    int frow = 2;  // fused: next RGBX row to fetch (the ring feeds luma row i+1 at row i)
    // ring rows travel in commit groups of two: one commit and one wait per two rows
    // (C2 DP 62.6 -> 61.4 us, C5 fused DP 1.53 -> 1.52 ms, 128 images 47.9 -> 46.8 ms;
    // groups of four measured 66.6 us at C2: the refill burst stalls the row)
    constexpr int RG = 2;
    constexpr bool PAIRS = RG > 1;
    static_assert(D % RG == 0 && K % RG == 0, "commit groups tile the ring and the K-blocks");
    auto fetch = [&](int u, bool commit = true) {  // this lane's C values of the next row -> ring stage u
        if constexpr (FUSED) {
            const uint32_t* src = rgbf + (long long)min(frow, H - 1) * p.rpitch;
            const uint32_t dst = ring_lane + uint32_t(u * 32 * C * RE);
            if constexpr (C == 2) cp_async8(dst, src);
            else {
#pragma unroll
                for (int k = 0; k < C; k += 4) cp_async16(dst + k * 4, src + k);
            }
            ++frow;
        } else {
            // this lane's C values of each plane: [plane 0 (C)][plane 1][plane 2] per stage
#pragma unroll
            for (int pl = 0; pl < (FWD ? 3 : 1); ++pl)
#pragma unroll
                for (int k = 0; k < C; k += 2)
                    cp_async16(ring_lane + uint32_t(u * 32 * C * RE + (pl * C + k) * 8), nrow + pl * p.cplane + k);
            nrow += p.epitch;
        }
        if (commit) cp_async_commit();
    };
    if constexpr (PAIRS) {
#pragma unroll
        for (int u = 0; u < D; ++u) fetch(u, u % RG == RG - 1);
    } else {
#pragma unroll
        for (int u = 0; u < D; ++u) fetch(u);
    }

    auto step = [&](int u, int i, int t) {
        if constexpr (PAIRS) {
            if (t % RG == 0) cp_async_wait<D / RG - 1>();  // the oldest group of rows has landed
        } else {
            cp_async_wait<D - 1>();  // the oldest of the D groups in flight has landed
        }
        double ev[C], fcl[C], fcu[C], fcr[C];  // energies, or forward transition costs (FWD)
        if constexpr (FUSED) {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(ring_b + ((size_t(warp) * D + u) * 32 + lane) * C * RE);
            uint32_t px[C];
#pragma unroll
            for (int k = 0; k < C; ++k) px[k] = src[k];
#pragma unroll
            for (int k = 0; k < C; ++k) { Lp[k] = Lc[k]; Lc[k] = Ln[k]; }
            luma_cols<C>(px, Ln);  // row i+1 (clamped at the bottom)
            if constexpr (FWD) fwd_cols<C>(Lp, Lc, oob, fcl, fcu, fcr);
            else energy_cols<C>(Lp, Lc, Ln, oob, ev);
        } else {
            const double* src = reinterpret_cast<const double*>(ring_b + ((size_t(warp) * D + u) * 32 + lane) * C * RE);
            if constexpr (FWD) {  // the ring row is cost row i of the three planes
#pragma unroll
                for (int k = 0; k < C; k += 2) {
                    const double2 a = *reinterpret_cast<const double2*>(src + k);
                    const double2 b = *reinterpret_cast<const double2*>(src + C + k);
                    const double2 c = *reinterpret_cast<const double2*>(src + 2 * C + k);
                    fcl[k] = a.x; fcl[k + 1] = a.y;
                    fcu[k] = b.x; fcu[k + 1] = b.y;
                    fcr[k] = c.x; fcr[k + 1] = c.y;
                }
                if (oob) {
#pragma unroll
                    for (int k = 0; k < C; ++k)
                        if (oob >> k & 1) fcl[k] = fcu[k] = fcr[k] = dinf();
                }
            } else {
#pragma unroll
                for (int k = 0; k < C; k += 2) {
                    const double2 x = *reinterpret_cast<const double2*>(src + k);
                    ev[k] = x.x;
                    ev[k + 1] = x.y;
                }
            }
        }
        const double lm = __shfl_up_sync(FULL, m[C - 1], 1);
        const int ll = __shfl_up_sync(FULL, lab[C - 1], 1);
        const double rm = __shfl_down_sync(FULL, m[0], 1);
        const int rl = __shfl_down_sync(FULL, lab[0], 1);
        double pm = lm;
        int pl = ll;
        uint32_t dbits = 0;
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const double cm = m[k];
            const int cl = lab[k];
            const double nm = (k + 1 < C) ? m[k + 1] : rm;
            const int nl = (k + 1 < C) ? lab[k + 1] : rl;
            int d;
            if constexpr (FWD) {
                if (k == 0) fwd_cell_left_last(pm, cm, nm, pl, cl, nl, fcl[k], fcu[k], fcr[k], m[k], lab[k], d);
                else fwd_cell(pm, cm, nm, pl, cl, nl, fcl[k], fcu[k], fcr[k], m[k], lab[k], d);
            } else {
                if (k == 0) dp_cell_left_last(pm, cm, nm, pl, cl, nl, ev[k], m[k], lab[k], d);
                else dp_cell(pm, cm, nm, pl, cl, nl, ev[k], m[k], lab[k], d);
            }
            dbits |= uint32_t(d) << (2 * k);
            pm = cm;
            pl = cl;
        }
        if constexpr (TABLES) {  // parity API only: full cost / predecessor tables
#pragma unroll
            for (int k = 0; k < C; ++k)
                if (useful >> k & 1) {
                    p.m_out[(long long)i * W + col0 + k] = m[k];
                    p.b_out[(long long)i * W + col0 + k] = col0 + k + int(dbits >> (2 * k) & 3) - 1;
                }
        }
        (void)dbits;
        if constexpr (PAIRS) {
            if (t % RG == RG - 1) {  // every row of the group consumed: refill the group
#pragma unroll
                for (int r = RG - 1; r >= 0; --r) fetch(u - r, r == 0);
            }
        } else {
            fetch(u);  // refill this stage with row i + D (own lane's bytes only: no cross-lane hazard)
        }
    };
    // block-end stores: shared-space label address and a running M-boundary
    // pointer, both hoisted (the generic->shared conversion was per call)
    const uint32_t lbl_s = smem_u32(labels + (col0 - cta_col0));
    double* mb_row = mbound + p.mpitch + col0;  // M row 32*(blk+1), advanced per label block
    auto block_end = [&](int i, int blk) {  // last row of a label block: labels to smem, M to global
        if constexpr (GLAB) {  // the table lives in global memory
#pragma unroll
            for (int k = 0; k < C; ++k)
                if (useful >> k & 1) glab[(long long)blk * (G * S) + col0 + k] = int8_t(lab[k] - (col0 + k));
        } else {
#pragma unroll
            for (int k = 0; k < C; ++k)
                if (useful >> k & 1)
                    asm volatile("st.shared.u8 [%0], %1;" ::"r"(lbl_s + uint32_t(blk * SM::COLS + k)),
                                 "r"(uint32_t(lab[k] - (col0 + k)))
                                 : "memory");
        }
        if (i != H - 1) {
#pragma unroll
            for (int k = 0; k < C; ++k)
                if (useful >> k & 1) mb_row[k] = m[k];
        }
        mb_row += p.mpitch;
    };
    auto reset_labels = [&]() {
#pragma unroll
        for (int k = 0; k < C; ++k) lab[k] = col0 + k;
    };
    int par = 0;
    uint32_t phases = 0;  // bit p: phase parity of my mbarrier for mailbox parity p
    // Per-lane exchange roles, hoisted out of the row loop. C divides K, so a
    // lane's C columns are either all halo, all edge-of-segment, or neither.
    const int wi0 = lane * C;  // my first column's index within the warp's 32*C
    const bool sendL = gl >= 0 && wi0 >= K && wi0 < 2 * K;
    const bool sendR = gr < G && wi0 >= 32 * C - 2 * K && wi0 < 32 * C - K;
    const bool recvL = lane < KL, recvR = lane >= 32 - KL;
    const uint32_t aLm = nl_m + uint32_t(wi0 - K) * 8, aLl = nl_l + uint32_t(wi0 - K) * 4;
    const uint32_t aRm = nr_m + uint32_t(wi0 - (32 * C - 2 * K)) * 8, aRl = nr_l + uint32_t(wi0 - (32 * C - 2 * K)) * 4;
    const double* rLm = my_m + wi0;                       // side 0 (+ parity*PSTRIDE)
    const int* rLl = my_l + wi0;
    const double* rRm = my_m + K + (wi0 - (32 * C - K));  // side 1
    const int* rRl = my_l + K + (wi0 - (32 * C - K));
    // A lane sends to at most one side and receives from at most one side (4K <= 32C,
    // K <= 16C), so each role is one predicated vector store / one selected load.
    static_assert(4 * K <= 32 * C && K <= 16 * C, "exchange roles must not overlap");
    const bool snd = sendL || sendR, rcv = recvL || recvR;
    const uint32_t s_m = sendL ? aLm : aRm, s_l = sendL ? aLl : aRl, s_b = sendL ? nl_b : nr_b;
    // non-receiving lanes read their own first mailbox slot (valid memory) and discard it
    const double* r_m = recvL ? rLm : recvR ? rRm : my_m;
    const int* r_l = recvL ? rLl : recvR ? rRl : my_l;
    const bool r_inf = recvL ? gl < 0 : (recvR && gr >= G);  // no neighbour on that side: +inf halo
    // exchange, split in two so the block-end bookkeeping runs under the DSMEM latency:
    auto send = [&]() {
        // send my K leftmost / rightmost useful columns straight into the
        // neighbours' halo mailboxes; each store completes bytes on the
        // neighbour's mbarrier (no cluster-wide barrier, no memory fence)
        const uint32_t po8 = uint32_t(par * PSTRIDE * 8), po4 = uint32_t(par * PSTRIDE * 4);
        const uint32_t mb = s_b + par * 8;
#pragma unroll
        for (int k = 0; k < C; k += 2) {
            st_async_v2_b64_if(snd, s_m + po8 + k * 8, m[k], m[k + 1], mb);
            st_async_v2_b32_if(snd, s_l + po4 + k * 4, uint32_t(lab[k]), uint32_t(lab[k + 1]), mb);
        }
    };
    auto recv = [&]() {
        // wait until both neighbours' halos for this parity have landed here
        if (lane == 0) mbar_arrive_expect_tx(my_b + par * 8, halo_tx);
        long long w0 = 0;
        if constexpr (PROF) w0 = clock64();
        while (!mbar_try_wait(my_b + par * 8, (phases >> par) & 1)) {
        }
        if constexpr (PROF) pf_wait += clock64() - w0;
        phases ^= 1u << par;
        // every lane loads (asm volatile: the loads cannot be skipped, so no branch), the
        // non-receiving lanes discard the values with selects
#pragma unroll
        for (int k = 0; k < C; k += 2) {
            double v0, v1;
            uint32_t l0, l1;
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                         : "=d"(v0), "=d"(v1)
                         : "r"(smem_u32(r_m + par * PSTRIDE + k)));
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                         : "=r"(l0), "=r"(l1)
                         : "r"(smem_u32(r_l + par * PSTRIDE + k)));
            m[k] = rcv ? (r_inf ? dinf() : v0) : m[k];
            m[k + 1] = rcv ? (r_inf ? dinf() : v1) : m[k + 1];
            lab[k] = rcv ? int(l0) : lab[k];
            lab[k + 1] = rcv ? int(l1) : lab[k + 1];
        }
        par ^= 1;
    };

    static_assert(LBLK % K == 0 && (D <= K ? K % D == 0 : D % K == 0),
                  "K-blocks tile label blocks; ring and K-blocks tile each other");
    // a ring deeper than a K-block (D = QB*K) cycles through QB block positions;
    // each gets its own unrolled body so ring slots stay compile-time offsets
    constexpr int QB = D > K ? D / K : 1;
    auto kblock = [&](auto qq, int i0) {
#pragma unroll
        for (int t = 0; t < K; ++t) step((decltype(qq)::value * K + t) % D, i0 + t, t);
    };
    const int nkb = (H - 1) / K;  // full K-row blocks
    for (int q = 0; q < nkb; ++q) {
        const int i0 = 1 + q * K;
        const int lpos = (q * K) % LBLK, blk = (q * K) / LBLK;
        if (lpos == 0) reset_labels();
        if constexpr (QB == 1) kblock(std::integral_constant<int, 0>{}, i0);
        else if constexpr (QB == 2) {
            if (q & 1) kblock(std::integral_constant<int, 1>{}, i0);
            else kblock(std::integral_constant<int, 0>{}, i0);
        } else {
            static_assert(QB == 4, "ring depth must be K, 2K or 4K when deeper than a K-block");
            switch (q & 3) {
                case 0: kblock(std::integral_constant<int, 0>{}, i0); break;
                case 1: kblock(std::integral_constant<int, 1>{}, i0); break;
                case 2: kblock(std::integral_constant<int, 2>{}, i0); break;
                default: kblock(std::integral_constant<int, 3>{}, i0); break;
            }
        }
        // K divides LBLK, so label blocks end only on a K-block's last row. The halo
        // lanes that recv() overwrites are never useful, so block_end may run in between.
        const bool more = i0 + K < H;
        if (more) send();
        if (lpos + K == LBLK || i0 + K - 1 == H - 1) block_end(i0 + K - 1, blk);
        if (more) recv();
    }
    {  // tail: the last (H-1) % K rows
        const int i0 = 1 + nkb * K;
        if (i0 < H) {
            const int lpos = (nkb * K) % LBLK, blk = (nkb * K) / LBLK;
            if (lpos == 0) reset_labels();
#pragma unroll
            for (int t = 0; t < K; ++t) {
                if (i0 + t >= H) break;
                step(((nkb % QB) * K + t) % D, i0 + t, t);
            }
            block_end(H - 1, blk);  // the tail always ends the image (and its label block)
        }
    }

    cp_async_wait<0>();  // the ring's trailing prefetches (rows past H-1) land before the region is reused
    long long pf_fwd = 0;
    if constexpr (PROF) pf_fwd = clock64();
    // Small label tables are gathered into CTA 0 (plain DSMEM word stores, ordered
    // by the cluster barrier below) so phase 1's block-to-block hops are local.
    int8_t* gtab = reinterpret_cast<int8_t*>(ring_b + SM::ring_bytes(D));
    const int GS = G * S;  // gathered row stride (bytes)
    if (p.gather) {
        __syncthreads();  // every warp of this CTA has stored its block-end labels
        uint32_t* dst0 = reinterpret_cast<uint32_t*>(cluster.map_shared_rank(gtab, 0));
        const uint32_t* src = reinterpret_cast<const uint32_t*>(labels);
        constexpr int WPR = SM::COLS / 4;  // words per label row of this CTA
        for (int idx = threadIdx.x; idx < nblk * WPR; idx += NWARP * 32) {
            const int b = idx / WPR, w = idx - b * WPR;
            dst0[(b * GS + cta * SM::COLS) / 4 + w] = src[idx];
        }
    }

    // ---- K3a: argmin of the bottom row over useful columns (solvers.hpp:94-99)
    double bv = dinf();
    int bi = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < C; ++k)
        if ((useful >> k & 1) && m[k] < bv) { bv = m[k]; bi = col0 + k; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) argmin_combine(bv, bi, __shfl_xor_sync(FULL, bv, o), __shfl_xor_sync(FULL, bi, o));
    if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
    __syncthreads();
    // per-CTA results go straight into CTA 0's slots (DSMEM stores, ordered by the barrier)
    double* cl_v = red_v + 96;
    int* cl_i = reinterpret_cast<int*>(red_v + 112);
    if (threadIdx.x == 0) {
        for (int w = 1; w < NWARP; ++w) argmin_combine(bv, bi, red_v[w], red_i[w]);
        cluster.map_shared_rank(cl_v, 0)[cta] = bv;
        cluster.map_shared_rank(cl_i, 0)[cta] = bi;
    }
    // the cluster barrier (arrive.release / wait.acquire at cluster scope) orders these
    // DSMEM stores and phase 1's seam stores below; no gpu-scope fence is needed
    if (ncl > 1) cluster.sync();
    else __syncthreads();

    // ---- K3b phase 1: block-boundary columns through the labels. Tables left
    // distributed over the cluster: the walk moves with the seam — each CTA's thread 0
    // follows the labels while the column is its own and hands the (block, column)
    // token to the owning CTA (st.async + mbarrier) when the seam crosses over, so hops
    // read local shared memory instead of one remote DSMEM load each.
    // The whole of warp 0 runs the walk (uniform control flow, lane 0 stores and sends):
    // a single diverged lane left warp 0 running phase 2 split, 3x slower.
    const bool handoff = !GLAB && !p.gather && ncl > 1 && nblk > 0 && !(p.dbg & 2);
    if (handoff && warp == 0) {
        constexpr int DONE = -2;
        auto send = [&](int to, int b, int c) {
            st_async_v2_b32_if(lane == 0, mapa_u32(smem_u32(p1msg), uint32_t(to)), uint32_t(b), uint32_t(c),
                               mapa_u32(smem_u32(p1bar), uint32_t(to)));
        };
        if (cta == 0) {
            bv = cl_v[0];
            bi = cl_i[0];
            for (int r = 1; r < ncl; ++r) argmin_combine(bv, bi, cl_v[r], cl_i[r]);
            if (lane == 0) seam[H - 1] = bi;
            send((bi / S) / NWARP, nblk - 1, bi);
        }
        const uint32_t bar = smem_u32(p1bar);
        for (uint32_t ph = 0;; ph ^= 1) {
            if (lane == 0) mbar_arrive_expect_tx(bar, 8);
            while (!mbar_try_wait(bar, ph)) {
            }
            int b = ld_shared_s32(smem_u32(p1msg)), c = ld_shared_s32(smem_u32(p1msg) + 4);
            if (b == DONE) break;
            while (b >= 0 && (c / S) / NWARP == cta) {
                c += labels[b * SM::COLS + (c - cta * SM::COLS)];
                if (b > 0 && lane == 0) seam[LBLK * b] = c;  // row 32b = last row of block b-1
                --b;
            }
            if (b >= 0) {
                send((c / S) / NWARP, b, c);
                continue;
            }
            if (lane == 0) seam[0] = c;
            for (int r = 0; r < ncl; ++r)
                if (r != cta) send(r, DONE, 0);
            break;
        }
    }
    if (!handoff && cta == 0 && threadIdx.x == 0 && !(p.dbg & 2)) {
        bv = cl_v[0];
        bi = cl_i[0];
        for (int r = 1; r < ncl; ++r) argmin_combine(bv, bi, cl_v[r], cl_i[r]);
        int c = bi;
        seam[H - 1] = c;
        if constexpr (GLAB) {  // written by every CTA before the cluster barrier: read through L2
            for (int b = nblk - 1; b >= 0; --b) {
                c += __ldcg(glab + (long long)b * GS + c);
                if (b > 0) seam[LBLK * b] = c;  // row 32b = last row of block b-1
            }
        } else if (p.gather) {
            for (int b = nblk - 1; b >= 0; --b) {
                c += gtab[b * GS + c];
                if (b > 0) seam[LBLK * b] = c;  // row 32b = last row of block b-1
            }
        } else {
            for (int b = nblk - 1; b >= 0; --b) {
                const int owner = (c / S) / NWARP;
                const int8_t* lb = cluster.map_shared_rank(labels, owner);
                c += lb[b * SM::COLS + (c - owner * SM::COLS)];
                if (b > 0) seam[LBLK * b] = c;  // row 32b = last row of block b-1
            }
        }
        if (nblk > 0) seam[0] = c;
    }
    // after this barrier no CTA touches another CTA's shared memory, so CTAs
    // may finish phase 2 and exit independently
    if (ncl > 1) cluster.sync();
    else __syncthreads();

    long long pf_p1 = 0;
    if constexpr (PROF) pf_p1 = clock64();
    // ---- K3b phase 2: every warp recomputes blocks g, g+G, ... in a 128-column window
    long long q0t = 0, q1t = 0, q2t = 0, q3t = 0;  // MODE 2: the first block's sub-phases
    {
        uint8_t* dirs = p2 + size_t(warp) * LBLK * P2_COLS;
        // phase-2 ring: this warp's forward-ring region, P2D rows of 128 columns
        constexpr int P2D = (D * C) / 4;
        constexpr int P2STAGE = P2_COLS * RE;  // bytes per phase-2 ring row
        static_assert(P2D >= 2, "phase-2 ring needs at least two stages");
        const unsigned char* p2ring_ptr = ring_b + size_t(warp) * D * 32 * C * RE + lane * 4 * RE;
        const uint32_t p2ring = smem_u32(p2ring_ptr);
        for (int b = g; b < nblk && !(p.dbg & 1); b += G) {
            if constexpr (PROF) { if (b == g) q0t = clock64(); }
            const int r0 = 1 + LBLK * b, r1 = min(LBLK * (b + 1), H - 1);
            const int c1 = __ldcg(seam + r1);  // phase 1 left the block's bottom column in global memory
            // 16-byte aligned lane slices: even column for double2 energies, multiple of 4 for RGBX
            const int wbase = (c1 - P2_COLS / 2) & (FUSED ? ~3 : ~1);
            const int wc0 = wbase + lane * 4;
            // fused: the backtrack from c1 at row r1 only reads cells within c1 +- 32 of
            // the block's cone (LBLK rows), which need RGBX columns c1 +- 33; lanes clear of
            // c1 +- (LBLK + 4) (and of the image) skip their reads — the wrong values their
            // stale stage bytes produce spread one column per row and stay outside the cone.
            // Only in the two-CTAs-per-SM batch shape (MINB 2), where it measured faster
            // (C5 DP 1.555 -> 1.541 ms, DRAM 4.46 -> 4.29 GB per launch); the small-batch
            // cluster shape measured 6 % slower with it (tools/ab_libs.sh)
            const bool qneed = MINB < 2 || (wc0 + 3 >= max(c1 - (LBLK + 4), -1) && wc0 <= min(c1 + LBLK + 4, W));
            double mm[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int j = wc0 + k;
                mm[k] = (j >= 0 && j < W) ? mbound[(long long)b * p.mpitch + j] : dinf();
            }
            // the block's energy rows stream through this warp's (now idle) forward ring,
            // P2D rows in flight via cp.async
            // fused: rolling luma rows of the window; the ring carries RGBX row r+1 at row r
            double QLp[4], QLc[4], QLn[4];
            uint32_t qoob = 0;
            const uint32_t* wrgb = FUSED ? p.rgb + img * p.rgb_istride + wc0 : nullptr;
            if constexpr (FUSED) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (wc0 + k < 0 || wc0 + k >= W) qoob |= 1u << k;
                uint32_t px[4];
                const uint32_t* ra = wrgb + (long long)(r0 - 1) * p.rpitch;
#pragma unroll
                for (int k = 0; k < 4; ++k) px[k] = qneed ? __ldg(ra + k) : 0u;
                luma_cols<4>(px, QLp);
                const uint32_t* rb = wrgb + (long long)r0 * p.rpitch;
#pragma unroll
                for (int k = 0; k < 4; ++k) px[k] = qneed ? __ldg(rb + k) : 0u;
                luma_cols<4>(px, QLc);
            } else if constexpr (FWD) {  // cost planes: columns outside the image are +inf
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (wc0 + k < 0 || wc0 + k >= W) qoob |= 1u << k;
            }
            auto p2fetch = [&](int r, int slot) {
                const uint32_t dst = p2ring + uint32_t(slot * P2STAGE);
                if constexpr (FUSED) {
                    cp_async16_if(qneed, dst, wrgb + (long long)min(r + 1, H - 1) * p.rpitch);
                } else {
                    const double* src = e + (long long)min(r, r1) * p.epitch + wc0;
#pragma unroll
                    for (int pl = 0; pl < (FWD ? 3 : 1); ++pl) {
                        cp_async16(dst + pl * 32, src + pl * p.cplane);
                        cp_async16(dst + pl * 32 + 16, src + pl * p.cplane + 2);
                    }
                }
                cp_async_commit();
            };
#pragma unroll
            for (int u = 0; u < P2D; ++u) p2fetch(r0 + u, u);
            // one ring row -> this lane's 4 energies (or forward costs); rows in order (the
            // fused luma rows roll)
            auto p2load = [&](int slot, double (&ec)[4], double (&qcl)[4], double (&qcu)[4], double (&qcr)[4]) {
                if constexpr (FUSED) {
                    const uint4 q = *reinterpret_cast<const uint4*>(p2ring_ptr + slot * P2STAGE);
                    const uint32_t px[4] = {q.x, q.y, q.z, q.w};
                    luma_cols<4>(px, QLn);
                    if constexpr (FWD) fwd_cols<4>(QLp, QLc, qoob, qcl, qcu, qcr);
                    else energy_cols<4>(QLp, QLc, QLn, qoob, ec);
#pragma unroll
                    for (int k = 0; k < 4; ++k) { QLp[k] = QLc[k]; QLc[k] = QLn[k]; }
                } else {
                    const double* src = reinterpret_cast<const double*>(p2ring_ptr + slot * P2STAGE);
                    const double2 x0 = *reinterpret_cast<const double2*>(src);
                    const double2 x1 = *reinterpret_cast<const double2*>(src + 2);
                    ec[0] = x0.x; ec[1] = x0.y; ec[2] = x1.x; ec[3] = x1.y;
                    if constexpr (FWD) {  // cost row r of the three planes
                        const double2 y0 = *reinterpret_cast<const double2*>(src + 4);
                        const double2 y1 = *reinterpret_cast<const double2*>(src + 6);
                        const double2 z0 = *reinterpret_cast<const double2*>(src + 8);
                        const double2 z1 = *reinterpret_cast<const double2*>(src + 10);
                        qcl[0] = x0.x; qcl[1] = x0.y; qcl[2] = x1.x; qcl[3] = x1.y;
                        qcu[0] = y0.x; qcu[1] = y0.y; qcu[2] = y1.x; qcu[3] = y1.y;
                        qcr[0] = z0.x; qcr[1] = z0.y; qcr[2] = z1.x; qcr[3] = z1.y;
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (qoob >> k & 1) qcl[k] = qcu[k] = qcr[k] = dinf();
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {  // the slot's values are in registers before its refill
                    if constexpr (FWD) asm volatile("" ::"d"(qcl[k]), "d"(qcu[k]), "d"(qcr[k]));
                    else asm volatile("" ::"d"(ec[k]));
                }
            };
            // row r's cells from the previous row (mm) and its energies / costs
            auto p2cells = [&](int r, const double (&ec)[4], const double (&qcl)[4], const double (&qcu)[4],
                               const double (&qcr)[4]) {
                const double lm = __shfl_up_sync(FULL, mm[3], 1);
                const double rm = __shfl_down_sync(FULL, mm[0], 1);
                double pm = lane == 0 ? dinf() : lm;
                const double rr = lane == 31 ? dinf() : rm;
                uint32_t db = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double cm = mm[k];
                    const double nm = (k + 1 < 4) ? mm[k + 1] : rr;
                    int d, dummy;
                    // k = 0: the shuffled left operand is compared last (same cell, see
                    // dp_cell_left_last), so one compare-select follows the shuffle
                    if constexpr (FWD) {
                        if (k == 0) fwd_cell_left_last(pm, cm, nm, 0, 0, 0, qcl[k], qcu[k], qcr[k], mm[k], dummy, d);
                        else fwd_cell(pm, cm, nm, 0, 0, 0, qcl[k], qcu[k], qcr[k], mm[k], dummy, d);
                    } else {
                        if (k == 0) dp_cell_left_last(pm, cm, nm, 0, 0, 0, ec[k], mm[k], dummy, d);
                        else dp_cell(pm, cm, nm, 0, 0, 0, ec[k], mm[k], dummy, d);
                    }
                    db |= uint32_t(d) << (8 * k);
                    pm = cm;
                }
                reinterpret_cast<uint32_t*>(dirs + (r - r0) * P2_COLS)[lane] = db;
            };
            const bool refill = !(PROF && (p.dbg & 16));  // dbg bit 4 (MODE 2): timing without refills
            if (r1 - r0 + 1 == LBLK) {
                // full block: unrolled (compile-time ring slots) and software-pipelined — row
                // t+1's ring read (and fused luma/e1) is issued before row t's cells, so the
                // shared-memory latency stays off the row-to-row chain
                double ea[4], la[4], ua[4], ra[4];
                cp_async_wait<P2D - 1>();
                p2load(0, ea, la, ua, ra);
                if constexpr (PROF) { if (b == g) { asm volatile("" ::"d"(mm[0])); q1t = clock64(); } }
#pragma unroll
                for (int t = 0; t < LBLK; ++t) {
                    double eb[4], lb[4], ub[4], rb[4];
                    if (t + 1 < LBLK) {
                        cp_async_wait<P2D - 2>();
                        p2load((t + 1) % P2D, eb, lb, ub, rb);
                    }
                    if (refill) p2fetch(r0 + t + P2D, t % P2D);
                    p2cells(r0 + t, ea, la, ua, ra);
#pragma unroll
                    for (int k = 0; k < 4; ++k) { ea[k] = eb[k]; la[k] = lb[k]; ua[k] = ub[k]; ra[k] = rb[k]; }
                }
            } else {
                for (int r = r0; r <= r1; ++r) {
                    const int slot = (r - r0) % P2D;
                    double ec[4], qcl[4], qcu[4], qcr[4];
                    cp_async_wait<P2D - 1>();
                    p2load(slot, ec, qcl, qcu, qcr);
                    if constexpr (PROF) { if (b == g && r == r0) { asm volatile("" ::"d"(mm[0])); q1t = clock64(); } }
                    if (refill) p2fetch(r + P2D, slot);
                    p2cells(r, ec, qcl, qcu, qcr);
                }
            }
            cp_async_wait<0>();
            __syncwarp();
            if constexpr (PROF) { if (b == g) q2t = clock64(); }
            if (lane == 0 && !(p.dbg & 4)) {
                int c = c1;
                for (int r = r1; r >= r0; --r) {
                    c += int(dirs[(r - r0) * P2_COLS + (c - wbase)]) - 1;
                    if (r - 1 != LBLK * b || b == 0) seam[r - 1] = c;
                }
            }
            __syncwarp();
            if constexpr (PROF) { if (b == g) q3t = clock64(); }
        }
    }
    if constexpr (PROF) {
        if (lane == 0) {
            long long* o = p.prof + g * 8;
            o[0] = pf_fwd - pf_t0;   // forward pass (incl. waits)
            o[1] = pf_wait;          // of which: waiting for halos
            o[2] = pf_p1 - pf_fwd;   // argmin + phase 1 + barriers
            o[3] = clock64() - pf_p1;  // phase 2
            o[4] = H;
            o[5] = q1t - q0t;  // first phase-2 block: start -> first row's data ready
            o[6] = q2t - q1t;  //   row recompute
            o[7] = q3t - q2t;  //   walk
        }
    }
    if (p.stamps) {
        if (ncl > 1) cluster.sync();
        else __syncthreads();
        if (cta == 0 && threadIdx.x == 0) p.stamps[img * p.st_istride + 3] = globaltimer();
    }
}

}  // namespace carve_dev
