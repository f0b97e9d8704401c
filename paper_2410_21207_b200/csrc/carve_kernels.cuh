// carve_kernels.cuh — the four sm_100a kernels of the seam-carving hot path.
//
//   K1  energy stencil        k_energy_full   (energy.hpp:82-98 + raster.hpp:61-71)
//       + 2-column fix-up     prologue of k_dp2
//   K2  cumulative-energy DP  k_dp2 (dp_cluster.cuh) (solvers.hpp:116-157, 263-289)
//   K3  argmin + backtrack    tail of k_dp2 (solvers.hpp:94-111)
//   K4  seam removal          k_compact_bulk (carve loop, TMA), k_compact (the
//                             remove_seam API) (carver.hpp:71-98); transpose
//                             kernels for horizontal seams (carver.hpp:216-222)
//
// Arithmetic contract: every FP64 operation is an
// explicit round-to-nearest intrinsic (__dmul_rn/__dadd_rn/__dsub_rn) so no
// FMA contraction can occur, matching the reference built for baseline
// x86-64. The whole library is also compiled with -fmad=false.
//
// Device layout: pixels are RGBX uint32 (r | g<<8 | b<<16),
// energy is FP64, both row-major with a fixed pitch (a multiple of 32
// elements) that does not change as the width shrinks; DP directions are one
// byte per cell (0: from j-1, 1: from j, 2: from j+1).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace carve_dev {

constexpr unsigned FULL = 0xffffffffu;

// Energy-plane padding: every FP64 energy row carries EPAD_L
// columns of +inf before logical column 0 and at least EPAD_R columns of +inf
// after the last live column, and the plane has EPAD_B spare rows at the
// bottom, so the DP's row loads are unconditional aligned 128-bit loads and
// out-of-image neighbours are +inf by construction (SPEC.md:315 exclusion).
// EPAD_R covers the widest overhang of a DP cluster past the image edge
// (one CTA's useful columns + halo + a warp's span; checked on the host).
constexpr int EPAD_L = 128, EPAD_R = 2304, EPAD_B = 16;

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// Programmatic dependent launch: a seam's DP and removal kernels are launched
// with programmatic stream serialization, so each is scheduled while its
// predecessor drains; pdl_wait() blocks until the predecessor grid has
// completed and its writes are visible (a no-op for ordinary launches).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Optional end-of-kernel timestamp: thread 0 of every block raises *p to its exit
// time on every return path (the kernel's end = the last block's exit).
struct EndStamp {
    unsigned long long* p;
    __device__ ~EndStamp() {
        if (p && threadIdx.x == 0) atomicMax(p, (unsigned long long)globaltimer());
    }
};

// raster.hpp:68 — 0.299*r + 0.587*g + 0.114*b, left to right, no contraction.
// byte `B` of p as an exact double: one I2F.F64.U8 with a byte selector (R.B1,
// R.B2) instead of shift + mask + I2F.F64.U32 (5 integer ops per pixel saved)
template <int B>
__device__ __forceinline__ double byte_f64(uint32_t p) {
    double d;
    asm("{.reg .u16 t; cvt.u16.u32 t, %1; cvt.rn.f64.u8 %0, t;}" : "=d"(d) : "r"(p >> (8 * B)));
    return d;
}
__device__ __forceinline__ double luma(uint32_t p) {
    const double r = byte_f64<0>(p), g = byte_f64<1>(p), b = byte_f64<2>(p);
    return __dadd_rn(__dadd_rn(__dmul_rn(0.299, r), __dmul_rn(0.587, g)), __dmul_rn(0.114, b));
}

// energy.hpp:95 — |gx| + |gy|, x term first.
__device__ __forceinline__ double e1(double l_left, double l_right, double l_up, double l_down) {
    return __dadd_rn(fabs(__dsub_rn(l_right, l_left)), fabs(__dsub_rn(l_down, l_up)));
}

// The DP variant translation units (dp_variants_*.cu) need only the helpers above.
#ifndef CARVE_KERNELS_HELPERS_ONLY

// ---------------------------------------------------------------------------
// layout conversion (host boundary): packed RGB bytes <-> RGBX plane

// Both conversions move 4 pixels per thread: 12 packed bytes as three 32-bit
// words (when the image base is 4-byte aligned) and the 4 RGBX words as one
// 128-bit access when the group stays inside one plane row; one 32-bit divide
// per group places it. Groups that straddle a row or the image end go per pixel.
__device__ __forceinline__ void rgb12_to_px(uint32_t a, uint32_t b, uint32_t c, uint32_t (&px)[4]) {
    px[0] = a & 0xFFFFFFu;
    px[1] = (a >> 24) | ((b & 0xFFFFu) << 8);
    px[2] = (b >> 16) | ((c & 0xFFu) << 16);
    px[3] = c >> 8;
}

__global__ void k_unpack(const uint8_t* __restrict__ in, int W, int H, uint32_t* __restrict__ out, int pitch,
                         long long in_istride, long long out_istride) {
    in += blockIdx.y * in_istride;
    out += blockIdx.y * out_istride;
    const unsigned n = unsigned(W) * unsigned(H), ng = (n + 3) / 4;
    const bool in_al = (reinterpret_cast<uintptr_t>(in) & 3) == 0;
    for (unsigned g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
        const unsigned k = 4 * g, i = k / unsigned(W), j = k - i * unsigned(W);
        uint32_t px[4];
        if (in_al && k + 3 < n) {
            const uint32_t* w3 = reinterpret_cast<const uint32_t*>(in + 3ull * k);
            rgb12_to_px(w3[0], w3[1], w3[2], px);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint8_t* p = in + 3ull * min(k + u, n - 1);
                px[u] = uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16);
            }
        }
        uint32_t* o = out + (size_t)i * pitch + j;
        if (j + 3 < unsigned(W) && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
            *reinterpret_cast<uint4*>(o) = make_uint4(px[0], px[1], px[2], px[3]);
        } else {
            unsigned ii = i, jj = j;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (k + u < n) out[(size_t)ii * pitch + jj] = px[u];
                if (++jj == unsigned(W)) { jj = 0; ++ii; }
            }
        }
    }
}

// transposed==true: the plane holds the image transposed (plane row = image column).
template <bool transposed>
__global__ void k_pack(const uint32_t* __restrict__ in, int pitch, int W, int H, uint8_t* __restrict__ out,
                       long long in_istride, long long out_istride) {
    in += blockIdx.y * in_istride;
    out += blockIdx.y * out_istride;
    const unsigned n = unsigned(W) * unsigned(H), ng = (n + 3) / 4;
    const bool out_al = (reinterpret_cast<uintptr_t>(out) & 3) == 0;
    for (unsigned g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
        const unsigned k = 4 * g, i = k / unsigned(W), j = k - i * unsigned(W);
        uint32_t px[4];
        const uint32_t* row = in + (size_t)i * pitch + j;
        if (!transposed && j + 3 < unsigned(W) && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
            const uint4 v = *reinterpret_cast<const uint4*>(row);
            px[0] = v.x; px[1] = v.y; px[2] = v.z; px[3] = v.w;
        } else {
            unsigned ii = i, jj = j;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const unsigned ci = min(ii, unsigned(H) - 1);
                px[u] = transposed ? in[(size_t)jj * pitch + ci] : in[(size_t)ci * pitch + jj];
                if (++jj == unsigned(W)) { jj = 0; ++ii; }
            }
        }
        if (out_al && k + 3 < n) {
            uint32_t* w3 = reinterpret_cast<uint32_t*>(out + 3ull * k);
            w3[0] = (px[0] & 0xFFFFFFu) | (px[1] << 24);
            w3[1] = ((px[1] >> 8) & 0xFFFFu) | (px[2] << 16);
            w3[2] = ((px[2] >> 16) & 0xFFu) | (px[3] << 8);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (k + u >= n) break;
                uint8_t* o = out + 3ull * (k + u);
                o[0] = uint8_t(px[u]);
                o[1] = uint8_t(px[u] >> 8);
                o[2] = uint8_t(px[u] >> 16);
            }
        }
    }
}

// 32x32 tiled transpose of an RGBX plane (raster.hpp:73-79): out(j, i) = in(i, j).
__global__ void k_transpose(const uint32_t* __restrict__ in, int ipitch, int W, int H, uint32_t* __restrict__ out,
                            int opitch, long long in_istride, long long out_istride) {
    __shared__ uint32_t tile[32][33];
    in += blockIdx.z * in_istride;
    out += blockIdx.z * out_istride;
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = by + r, j = bx + threadIdx.x;
        if (i < H && j < W) tile[r][threadIdx.x] = in[(long long)i * ipitch + j];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int j = bx + r, i = by + threadIdx.x;  // out row j, col i
        if (i < H && j < W) out[(long long)j * opitch + i] = tile[threadIdx.x][r];
    }
}

// ---------------------------------------------------------------------------
// K1 — full energy map. 64x16 output tile per 256-thread CTA; the (16+2) x
// (64+2) luma tile (edge-replicated, raster.hpp:54-58) is staged in shared
// memory from 128-bit coalesced RGBX loads; each thread writes 4 energies as
// two 128-bit stores. Algorithmic traffic: 4 B read + 8 B written per pixel.

constexpr int K1_TW = 64, K1_TH = 16;

__device__ __forceinline__ void k1_tile(const uint32_t* __restrict__ rgb, int pitch, int W, int H,
                                        double* __restrict__ e, int epitch, int i0, int j0,
                                        double (*L)[K1_TW + 2]) {
    const int t = threadIdx.x;
    // interior columns: 18 rows x 16 chunks of 4 pixels
    for (int item = t; item < (K1_TH + 2) * (K1_TW / 4); item += blockDim.x) {
        const int r = item / (K1_TW / 4), q = item % (K1_TW / 4);
        const int gi = min(max(i0 + r - 1, 0), H - 1);
        const int gj = j0 + 4 * q;
        const uint32_t* row = rgb + (long long)gi * pitch;
        uint32_t px[4];
        if (gj + 3 < W) {
            const uint4 v = *reinterpret_cast<const uint4*>(row + gj);
            px[0] = v.x; px[1] = v.y; px[2] = v.z; px[3] = v.w;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) px[u] = row[min(gj + u, W - 1)];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) L[r][1 + 4 * q + u] = luma(px[u]);
    }
    // halo columns j0-1 and j0+64
    for (int item = t; item < (K1_TH + 2) * 2; item += blockDim.x) {
        const int r = item >> 1, side = item & 1;
        const int gi = min(max(i0 + r - 1, 0), H - 1);
        const int gj = side ? min(j0 + K1_TW, W - 1) : max(j0 - 1, 0);
        L[r][side ? K1_TW + 1 : 0] = luma(rgb[(long long)gi * pitch + gj]);
    }
    __syncthreads();
    {
        const int r = t / (K1_TW / 4), q = t % (K1_TW / 4);
        const int gi = i0 + r;
        if (gi < H) {
            double out[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = 1 + 4 * q + u;
                // clamped columns: for the last real column the right neighbour
                // must be itself (at_clamped); smem col c+1 holds column gj+1
                // clamped only at the tile edge, so clamp explicitly here.
                const int gj = j0 + 4 * q + u;
                const int cr = (gj + 1 < W) ? c + 1 : c;
                const int cl = (gj - 1 >= 0) ? c - 1 : c;
                out[u] = e1(L[r + 1][cl], L[r + 1][cr], L[r][c], L[r + 2][c]);
            }
            double* erow = e + (long long)gi * epitch;
            const int gj = j0 + 4 * q;
            if (gj + 3 < W) {
                *reinterpret_cast<double2*>(erow + gj) = make_double2(out[0], out[1]);
                *reinterpret_cast<double2*>(erow + gj + 2) = make_double2(out[2], out[3]);
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (gj + u < W) erow[gj + u] = out[u];
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_energy_full(const uint32_t* __restrict__ rgb, int pitch, int W, int H,
                                                     double* __restrict__ e, int epitch, long long rgb_istride,
                                                     long long e_istride) {
    __shared__ double L[K1_TH + 2][K1_TW + 2];
    rgb += blockIdx.z * rgb_istride;
    e += blockIdx.z * e_istride;
    k1_tile(rgb, pitch, W, H, e, epitch, blockIdx.y * K1_TH, blockIdx.x * K1_TW, L);
}

// K1, row-streaming form (the default): one warp owns a 128-column strip
// (4 columns per lane) for a run of R rows. RGBX rows stream through registers
// two rows ahead, the three luma rows (i-1, i, i+1) roll in registers, lane
// neighbours come by shuffle and the strip's outer neighbours from one extra
// pixel loaded by lanes 0 and 31, so every pixel's luma is computed about
// once and there is no shared memory or barrier. Clamping follows at_clamped
// (raster.hpp:54-58): rows outside [0, H) and columns outside [0, W) read the
// nearest edge. Loads never leave [0, W) x [0, H), so unpadded planes work.
constexpr int K1S_C = 4, K1S_COLS = 32 * K1S_C;
template <int MINB, int PF>
__global__ void __launch_bounds__(256, MINB) k_energy_rows(const uint32_t* __restrict__ rgb, int pitch, int W, int H,
                                                     double* __restrict__ e, int epitch, long long rgb_istride,
                                                     long long e_istride, int nstrips, int R,
                                                     unsigned long long* stamps = nullptr, long long st_is = 0) {
    // optional [start, end] stamps of the phase's first seam (its energy_s)
    if (stamps && blockIdx.x == 0 && threadIdx.x == 0)
        atomicCAS(&stamps[blockIdx.y * st_is], 0ull, (unsigned long long)globaltimer());
    EndStamp end_stamp{stamps ? stamps + blockIdx.y * st_is + 1 : nullptr};
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int strip = gw % nstrips, i0 = (gw / nstrips) * R;
    if (i0 >= H) return;
    rgb += blockIdx.y * rgb_istride;
    e += blockIdx.y * e_istride;
    const int s0 = strip * K1S_COLS, col0 = s0 + lane * K1S_C;
    const bool vec = col0 + K1S_C <= W;
    uint32_t lcl = 0, rcl = 0, live = 0;
#pragma unroll
    for (int k = 0; k < K1S_C; ++k) {
        if (col0 + k == 0) lcl |= 1u << k;
        if (col0 + k == W - 1) rcl |= 1u << k;
        if (col0 + k < W) live |= 1u << k;
    }
    // lanes 0 / 31: the column just outside the strip (clamped into the image)
    const bool xl = lane == 0 || lane == 31;
    const int xcol = lane == 0 ? max(s0 - 1, 0) : min(s0 + K1S_COLS, W - 1);
    auto load = [&](int r, uint32_t (&px)[K1S_C], uint32_t& x) {
        const uint32_t* row = rgb + (long long)min(max(r, 0), H - 1) * pitch;
        if (vec) {
            const uint4 v = *reinterpret_cast<const uint4*>(row + col0);
            px[0] = v.x; px[1] = v.y; px[2] = v.z; px[3] = v.w;
        } else {
#pragma unroll
            for (int k = 0; k < K1S_C; ++k) px[k] = row[min(col0 + k, W - 1)];
        }
        if (xl) x = row[xcol];
    };
    double Lp[K1S_C], Lc[K1S_C], Ln[K1S_C], xc = 0.0, xn = 0.0;
    uint32_t pbuf[PF][K1S_C], xbuf[PF];
    auto to_luma = [&](const uint32_t (&px)[K1S_C], uint32_t x, double (&L)[K1S_C], double& xlum) {
#pragma unroll
        for (int k = 0; k < K1S_C; ++k) L[k] = luma(px[k]);
        if (xl) xlum = luma(x);
    };
    load(i0 - 1, pbuf[0], xbuf[0]);
    to_luma(pbuf[0], xbuf[0], Lp, xc);
    load(i0, pbuf[0], xbuf[0]);
    to_luma(pbuf[0], xbuf[0], Lc, xc);
    const int i1 = min(i0 + R, H);
#pragma unroll
    for (int u = 0; u < PF; ++u) load(i0 + 1 + u, pbuf[u], xbuf[u]);  // rows i+1 .. i+PF in flight at row i
    auto row_step = [&](int i, uint32_t (&px)[K1S_C], uint32_t& x) {
        to_luma(px, x, Ln, xn);
        load(i + 1 + PF, px, x);  // refill this buffer (clamped past the bottom; unused there)
        double lL = __shfl_up_sync(FULL, Lc[K1S_C - 1], 1);
        double lR = __shfl_down_sync(FULL, Lc[0], 1);
        if (lane == 0) lL = xc;
        if (lane == 31) lR = xc;
        double out[K1S_C];
#pragma unroll
        for (int k = 0; k < K1S_C; ++k) {
            double left = k > 0 ? Lc[k - 1] : lL;
            double right = k + 1 < K1S_C ? Lc[k + 1] : lR;
            if (lcl >> k & 1) left = Lc[k];
            if (rcl >> k & 1) right = Lc[k];
            out[k] = e1(left, right, Lp[k], Ln[k]);
        }
        double* erow = e + (long long)i * epitch + col0;
        if (live == (1u << K1S_C) - 1) {
            *reinterpret_cast<double2*>(erow) = make_double2(out[0], out[1]);
            *reinterpret_cast<double2*>(erow + 2) = make_double2(out[2], out[3]);
        } else {
#pragma unroll
            for (int k = 0; k < K1S_C; ++k)
                if (live >> k & 1) erow[k] = out[k];
        }
#pragma unroll
        for (int k = 0; k < K1S_C; ++k) { Lp[k] = Lc[k]; Lc[k] = Ln[k]; }
        xc = xn;
    };
    for (int i = i0; i < i1; i += PF) {
#pragma unroll
        for (int u = 0; u < PF; ++u)
            if (i + u < i1) row_step(i + u, pbuf[u], xbuf[u]);
    }
}

// K1 with a shared-memory row ring (CARVE_K1V=4 / the large-plane default): the same
// strip decomposition and arithmetic as k_energy_rows, but each lane's 4 RGBX pixels of
// rows i+1 .. i+DK (and lanes 0/31's strip-edge pixel) are in flight through cp.async
// instead of registers: DK x 512 B per warp, so a 3-CTA SM has ~100 KB of loads in
// flight (Little's law at HBM latency) where the register version had ~24 KB. Pixels
// right of the image (the padded pitch, or the next 4-pixel group of an unpadded row)
// are loaded but never used: the right-edge column clamps to itself.
template <int MINB, int DK>
__global__ void __launch_bounds__(256, MINB) k_energy_ring(const uint32_t* __restrict__ rgb, int pitch, int W, int H,
                                                     double* __restrict__ e, int epitch, long long rgb_istride,
                                                     long long e_istride, int nstrips, int R,
                                                     unsigned long long* stamps = nullptr, long long st_is = 0) {
    extern __shared__ __align__(16) uint32_t kr_sm[];  // [8 warps][DK][K1S_COLS + 4]
    if (stamps && blockIdx.x == 0 && threadIdx.x == 0)
        atomicCAS(&stamps[blockIdx.y * st_is], 0ull, (unsigned long long)globaltimer());
    EndStamp end_stamp{stamps ? stamps + blockIdx.y * st_is + 1 : nullptr};
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * (blockDim.x >> 5) + wib;
    const int strip = gw % nstrips, i0 = (gw / nstrips) * R;
    if (i0 >= H) return;
    rgb += blockIdx.y * rgb_istride;
    e += blockIdx.y * e_istride;
    const int s0 = strip * K1S_COLS, col0 = s0 + lane * K1S_C;
    constexpr int RS = K1S_COLS + 4;  // ring row stride (words): 128 strip pixels + the edge pixel
    uint32_t* ring = kr_sm + wib * DK * RS;
    const uint32_t ring_s = uint32_t(__cvta_generic_to_shared(ring));
    uint32_t lcl = 0, rcl = 0, live = 0;
#pragma unroll
    for (int k = 0; k < K1S_C; ++k) {
        if (col0 + k == 0) lcl |= 1u << k;
        if (col0 + k == W - 1) rcl |= 1u << k;
        if (col0 + k < W) live |= 1u << k;
    }
    const bool xl = lane == 0 || lane == 31;
    const int xcol = lane == 0 ? max(s0 - 1, 0) : min(s0 + K1S_COLS, W - 1);
    const bool in_row = col0 < W;  // groups fully right of the image read nothing
    auto fetch = [&](int r, int slot) {  // row r (clamped) -> ring slot, one commit group per row
        const uint32_t* row = rgb + (long long)min(max(r, 0), H - 1) * pitch;
        const uint32_t dst = ring_s + uint32_t((slot * RS + lane * K1S_C) * 4);
        if (in_row) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(row + col0) : "memory");
        if (xl)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ring_s + uint32_t((slot * RS + K1S_COLS +
                                                                                                (lane == 31)) * 4)),
                         "l"(row + xcol)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto take = [&](int slot, double (&L)[K1S_C], double& xlum) {  // ring slot -> lumas
        const uint4 v = *reinterpret_cast<const uint4*>(ring + slot * RS + lane * K1S_C);
        const uint32_t px[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < K1S_C; ++k) L[k] = luma(px[k]);
        if (xl) xlum = luma(ring[slot * RS + K1S_COLS + (lane == 31)]);
    };
    double Lp[K1S_C], Lc[K1S_C], Ln[K1S_C], xc = 0.0, xn = 0.0, xp = 0.0;
    const int i1 = min(i0 + R, H);
    // slots: row i0 - 1 + t lives in slot t % DK; rows i0-1 .. i0-2+DK in flight at first
#pragma unroll
    for (int t = 0; t < DK; ++t) fetch(i0 - 1 + t, t);
    asm volatile("cp.async.wait_group %0;" ::"n"(DK - 1) : "memory");
    take(0, Lp, xp);
    fetch(i0 - 1 + DK, 0);
    asm volatile("cp.async.wait_group %0;" ::"n"(DK - 1) : "memory");
    take(1, Lc, xc);
    fetch(i0 + DK, 1);
    for (int i = i0; i < i1; ++i) {
        const int t = i - i0 + 2;  // ring index of row i + 1
        asm volatile("cp.async.wait_group %0;" ::"n"(DK - 1) : "memory");
        take(t % DK, Ln, xn);
        fetch(i + 1 + DK, t % DK);  // refill the slot with row i + 1 + DK
        double lL = __shfl_up_sync(FULL, Lc[K1S_C - 1], 1);
        double lR = __shfl_down_sync(FULL, Lc[0], 1);
        if (lane == 0) lL = xc;
        if (lane == 31) lR = xc;
        double out[K1S_C];
#pragma unroll
        for (int k = 0; k < K1S_C; ++k) {
            double left = k > 0 ? Lc[k - 1] : lL;
            double right = k + 1 < K1S_C ? Lc[k + 1] : lR;
            if (lcl >> k & 1) left = Lc[k];
            if (rcl >> k & 1) right = Lc[k];
            out[k] = e1(left, right, Lp[k], Ln[k]);
        }
        double* erow = e + (long long)i * epitch + col0;
        if (live == (1u << K1S_C) - 1) {
            *reinterpret_cast<double2*>(erow) = make_double2(out[0], out[1]);
            *reinterpret_cast<double2*>(erow + 2) = make_double2(out[2], out[3]);
        } else {
#pragma unroll
            for (int k = 0; k < K1S_C; ++k)
                if (live >> k & 1) erow[k] = out[k];
        }
#pragma unroll
        for (int k = 0; k < K1S_C; ++k) { Lp[k] = Lc[k]; Lc[k] = Ln[k]; }
        xp = xc;
        xc = xn;
    }
    (void)xp;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// +inf into the left/right pad columns of rows [0, H) (e points at logical column 0)
__global__ void k_fill_pads(double* __restrict__ e, int epitch, int W, int H, long long e_istride) {
    e += blockIdx.y * e_istride;
    const double inf = dinf();
    constexpr int N = EPAD_L + EPAD_R;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < (long long)H * N;
         k += (long long)gridDim.x * blockDim.x) {
        const int i = int(k / N), c = int(k - (long long)i * N);
        const int j = c < EPAD_L ? c - EPAD_L : W + (c - EPAD_L);
        e[(long long)i * epitch + j] = inf;
    }
}

// Luma plane -> e1 (the LumaGrid overload of energy_e1, energy.hpp:89-98).
__global__ void k_energy_luma(const double* __restrict__ l, int W, int H, double* __restrict__ e) {
    const long long n = (long long)W * H;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = int(k / W), j = int(k - (long long)i * W);
        const double* row = l + (long long)i * W;
        const double lft = row[max(j - 1, 0)], rgt = row[min(j + 1, W - 1)];
        const double up = l[(long long)max(i - 1, 0) * W + j], dn = l[(long long)min(i + 1, H - 1) * W + j];
        e[k] = e1(lft, rgt, up, dn);
    }
}

__global__ void k_luma(const uint32_t* __restrict__ rgb, int pitch, int W, int H, double* __restrict__ out) {
    const long long n = (long long)W * H;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = int(k / W), j = int(k - (long long)i * W);
        out[k] = luma(rgb[(long long)i * pitch + j]);
    }
}

// ---------------------------------------------------------------------------
// K4 — seam removal: out[i][j] = in[i][j < s[i] ? j : j+1] (carver.hpp:71-82)
// for the RGBX plane and the FP64 energy plane, fused with the K1 fix-up of
// the (at most) two new-grid columns s[i]-1 and s[i] whose stencil changed
// (every other cell keeps its old energy bitwise).
// One warp per row; each lane produces one 16-byte output chunk per step
// from its aligned 16-byte input chunk plus the next lane's first element.

template <typename T>
struct Vec16;
template <>
struct Vec16<uint32_t> {
    static constexpr int N = 4;
    using V = uint4;
    __device__ static void unpack(const V& v, uint32_t (&a)[4]) { a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w; }
    __device__ static V pack(const uint32_t (&a)[4]) { return make_uint4(a[0], a[1], a[2], a[3]); }
};
template <>
struct Vec16<double> {
    static constexpr int N = 2;
    using V = double2;
    __device__ static void unpack(const V& v, double (&a)[2]) { a[0] = v.x; a[1] = v.y; }
    __device__ static V pack(const double (&a)[2]) { return make_double2(a[0], a[1]); }
};

// energy of new-grid cell (i, x) recomputed from the pre-removal RGBX plane
__device__ __forceinline__ double fixup_energy(const uint32_t* __restrict__ rgb, int pitch, int Wn, int H,
                                               const int* __restrict__ seam, int i, int x) {
    auto old = [&](int r, int c) { return rgb[(long long)r * pitch + c + (c >= __ldg(seam + r) ? 1 : 0)]; };
    const int xl = max(x - 1, 0), xr = min(x + 1, Wn - 1);
    const int iu = max(i - 1, 0), id = min(i + 1, H - 1);
    return e1(luma(old(i, xl)), luma(old(i, xr)), luma(old(iu, x)), luma(old(id, x)));
}

template <typename T>
__device__ __forceinline__ void compact_row(const T* __restrict__ in, T* __restrict__ out, int W, int s, int lane,
                                            const uint32_t* __restrict__ rgb_old, int rpitch, int H,
                                            const int* __restrict__ seam, int i, bool fix) {
    using VT = Vec16<T>;
    constexpr int N = VT::N;
    const int Wn = W - 1;
    for (int q0 = 0; q0 * N < Wn; q0 += 32) {
        const int base = (q0 + lane) * N;
        const bool active = base < Wn;
        T a[N];
        // load whenever the chunk holds an input element: the previous lane's
        // last output may need this chunk's first element even when no output
        // position of this chunk survives
        if (base < W) VT::unpack(*reinterpret_cast<const typename VT::V*>(in + base), a);
        else {
#pragma unroll
            for (int u = 0; u < N; ++u) a[u] = T(0);
        }
        T nxt = __shfl_down_sync(FULL, a[0], 1);
        if (lane == 31 && active && base + N < W) nxt = in[base + N];
        T o[N];
#pragma unroll
        for (int u = 0; u < N; ++u) {
            const T hi = (u + 1 < N) ? a[u + 1] : nxt;
            o[u] = (base + u >= s) ? hi : a[u];
        }
        if (fix) {
#pragma unroll
            for (int u = 0; u < N; ++u) {
                const int x = base + u;
                if ((x == s - 1 || x == s) && x < Wn)
                    o[u] = T(fixup_energy(rgb_old, rpitch, Wn, H, seam, i, x));
            }
        }
        if (base + N <= Wn) *reinterpret_cast<typename VT::V*>(out + base) = VT::pack(o);
        else if (active) {
#pragma unroll
            for (int u = 0; u < N; ++u)
                if (base + u < Wn) out[base + u] = o[u];
        }
    }
}

struct CompactParams {
    const uint32_t* rgb_in;
    uint32_t* rgb_out;
    const double* e_in;  // nullable: RGB-only removal
    double* e_out;
    int pitch;   // RGBX plane pitch (elements)
    int epitch;  // energy plane pitch (doubles); e_in/e_out point at logical column 0
    int rgb_edges;  // in-place kernel: keep the RGBX replica columns -1 and W-1 (fused DP)
    int W, H;
    const int* seam;
    unsigned long long* stamps;  // optional [start, end] per image (written by block 0 / last block)
    long long p_istride, e_istride, s_istride, st_istride;
    const int* stop;  // optional device flag: nonzero = return at once (data-dependent loops)
};

// One thread per 4-pixel output chunk: 128-bit RGBX load + the next pixel,
// two 128-bit energy loads + the next energy, 128-bit stores. Every thread is
// independent, so a row is served by many warps with all loads in flight
// (the earlier one-warp-per-row loop was latency-bound at ~0.25 IPC).
constexpr int CP_CHUNK = 4, CP_THREADS = 256;

__global__ void __launch_bounds__(CP_THREADS) k_compact(CompactParams p) {
    const int img = blockIdx.z;
    const int i = blockIdx.y;
    const uint32_t* __restrict__ rgb_in = p.rgb_in + img * p.p_istride;
    uint32_t* __restrict__ rgb_out = p.rgb_out + img * p.p_istride;
    const int* __restrict__ seam = p.seam + img * p.s_istride;
    if (p.stamps && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
        atomicCAS(&p.stamps[img * p.st_istride + 0], 0ull, (unsigned long long)globaltimer());
    const int W = p.W, Wn = W - 1;
    const int base = (blockIdx.x * CP_THREADS + threadIdx.x) * CP_CHUNK;
    if (base < Wn) {
        const int s = __ldg(seam + i);
        // RGBX plane
        {
            const uint32_t* in = rgb_in + (long long)i * p.pitch;
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(in + base));
            const uint32_t a[5] = {v.x, v.y, v.z, v.w, base + 4 < W ? __ldg(in + base + 4) : 0u};
            uint32_t o[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) o[u] = (base + u >= s) ? a[u + 1] : a[u];
            uint32_t* out = rgb_out + (long long)i * p.pitch;
            if (base + 4 <= Wn) *reinterpret_cast<uint4*>(out + base) = make_uint4(o[0], o[1], o[2], o[3]);
            else
                for (int u = 0; u < 4 && base + u < Wn; ++u) out[base + u] = o[u];
        }
        if (p.e_in) {
            const long long eo = img * p.e_istride + (long long)i * p.epitch;
            const double* in = p.e_in + eo;
            const double2 v0 = __ldg(reinterpret_cast<const double2*>(in + base));
            const double2 v1 = __ldg(reinterpret_cast<const double2*>(in + base + 2));
            const double a[5] = {v0.x, v0.y, v1.x, v1.y, base + 4 < W ? __ldg(in + base + 4) : 0.0};
            double o[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int x = base + u;
                o[u] = (x >= s) ? a[u + 1] : a[u];
                // K1 fix-up: the two new-grid columns whose stencil changed
                if ((x == s - 1 || x == s) && x < Wn) o[u] = fixup_energy(rgb_in, p.pitch, Wn, p.H, seam, i, x);
            }
            double* out = p.e_out + eo;
            if (base + 4 <= Wn) {
                *reinterpret_cast<double2*>(out + base) = make_double2(o[0], o[1]);
                *reinterpret_cast<double2*>(out + base + 2) = make_double2(o[2], o[3]);
            } else {
                for (int u = 0; u < 4 && base + u < Wn; ++u) out[base + u] = o[u];
            }
            // the vacated column joins the +inf pad; so does the column this plane
            // last held live (planes alternate, so it may still be stale)
            if (base + 4 >= Wn) {
                out[Wn] = dinf();
                out[W] = dinf();
            }
        }
    }
    if (p.stamps && threadIdx.x == 0) atomicMax(&p.stamps[img * p.st_istride + 1], (unsigned long long)globaltimer());
}

// K4 in place (the carve loop's removal): RPB rows per CTA; only pixels at or
// right of the seam move (on average half the row), RGBX and FP64 energy.
// Every thread loads its shifted source chunk, the CTA synchronises, then the
// chunks are stored back, so the left shift by one is race-free within the row
// and rows are independent. The energy fix-up of the two new-grid columns runs
// in the next DP launch (Dp2Params::prev_seam), once every row is compacted.
template <int CH, int RPB>  // pixels per thread, rows per CTA (loads of all rows in flight before one barrier)
__global__ void __launch_bounds__(1024) k_compact_inplace(CompactParams p) {
    const int img = blockIdx.y;
    const int W = p.W, Wn = W - 1;
    const int base = threadIdx.x * CH;
    if (p.stamps && blockIdx.x == 0 && threadIdx.x == 0)
        atomicCAS(&p.stamps[img * p.st_istride + 0], 0ull, (unsigned long long)globaltimer());
    uint32_t o[RPB][CH];
    double oe[RPB][CH];
    bool act[RPB];
#pragma unroll
    for (int r = 0; r < RPB; ++r) {
        const int i = blockIdx.x * RPB + r;
        act[r] = false;
        if (i >= p.H) continue;
        const int s = __ldg(p.seam + img * p.s_istride + i);
        act[r] = base + CH > s && base < Wn;
        if (!act[r]) continue;
        const uint32_t* rgb = p.rgb_out + img * p.p_istride + (long long)i * p.pitch;
        uint32_t a[CH + 1];
#pragma unroll
        for (int q = 0; q < CH; q += 4) {
            const uint4 v = *reinterpret_cast<const uint4*>(rgb + base + q);
            a[q] = v.x; a[q + 1] = v.y; a[q + 2] = v.z; a[q + 3] = v.w;
        }
        a[CH] = base + CH < W ? rgb[base + CH] : 0u;
#pragma unroll
        for (int u = 0; u < CH; ++u) o[r][u] = (base + u >= s) ? a[u + 1] : a[u];
        if (p.e_out) {
            const double* e = p.e_out + img * p.e_istride + (long long)i * p.epitch;
            double b[CH + 1];
#pragma unroll
            for (int q = 0; q < CH; q += 2) {
                const double2 v = *reinterpret_cast<const double2*>(e + base + q);
                b[q] = v.x; b[q + 1] = v.y;
            }
            b[CH] = base + CH < W ? e[base + CH] : 0.0;
#pragma unroll
            for (int u = 0; u < CH; ++u) oe[r][u] = (base + u >= s) ? b[u + 1] : b[u];
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RPB; ++r) {
        const int i = blockIdx.x * RPB + r;
        if (i >= p.H) continue;
        double* e = p.e_out ? p.e_out + img * p.e_istride + (long long)i * p.epitch : nullptr;
        if (act[r]) {
            uint32_t* rgb = p.rgb_out + img * p.p_istride + (long long)i * p.pitch;
            if (base + CH <= Wn) {
#pragma unroll
                for (int q = 0; q < CH; q += 4)
                    *reinterpret_cast<uint4*>(rgb + base + q) =
                        make_uint4(o[r][q], o[r][q + 1], o[r][q + 2], o[r][q + 3]);
                if (e) {
#pragma unroll
                    for (int q = 0; q < CH; q += 2)
                        *reinterpret_cast<double2*>(e + base + q) = make_double2(oe[r][q], oe[r][q + 1]);
                }
            } else {
#pragma unroll
                for (int u = 0; u < CH; ++u)
                    if (base + u < Wn) {
                        rgb[base + u] = o[r][u];
                        if (e) e[base + u] = oe[r][u];
                    }
            }
        }
        if (e && threadIdx.x == 0) e[Wn] = dinf();  // the vacated column joins the +inf pad
    }
    if (p.rgb_edges) {  // replica columns for the fused DP's clamped stencil (raster.hpp:54-58)
        __syncthreads();
        if (threadIdx.x < RPB) {
            const int i = blockIdx.x * RPB + threadIdx.x;
            if (i < p.H) {
                uint32_t* rgb = p.rgb_out + img * p.p_istride + (long long)i * p.pitch;
                rgb[-1] = rgb[0];
                rgb[Wn] = rgb[Wn - 1];
            }
        }
    }
    if (p.stamps && threadIdx.x == 0) atomicMax(&p.stamps[img * p.st_istride + 1], (unsigned long long)globaltimer());
}

// RGBX replica columns -1 and W (edge replication, raster.hpp:54-58) for the fused DP.
__global__ void k_rgb_edges(uint32_t* __restrict__ rgb, int pitch, int W, int H, long long istride) {
    rgb += blockIdx.y * istride;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < H; i += gridDim.x * blockDim.x) {
        uint32_t* row = rgb + (long long)i * pitch;
        row[-1] = row[0];
        row[W] = row[W - 1];
    }
}

// K4, last removal of a phase, fused with the layout change that follows it
// (carver.hpp:216-222 transpose sandwich; raster.hpp:73-79):
//   OUT_PLANE : out(j, i) = in(i, j + [j >= s_i])  -> the transposed RGBX plane
//               the height phase carves (j < W-1, i < H)
//   OUT_PACKED: the final image in packed RGB, transposed back (height phase)
//   OUT_ROWS  : the final image in packed RGB, not transposed (width-only carves)
// A 32x32 tile goes through shared memory, so the row-major reads of the
// shifted row and the transposed writes are both coalesced.
enum { OUT_PLANE = 0, OUT_PACKED = 1, OUT_ROWS = 2 };

template <int MODE>
__global__ void k_compact_transpose(const uint32_t* __restrict__ in, int ipitch, int W, int H,
                                    const int* __restrict__ seam, uint32_t* __restrict__ out, int opitch,
                                    uint8_t* __restrict__ packed, long long in_is, long long out_is, long long seam_is,
                                    long long pk_is, unsigned long long* stamps, long long st_is) {
    __shared__ uint32_t tile[32][33];
    const int img = blockIdx.z;
    in += img * in_is;
    seam += img * seam_is;
    if (stamps && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0)
        atomicCAS(&stamps[img * st_is + 0], 0ull, (unsigned long long)globaltimer());
    const int Wn = W - 1;
    const int bj = blockIdx.x * 32, bi = blockIdx.y * 32;  // output-column (j) and row (i) tile origins
    if (MODE == OUT_ROWS) {
        // no transpose: rows stay rows; one thread per output pixel, packed write
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int i = bi + r, j = bj + threadIdx.x;
            if (i < H && j < Wn) {
                const int sp = __ldg(seam + i);
                const uint32_t v = in[(long long)i * ipitch + j + (j >= sp ? 1 : 0)];
                uint8_t* o = packed + img * pk_is + ((long long)i * Wn + j) * 3;
                o[0] = uint8_t(v);
                o[1] = uint8_t(v >> 8);
                o[2] = uint8_t(v >> 16);
            }
        }
    } else {
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int i = bi + r, j = bj + threadIdx.x;
            if (i < H && j < Wn) {
                const int sp = __ldg(seam + i);
                tile[r][threadIdx.x] = in[(long long)i * ipitch + j + (j >= sp ? 1 : 0)];
            }
        }
        __syncthreads();
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int j = bj + r, i = bi + threadIdx.x;  // output row j, column i
            if (i < H && j < Wn) {
                const uint32_t v = tile[threadIdx.x][r];
                if (MODE == OUT_PLANE) {
                    out[img * out_is + (long long)j * opitch + i] = v;
                } else {
                    uint8_t* o = packed + img * pk_is + ((long long)j * H + i) * 3;
                    o[0] = uint8_t(v);
                    o[1] = uint8_t(v >> 8);
                    o[2] = uint8_t(v >> 16);
                }
            }
        }
    }
    if (stamps && threadIdx.x == 0 && threadIdx.y == 0)
        atomicMax(&stamps[img * st_is + 1], (unsigned long long)globaltimer());
}

// K4 in place, one warp per row: the warp walks the part of the row right of
// the seam in batches of NB chunks per lane; all loads of a batch are issued
// before its stores, and batch b+1's loads only touch elements at or beyond
// the last element batch b read, so the left shift is race-free in program
// order without any CTA barrier. Rows are independent.
// HAS_E: the FP64 energy plane moves too (single-image mode); without it the
// kernel stays small enough for full occupancy (batches, RGBX only). The RGBX
// replica columns -1 / W-1 the fused DP reads are written by the lanes that
// store columns 0 / Wn-1 (no extra dependent load at the end of the row).
// One row's in-place removal by one warp (the body of k_compact_warp, also run
// by the fused batch DP after its backtrack): the part right of seam column s
// moves left by one, in batches of NB 4-pixel chunks per lane.
template <int NB, bool HAS_E>
__device__ __forceinline__ void compact_row_warp(uint32_t* __restrict__ rgb, double* __restrict__ e, int W, int s,
                                                 int lane, bool edges) {
    const int Wn = W - 1;
    // first 4-aligned chunk that changes
    const int q0 = (s >> 2);
    for (int qb = q0; qb * 4 < Wn; qb += 32 * NB) {
        uint32_t o[NB][4];
        double oe[HAS_E ? NB : 1][4];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int base = (qb + u * 32 + lane) * 4;
            if (base < Wn) {
                const uint4 v = *reinterpret_cast<const uint4*>(rgb + base);
                const uint32_t a[5] = {v.x, v.y, v.z, v.w, base + 4 < W ? rgb[base + 4] : 0u};
#pragma unroll
                for (int t = 0; t < 4; ++t) o[u][t] = (base + t >= s) ? a[t + 1] : a[t];
                if constexpr (HAS_E) {
                    const double2 v0 = *reinterpret_cast<const double2*>(e + base);
                    const double2 v1 = *reinterpret_cast<const double2*>(e + base + 2);
                    const double b[5] = {v0.x, v0.y, v1.x, v1.y, base + 4 < W ? e[base + 4] : 0.0};
#pragma unroll
                    for (int t = 0; t < 4; ++t) oe[u][t] = (base + t >= s) ? b[t + 1] : b[t];
                }
            }
        }
        __syncwarp();  // every lane's loads of this batch precede any store of it
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int base = (qb + u * 32 + lane) * 4;
            if (base + 4 <= Wn) {
                *reinterpret_cast<uint4*>(rgb + base) = make_uint4(o[u][0], o[u][1], o[u][2], o[u][3]);
                if constexpr (HAS_E) {
                    *reinterpret_cast<double2*>(e + base) = make_double2(oe[u][0], oe[u][1]);
                    *reinterpret_cast<double2*>(e + base + 2) = make_double2(oe[u][2], oe[u][3]);
                }
            } else if (base < Wn) {
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (base + t < Wn) {
                        rgb[base + t] = o[u][t];
                        if constexpr (HAS_E) e[base + t] = oe[u][t];
                    }
            }
            if (edges && base < Wn) {  // replica columns (raster.hpp:54-58 clamping)
                if (base == 0 && s == 0) rgb[-1] = o[u][0];
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (base + t == Wn - 1) rgb[Wn] = o[u][t];
            }
        }
        __syncwarp();  // this batch's stores precede the next batch's loads
    }
    // seam in the row's last chunk: nothing moved, but the right replica follows column Wn-1
    if (edges && lane == 0 && q0 * 4 >= Wn) rgb[Wn] = rgb[Wn - 1];
    if constexpr (HAS_E) {
        if (lane == 0) e[Wn] = dinf();  // the vacated column joins the +inf pad
    }
}

// R rows' in-place RGBX removal by one warp at once (the fused batch DP's
// epilogue): every lane holds one 4-pixel chunk of each of the R rows per
// batch, so R x 512 B of loads are in flight per warp before any store. Same
// semantics as compact_row_warp<.., false> with edges (replica columns).
template <int R>
__device__ __forceinline__ void compact_rows_warp(uint32_t* __restrict__ plane, long long pitch, int W, const int (&s)[R],
                                                  int lane) {
    const int Wn = W - 1;
    int q0[R], nb = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        q0[r] = s[r] >> 2;
        nb = max(nb, (Wn - 1 - q0[r] * 4 + 128) / 128);  // batches of 32 chunks this row needs (>= 0)
    }
    for (int t = 0; t < nb; ++t) {
        uint32_t o[R][4];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t* row = plane + r * pitch;
            const int base = (q0[r] + t * 32 + lane) * 4;
            if (base < Wn) {
                const uint4 v = *reinterpret_cast<const uint4*>(row + base);
                const uint32_t a[5] = {v.x, v.y, v.z, v.w, base + 4 < W ? row[base + 4] : 0u};
#pragma unroll
                for (int u = 0; u < 4; ++u) o[r][u] = (base + u >= s[r]) ? a[u + 1] : a[u];
            }
        }
        __syncwarp();  // every lane's loads of this batch precede any store of it
#pragma unroll
        for (int r = 0; r < R; ++r) {
            uint32_t* row = plane + r * pitch;
            const int base = (q0[r] + t * 32 + lane) * 4;
            if (base + 4 <= Wn) {
                *reinterpret_cast<uint4*>(row + base) = make_uint4(o[r][0], o[r][1], o[r][2], o[r][3]);
            } else if (base < Wn) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (base + u < Wn) row[base + u] = o[r][u];
            }
            if (base < Wn) {  // replica columns (raster.hpp:54-58 clamping)
                if (base == 0 && s[r] == 0) row[-1] = o[r][0];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (base + u == Wn - 1) row[Wn] = o[r][u];
            }
        }
        __syncwarp();  // this batch's stores precede the next batch's loads
    }
#pragma unroll
    for (int r = 0; r < R; ++r)  // seam in the row's last chunk: only the right replica changes
        if (lane == 0 && q0[r] * 4 >= Wn) plane[r * pitch + Wn] = plane[r * pitch + Wn - 1];
}

template <int NB, bool HAS_E>
__global__ void __launch_bounds__(256) k_compact_warp(CompactParams p) {
    const int img = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    pdl_wait();  // the DP that produced this seam has completed
    pdl_launch_dependents();
    if (p.stop && *p.stop) return;  // uniform over the grid (set by an earlier kernel)
    if (p.stamps && blockIdx.x == 0 && threadIdx.x == 0)
        atomicCAS(&p.stamps[img * p.st_istride + 0], 0ull, (unsigned long long)globaltimer());
    if (i < p.H) {
        const int s = __ldg(p.seam + img * p.s_istride + i);
        uint32_t* rgb = p.rgb_out + img * p.p_istride + (long long)i * p.pitch;
        double* e = HAS_E ? p.e_out + img * p.e_istride + (long long)i * p.epitch : nullptr;
        compact_row_warp<NB, HAS_E>(rgb, e, p.W, s, lane, p.rgb_edges);
    }
    if (p.stamps && threadIdx.x == 0) atomicMax(&p.stamps[img * p.st_istride + 1], (unsigned long long)globaltimer());
}

// Batches (RGBX only, replica columns refreshed): one warp removes the seam
// from R consecutive rows at once, so R x 512 B of loads are in flight per warp
// and the per-row seam load / ramp is amortised over R rows.
template <int R>
__global__ void __launch_bounds__(256) k_compact_rows(CompactParams p) {
    const int img = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int i0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * R;
    pdl_wait();  // the DP that produced this seam has completed
    pdl_launch_dependents();
    if (p.stamps && blockIdx.x == 0 && threadIdx.x == 0)
        atomicCAS(&p.stamps[img * p.st_istride + 0], 0ull, (unsigned long long)globaltimer());
    const int* seam = p.seam + img * p.s_istride;
    uint32_t* plane = p.rgb_out + img * p.p_istride;
    if (i0 + R <= p.H) {
        int sr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) sr[r] = __ldg(seam + i0 + r);
        compact_rows_warp<R>(plane + (long long)i0 * p.pitch, p.pitch, p.W, sr, lane);
    } else {
        for (int i = i0; i < p.H; ++i)
            compact_row_warp<4, false>(plane + (long long)i * p.pitch, nullptr, p.W, __ldg(seam + i), lane, true);
    }
    if (p.stamps && threadIdx.x == 0) atomicMax(&p.stamps[img * p.st_istride + 1], (unsigned long long)globaltimer());
}

// Batches (RGBX only, replica columns refreshed): the moving part of each row is
// fetched by the TMA engine (cp.async.bulk global -> shared, mbarrier completion)
// SLOTS rows ahead, so many rows' loads are in flight per CTA without holding
// registers; the CTA's threads then store the row shifted left by one pixel from
// shared memory (128-bit coalesced stores). In place: a row's stores start only
// after its whole right part has landed in shared memory.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
// HAS_E: the FP64 energy plane moves too (single images; its vacated column becomes
// the +inf pad) and the replica columns are left alone; without it (batches, fused DP)
// the RGBX replica columns -1 / W-1 are refreshed. Shared memory per slot: the RGBX
// part (slot_words) then, with HAS_E, the energy part (slot_words doubles).
constexpr int CB_MAX_SLOTS = 4;
template <bool HAS_E>
__global__ void __launch_bounds__(128) k_compact_bulk(CompactParams p, int rows_per_cta, int slot_words, int slots) {
    extern __shared__ __align__(128) uint32_t cb_sm[];
    __shared__ __align__(8) uint64_t cb_bar[CB_MAX_SLOTS];
    const int img = blockIdx.y;
    const int row0 = blockIdx.x * rows_per_cta;
    const int nrows = min(rows_per_cta, p.H - row0);
    const int W = p.W, Wn = W - 1;
    const int* seam = p.seam + img * p.s_istride + row0;
    uint32_t* plane = p.rgb_out + img * p.p_istride + (long long)row0 * p.pitch;
    double* eplane = HAS_E ? p.e_out + img * p.e_istride + (long long)row0 * p.epitch : nullptr;
    const int slot_bytes = slot_words * (HAS_E ? 12 : 4);
    const uint32_t bar0 = uint32_t(__cvta_generic_to_shared(cb_bar));
    const uint32_t sm0 = uint32_t(__cvta_generic_to_shared(cb_sm));
    if (threadIdx.x == 0) {
        for (int k = 0; k < slots; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * k) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();  // the DP that produced this seam has completed
    pdl_launch_dependents();
    if (p.stop && *p.stop) return;  // uniform over the grid (set by an earlier kernel)
    if (p.stamps && blockIdx.x == 0 && threadIdx.x == 0)
        atomicCAS(&p.stamps[img * p.st_istride + 0], 0ull, (unsigned long long)globaltimer());
    // row r's moving part: 16-byte aligned from a = floor4(s) to W (rounded up to 4 pixels;
    // the padded pitches cover the overhang)
    auto issue = [&](int r) {
        const int a = __ldg(seam + r) & ~3;
        const uint32_t n4 = uint32_t((W - a + 3) & ~3);
        const uint32_t b = bar0 + 8 * (r % slots);
        const uint32_t dst = sm0 + uint32_t((r % slots) * slot_bytes);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n4 * (HAS_E ? 12 : 4))
                     : "memory");
        bulk_g2s(dst, plane + (long long)r * p.pitch + a, n4 * 4, b);
        if constexpr (HAS_E) bulk_g2s(dst + uint32_t(slot_words * 4), eplane + (long long)r * p.epitch + a, n4 * 8, b);
    };
    if (threadIdx.x == 0)
        for (int r = 0; r < min(slots, nrows); ++r) issue(r);
    for (int r = 0; r < nrows; ++r) {
        const int k = r % slots;
        const uint32_t parity = uint32_t(r / slots) & 1u;
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                         : "=r"(ok)
                         : "r"(bar0 + 8 * k), "r"(parity)
                         : "memory");
        const int s = __ldg(seam + r), a = s & ~3;
        const unsigned char* slot = reinterpret_cast<const unsigned char*>(cb_sm) + size_t(k) * slot_bytes;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(slot) - a;  // src[j] = old pixel j, j in [a, W)
        const double* esrc = reinterpret_cast<const double*>(slot + slot_words * 4) - a;
        uint32_t* row = plane + (long long)r * p.pitch;
        double* erow = HAS_E ? eplane + (long long)r * p.epitch : nullptr;
        for (int c = a + 4 * int(threadIdx.x); c < Wn; c += 4 * int(blockDim.x)) {
            uint32_t o[4];
            double oe[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                o[u] = src[c + u + (c + u >= s ? 1 : 0)];
                if constexpr (HAS_E) oe[u] = esrc[c + u + (c + u >= s ? 1 : 0)];
            }
            if (c + 4 <= Wn) {
                *reinterpret_cast<uint4*>(row + c) = make_uint4(o[0], o[1], o[2], o[3]);
                if constexpr (HAS_E) {
                    *reinterpret_cast<double2*>(erow + c) = make_double2(oe[0], oe[1]);
                    *reinterpret_cast<double2*>(erow + c + 2) = make_double2(oe[2], oe[3]);
                }
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (c + u < Wn) {
                        row[c + u] = o[u];
                        if constexpr (HAS_E) erow[c + u] = oe[u];
                    }
            }
            if constexpr (!HAS_E) {
                if (c == 0 && s == 0) row[-1] = o[0];  // replica columns (raster.hpp:54-58 clamping)
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (c + u == Wn - 1) row[Wn] = o[u];
            }
        }
        if (threadIdx.x == 0) {
            if constexpr (HAS_E) erow[Wn] = dinf();  // the vacated column joins the +inf pad
            // the seam is in the row's last 4-pixel chunk past Wn-1: nothing moves, only the right
            // replica follows column Wn-1 (unchanged in global memory, before the loaded part)
            else if (a >= Wn) row[Wn] = row[Wn - 1];
        }
        __syncthreads();  // every thread is done with slot k
        if (threadIdx.x == 0 && r + slots < nrows) issue(r + slots);
    }
    if (p.stamps && threadIdx.x == 0) atomicMax(&p.stamps[img * p.st_istride + 1], (unsigned long long)globaltimer());
}

// ---------------------------------------------------------------------------
// Object removal: masks travel in the RGBX planes' spare
// byte (bit 24), so every removal and transpose kernel carries them for free.

constexpr uint32_t MASK_BIT = 1u << 24;

// packed RGB + u8 flags (nonzero = remove, energy.hpp:25-37) -> RGBX with the mask bit
__global__ void k_unpack_masked(const uint8_t* __restrict__ in, const uint8_t* __restrict__ mask, int W, int H,
                                uint32_t* __restrict__ out, int pitch) {
    const long long n = (long long)W * H;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = int(k / W), j = int(k - (long long)i * W);
        const uint8_t* p = in + 3 * k;
        out[(long long)i * pitch + j] = uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) |
                                        (mask[k] ? MASK_BIT : 0u);
    }
}

// mask_from_image (energy.hpp:244-253): FP64 luma >= 128 marks a pixel
__global__ void k_mask_from_rgb(const uint8_t* __restrict__ in, long long n, uint8_t* __restrict__ flags) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const uint8_t* p = in + 3 * k;
        flags[k] = luma(uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16)) >= 128.0 ? 1 : 0;
    }
}

// apply_mask's reductions (energy.hpp:224-233) over the live W x H: energies are
// >= +0, so their IEEE bit patterns order like the values and atomicMax on the
// bits is an exact max.
struct MaskStats {
    unsigned long long max_unmasked, max_all, marked;
    int any_unmasked;
};

template <bool U8>  // mask from a u8 plane (API) or the RGBX mask bit (carve loop)
__device__ __forceinline__ bool masked_at(const uint8_t* m8, const uint32_t* rgb, int rpitch, int i, int j, int W) {
    if constexpr (U8) return m8[(long long)i * W + j] != 0;
    else return (rgb[(long long)i * rpitch + j] & MASK_BIT) != 0;
}

template <bool U8>
__global__ void k_mask_stats(const double* __restrict__ e, int epitch, const uint8_t* __restrict__ m8,
                             const uint32_t* __restrict__ rgb, int rpitch, int W, int H, MaskStats* st,
                             const int* stop = nullptr, unsigned long long* stamps = nullptr) {
    if (stop && *stop) return;
    if (stamps && blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(stamps, 0ull, (unsigned long long)globaltimer());
    unsigned long long mu = 0, ma = 0, cnt = 0;
    int any = 0;
    const long long n = (long long)W * H;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = int(k / W), j = int(k - (long long)i * W);
        // std::max(0.0, v) semantics (the reference's maxima start at 0.0): only
        // positive values can raise them, and their bit patterns order like values
        const double v = e[(long long)i * epitch + j];
        const unsigned long long b = v > 0.0 ? (unsigned long long)__double_as_longlong(v) : 0ull;
        ma = b > ma ? b : ma;
        if (masked_at<U8>(m8, rgb, rpitch, i, j, W)) ++cnt;
        else {
            mu = b > mu ? b : mu;
            any = 1;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(FULL, mu, o), c = __shfl_xor_sync(FULL, ma, o);
        mu = a > mu ? a : mu;
        ma = c > ma ? c : ma;
        cnt += __shfl_xor_sync(FULL, cnt, o);
        any |= __shfl_xor_sync(FULL, any, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (mu) atomicMax(&st->max_unmasked, mu);
        if (ma) atomicMax(&st->max_all, ma);
        if (cnt) atomicAdd(&st->marked, cnt);
        if (any) atomicOr(&st->any_unmasked, 1);
    }
}

// k = 1000 * (h * m + 1), left to right, no contraction (energy.hpp:234-235)
__device__ __forceinline__ double mask_bias(const MaskStats* st, int H) {
    const double m = __longlong_as_double((long long)(st->any_unmasked ? st->max_unmasked : st->max_all));
    return __dmul_rn(1000.0, __dadd_rn(__dmul_rn(double(H), m), 1.0));
}

// biased map (energy.hpp:237-240): masked cells -> -k; in the carve loop also
// column W (the one the last removal vacated) -> +inf pad
// the removal loop's stop test, one thread: no marked pixel left -> *done = 1 (every
// later kernel of the loop returns at once); else one more seam (*count)
__global__ void k_mask_decide(const MaskStats* st, int* done, int* count) {
    if (*done) return;
    if (st->marked == 0) *done = 1;
    else ++*count;
}

template <bool U8>
__global__ void k_apply_mask(const double* __restrict__ e, int epitch, const uint8_t* __restrict__ m8,
                             const uint32_t* __restrict__ rgb, int rpitch, int W, int H, const MaskStats* st,
                             double* __restrict__ out, int opitch, int pad_col, const int* stop = nullptr,
                             unsigned long long* stamp_end = nullptr) {
    if (stop && *stop) return;
    EndStamp end_stamp{stamp_end};
    const double negk = -mask_bias(st, H);
    const long long n = (long long)W * H;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = int(k / W), j = int(k - (long long)i * W);
        out[(long long)i * opitch + j] = masked_at<U8>(m8, rgb, rpitch, i, j, W) ? negk : e[(long long)i * epitch + j];
        if (pad_col && j == W - 1) out[(long long)i * opitch + W] = dinf();
    }
}

// K1 fix-up of the two new-grid columns around a removed seam (SURVEY.md
// Appendix A.4), standalone: the object-removal loop solves on a biased copy,
// so the DP prologue's in-place fix-up does not apply there.
__global__ void k_fixup_energy(double* __restrict__ e, int epitch, const uint32_t* __restrict__ rgb, int rpitch, int W,
                               int H, const int* __restrict__ seam, const int* stop = nullptr,
                               unsigned long long* stamp_end = nullptr) {
    if (stop && *stop) return;
    EndStamp end_stamp{stamp_end};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < H; i += gridDim.x * blockDim.x) {
        const int sp = seam[i];
        const uint32_t* row = rgb + (long long)i * rpitch;
        const uint32_t* up = rgb + (long long)max(i - 1, 0) * rpitch;
        const uint32_t* dn = rgb + (long long)min(i + 1, H - 1) * rpitch;
        for (int x = sp - 1; x <= sp; ++x)
            if (x >= 0 && x < W)
                e[(long long)i * epitch + x] =
                    e1(luma(row[max(x - 1, 0)]), luma(row[min(x + 1, W - 1)]), luma(up[x]), luma(dn[x]));
    }
}

// ---------------------------------------------------------------------------
// Forward energy helpers

// forward_costs (energy.hpp:196-216): cu = |R - L|, cl = cu + |A - L|,
// cr = cu + |A - R| over clamped neighbours (at_clamped, raster.hpp:54-58),
// left to right, no contraction
__device__ __forceinline__ void fwd_costs_of(double l, double r, double a, double& cl, double& cu, double& cr) {
    cu = fabs(__dsub_rn(r, l));
    cl = __dadd_rn(cu, fabs(__dsub_rn(a, l)));
    cr = __dadd_rn(cu, fabs(__dsub_rn(a, r)));
}

// ... of an arbitrary luma plane (pitch W in, pitch opitch out; the API entry and
// the dp_seam_forward(gray) path; the default forward carve loop computes the
// same costs in registers inside the fused DP)
__global__ void k_forward_costs(const double* __restrict__ g, int W, int H, double* __restrict__ left,
                                double* __restrict__ up, double* __restrict__ right, int opitch) {
    const long long n = (long long)W * H;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = int(k / W), j = int(k - (long long)i * W);
        const double* row = g + (long long)i * W;
        const double l = row[max(j - 1, 0)], r = row[min(j + 1, W - 1)];
        const double a = g[(long long)max(i - 1, 0) * W + j];
        const long long o = (long long)i * opitch + j;
        fwd_costs_of(l, r, a, left[o], up[o], right[o]);
    }
}

// ... of to_grayscale of an RGBX plane, into three padded planes (plane stride
// cplane): the recompute=false forward loop's cost state at the start of a phase
__global__ void k_forward_costs_rgbx(const uint32_t* __restrict__ rgb, int rpitch, int W, int H,
                                     double* __restrict__ costs, int epitch, long long cplane) {
    const long long n = (long long)W * H;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = int(k / W), j = int(k - (long long)i * W);
        const uint32_t* row = rgb + (long long)i * rpitch;
        const double l = luma(row[max(j - 1, 0)]), r = luma(row[min(j + 1, W - 1)]);
        const double a = luma(rgb[(long long)max(i - 1, 0) * rpitch + j]);
        const long long o = (long long)i * epitch + j;
        fwd_costs_of(l, r, a, costs[o], costs[o + cplane], costs[o + 2 * cplane]);
    }
}

// detail::drop_columns (carver.hpp:57-67) on `np` FP64 planes at once (plane
// stride pstride, pitch `pitch`, out of place): out[i][j] = in[i][j + (j >= s_i)]
// for j < W - 1. One CTA row per image row, consecutive columns per thread.
__global__ void k_drop_col_planes(const double* __restrict__ in, double* __restrict__ out, int pitch,
                                  long long pstride, int W, int H, const int* __restrict__ seam) {
    const int i = blockIdx.y, pl = blockIdx.z;
    const int s = __ldg(seam + i);
    const double* src = in + pl * pstride + (long long)i * pitch;
    double* dst = out + pl * pstride + (long long)i * pitch;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < W - 1; j += gridDim.x * blockDim.x)
        dst[j] = src[j + (j >= s ? 1 : 0)];
}

// remove_seam(LumaGrid / EnergyMap / RemovalMask) (carver.hpp:84-112): the
// row-major w x h plane minus column s_i of every row, out of place, packed
// pitch w - 1. One thread per output element; T = double or uint8_t.
template <typename T>
__global__ void k_drop_columns(const T* __restrict__ in, int W, int H, const int* __restrict__ seam,
                               T* __restrict__ out) {
    const long long n = (long long)(W - 1) * H;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = int(k / (W - 1)), j = int(k - (long long)i * (W - 1));
        out[k] = in[(long long)i * W + j + (j >= __ldg(seam + i) ? 1 : 0)];
    }
}

// columns -1 and W of a padded FP64 plane replicate columns 0 and W-1
__global__ void k_edge_replicas_f64(double* __restrict__ e, int epitch, int W, int H) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < H; i += gridDim.x * blockDim.x) {
        double* row = e + (long long)i * epitch;
        row[-1] = row[0];
        row[W] = row[W - 1];
    }
}

// ---------------------------------------------------------------------------
// Seam recording and enlargement

// record_seams (carver.hpp:226-262) reports each seam in original-image
// coordinates via per-row survivor lists. The device carve loop logs seam t in
// the coordinates of the grid it was found on; column x of grid u+1 is column
// x + (x >= s_u) of grid u (remove_seam, carver.hpp:71-82), so walking back
// through the row's earlier seams recovers the survivor index. One thread per
// (seam, row); the log is read row-coalesced.
__global__ void k_seams_to_original(const int* __restrict__ log, int count, int H, int* __restrict__ out) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= (long long)count * H) return;
    const int t = int(idx / H), i = int(idx - (long long)t * H);
    int x = log[idx];
    for (int u = t - 1; u >= 0; --u) x += x >= log[(long long)u * H + i] ? 1 : 0;
    out[idx] = x;
}

// enlarge_to_width's replay (carver.hpp:266-285) in closed form. Recorded
// columns of one row are distinct original columns, and the replay's shift
// rule keeps every later seam pointing at the same original pixel, so seam t
// always inserts immediately right of original column o_t, whose right
// neighbour at that moment is still original column o_t + 1 (nothing else has
// been inserted after o_t; clamped at the border). The enlarged row is thus
// the original row with insert_columns' rounded mean (carver.hpp:124-128) of
// p[o] and p[min(o+1, W-1)] after every recorded column o — independent of the
// replay order. One warp per row: the recorded columns become a bitmap in
// shared memory; a warp scan of word popcounts gives every column's output
// position; lanes walk the row with consecutive columns (coalesced reads).
// cols[t * cstride + i] is row i's column of seam t. Packed RGB in and out.
__global__ void k_expand_rows(const uint8_t* __restrict__ in, int W, int H, const int* __restrict__ cols, int count,
                              long long cstride, uint8_t* __restrict__ out) {
    extern __shared__ uint32_t bm_all[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int i = blockIdx.x * (blockDim.x >> 5) + wib;
    const int nw = (W + 31) >> 5;
    uint32_t* bm = bm_all + wib * nw;
    if (i >= H) return;
    for (int k = lane; k < nw; k += 32) bm[k] = 0u;
    __syncwarp();
    for (int t = lane; t < count; t += 32) {
        const int o = cols[(long long)t * cstride + i];
        atomicOr(&bm[o >> 5], 1u << (o & 31));
    }
    __syncwarp();
    const uint8_t* src = in + (long long)i * W * 3;
    uint8_t* dst = out + (long long)i * (W + count) * 3;
    int running = 0;  // inserted pixels left of this group of 32 words
    for (int wb = 0; wb < nw; wb += 32) {
        const uint32_t word = wb + lane < nw ? bm[wb + lane] : 0u;
        const int cnt = __popc(word);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
        }
        const int pre = running + incl - cnt;  // inserted pixels left of my word
        for (int u = 0; u < 32 && wb + u < nw; ++u) {
            const uint32_t wu = __shfl_sync(FULL, word, u);
            const int pu = __shfl_sync(FULL, pre, u);
            const int j = (wb + u) * 32 + lane;
            if (j < W) {
                const int pos = j + pu + __popc(wu & ((1u << lane) - 1u));
                const uint8_t* a = src + 3 * j;
                uint8_t* d = dst + 3 * pos;
                d[0] = a[0];
                d[1] = a[1];
                d[2] = a[2];
                if (wu >> lane & 1u) {
                    const uint8_t* b = src + 3 * min(j + 1, W - 1);
                    d[3] = uint8_t((a[0] + b[0] + 1) / 2);
                    d[4] = uint8_t((a[1] + b[1] + 1) / 2);
                    d[5] = uint8_t((a[2] + b[2] + 1) / 2);
                }
            }
        }
        running += __shfl_sync(FULL, incl, 31);
    }
}

#endif  // CARVE_KERNELS_HELPERS_ONLY

}  // namespace carve_dev
