/* carve_cuda.h — C ABI of libcarve_cuda.so, the B200 (sm_100a) seam-carving engine.
 *
 * This is the drop-in boundary. Each entry point replaces the
 * body of one reference function in /root/reference/proj/include/carve/ and
 * keeps its argument meaning and error behaviour; the C++ headers in
 * include/carve/ wrap these calls under the reference's own names and throw
 * carve::Error exactly where the reference does.
 *
 * Conventions
 *  - Images are packed 8-bit RGB, row-major, 3 bytes per pixel
 *    (raster.hpp:19-42 `Rgb`/`PixelGrid`). Scalar planes are row-major
 *    doubles (raster.hpp:45-59 `LumaGrid`, energy.hpp:16-23 `EnergyMap`).
 *  - Host pointers are caller-owned; outputs are preallocated by the caller.
 *    Pinned host memory makes the copies asynchronous, pageable works too.
 *  - Every call is synchronous (returns after its stream has drained) and
 *    thread-safe: each calling thread owns one context per device (stream,
 *    cached device buffers, pinned staging).
 *  - Return value: CARVE_OK, or 1 + the reference `carve::Errc` ordinal
 *    (error.hpp:8-26), or CARVE_E_CUDA for a device/runtime failure (which
 *    the reference CLI would report as a runtime error, exit code 2).
 *    carve_cuda_last_error() returns the thread's last message.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns CARVE_E_CUDA.
 */
#ifndef CARVE_CUDA_H
#define CARVE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int carve_status;

enum {
    CARVE_OK = 0,
    /* 1 + carve::Errc (error.hpp:8-26) */
    CARVE_E_FILE_NOT_FOUND = 1,
    CARVE_E_UNSUPPORTED_FORMAT = 2,
    CARVE_E_CORRUPT_IMAGE = 3,
    CARVE_E_IO_FAILURE = 4,
    CARVE_E_DIMENSION_MISMATCH = 5,
    CARVE_E_INVALID_SEAM = 6,
    CARVE_E_IMAGE_TOO_LARGE = 7,
    CARVE_E_EMPTY_IMAGE = 8,
    CARVE_E_WIDTH_TOO_SMALL = 9,
    CARVE_E_INVALID_TARGET = 10,
    CARVE_E_TARGET_TOO_LARGE = 11,
    CARVE_E_EMPTY_MASK = 12,
    CARVE_E_INSUFFICIENT_DATA = 13,
    CARVE_E_SIZE_EXCEEDS_SOURCE = 14,
    CARVE_E_SOLVER_CAP_VIOLATED = 15,
    CARVE_E_EMPTY_INPUT = 16,
    CARVE_E_USAGE_ERROR = 17,
    /* device / runtime failure (no reference equivalent) */
    CARVE_E_CUDA = 100
};

/* Per-seam timing, filled from device %globaltimer stamps
 * (replaces carver.hpp:23-27 SeamTiming laps). Seconds. */
/* The CarveConfig fields that change results (carver.hpp:15-24); NULL = the
 * reference defaults {forward = 0, recompute = 1}. solver/workers/energy_fn
 * have no output effect on this path (dp == pardp; e1 only). */
typedef struct carve_cuda_config {
    int forward;   /* forward energy: dp_seam_forward on forward_costs(to_grayscale(current)) */
    int recompute; /* 0: the phase's first e1 map (or, with forward, its three forward-cost
                      planes) is computed once and then only carved (carver.hpp:175-188) */
} carve_cuda_config;

typedef struct carve_seam_timing {
    double energy_s; /* K1 full map for a phase's first seam, the DP prologue's
                        2-column fix-up for the others; 0 where the energy is
                        computed inside the DP (batches, forward energy) or not
                        recomputed (recompute = 0) */
    double solve_s;  /* DP + argmin + backtrack (K2+K3) */
    double remove_s; /* compaction (K4) */
} carve_seam_timing;

/* ---- library ----------------------------------------------------------- */
const char* carve_cuda_last_error(void);
const char* carve_cuda_version(void);
/* Number of usable CUDA devices (0 when none). */
int carve_cuda_device_count(void);
/* Select the device used by this thread's subsequent calls (default 0). */
carve_status carve_cuda_set_device(int device);
/* Number of kernels this library launched on this thread since the last reset. */
uint64_t carve_cuda_launch_count(void);
void carve_cuda_reset_launch_count(void);
/* Profiling mode for the bench: when on, every kernel the carve driver
 * launches on this thread's current device is bracketed by a CUDA event pair
 * on its stream. Turning it on or off clears the collected records. */
carve_status carve_cuda_set_kernel_events(int on);
/* Sum over the collected launches of one kernel kind (0 energy full map,
 * 1 DP+argmin+backtrack, 2 removal+fix-up, 3 unpack, 4 pack, 5 transpose):
 * total event time (ms), launch count, total algorithmic bytes
 * (SURVEY.md §8d). Synchronizes the context stream. */
carve_status carve_cuda_kernel_event_stats(int kind, double* ms_total, uint64_t* launches, double* bytes_total);

/* ---- raster / energy (raster.hpp:61-79, energy.hpp:89-98,186-194) ------ */
/* replaces to_grayscale (raster.hpp:61-71) */
carve_status carve_cuda_to_grayscale(const uint8_t* rgb, int w, int h, double* luma_out);
/* replaces energy_e1(to_grayscale(img)) (energy.hpp:89-98 + raster.hpp:61-71) */
carve_status carve_cuda_energy_e1_rgb(const uint8_t* rgb, int w, int h, double* e_out);
/* replaces energy_e1(const LumaGrid&) on an arbitrary luma plane (energy.hpp:89-98) */
carve_status carve_cuda_energy_e1_luma(const double* luma, int w, int h, double* e_out);
/* replaces transpose (raster.hpp:73-79) */
carve_status carve_cuda_transpose_rgb(const uint8_t* rgb, int w, int h, uint8_t* out);

/* ---- solver (solvers.hpp:69-111, 263-289, 331-358) --------------------- */
/* replaces dp_seam / parallel_dp_seam (solvers.hpp:263-289, 331-347): the
 * cost table m (w*h doubles) and predecessor table b (w*h ints) are written
 * when non-NULL; seam_out receives h column indices, top row first.
 * Bit-identical for every input and independent of any worker count. */
carve_status carve_cuda_dp_seam(const double* e, int w, int h, double* m_out, int32_t* b_out, int32_t* seam_out);
/* Tools: run the DP once on e with per-warp clock64 phase counters
 * ([warp][8]: forward, halo wait, argmin+phase1, phase2, H). */
carve_status carve_cuda_dp_profile(const double* e, int w, int h, long long* counters, int ncounters, int* warps);
/* replaces validate_seam (solvers.hpp:69-78); pure host check */
carve_status carve_cuda_validate_seam(const int32_t* seam, int n, int w, int h);

/* ---- forward energy (energy.hpp:196-216, solvers.hpp:294-326) ---------- */
/* replaces forward_costs(const LumaGrid&); outputs w*h doubles each */
carve_status carve_cuda_forward_costs(const double* luma, int w, int h, double* left, double* up, double* right);
/* replaces dp_seam_forward(gray, forward_costs(gray)): table (nullable pair)
 * and seam, bit-identical. */
carve_status carve_cuda_dp_seam_forward(const double* luma, int w, int h, double* m_out, int32_t* b_out,
                                        int32_t* seam_out);
/* replaces dp_seam_forward(gray, costs) for arbitrary caller-given costs
 * (solvers.hpp:294-326; gray only supplies the dimensions there): three w*h
 * planes, row-major. Finite costs only: a non-finite cost returns
 * CARVE_E_USAGE_ERROR (the reference's best = +inf start would then differ). */
carve_status carve_cuda_dp_seam_forward_costs(const double* left, const double* up, const double* right, int w,
                                              int h, double* m_out, int32_t* b_out, int32_t* seam_out);

/* ---- object removal (energy.hpp:220-253, carver.hpp:287-340) ---------- */
/* replaces mask_from_image: flags (w*h bytes) = luma >= 128 */
carve_status carve_cuda_mask_from_rgb(const uint8_t* rgb, int w, int h, uint8_t* flags);
/* replaces apply_mask(energy, mask): masked cells -> -1000*(h*m+1) */
carve_status carve_cuda_apply_mask(const double* e, int w, int h, const uint8_t* mask, double* out);
/* replaces remove_object(grid, mask, cfg, restore) (carver.hpp:327-340).
 * mask: w*h flags (nonzero = remove). rgb_out: caller buffer of w*h*3 bytes,
 * the result is *out_w x *out_h. seams_out (nullable): w*h ints, receives the
 * report's seams concatenated (length h each for vertical removal, w each when
 * the mask's bounding box is wider than tall); *nseams (nullable) their count. */
carve_status carve_cuda_remove_object(const uint8_t* rgb, int w, int h, const uint8_t* mask,
                                      const carve_cuda_config* cfg, int restore, uint8_t* rgb_out, int* out_w,
                                      int* out_h, int32_t* seams_out, int* nseams);
/* remove_object with the report's per-seam timings (timings_out: nullable, w*h
 * entries at most; energy = the mask statistics + biased map, solve = the DP,
 * remove = removal + 2-column fix-up) and an orientation: 0 = remove_object
 * (auto, by mask_bounds), 1 = detail::remove_object_vertical (carver.hpp:289-321;
 * an empty mask carves nothing instead of failing). The loop length is
 * data-dependent, yet there is no host round trip per seam: the stop test is a
 * device flag every kernel of the loop checks; the host reads it once per batch
 * of iterations. */
carve_status carve_cuda_remove_object_ex(const uint8_t* rgb, int w, int h, const uint8_t* mask,
                                         const carve_cuda_config* cfg, int restore, int orientation,
                                         uint8_t* rgb_out, int* out_w, int* out_h, int32_t* seams_out, int* nseams,
                                         carve_seam_timing* timings_out);

/* ---- seam recording and enlargement (carver.hpp:114-140, 226-285; cli.hpp:262-277, 301-309) */
/* replaces insert_seam (carver.hpp:137-140: validate_seam + detail::insert_columns
 * :117-130); out is (w+1)*h*3 bytes */
carve_status carve_cuda_insert_seam_rgb(const uint8_t* rgb, int w, int h, const int32_t* seam, int n,
                                        uint8_t* out);
/* replaces detail::insert_columns (carver.hpp:118-132): as insert_seam but
 * without the connectivity check (replayed recorded seams may jump); columns
 * must lie in [0, w) (CARVE_E_INVALID_SEAM otherwise) */
carve_status carve_cuda_insert_columns_rgb(const uint8_t* rgb, int w, int h, const int32_t* cols, int n,
                                           uint8_t* out);
/* replaces record_seams (carver.hpp:226-262) with the default CarveConfig:
 * seams_out receives count*h ints, seam t's column of row i at [t*h + i], in
 * original-image coordinates. timings_out (nullable): count entries. */
carve_status carve_cuda_record_seams(const uint8_t* rgb, int w, int h, int count, const carve_cuda_config* cfg,
                                     int32_t* seams_out, carve_seam_timing* timings_out);
/* replaces run_enlarge (cli.hpp:262-277): enlarge_to_width(target_w)
 * (carver.hpp:266-285) if target_w != w, then enlarge_to_width of the
 * transpose to target_h if target_h != h. rgb_out: target_w*target_h*3 bytes.
 * seams_out (nullable): (target_w-w)*h + (target_h-h)*target_w ints — each
 * phase's recorded seams (its CarveReport.seams), concatenated. */
carve_status carve_cuda_enlarge(const uint8_t* rgb, int w, int h, int target_w, int target_h,
                                const carve_cuda_config* cfg, uint8_t* rgb_out, int32_t* seams_out);
/* carve_cuda_enlarge plus each recording's per-seam timings (the CarveReport
 * per_seam of record_seams, carver.hpp:226-262): timings_out (nullable) receives
 * (target_w-w) + (target_h-h) entries, width phase first. */
carve_status carve_cuda_enlarge_timed(const uint8_t* rgb, int w, int h, int target_w, int target_h,
                                      const carve_cuda_config* cfg, uint8_t* rgb_out, int32_t* seams_out,
                                      carve_seam_timing* timings_out);

/* ---- pipelines (carver.hpp:71-82, 191-222; cli.hpp:242-259) ----------- */
/* replaces remove_seam(PixelGrid) (carver.hpp:71-82); out is (w-1)*h*3 bytes */
carve_status carve_cuda_remove_seam_rgb(const uint8_t* rgb, int w, int h, const int32_t* seam, int n,
                                        uint8_t* out);
/* replace remove_seam(LumaGrid) / remove_seam(EnergyMap) (f64) and
 * remove_seam(RemovalMask) (u8) = detail::drop_columns (carver.hpp:57-67,
 * 84-112): the w*h plane minus column seam[i] of row i, out is (w-1)*h values.
 * Like the reference these do not require a connected seam; n must equal h and
 * every column must lie in [0, w) (CARVE_E_INVALID_SEAM otherwise). */
carve_status carve_cuda_remove_seam_f64(const double* in, int w, int h, const int32_t* seam, int n, double* out);
carve_status carve_cuda_remove_seam_u8(const uint8_t* in, int w, int h, const int32_t* seam, int n, uint8_t* out);
/* replaces run_resize's carving (cli.hpp:249-256): carve_to_width(target_w)
 * then, if target_h != h, carve_to_height(target_h) (carver.hpp:191-222).
 * rgb_out: target_w*target_h*3 bytes.
 * seams_out (nullable): (w-target_w)*h + (h-target_h)*target_w ints — every
 *   seam in removal order, as CarveReport.seams holds them (carver.hpp:31).
 * timings_out (nullable): (w-target_w)+(h-target_h) entries.
 * The whole loop runs on the device; no host round trip per seam. */
/* carve_cuda_carve with a CarveConfig (forward energy, recompute) */
carve_status carve_cuda_carve_cfg(const uint8_t* rgb, int w, int h, int target_w, int target_h,
                                  const carve_cuda_config* cfg, uint8_t* rgb_out, int32_t* seams_out,
                                  carve_seam_timing* timings_out);
carve_status carve_cuda_carve(const uint8_t* rgb, int w, int h, int target_w, int target_h, uint8_t* rgb_out,
                              int32_t* seams_out, carve_seam_timing* timings_out);

/* Batch of n same-size images carved to target_w x target_h across `ndev`
 * devices (devices == NULL: 0..ndev-1; ndev <= 0: all; a device may be listed
 * more than once). One host thread per listed device claims chunks of whole
 * images from a shared atomic counter (SURVEY.md §8e work queue) and runs P
 * copy/compute pipelines on them: chunk uploads, carves and downloads overlap.
 * No inter-device communication. */
carve_status carve_cuda_carve_batch(const uint8_t* const* rgb, int n, int w, int h, int target_w, int target_h,
                                    uint8_t* const* rgb_out, const int* devices, int ndev);
/* The host pipeline shape carve_cuda_carve_batch uses for n images over ndev
 * devices: pipelines per device and images per chunk (pure host logic; honours
 * CARVE_PIPELINES / CARVE_PIPE_CHUNK). */
carve_status carve_cuda_batch_plan(int n, int w, int h, int target_w, int target_h, int ndev, int* pipes,
                                   int* chunk);

/* ---- device-resident entry points (inputs already in HBM) --------------
 * d_rgb / d_out are device pointers to packed RGB on the current device;
 * `stream` is a cudaStream_t (NULL = the legacy default stream). These
 * enqueue work and return without synchronizing (the bench times them with
 * CUDA events on `stream`). The work runs on library-owned streams forked
 * from `stream` by an event and joined back into it, so the library's scratch
 * is always ordered on one stream: later calls of this thread (synchronous or
 * asynchronous, on any stream) wait for it. d_seams (nullable) receives seams
 * as above. */
carve_status carve_cuda_carve_device(const uint8_t* d_rgb, int w, int h, int target_w, int target_h,
                                     uint8_t* d_out, int32_t* d_seams, void* stream);
carve_status carve_cuda_carve_batch_device(const uint8_t* d_rgb, int n, int w, int h, int target_w, int target_h,
                                           uint8_t* d_out, void* stream);

/* ---- bench fixture (bench.hpp:67-94) ------------------------------------ */
/* make_test_image byte for byte; variant k > 0 xors k into the seed (the
 * C5 batch extension). Host-side generator. */
carve_status carve_make_test_image(int w, int h, uint32_t variant, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif /* CARVE_CUDA_H */
