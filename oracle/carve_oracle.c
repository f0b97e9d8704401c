/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into the product;
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * A plain-C restatement of the reference hot path (seam carving with e1
 * energy and the dynamic-programming solver), following the reference
 * arithmetic operation for operation so results are FP64-bit-identical.
 * Built by oracle/Makefile with gcc -O2 -ffp-contract=off and no -march
 * (FMA contraction changes luma bits).
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * the reference itself compiled from /root/reference (oracle/_ref, built by
 * oracle/Makefile from ref_shim.cpp) and against the committed golden
 * vectors in tests/golden/ generated from that build.
 *
 * Status codes: 0 ok, 1 + Errc (error.hpp:8-26) on a reference error.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* error.hpp:8-26 ordinal + 1 */
enum {
    OR_OK = 0,
    OR_DIMENSION_MISMATCH = 1 + 4,
    OR_INVALID_SEAM = 1 + 5,
    OR_EMPTY_IMAGE = 1 + 7,
    OR_WIDTH_TOO_SMALL = 1 + 8,
    OR_INVALID_TARGET = 1 + 9,
    OR_TARGET_TOO_LARGE = 1 + 10,
    OR_EMPTY_MASK = 1 + 11,
    OR_NO_MEMORY = 100,
};

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* bench.hpp:67-94 make_test_image; `variant` k > 0 XORs k into the xorshift
 * seed (the documented C5 batch extension); k = 0 is the
 * reference fixture byte for byte. */
int or_make_test_image(int w, int h, uint32_t variant, uint8_t* out) {
    if (w < 1 || h < 1) return OR_EMPTY_IMAGE;
    uint32_t s = 0x9E3779B9u ^ ((uint32_t)w * 2654435761u) ^ (uint32_t)h;
    if (variant) {
        s ^= variant;
        if (!s) s = 1u;
    }
    const double pi = 3.14159265358979323846;
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) {
            const double u = (double)i / (double)(h - 1 > 1 ? h - 1 : 1);
            const double v = (double)j / (double)(w - 1 > 1 ? w - 1 : 1);
            double base = 60.0 + 70.0 * (u + v) / 2.0 + 45.0 * sin(3.0 * pi * u) * cos(3.0 * pi * v);
            if (u > 0.33 && u < 0.66 && v > 0.25 && v < 0.75) base += (((i / 3) + (j / 3)) % 2) ? 55.0 : -55.0;
            int n[3];
            for (int c = 0; c < 3; ++c) {
                s ^= s << 13;
                s ^= s >> 17;
                s ^= s << 5;
                n[c] = (int)(s % 37u) - 18;
            }
            uint8_t* p = out + ((size_t)i * w + j) * 3;
            p[0] = (uint8_t)clampd(base + n[0], 0.0, 255.0);
            p[1] = (uint8_t)clampd(base * 0.85 + 24.0 + n[1], 8.0, 255.0);
            p[2] = (uint8_t)clampd(210.0 - base * 0.55 + n[2], 0.0, 255.0);
        }
    return OR_OK;
}

/* raster.hpp:61-71 — BT.601 luma, evaluated left to right, no FMA. */
static double luma_of(const uint8_t* p) { return 0.299 * p[0] + 0.587 * p[1] + 0.114 * p[2]; }

int or_to_grayscale(const uint8_t* rgb, int w, int h, double* out) {
    for (size_t k = 0; k < (size_t)w * h; ++k) out[k] = luma_of(rgb + 3 * k);
    return OR_OK;
}

/* energy.hpp:82-98 — clamped central differences (raster.hpp:54-58), no /2,
 * e = |gx| + |gy| with the x term first. */
int or_energy_e1_luma(const double* g, int w, int h, double* out) {
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) {
            const double gx = g[(size_t)i * w + clampi(j + 1, 0, w - 1)] - g[(size_t)i * w + clampi(j - 1, 0, w - 1)];
            const double gy = g[(size_t)clampi(i + 1, 0, h - 1) * w + j] - g[(size_t)clampi(i - 1, 0, h - 1) * w + j];
            out[(size_t)i * w + j] = fabs(gx) + fabs(gy);
        }
    return OR_OK;
}

int or_energy_e1_rgb(const uint8_t* rgb, int w, int h, double* out) {
    double* l = (double*)malloc(sizeof(double) * (size_t)w * h);
    if (!l) return OR_NO_MEMORY;
    or_to_grayscale(rgb, w, h, l);
    or_energy_e1_luma(l, w, h, out);
    free(l);
    return OR_OK;
}

/* solvers.hpp:263-289 dp_seam + :94-111 argmin_row/backtrack.
 * Candidates k in [max(0,j-1), min(w-1,j+1)] scanned upward with strict <,
 * so the smallest column wins ties; argmin is the first index of the min.
 * m/b may be NULL (then scratch tables are used). */
int or_dp_seam(const double* e, int w, int h, double* m_out, int* b_out, int* seam) {
    if (w < 1 || h < 1) return OR_EMPTY_IMAGE;
    double* m = m_out ? m_out : (double*)malloc(sizeof(double) * (size_t)w * h);
    int* b = b_out ? b_out : (int*)malloc(sizeof(int) * (size_t)w * h);
    if (!m || !b) return OR_NO_MEMORY;
    for (int j = 0; j < w; ++j) {
        m[j] = e[j];
        b[j] = j;
    }
    for (int i = 1; i < h; ++i) {
        const double* prev = m + (size_t)(i - 1) * w;
        for (int j = 0; j < w; ++j) {
            int from = -1;
            double best = INFINITY;
            const int lo = j - 1 < 0 ? 0 : j - 1, hi = j + 1 > w - 1 ? w - 1 : j + 1;
            for (int k = lo; k <= hi; ++k)
                if (prev[k] < best) {
                    best = prev[k];
                    from = k;
                }
            m[(size_t)i * w + j] = e[(size_t)i * w + j] + best;
            b[(size_t)i * w + j] = from;
        }
    }
    const double* last = m + (size_t)(h - 1) * w;
    int col = 0;
    for (int j = 1; j < w; ++j)
        if (last[j] < last[col]) col = j;
    seam[h - 1] = col;
    for (int i = h - 1; i >= 1; --i) {
        col = b[(size_t)i * w + col];
        seam[i - 1] = col;
    }
    if (!m_out) free(m);
    if (!b_out) free(b);
    return OR_OK;
}

/* solvers.hpp:69-78 */
int or_validate_seam(const int* seam, int n, int w, int h) {
    if (n != h) return OR_INVALID_SEAM;
    for (int i = 0; i < n; ++i) {
        if (seam[i] < 0 || seam[i] >= w) return OR_INVALID_SEAM;
        if (i > 0 && abs(seam[i] - seam[i - 1]) > 1) return OR_INVALID_SEAM;
    }
    return OR_OK;
}

/* carver.hpp:71-82 — out[i][j] = in[i][j < s[i] ? j : j + 1]. */
int or_remove_seam(const uint8_t* in, int w, int h, const int* seam, int n, uint8_t* out) {
    int st = or_validate_seam(seam, n, w, h);
    if (st) return st;
    if (w < 2) return OR_WIDTH_TOO_SMALL;
    for (int i = 0; i < h; ++i) {
        const uint8_t* src = in + (size_t)i * w * 3;
        uint8_t* dst = out + (size_t)i * (w - 1) * 3;
        memcpy(dst, src, (size_t)seam[i] * 3);
        memcpy(dst + (size_t)seam[i] * 3, src + (size_t)(seam[i] + 1) * 3, (size_t)(w - seam[i] - 1) * 3);
    }
    return OR_OK;
}

/* raster.hpp:73-79 */
int or_transpose(const uint8_t* in, int w, int h, uint8_t* out) {
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) memcpy(out + ((size_t)j * h + i) * 3, in + ((size_t)i * w + j) * 3, 3);
    return OR_OK;
}

/* carver.hpp:191-214 carve_to_width with the default config (recompute=true,
 * e1, dp): every seam recomputes luma+energy on the current grid, solves,
 * removes. `work` holds the current grid in place. */
static int carve_width_inplace(uint8_t* work, int w, int h, int target_w, int** seams_cursor) {
    double* e = (double*)malloc(sizeof(double) * (size_t)w * h);
    uint8_t* tmp = (uint8_t*)malloc((size_t)w * h * 3);
    int* seam = (int*)malloc(sizeof(int) * (size_t)h);
    if (!e || !tmp || !seam) return OR_NO_MEMORY;
    for (int cw = w; cw > target_w; --cw) {
        or_energy_e1_rgb(work, cw, h, e);
        or_dp_seam(e, cw, h, NULL, NULL, seam);
        or_remove_seam(work, cw, h, seam, h, tmp);
        memcpy(work, tmp, (size_t)(cw - 1) * h * 3);
        if (seams_cursor && *seams_cursor) {
            memcpy(*seams_cursor, seam, sizeof(int) * (size_t)h);
            *seams_cursor += h;
        }
    }
    free(e);
    free(tmp);
    free(seam);
    return OR_OK;
}

/* run_resize (cli.hpp:242-259): width phase, then carve_to_height
 * (carver.hpp:216-222) as transpose ∘ carve_to_width ∘ transpose. */
int or_carve(const uint8_t* rgb, int w, int h, int target_w, int target_h, uint8_t* out, int* seams_out) {
    if (w < 1 || h < 1) return OR_EMPTY_IMAGE;
    if (target_w < 1 || target_w > w) return OR_INVALID_TARGET;
    if (target_h < 1 || target_h > h) return OR_INVALID_TARGET;
    uint8_t* work = (uint8_t*)malloc((size_t)w * h * 3);
    if (!work) return OR_NO_MEMORY;
    memcpy(work, rgb, (size_t)w * h * 3);
    int* cursor = seams_out;
    int st = carve_width_inplace(work, w, h, target_w, &cursor);
    int cw = target_w;
    if (!st && target_h != h) {
        uint8_t* t = (uint8_t*)malloc((size_t)cw * h * 3);
        if (!t) return OR_NO_MEMORY;
        or_transpose(work, cw, h, t);
        st = carve_width_inplace(t, h, cw, target_h, &cursor);
        or_transpose(t, target_h, cw, work);
        free(t);
    }
    if (!st) memcpy(out, work, (size_t)cw * target_h * 3);
    free(work);
    return st;
}

/* energy.hpp:196-216 forward_costs: at_clamped neighbours, cu = |right - left|,
 * cl = cu + |above - left|, cr = cu + |above - right|. */
int or_forward_costs(const double* g, int w, int h, double* left, double* up, double* right) {
    if (w < 1 || h < 1) return OR_EMPTY_IMAGE;
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) {
            const double l = g[(size_t)i * w + clampi(j - 1, 0, w - 1)];
            const double r = g[(size_t)i * w + clampi(j + 1, 0, w - 1)];
            const double a = g[(size_t)clampi(i - 1, 0, h - 1) * w + j];
            const size_t idx = (size_t)i * w + j;
            const double cu = fabs(r - l);
            up[idx] = cu;
            left[idx] = cu + fabs(a - l);
            right[idx] = cu + fabs(a - r);
        }
    return OR_OK;
}

/* solvers.hpp:294-326 dp_seam_forward(gray, costs) for arbitrary costs (gray
 * only supplies the dimensions): candidates prev + transition cost in the
 * order left, up, right, strict <, best starting at +inf. m/b nullable. */
int or_dp_seam_forward_costs(const double* cl, const double* cu, const double* cr, int w, int h, double* m_out,
                             int* b_out, int* seam) {
    if (w < 1 || h < 1) return OR_EMPTY_IMAGE;
    const size_t n = (size_t)w * h;
    double* m = m_out ? m_out : (double*)malloc(n * 8);
    int* b = b_out ? b_out : (int*)malloc(n * 4);
    if (!m || !b) return OR_NO_MEMORY;
    for (int j = 0; j < w; ++j) {
        m[j] = cu[j];
        b[j] = j;
    }
    for (int i = 1; i < h; ++i) {
        const double* prev = m + (size_t)(i - 1) * w;
        for (int j = 0; j < w; ++j) {
            const size_t idx = (size_t)i * w + j;
            int from = -1;
            double best = INFINITY;
            if (j > 0 && prev[j - 1] + cl[idx] < best) {
                best = prev[j - 1] + cl[idx];
                from = j - 1;
            }
            if (prev[j] + cu[idx] < best) {
                best = prev[j] + cu[idx];
                from = j;
            }
            if (j < w - 1 && prev[j + 1] + cr[idx] < best) {
                best = prev[j + 1] + cr[idx];
                from = j + 1;
            }
            m[idx] = best;
            b[idx] = from;
        }
    }
    /* solvers.hpp:94-111 argmin (first index) + backtrack */
    const double* last = m + (size_t)(h - 1) * w;
    int c = 0;
    for (int j = 1; j < w; ++j)
        if (last[j] < last[c]) c = j;
    seam[h - 1] = c;
    for (int i = h - 1; i > 0; --i) seam[i - 1] = b[(size_t)i * w + seam[i]];
    if (!m_out) free(m);
    if (!b_out) free(b);
    return OR_OK;
}

/* solvers.hpp:294-326 dp_seam_forward(g, forward_costs(g)) */
int or_dp_seam_forward(const double* g, int w, int h, double* m_out, int* b_out, int* seam) {
    if (w < 1 || h < 1) return OR_EMPTY_IMAGE;
    const size_t n = (size_t)w * h;
    double* cl = (double*)malloc(n * 8);
    double* cu = (double*)malloc(n * 8);
    double* cr = (double*)malloc(n * 8);
    if (!cl || !cu || !cr) return OR_NO_MEMORY;
    or_forward_costs(g, w, h, cl, cu, cr);
    const int st = or_dp_seam_forward_costs(cl, cu, cr, w, h, m_out, b_out, seam);
    free(cl);
    free(cu);
    free(cr);
    return st;
}

/* carver.hpp:57-67 detail::drop_columns, the body of remove_seam(LumaGrid /
 * EnergyMap) (:84-98) and of remove_seam(RemovalMask) (:100-112): row i loses
 * column seam[i]; no connectivity requirement (the reference does not
 * validate these overloads). elem = 8 (doubles) or 1 (mask bytes). */
int or_drop_columns(const void* in, int w, int h, const int* seam, int n, int elem, void* out) {
    if (n != h) return OR_INVALID_SEAM;
    for (int i = 0; i < h; ++i) {
        if (seam[i] < 0 || seam[i] >= w) return OR_INVALID_SEAM;
        const uint8_t* src = (const uint8_t*)in + (size_t)i * w * elem;
        uint8_t* dst = (uint8_t*)out + (size_t)i * (w - 1) * elem;
        memcpy(dst, src, (size_t)seam[i] * elem);
        memcpy(dst + (size_t)seam[i] * elem, src + (size_t)(seam[i] + 1) * elem, (size_t)(w - seam[i] - 1) * elem);
    }
    return OR_OK;
}

/* carver.hpp:191-214 carve_to_width with CarveConfig::forward / ::recompute
 * (solve_step :153-173, carve_cached_state :176-188): forward solves
 * dp_seam_forward on the current image's luma (recompute=true); recompute=false
 * (backward) computes e1 once and then carves the map alongside the image. */
static int carve_width_cfg(uint8_t* work, int w, int h, int target_w, int forward, int recompute,
                           int** seams_cursor) {
    double* e = (double*)malloc(sizeof(double) * (size_t)w * h);
    double* e2 = (double*)malloc(sizeof(double) * (size_t)w * h);
    uint8_t* tmp = (uint8_t*)malloc((size_t)w * h * 3);
    int* seam = (int*)malloc(sizeof(int) * (size_t)h);
    /* forward + recompute=false: the cached ForwardCosts (carver.hpp:157-160, 177-183) */
    double* fc[3] = {NULL, NULL, NULL};
    if (!e || !e2 || !tmp || !seam) return OR_NO_MEMORY;
    if (!recompute && !forward) or_energy_e1_rgb(work, w, h, e);
    if (!recompute && forward) {
        for (int k = 0; k < 3; ++k)
            if (!(fc[k] = (double*)malloc(sizeof(double) * (size_t)w * h))) return OR_NO_MEMORY;
        or_to_grayscale(work, w, h, e);
        or_forward_costs(e, w, h, fc[0], fc[1], fc[2]);
    }
    for (int cw = w; cw > target_w; --cw) {
        if (forward && !recompute) {
            or_dp_seam_forward_costs(fc[0], fc[1], fc[2], cw, h, NULL, NULL, seam);
            for (int k = 0; k < 3; ++k) { /* drop_columns on each cost plane (carver.hpp:179-181) */
                or_drop_columns(fc[k], cw, h, seam, h, 8, e2);
                memcpy(fc[k], e2, sizeof(double) * (size_t)(cw - 1) * h);
            }
        } else if (forward) {
            or_to_grayscale(work, cw, h, e);
            or_dp_seam_forward(e, cw, h, NULL, NULL, seam);
        } else {
            if (recompute) or_energy_e1_rgb(work, cw, h, e);
            or_dp_seam(e, cw, h, NULL, NULL, seam);
        }
        or_remove_seam(work, cw, h, seam, h, tmp);
        memcpy(work, tmp, (size_t)(cw - 1) * h * 3);
        if (!recompute && !forward) { /* drop_columns (carver.hpp:57-67) on the cached map */
            for (int i = 0; i < h; ++i) {
                const double* src = e + (size_t)i * cw;
                double* dst = e2 + (size_t)i * (cw - 1);
                memcpy(dst, src, sizeof(double) * (size_t)seam[i]);
                memcpy(dst + seam[i], src + seam[i] + 1, sizeof(double) * (size_t)(cw - seam[i] - 1));
            }
            memcpy(e, e2, sizeof(double) * (size_t)(cw - 1) * h);
        }
        if (seams_cursor && *seams_cursor) {
            memcpy(*seams_cursor, seam, sizeof(int) * (size_t)h);
            *seams_cursor += h;
        }
    }
    free(e);
    free(e2);
    free(tmp);
    free(seam);
    for (int k = 0; k < 3; ++k) free(fc[k]);
    return OR_OK;
}

/* run_resize (cli.hpp:242-259) with a CarveConfig (forward, recompute) */
int or_carve_cfg(const uint8_t* rgb, int w, int h, int target_w, int target_h, int forward, int recompute,
                 uint8_t* out, int* seams_out) {
    if (w < 1 || h < 1) return OR_EMPTY_IMAGE;
    if (target_w < 1 || target_w > w) return OR_INVALID_TARGET;
    if (target_h < 1 || target_h > h) return OR_INVALID_TARGET;
    uint8_t* work = (uint8_t*)malloc((size_t)w * h * 3);
    if (!work) return OR_NO_MEMORY;
    memcpy(work, rgb, (size_t)w * h * 3);
    int* cursor = seams_out;
    int st = carve_width_cfg(work, w, h, target_w, forward, recompute, &cursor);
    const int cw = target_w;
    if (!st && target_h != h) {
        uint8_t* t = (uint8_t*)malloc((size_t)cw * h * 3);
        if (!t) return OR_NO_MEMORY;
        or_transpose(work, cw, h, t);
        st = carve_width_cfg(t, h, cw, target_h, forward, recompute, &cursor);
        or_transpose(t, target_h, cw, work);
        free(t);
    }
    if (!st) memcpy(out, work, (size_t)cw * target_h * 3);
    free(work);
    return st;
}

/* energy.hpp:220-241 apply_mask: masked cells become -k, k = 1000*(h*m + 1),
 * m = max over unmasked cells (over all cells when every cell is masked). */
int or_apply_mask(const double* e, int w, int h, const uint8_t* mask, double* out) {
    double max_unmasked = 0.0, max_all = 0.0;
    int any_unmasked = 0;
    const size_t n = (size_t)w * h;
    for (size_t i = 0; i < n; ++i) {
        if (e[i] > max_all) max_all = e[i];
        if (!mask[i]) {
            if (e[i] > max_unmasked) max_unmasked = e[i];
            any_unmasked = 1;
        }
    }
    const double m = any_unmasked ? max_unmasked : max_all;
    const double k = 1000.0 * ((double)h * m + 1.0);
    for (size_t i = 0; i < n; ++i) out[i] = mask[i] ? -k : e[i];
    return OR_OK;
}

/* energy.hpp:244-253 mask_from_image: luma >= 128 marks a pixel */
int or_mask_from_image(const uint8_t* rgb, int w, int h, uint8_t* flags) {
    for (size_t i = 0; i < (size_t)w * h; ++i) flags[i] = luma_of(rgb + 3 * i) >= 128.0 ? 1 : 0;
    return OR_OK;
}

static void transpose_u8(const uint8_t* in, int w, int h, uint8_t* out) {
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) out[(size_t)j * h + i] = in[(size_t)i * w + j];
}

static int enlarge_width(const uint8_t* in, int w, int h, int target_w, int forward, uint8_t* out,
                         int** seams_cursor);

/* carver.hpp:287-315 remove_object_vertical: per seam e1 of the current image,
 * apply_mask with the remaining mask, dp seam, remove from image and mask; until
 * no marked cell remains. Then (restore) enlarge_to_width back to w. `forward`
 * only affects the restoring enlargement (record_seams with cfg). */
static int remove_object_vertical(uint8_t* work, int w, int h, uint8_t* mask, int forward, int restore, int* out_w,
                                  int* seams_out, int* nseams, uint8_t* out) {
    double* e = (double*)malloc((size_t)w * h * 8);
    double* eb = (double*)malloc((size_t)w * h * 8);
    uint8_t* tmp = (uint8_t*)malloc((size_t)w * h * 3);
    uint8_t* mtmp = (uint8_t*)malloc((size_t)w * h);
    int* seam = (int*)malloc(sizeof(int) * (size_t)h);
    if (!e || !eb || !tmp || !mtmp || !seam) return OR_NO_MEMORY;
    int cw = w, ns = 0, st = OR_OK;
    for (;;) {
        size_t marked = 0;
        for (size_t i = 0; i < (size_t)cw * h; ++i) marked += mask[i] != 0;
        if (!marked) break;
        if (cw < 2) { st = OR_WIDTH_TOO_SMALL; break; }
        or_energy_e1_rgb(work, cw, h, e);
        or_apply_mask(e, cw, h, mask, eb);
        or_dp_seam(eb, cw, h, NULL, NULL, seam);
        or_remove_seam(work, cw, h, seam, h, tmp);
        memcpy(work, tmp, (size_t)(cw - 1) * h * 3);
        for (int i = 0; i < h; ++i) { /* remove_seam(RemovalMask) carver.hpp:100-112 */
            const uint8_t* src = mask + (size_t)i * cw;
            uint8_t* dst = mtmp + (size_t)i * (cw - 1);
            memcpy(dst, src, (size_t)seam[i]);
            memcpy(dst + seam[i], src + seam[i] + 1, (size_t)(cw - seam[i] - 1));
        }
        memcpy(mask, mtmp, (size_t)(cw - 1) * h);
        memcpy(seams_out + (size_t)ns * h, seam, sizeof(int) * (size_t)h);
        ++ns;
        --cw;
    }
    *nseams = ns;
    if (!st) {
        if (restore && cw < w) {
            int* none = NULL;
            st = enlarge_width(work, cw, h, w, forward, out, &none);
            *out_w = w;
        } else {
            memcpy(out, work, (size_t)cw * h * 3);
            *out_w = cw;
        }
    }
    free(e);
    free(eb);
    free(tmp);
    free(mtmp);
    free(seam);
    return st;
}

/* carver.hpp:327-340 remove_object. out: w*h*3 bytes; out_dims {w, h};
 * seams_out: w*h ints (the report's seams, concatenated); nseams. */
int or_remove_object(const uint8_t* rgb, int w, int h, const uint8_t* mask_in, int forward, int restore, uint8_t* out,
                     int* out_dims, int* seams_out, int* nseams) {
    int top = h, left = w, bottom = -1, right = -1;
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j)
            if (mask_in[(size_t)i * w + j]) {
                if (i < top) top = i;
                if (j < left) left = j;
                if (i > bottom) bottom = i;
                if (j > right) right = j;
            }
    if (bottom < top) return OR_EMPTY_MASK;
    uint8_t* work = (uint8_t*)malloc((size_t)w * h * 3);
    uint8_t* mask = (uint8_t*)malloc((size_t)w * h);
    if (!work || !mask) return OR_NO_MEMORY;
    int st, ow;
    if (right - left + 1 <= bottom - top + 1) {
        memcpy(work, rgb, (size_t)w * h * 3);
        memcpy(mask, mask_in, (size_t)w * h);
        st = remove_object_vertical(work, w, h, mask, forward, restore, &ow, seams_out, nseams, out);
        out_dims[0] = ow;
        out_dims[1] = h;
    } else {
        uint8_t* res = (uint8_t*)malloc((size_t)w * h * 3);
        if (!res) return OR_NO_MEMORY;
        or_transpose(rgb, w, h, work);
        transpose_u8(mask_in, w, h, mask);
        st = remove_object_vertical(work, h, w, mask, forward, restore, &ow, seams_out, nseams, res);
        if (!st) or_transpose(res, ow, w, out);
        out_dims[0] = w;
        out_dims[1] = ow;
        free(res);
    }
    free(work);
    free(mask);
    return st;
}

/* carver.hpp:117-130 detail::insert_columns: one pixel per row right of
 * column cols[i] (stride `cs` between rows' entries), the channel-wise rounded
 * mean of its left and right neighbours, the right one clamped at the border. */
static void insert_columns(const uint8_t* in, int w, int h, const int* cols, size_t cs, uint8_t* out) {
    for (int i = 0; i < h; ++i) {
        const int c = cols[(size_t)i * cs];
        const uint8_t* src = in + (size_t)i * w * 3;
        uint8_t* dst = out + (size_t)i * (w + 1) * 3;
        memcpy(dst, src, (size_t)(c + 1) * 3);
        const uint8_t* a = src + (size_t)c * 3;
        const uint8_t* b = src + (size_t)(c + 1 < w ? c + 1 : w - 1) * 3;
        for (int ch = 0; ch < 3; ++ch) dst[(size_t)(c + 1) * 3 + ch] = (uint8_t)((a[ch] + b[ch] + 1) / 2);
        memcpy(dst + (size_t)(c + 2) * 3, src + (size_t)(c + 1) * 3, (size_t)(w - c - 1) * 3);
    }
}

/* carver.hpp:137-140 insert_seam */
int or_insert_seam(const uint8_t* in, int w, int h, const int* seam, int n, uint8_t* out) {
    int st = or_validate_seam(seam, n, w, h);
    if (st) return st;
    insert_columns(in, w, h, seam, 1, out);
    return OR_OK;
}

/* carver.hpp:226-262 record_seams (default config): the removal loop on a
 * scratch copy, each seam mapped to original coordinates through per-row
 * survivor lists (survivor[i][seam[i]], then erase). seams_out: count*h ints. */
static int carve_width_cfg(uint8_t* work, int w, int h, int target_w, int forward, int recompute,
                           int** seams_cursor);

static int record_seams_cfg(const uint8_t* rgb, int w, int h, int count, int forward, int* seams_out);

int or_record_seams(const uint8_t* rgb, int w, int h, int count, int* seams_out) {
    return record_seams_cfg(rgb, w, h, count, 0, seams_out);
}

static int record_seams_cfg(const uint8_t* rgb, int w, int h, int count, int forward, int* seams_out) {
    if (w < 1 || h < 1) return OR_EMPTY_IMAGE;
    if (count < 0 || count > w - 1) return OR_INVALID_TARGET;
    uint8_t* work = (uint8_t*)malloc((size_t)w * h * 3);
    int* cur = (int*)malloc(sizeof(int) * ((size_t)count * h + 1));
    int* surv = (int*)malloc(sizeof(int) * (size_t)w * h);
    if (!work || !cur || !surv) return OR_NO_MEMORY;
    memcpy(work, rgb, (size_t)w * h * 3);
    int* cursor = cur;
    int st = carve_width_cfg(work, w, h, w - count, forward, 1, &cursor);
    for (int i = 0; i < h && !st; ++i) {
        int* row = surv + (size_t)i * w;
        int len = w;
        for (int j = 0; j < w; ++j) row[j] = j;
        for (int t = 0; t < count; ++t) {
            const int c = cur[(size_t)t * h + i];
            seams_out[(size_t)t * h + i] = row[c];
            memmove(row + c, row + c + 1, sizeof(int) * (size_t)(len - c - 1));
            --len;
        }
    }
    free(work);
    free(cur);
    free(surv);
    return st;
}

/* carver.hpp:266-285 enlarge_to_width: record k seams, then replay them
 * oldest-first through insert_columns, shifting every later recorded column
 * right by one where it lands at-or-right-of the inserted column. `seams_out`
 * (nullable) receives the recorded (unshifted) seams. */
static int enlarge_width(const uint8_t* in, int w, int h, int target_w, int forward, uint8_t* out,
                         int** seams_cursor) {
    const int k = target_w - w;
    if (k < 0) return OR_INVALID_TARGET;
    if (target_w > 2 * w - 1) return OR_TARGET_TOO_LARGE;
    int* seams = (int*)malloc(sizeof(int) * ((size_t)k * h + 1));
    uint8_t* a = (uint8_t*)malloc((size_t)target_w * h * 3);
    uint8_t* b = (uint8_t*)malloc((size_t)target_w * h * 3);
    if (!seams || !a || !b) return OR_NO_MEMORY;
    int st = record_seams_cfg(in, w, h, k, forward, seams);
    if (!st && seams_cursor && *seams_cursor) {
        memcpy(*seams_cursor, seams, sizeof(int) * (size_t)k * h);
        *seams_cursor += (size_t)k * h;
    }
    memcpy(a, in, (size_t)w * h * 3);
    for (int t = 0; t < k && !st; ++t) {
        insert_columns(a, w + t, h, seams + (size_t)t * h, 1, b);
        memcpy(a, b, (size_t)(w + t + 1) * h * 3);
        for (int u = t + 1; u < k; ++u)
            for (int i = 0; i < h; ++i)
                if (seams[(size_t)u * h + i] >= seams[(size_t)t * h + i]) ++seams[(size_t)u * h + i];
    }
    if (!st) memcpy(out, a, (size_t)target_w * h * 3);
    free(seams);
    free(a);
    free(b);
    return st;
}

/* run_enlarge (cli.hpp:262-277): enlarge_to_width on the width, then on the
 * transpose for the height. */
int or_enlarge(const uint8_t* rgb, int w, int h, int target_w, int target_h, uint8_t* out, int* seams_out) {
    if (w < 1 || h < 1) return OR_EMPTY_IMAGE;
    int* cursor = seams_out;
    int cw = w, st = OR_OK;
    uint8_t* work = (uint8_t*)malloc((size_t)(target_w > w ? target_w : w) * h * 3);
    if (!work) return OR_NO_MEMORY;
    if (target_w != w) {
        st = enlarge_width(rgb, w, h, target_w, 0, work, &cursor);
        cw = target_w;
    } else {
        memcpy(work, rgb, (size_t)w * h * 3);
    }
    if (!st && target_h != h) {
        const size_t big = (size_t)cw * (target_h > h ? target_h : h) * 3;
        uint8_t* t = (uint8_t*)malloc(big);
        uint8_t* t2 = (uint8_t*)malloc(big);
        if (!t || !t2) return OR_NO_MEMORY;
        or_transpose(work, cw, h, t);
        st = enlarge_width(t, h, cw, target_h, 0, t2, &cursor);
        if (!st) {
            free(work);
            work = (uint8_t*)malloc(big);
            if (!work) return OR_NO_MEMORY;
            or_transpose(t2, target_h, cw, work);
        }
        free(t);
        free(t2);
    }
    if (!st) memcpy(out, work, (size_t)cw * target_h * 3);
    free(work);
    return st;
}

/* FNV-1a-64 of a byte buffer (the survey's output-hash convention). */
uint64_t or_fnv1a64(const uint8_t* p, size_t n) {
    uint64_t hsh = 0xcbf29ce484222325ull;
    for (size_t k = 0; k < n; ++k) {
        hsh ^= p[k];
        hsh *= 0x100000001b3ull;
    }
    return hsh;
}
