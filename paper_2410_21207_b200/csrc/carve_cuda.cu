// carve_cuda.cu — host side of libcarve_cuda.so: per-thread device contexts,
// the device-resident carve driver, and the extern "C" boundary declared in
// include/carve_cuda.h. No CPU compute path exists: every compute entry point
// runs the sm_100a kernels in carve_kernels.cuh or returns CARVE_E_CUDA.
#include "carve_cuda.h"
#include "carve_kernels.cuh"
#include "dp_cluster.cuh"
#include "dp_variants.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>  // environ

namespace {

using namespace carve_dev;

thread_local std::string t_err;
thread_local int t_device = 0;
thread_local uint64_t t_launches = 0;

struct Fail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Fail{code, msg}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(CARVE_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool sync_debug() {
    static const bool on = [] {
        const char* e = std::getenv("CARVE_SYNC_DEBUG");
        return e && *e == '1';
    }();
    return on;
}

thread_local long long t_dbg_tag = 0;  // caller-set context for CARVE_SYNC_DEBUG reports

#define LAUNCHED(what)                                                                            \
    do {                                                                                          \
        ++t_launches;                                                                             \
        ck(cudaGetLastError(), "launch " what);                                                   \
        if (sync_debug())                                                                         \
            ck(cudaDeviceSynchronize(), (std::string("after " what " tag ") + std::to_string(t_dbg_tag)).c_str()); \
    } while (0)

template <class F>
int guarded(F&& f) {
    try {
        f();
        return CARVE_OK;
    } catch (const Fail& e) {
        t_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        t_err = "host allocation failed";
        return CARVE_E_CUDA;
    } catch (const std::exception& e) {
        t_err = e.what();
        return CARVE_E_CUDA;
    }
}

size_t round_up(size_t x, size_t m) { return (x + m - 1) / m * m; }

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* ensure(size_t n) {
        if (n > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            ck(cudaMalloc(&p, n), "cudaMalloc");
            cap = n;
        }
        return p;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    DevBuf packed_in, packed_out, rgb[2], e[2], dir, seams, stamps, scratch_a, scratch_b, mbound;
    DevBuf rec, enl[3];  // recorded seams (original coordinates), enlargement intermediates
    DevBuf glab;         // DP label tables in global memory (images whose table exceeds shared memory)
    DevBuf stats;        // object removal: MaskStats
    int max_smem_optin = 0;
    std::map<const void*, int> smem_set;  // kernel -> dynamic smem attribute set
    // kernel-event profiling mode (bench attribution): one event pair per launch
    bool prof = false;
    struct ProfRec {
        int kind;
        double bytes;
        cudaEvent_t a, b;
    };
    std::vector<ProfRec> prof_recs;
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t ev() {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "cudaEventCreate");
        return e;
    }
    explicit Ctx(int dev) : device(dev) {
        ck(cudaSetDevice(dev), "cudaSetDevice");
        cudaDeviceProp prop{};
        ck(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
        if (prop.major < 10)
            fail(CARVE_E_CUDA, "device " + std::to_string(dev) + " (" + prop.name +
                                   ") is not sm_100-class; libcarve_cuda is built for sm_100a only");
        max_smem_optin = int(prop.sharedMemPerBlockOptin);
        ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    // CUDA graphs of whole device-resident carves (run_graphed), keyed by geometry, the
    // buffers they touch and the CARVE_* environment
    struct GraphEntry {
        std::vector<uintptr_t> key;
        cudaGraphExec_t exec;
        uint64_t launches;
    };
    std::vector<GraphEntry> graphs;
    // batch pipelining: host->device and device->host copies on their own streams
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t pipe_ev[3][2] = {};  // [h2d done, compute done, d2h done][buffer]
    DevBuf pin_in[2], pin_out[2];    // double-buffered packed images
    void ensure_pipeline() {
        if (h2d) return;
        ck(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking), "cudaStreamCreate(h2d)");
        ck(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking), "cudaStreamCreate(d2h)");
        for (auto& row : pipe_ev)
            for (auto& e : row) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    }
    ~Ctx() {
        for (auto& ge : graphs) cudaGraphExecDestroy(ge.exec);
        for (auto& row : pipe_ev)
            for (auto& e : row)
                if (e) cudaEventDestroy(e);
        if (h2d) cudaStreamDestroy(h2d);
        if (d2h) cudaStreamDestroy(d2h);
        if (stream) cudaStreamDestroy(stream);
    }
};

thread_local std::map<int, std::unique_ptr<Ctx>> t_ctx;

void init_kernel_attributes(Ctx& c);  // defined after the kernel tables

// shared memory for the bulk removal's row slots (RGBX + optional FP64 part per slot)
constexpr size_t kCompactBulkSmem = 200 * 1024;

enum KernelKind { KK_ENERGY = 0, KK_DP = 1, KK_COMPACT = 2, KK_UNPACK = 3, KK_PACK = 4, KK_TRANSPOSE = 5, KK_N = 6 };

// RAII bracket: records an event pair around one launch when profiling is on
struct Prof {
    Ctx& c;
    cudaStream_t s;
    int kind;
    double bytes;
    cudaEvent_t a = nullptr;
    Prof(Ctx& c_, cudaStream_t s_, int kind_, double bytes_) : c(c_), s(s_), kind(kind_), bytes(bytes_) {
        if (c.prof) {
            a = c.ev();
            ck(cudaEventRecord(a, s), "cudaEventRecord");
        }
    }
    ~Prof() {
        if (a) {
            cudaEvent_t b = c.ev();
            cudaEventRecord(b, s);
            c.prof_recs.push_back({kind, bytes, a, b});
        }
    }
};

// batch pipelines run on long-lived contexts keyed by (device, pipeline) instead
// of the calling thread's, so their worker threads (created per call) reuse the
// streams and device buffers; each slot's mutex serialises concurrent callers
thread_local Ctx* t_ctx_override = nullptr;
constexpr int CARVE_MAX_PIPELINES = 4;  // concurrent pipelines / sub-batches per device
struct PipeSlot {
    std::mutex m;
    std::unique_ptr<Ctx> c;
};
PipeSlot& pipe_slot(int dev, int pipe) {
    static std::mutex gm;
    static std::map<std::pair<int, int>, std::unique_ptr<PipeSlot>> slots;
    std::lock_guard<std::mutex> lk(gm);
    auto& p = slots[{dev, pipe}];
    if (!p) p = std::make_unique<PipeSlot>();
    return *p;
}

Ctx& ctx() {
    if (t_ctx_override) {
        ck(cudaSetDevice(t_ctx_override->device), "cudaSetDevice");
        return *t_ctx_override;
    }
    auto it = t_ctx.find(t_device);
    if (it == t_ctx.end()) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) fail(CARVE_E_CUDA, "no CUDA device available");
        if (t_device < 0 || t_device >= n) fail(CARVE_E_CUDA, "invalid device index");
        it = t_ctx.emplace(t_device, std::make_unique<Ctx>(t_device)).first;
        // kernel attributes are set once, before any launch on this context
        init_kernel_attributes(*it->second);
    }
    ck(cudaSetDevice(it->second->device), "cudaSetDevice");
    return *it->second;
}

void sync(Ctx& c) { ck(cudaStreamSynchronize(c.stream), "cudaStreamSynchronize"); }

int grid_for(long long n, int block, int per_image_cap = 148 * 8) {
    long long g = (n + block - 1) / block;
    return int(std::max<long long>(1, std::min<long long>(g, per_image_cap)));
}

// ---------------------------------------------------------------------------
// kernel launchers

void launch_unpack(Ctx& c, const uint8_t* in, int W, int H, uint32_t* out, int pitch, int nimg, long long in_is,
                   long long out_is, cudaStream_t s) {
    dim3 grid(grid_for(((long long)W * H + 3) / 4, 256), nimg);
    k_unpack<<<grid, 256, 0, s>>>(in, W, H, out, pitch, in_is, out_is);
    LAUNCHED("k_unpack");
}

void launch_pack(Ctx& c, const uint32_t* in, int pitch, int W, int H, bool transposed, uint8_t* out, int nimg,
                 long long in_is, long long out_is, cudaStream_t s) {
    dim3 grid(grid_for(((long long)W * H + 3) / 4, 256), nimg);
    if (transposed) k_pack<true><<<grid, 256, 0, s>>>(in, pitch, W, H, out, in_is, out_is);
    else k_pack<false><<<grid, 256, 0, s>>>(in, pitch, W, H, out, in_is, out_is);
    LAUNCHED("k_pack");
}

void launch_transpose(const uint32_t* in, int ipitch, int W, int H, uint32_t* out, int opitch, int nimg,
                      long long in_is, long long out_is, cudaStream_t s) {
    dim3 grid((W + 31) / 32, (H + 31) / 32, nimg);
    k_transpose<<<grid, dim3(32, 8), 0, s>>>(in, ipitch, W, H, out, opitch, in_is, out_is);
    LAUNCHED("k_transpose");
}

int env_int(const char* name, int dflt);

void launch_energy(const uint32_t* rgb, int pitch, int W, int H, double* e, int epitch, int nimg, long long rgb_is,
                   long long e_is, cudaStream_t s, unsigned long long* st = nullptr, long long st_is = 0) {
    if (env_int("CARVE_K1", 1) == 0) {  // shared-memory tile version (kept for A/B)
        dim3 grid((W + K1_TW - 1) / K1_TW, (H + K1_TH - 1) / K1_TH, nimg);
        k_energy_full<<<grid, 256, 0, s>>>(rgb, pitch, W, H, e, epitch, rgb_is, e_is);
        LAUNCHED("k_energy_full");
        return;
    }
    // Rows per warp: one full wave of resident warps over the whole job (no
    // partial second wave), runs of at least 4 rows (vertical halo <= 50%).
    static const long long resident_warps = [] {
        int dev = 0, nsm = 0, per_sm = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        ck(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev), "SM count");
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_energy_rows<1, 2>, 256, 0), "K1 occupancy");
        return (long long)nsm * std::max(per_sm, 1) * 8;
    }();
    // Shape: 3 CTAs/SM (80 registers) on large planes (C3 K1 0.44 -> 0.49 of HBM peak,
    // C4 0.52 -> 0.61), 2 CTAs/SM with longer runs below 4 Mpx (C2 0.31 vs 0.22).
    // CARVE_K1V forces one: 0 = 2 CTAs/SM, 1 = prefetch 4, 2 = 3 CTAs/SM, 3 = half runs.
    const int k1v_env = env_int("CARVE_K1V", -1);  // read per call (tests switch it)
    // >= 4 Mpx: the shared-memory row ring with 8 rows in flight per warp, 3 CTAs/SM
    // (tools/k1_sweep.sh, B200: C3 0.46 -> 0.52, C4 0.59 -> 0.67 of the measured HBM peak;
    // 12 or 16 rows in flight measured lower)
    const int k1v = k1v_env >= 0 ? k1v_env : ((long long)W * H * nimg >= (4ll << 20) ? 4 : 0);
    static const long long resident_warps2 = [] {
        int dev = 0, nsm = 0, per_sm = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        ck(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev), "SM count");
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_energy_rows<3, 2>, 256, 0), "K1 occupancy");
        return (long long)nsm * std::max(per_sm, 1) * 8;
    }();
    const int nstrips = (W + K1S_COLS - 1) / K1S_COLS;
    const long long units = (long long)nstrips * H * nimg;  // warp-rows of work
    const long long rw = (k1v == 2 || k1v >= 4) ? resident_warps2 : resident_warps;
    int R = int(std::max<long long>(4, (units + rw - 1) / rw));
    if (k1v == 3) R = std::max(4, R / 2);
    R = k1v == 1 ? ((R + 3) & ~3) : ((R + 1) & ~1);
    const long long warps = (long long)nstrips * ((H + R - 1) / R);
    dim3 grid(unsigned((warps + 7) / 8), nimg);
    if (k1v >= 4 && k1v <= 6) {  // shared-memory row ring: 8 / 12 / 16 rows in flight per warp
        static const bool attrs = [] {
            ck(cudaFuncSetAttribute(k_energy_ring<3, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    8 * 12 * (K1S_COLS + 4) * 4),
               "cudaFuncSetAttribute(k_energy_ring)");
            ck(cudaFuncSetAttribute(k_energy_ring<3, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    8 * 16 * (K1S_COLS + 4) * 4),
               "cudaFuncSetAttribute(k_energy_ring)");
            return true;
        }();
        (void)attrs;
        if (k1v == 4)
            k_energy_ring<3, 8><<<grid, 256, 8 * 8 * (K1S_COLS + 4) * 4, s>>>(rgb, pitch, W, H, e, epitch, rgb_is, e_is,
                                                                          nstrips, R, st, st_is);
        else if (k1v == 5)
            k_energy_ring<3, 12><<<grid, 256, 8 * 12 * (K1S_COLS + 4) * 4, s>>>(rgb, pitch, W, H, e, epitch, rgb_is,
                                                                            e_is, nstrips, R, st, st_is);
        else
            k_energy_ring<3, 16><<<grid, 256, 8 * 16 * (K1S_COLS + 4) * 4, s>>>(rgb, pitch, W, H, e, epitch, rgb_is,
                                                                            e_is, nstrips, R, st, st_is);
        LAUNCHED("k_energy_ring");
        return;
    }
    if (k1v == 1) k_energy_rows<1, 4><<<grid, 256, 0, s>>>(rgb, pitch, W, H, e, epitch, rgb_is, e_is, nstrips, R, st, st_is);
    else if (k1v == 2)
        k_energy_rows<3, 2><<<grid, 256, 0, s>>>(rgb, pitch, W, H, e, epitch, rgb_is, e_is, nstrips, R, st, st_is);
    else k_energy_rows<1, 2><<<grid, 256, 0, s>>>(rgb, pitch, W, H, e, epitch, rgb_is, e_is, nstrips, R, st, st_is);
    LAUNCHED("k_energy_rows");
}

void launch_fill_pads(double* e, int epitch, int W, int H, int nimg, long long e_is, cudaStream_t s) {
    dim3 grid(grid_for((long long)H * (EPAD_L + EPAD_R), 256), nimg);
    k_fill_pads<<<grid, 256, 0, s>>>(e, epitch, W, H, e_is);
    LAUNCHED("k_fill_pads");
}

void launch_rgb_edges(uint32_t* rgb, int pitch, int W, int H, int nimg, long long is, cudaStream_t s) {
    dim3 grid(grid_for(H, 256), nimg);
    k_rgb_edges<<<grid, 256, 0, s>>>(rgb, pitch, W, H, is);
    LAUNCHED("k_rgb_edges");
}

int padded_epitch(int w) { return int(round_up(size_t(EPAD_L) + w + EPAD_R, 32)); }

constexpr int kDpSmemBudget = 220 * 1024;

// programmatic dependent launch for this thread's launches; run_carve turns it off
// for batches (t_pdl): there the dependent grid's early-launched CTAs wait on SMs the
// running grid's later CTAs need (measured on B200: 128 one-CTA images 64.9 -> 50.2 ms,
// C5 e2e 3.54K -> 3.65K images/s, single images unchanged)
thread_local bool t_pdl = true;
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("CARVE_PDL");
        return !(e && *e == '0');
    }();
    return on && t_pdl;
}

// ---- K2+K3 v2: cluster trapezoid DP (dp_cluster.cuh) ------------------------
// The variant table is instantiated in dp_variants_*.cu (separate translation
// units, compiled in parallel); indices are stable (CARVE_DP_VARIANT, orders below).
const std::vector<Dp2Variant>& dp2_variants() {
    static const std::vector<Dp2Variant> v = [] {
        std::vector<Dp2Variant> t;
        dp2_variants_a(t);
        dp2_variants_b(t);
        dp2_variants_c(t);
        dp2_variants_d(t);
        return t;
    }();
    return v;
}
#define kDp2Variants dp2_variants()

void init_kernel_attributes(Ctx& c) {
    ck(cudaFuncSetAttribute(k_compact_bulk<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCompactBulkSmem)),
       "cudaFuncSetAttribute(k_compact_bulk)");
    ck(cudaFuncSetAttribute(k_compact_bulk<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCompactBulkSmem)),
       "cudaFuncSetAttribute(k_compact_bulk)");
    for (const Dp2Variant& v : kDp2Variants)
        for (const void* fn :
             {v.fn, v.fn_tables, v.fn_prof, v.fn_fused, v.fn_fwd, v.fn_fwd_tables, v.fn_fwdp, v.fn_fwdp_tables}) {
            ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kDpSmemBudget),
               "cudaFuncSetAttribute(dp2 smem)");
            ck(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
               "cudaFuncSetAttribute(dp2 cluster)");
            c.smem_set[fn] = kDpSmemBudget;
        }
}

struct Dp2Plan {
    const Dp2Variant* v;
    int ncl, nblk;
    size_t smem;
    int gather;  // label table gathered into CTA 0 (fits in shared memory)
    int glab;    // label table in global memory (does not fit in shared memory)
};

int env_int(const char* name, int dflt) {
    const char* s = std::getenv(name);
    return s && *s ? std::atoi(s) : dflt;
}

// Preference orders (measured on B200: tools/sweep_dp.py, tools/sweep_batch.py;
// profiles/r01_dp_variant_sweep.jsonl): the first variant whose cluster fits
// wins. Single images are latency-bound and favour one C=2 warp per
// scheduler; batches are throughput-bound and favour less halo redundancy.
const int kDp2Order[] = {0, 12, 1, 11, 10, 2, 3, 4, 6, 5, 7, 8, 13, 14, 15, 16};
// large batches (>= one image per SM): one 10-warp CTA per image, 2 per SM;
// smaller batches spread each image over a 3-CTA cluster to fill the SMs
// (measured, tools/sweep_batch.py: 1024 images 2.05 -> 1.58 ms per seam with
// variant 9 <4,8,10,4>; 128 images 0.32 (v9) vs 0.28 ms (v5))
const int kDp2BatchOrder[] = {9, 5, 6, 0, 1, 2, 3, 4, 7, 8, 13, 14, 15, 16};
const int kDp2SmallBatchOrder[] = {5, 6, 0, 1, 2, 3, 4, 7, 8, 13, 14, 15, 16};

int device_sm_count() {
    int dev = 0, nsm = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    ck(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev), "SM count");
    return nsm;
}

// concurrent carves this thread's launches share the device with (pipelines or
// sub-batches of one batch call): the small-batch DP shapes exist to fill the GPU
// with few images, which the other carves already do
thread_local int t_concurrency = 1;

// ring kind of a DP launch: FP64 energy plane, RGBX rows (fused), three FP64 cost planes
enum RingKind { RING_ENERGY = 0, RING_RGBX = 1, RING_COSTS = 2 };

Dp2Plan dp2_plan(int W, int H, bool batch = false, int ring = RING_ENERGY, int nimg = 1) {
    const int nblk = H > 1 ? (H - 1 + LBLK - 1) / LBLK : 0;
    const int forced = env_int("CARVE_DP_VARIANT", -1);
    const int max_ncl = env_int("CARVE_DP_MAX_NCL", 16);
    // passes: label table in shared memory (preferred cluster sizes, then up to 16
    // CTAs), then the global-memory-table instances (tall or wide images; a forced
    // CARVE_DP_VARIANT of those, or CARVE_DP_GLABELS=1, selects them directly)
    const bool force_glab = env_int("CARVE_DP_GLABELS", 0) != 0 ||
                            (forced >= 0 && forced < int(dp2_variants().size()) && dp2_variants()[forced].glab);
    for (int pass = force_glab ? 2 : 0; pass < 3; ++pass) {
        const bool glab = pass == 2;
        std::vector<int> order;
        if (forced >= 0 && forced < int(dp2_variants().size())) order.push_back(forced);
        else if (batch && (long long)nimg * t_concurrency >= device_sm_count()) order.assign(std::begin(kDp2BatchOrder), std::end(kDp2BatchOrder));
        else if (batch) order.assign(std::begin(kDp2SmallBatchOrder), std::end(kDp2SmallBatchOrder));
        else order.assign(std::begin(kDp2Order), std::end(kDp2Order));
        for (int k : order) {
            const Dp2Variant& v = kDp2Variants[k];
            if (v.glab != glab) continue;
            const int ncl = (W + v.cols() - 1) / v.cols();
            const int nblk_smem = glab ? 0 : nblk;  // label rows kept on chip
            const size_t smem = ring == RING_RGBX    ? v.smem_fused(nblk_smem, v.D)
                                : ring == RING_COSTS ? v.smem_costs(nblk_smem, v.D)
                                                     : v.smem(nblk_smem, v.D);
            if (ncl > (pass == 0 ? max_ncl : 16) || smem > size_t(kDpSmemBudget)) continue;
            // columns read past the image edge must stay inside the +inf pad
            if (ncl * v.cols() - W + v.K + 32 * v.C > EPAD_R) continue;
            // gather the block-end labels into CTA 0 when the table is small; not for
            // batches, where the extra shared memory costs a CTA per SM (measured:
            // C5 2.33K -> 2.61K images/s without it) while phase 1 overlaps other images
            const size_t gbytes = round_up(size_t(nblk) * ncl * v.cols(), 16);
            const bool gather = !glab && nblk > 0 && gbytes <= size_t(96) * 1024 &&
                                smem + gbytes <= size_t(kDpSmemBudget) && env_int("CARVE_DP_GATHER", batch ? 0 : 1) != 0;
            return Dp2Plan{&v, ncl, nblk, smem + (gather ? gbytes : 0), gather ? 1 : 0, glab ? 1 : 0};
        }
    }
    fail(CARVE_E_IMAGE_TOO_LARGE, "no DP cluster configuration fits width " + std::to_string(W) + " x height " +
                                      std::to_string(H));
}

void launch_dp2(Ctx& c, const Dp2Plan& pl, Dp2Params p, int nimg, cudaStream_t s, bool fused = false,
                bool forward = false) {
    const Dp2Variant& v = *pl.v;
    p.G = pl.ncl * v.NW;
    p.nblk = pl.nblk;
    p.gather = pl.gather;
    if (pl.glab) {
        p.glab_istride = (long long)round_up(size_t(pl.nblk) * p.G * v.S(), 128);
        p.glab = static_cast<int8_t*>(c.glab.ensure(size_t(std::max<long long>(p.glab_istride, 128)) * nimg));
    } else {
        p.glab = nullptr;
    }
    p.dbg = env_int("CARVE_DP_DBG", 0);
    const void* fn = forward ? (fused ? (p.m_out ? v.fn_fwd_tables : v.fn_fwd) : (p.m_out ? v.fn_fwdp_tables : v.fn_fwdp))
                     : fused ? v.fn_fused : p.m_out ? v.fn_tables : (p.prof ? v.fn_prof : v.fn);
    if (c.smem_set.find(fn) == c.smem_set.end()) fail(CARVE_E_CUDA, "DP kernel attributes not initialised");
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(nimg * pl.ncl));
    cfg.blockDim = dim3(unsigned(v.NW * 32));
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(pl.ncl);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    void* args[] = {&p};
    ck(cudaLaunchKernelExC(&cfg, fn, args), "launch k_dp2");
    LAUNCHED("k_dp2");
}

template <bool HAS_E>
void launch_compact_bulk(cudaLaunchConfig_t cfg, const CompactParams& p, int nimg, int rpc) {
    const int slot_words = int(round_up(size_t(p.W) + 4, 32));
    const size_t slot_bytes = size_t(slot_words) * (HAS_E ? 12 : 4);
    // up to 4 rows in flight per CTA while two CTAs still fit per SM (C3's 3840-wide rows:
    // 2 slots; C4's 7680-wide rows: 2 slots, one CTA per SM)
    int slots = int(std::min<size_t>(CB_MAX_SLOTS, std::max<size_t>(2, (kCompactBulkSmem / 2) / slot_bytes)));
    slots = int(std::min<size_t>(size_t(slots), kCompactBulkSmem / slot_bytes));
    if (slots < 1) {  // a row does not fit one shared-memory slot: warp-per-row removal
        cfg.gridDim = dim3((p.H + 7) / 8, nimg);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = 0;
        ck(cudaLaunchKernelEx(&cfg, k_compact_warp<4, HAS_E>, p), "launch k_compact_warp");
        LAUNCHED("k_compact_warp");
        return;
    }
    cfg.gridDim = dim3((p.H + rpc - 1) / rpc, nimg);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = size_t(slots) * slot_bytes;
    ck(cudaLaunchKernelEx(&cfg, k_compact_bulk<HAS_E>, p, rpc, slot_words, slots), "launch k_compact_bulk");
    LAUNCHED("k_compact_bulk");
}

void launch_compact_inplace(const CompactParams& p, int nimg, cudaStream_t s) {
    if (env_int("CARVE_COMPACT", 2) == 2) {  // warp per row (default); 1 = CTA per row
        // warps per CTA: small CTAs spread few rows over all SMs (single images)
        const int wpb = env_int("CARVE_COMPACT_WPB", 8);
        const int nb = env_int("CARVE_COMPACT_NB", 4);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((p.H + wpb - 1) / wpb, nimg);
        cfg.blockDim = dim3(wpb * 32);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl_enabled() ? 1 : 0;
        if (p.e_out && env_int("CARVE_COMPACT_BULK", 1) != 0) {
            // rows per CTA: about two CTAs per SM over the job (C2 1080 rows: 4 -> 10.6 us;
            // C4 4320 rows: 15 -> 72.7 us, was 84.6 with the warp-per-row kernel)
            static const int nsm = device_sm_count();
            const int rpc_auto = std::max(2, std::min(16, int((p.H * (long long)nimg + 2 * nsm - 1) / (2 * nsm))));
            launch_compact_bulk<true>(cfg, p, nimg, env_int("CARVE_COMPACT_RPC_E", rpc_auto));
            return;
        }
        if (p.e_out) {
            if (nb == 8) ck(cudaLaunchKernelEx(&cfg, k_compact_warp<8, true>, p), "launch k_compact_warp");
            else if (nb == 2) ck(cudaLaunchKernelEx(&cfg, k_compact_warp<2, true>, p), "launch k_compact_warp");
            else ck(cudaLaunchKernelEx(&cfg, k_compact_warp<4, true>, p), "launch k_compact_warp");
        } else if (p.rgb_edges && env_int("CARVE_COMPACT_BULK", 1) != 0) {
            // batches: TMA bulk loads of each row's moving part, 4 rows in flight per CTA
            launch_compact_bulk<false>(cfg, p, nimg, env_int("CARVE_COMPACT_RPC", 8));  // C5: 8 0.541, 16 0.554 ms
            return;
        } else if (p.rgb_edges) {  // batches: R rows per warp
            const int R = env_int("CARVE_COMPACT_ROWS", 2);  // measured: R=2 0.712, 1 0.730, 4 0.954 ms per seam (C5)
            if (R > 1) {
                cfg.gridDim = dim3((p.H + wpb * R - 1) / (wpb * R), nimg);
                if (R == 2) ck(cudaLaunchKernelEx(&cfg, k_compact_rows<2>, p), "launch k_compact_rows");
                else if (R == 8) ck(cudaLaunchKernelEx(&cfg, k_compact_rows<8>, p), "launch k_compact_rows");
                else ck(cudaLaunchKernelEx(&cfg, k_compact_rows<4>, p), "launch k_compact_rows");
                LAUNCHED("k_compact_rows");
                return;
            }
            ck(cudaLaunchKernelEx(&cfg, k_compact_warp<4, false>, p), "launch k_compact_warp");
        } else {
            ck(cudaLaunchKernelEx(&cfg, k_compact_warp<4, false>, p), "launch k_compact_warp");
        }
        LAUNCHED("k_compact_warp");
        return;
    }
    // one row per CTA: measured faster than batching 2-4 rows per CTA (C2 10.5 vs 11.3 us)
    const int W = p.W;
    auto grid = [&](int rpb) { return dim3((p.H + rpb - 1) / rpb, nimg); };
    if (W <= 4 * 1024) {
        k_compact_inplace<4, 1><<<grid(1), int(round_up((W + 3) / 4, 32)), 0, s>>>(p);
    } else if (W <= 8 * 1024) {
        k_compact_inplace<8, 1><<<grid(1), int(round_up((W + 7) / 8, 32)), 0, s>>>(p);
    } else if (W <= 16 * 1024) {
        k_compact_inplace<16, 1><<<grid(1), int(round_up((W + 15) / 16, 32)), 0, s>>>(p);
    } else {
        fail(CARVE_E_IMAGE_TOO_LARGE, "width exceeds the in-place removal limit of 16384");
    }
    LAUNCHED("k_compact_inplace");
}

template <int MODE>
void launch_compact_transpose(const uint32_t* in, int ipitch, int W, int H, const int* seam, uint32_t* out,
                              int opitch, uint8_t* packed, int nimg, long long in_is, long long out_is,
                              long long seam_is, long long pk_is, unsigned long long* st, long long st_is,
                              cudaStream_t s) {
    dim3 grid((W - 1 + 31) / 32, (H + 31) / 32, nimg);
    k_compact_transpose<MODE><<<grid, dim3(32, 8), 0, s>>>(in, ipitch, W, H, seam, out, opitch, packed, in_is, out_is,
                                                           seam_is, pk_is, st, st_is);
    LAUNCHED("k_compact_transpose");
}

void launch_compact(const CompactParams& p, int nimg, cudaStream_t s) {
    const int per_cta = CP_THREADS * CP_CHUNK;
    dim3 grid((p.W - 1 + per_cta - 1) / per_cta, p.H, nimg);
    k_compact<<<grid, CP_THREADS, 0, s>>>(p);
    LAUNCHED("k_compact");
}

// ---------------------------------------------------------------------------
// the resident carve loop: nimg same-size images, packed RGB in -> packed out.
// Layout per image in the plane buffers: one plane of `plane` elements.

struct CarveGeometry {
    int w, h, tw, th;
    int pitch_a, pitch_b;
    size_t plane;     // elements per image plane (max over both orientations)
    int dpitch;       // bytes per direction row
    int dir_rows;
    size_t seam_ints; // per image
    int nseams;
    int mpitch;       // M-boundary row pitch (doubles)
    long long mb_istride;
    int epitch_a, epitch_b;  // padded energy-plane pitches per phase
    size_t eplane;           // doubles per image energy plane (max over phases, incl. pads)
};

CarveGeometry geometry(int w, int h, int tw, int th) {
    CarveGeometry g{};
    g.w = w;
    g.h = h;
    g.tw = tw;
    g.th = th;
    // RGBX planes share the energy planes' padded geometry: logical column 0 at
    // EPAD_L, >= EPAD_R columns after the live width, EPAD_B spare rows. The
    // fused DP reads RGBX rows exactly like energy rows (unconditional loads).
    g.pitch_a = padded_epitch(w);
    g.pitch_b = padded_epitch(h);
    g.plane = size_t(g.pitch_a) * (h + EPAD_B);
    if (th != h) g.plane = std::max(g.plane, size_t(g.pitch_b) * (tw + EPAD_B));
    g.dpitch = int(round_up(std::max(w, h), 16) + 128);
    g.dir_rows = std::max(h, tw);
    g.seam_ints = size_t(w - tw) * h + size_t(h - th) * tw;
    g.nseams = (w - tw) + (h - th);
    g.mpitch = std::max(g.pitch_a, g.pitch_b);
    g.epitch_a = padded_epitch(w);
    g.epitch_b = padded_epitch(h);
    g.eplane = size_t(g.epitch_a) * (h + EPAD_B);
    if (th != h) g.eplane = std::max(g.eplane, size_t(g.epitch_b) * (tw + EPAD_B));
    g.mb_istride = (long long)((g.dir_rows + LBLK - 1) / LBLK + 1) * g.mpitch;
    return g;
}

void check_targets(int w, int h, int tw, int th) {
    if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "PixelGrid dimensions must be >= 1");
    if (tw < 1 || tw > w) fail(CARVE_E_INVALID_TARGET, "target width must be in [1, width]");
    if (th < 1 || th > h) fail(CARVE_E_INVALID_TARGET, "target height must be in [1, height]");
    // DP configuration must exist for the widths the solver will see
    if (tw < w) dp2_plan(w, h);
    if (th < h) dp2_plan(h, tw);
}

// stamps layout per image: 6 per seam [energy start/end, solve start/end, remove
// start/end] (+ 4 spare). Energy: the K1 full map for a phase's first seam, the DP
// prologue's 2-column fix-up for the others; 0 where it is fused into the DP
// (batches, forward energy) or not recomputed (recompute=false).
constexpr int kStampsPerSeam = 6;
size_t stamp_words(const CarveGeometry& g) { return size_t(g.nseams) * kStampsPerSeam + 4; }

// CarveConfig fields that change the device loop (carver.hpp:15-24)
struct CarveOpts {
    bool forward = false;   // forward energy: dp_seam_forward on the current luma (fused DP, FWD cells)
    bool recompute = true;  // false: e1 once per phase, then the map is only carved (no fix-up)
};

CarveOpts opts_of(const carve_cuda_config* cfg) {
    CarveOpts o;
    if (cfg) {
        o.forward = cfg->forward != 0;
        o.recompute = cfg->recompute != 0;
    }
    return o;
}

void run_carve(Ctx& c, const uint8_t* d_in, uint8_t* d_out, int nimg, const CarveGeometry& g, int* d_seams,
               size_t seam_istride, unsigned long long* d_stamps, cudaStream_t s, CarveOpts o = {}) {
    const long long in_is = (long long)g.w * g.h * 3, out_is = (long long)g.tw * g.th * 3;
    struct PdlScope {
        bool prev;
        explicit PdlScope(bool on) : prev(t_pdl) { t_pdl = on; }
        ~PdlScope() { t_pdl = prev; }
    } pdl_scope(nimg == 1 || env_int("CARVE_PDL_BATCH", 0) != 0);
    // logical column 0 of each padded RGBX plane ([1]: transpose target only)
    uint32_t* rgb[2] = {c.rgb[0].as<uint32_t>() + EPAD_L, c.rgb[1].p ? c.rgb[1].as<uint32_t>() + EPAD_L : nullptr};
    double* e = c.e[0].as<double>() + EPAD_L;                                 // logical column 0
    const long long eis = (long long)g.eplane;
    const long long pis = (long long)g.plane;
    const size_t sw = stamp_words(g);
    int cur = 0;
    {
        Prof pr(c, s, KK_UNPACK, 7.0 * g.w * g.h * nimg);
        launch_unpack(c, d_in, g.w, g.h, rgb[cur], g.pitch_a, nimg, in_is, pis, s);
    }

    // One orientation's seam loop: K1 once, then per seam the DP (whose
    // prologue applies the previous removal's 2-column energy fix-up) and the
    // in-place removal. Nothing returns to the host between seams.
    // Batches run the fused DP (energy recomputed from RGBX, no energy plane);
    // single images keep the incremental energy plane. CARVE_FUSED=0/1 overrides.
    // Forward energy always runs fused (transition costs from the RGBX rows);
    // recompute=false needs the carried energy plane.
    const int fused_env = env_int("CARVE_FUSED", -1);
    // forward + recompute=false (carver.hpp:175-184): the forward costs of the phase's
    // first image are computed once into three planes and then only carved
    // (drop_columns), as the reference carves its cached ForwardCosts; the DP streams them
    const bool costs = o.forward && !o.recompute;
    const bool fused = (o.forward && o.recompute) || (o.recompute && (fused_env >= 0 ? fused_env != 0 : nimg > 1));
    // cost-plane sets A/B (3 padded planes each, ping-pong per seam)
    double* cset[2] = {costs ? c.e[0].as<double>() + EPAD_L : nullptr, costs ? c.e[1].as<double>() + EPAD_L : nullptr};
    const long long cplane = (long long)g.eplane;  // plane stride inside a set
    // `finish`: what the phase's last removal writes (fused with K4, see k_compact_transpose):
    // OUT_PLANE  the transposed RGBX plane for the height phase (rgb[cur ^ 1], pitch_b)
    // OUT_PACKED the final image, transposed back, packed RGB into d_out
    // OUT_ROWS   the final image, packed RGB into d_out
    auto phase = [&](int W0, int H, int ntake, int pitch, int epitch, int seam_base, int stamp_seam0, int finish) {
        if (ntake <= 0) return;
        int cs = 0;  // current cost-plane set
        if (costs) {
            for (int im = 0; im < nimg; ++im) {
                k_forward_costs_rgbx<<<grid_for((long long)W0 * H, 256), 256, 0, s>>>(
                    rgb[cur] + im * pis, pitch, W0, H, cset[0] + im * 3 * cplane, epitch, cplane);
                LAUNCHED("k_forward_costs_rgbx");
            }
        } else if (fused) {
            launch_rgb_edges(rgb[cur], pitch, W0, H, nimg, pis, s);
        } else {
            {
                // algorithmic bytes: 3 B RGB read + 8 B FP64 write per pixel
                Prof pr(c, s, KK_ENERGY, 11.0 * W0 * H * nimg);
                launch_energy(rgb[cur], pitch, W0, H, e, epitch, nimg, pis, eis, s,
                              d_stamps ? d_stamps + size_t(stamp_seam0) * kStampsPerSeam : nullptr, (long long)sw);
            }
            launch_fill_pads(e, epitch, W0, H, nimg, eis, s);
        }
        for (int k = 0; k < ntake; ++k) {
            const int W = W0 - k;
            t_dbg_tag = W;
            int* seam = d_seams + seam_base + size_t(k) * H;
            unsigned long long* st = d_stamps ? d_stamps + size_t(stamp_seam0 + k) * kStampsPerSeam : nullptr;
            {
                const Dp2Plan pl = dp2_plan(W, H, nimg > 1, fused ? RING_RGBX : costs ? RING_COSTS : RING_ENERGY, nimg);
                Dp2Params q{};
                q.e = costs ? cset[cs] : e;
                q.epitch = epitch;
                q.cplane = cplane;
                q.W = W;
                q.H = H;
                q.mbound = c.mbound.as<double>();
                q.mpitch = g.mpitch;
                q.seam = seam;
                q.stamps = st;
                q.e_istride = costs ? 3 * cplane : eis;
                q.mb_istride = g.mb_istride;
                q.s_istride = (long long)seam_istride;
                q.st_istride = (long long)sw;
                q.rgb = rgb[cur];
                q.rpitch = pitch;
                q.rgb_istride = pis;
                // fix up the energy around the previous seam (removed from width W + 1)
                if (k > 0 && !fused && !costs && o.recompute) q.prev_seam = seam - H;
                // algorithmic: 8 B FP64 energy read per cell (no direction
                // plane); fused: 4 B RGBX read per cell
                Prof pr(c, s, KK_DP, (fused ? 4.0 : 8.0) * W * H * nimg);
                launch_dp2(c, pl, q, nimg, s, fused, o.forward);
            }
            if (costs && k + 1 < ntake) {  // drop_columns of the three cost planes (carver.hpp:179-181)
                for (int im = 0; im < nimg; ++im) {
                    k_drop_col_planes<<<dim3(unsigned((W + 255) / 256), unsigned(H), 3u), 256, 0, s>>>(
                        cset[cs] + im * 3 * cplane, cset[cs ^ 1] + im * 3 * cplane, epitch, cplane, W, H,
                        seam + im * (long long)seam_istride);
                    LAUNCHED("k_drop_col_planes");
                }
                cs ^= 1;
            }
            CompactParams q{};
            const bool last = (k + 1 == ntake);
            q.rgb_in = q.rgb_out = rgb[cur];
            q.e_in = q.e_out = (last || fused || costs) ? nullptr : e;  // the final width needs no energy
            q.rgb_edges = (fused || costs) && !last;
            q.pitch = pitch;
            q.epitch = epitch;
            q.W = W;
            q.H = H;
            q.seam = seam;
            q.stamps = st ? st + 4 : nullptr;
            q.p_istride = pis;
            q.e_istride = eis;
            q.s_istride = (long long)seam_istride;
            q.st_istride = (long long)sw;
            if (!last) {
                // algorithmic: read W + write W-1 per row, 3 B RGB (+ 8 B FP64) per
                // element, although the in-place kernel moves only the part right of the seam
                Prof pr(c, s, KK_COMPACT, (fused ? 3.0 : 11.0) * H * (2.0 * W - 1) * nimg);
                launch_compact_inplace(q, nimg, s);
            } else {
                // the last removal writes the next layout directly (3 B RGB read + 3 B written per pixel)
                Prof pr(c, s, KK_COMPACT, 3.0 * H * (2.0 * W - 1) * nimg);
                unsigned long long* cst = st ? st + 4 : nullptr;
                const long long ls = (long long)seam_istride, lst = (long long)sw;
                if (finish == OUT_PLANE)
                    launch_compact_transpose<OUT_PLANE>(rgb[cur], pitch, W, H, seam, rgb[cur ^ 1], g.pitch_b, nullptr,
                                                        nimg, pis, pis, ls, 0, cst, lst, s);
                else if (finish == OUT_PACKED)
                    launch_compact_transpose<OUT_PACKED>(rgb[cur], pitch, W, H, seam, nullptr, 0, d_out, nimg, pis, 0,
                                                         ls, out_is, cst, lst, s);
                else
                    launch_compact_transpose<OUT_ROWS>(rgb[cur], pitch, W, H, seam, nullptr, 0, d_out, nimg, pis, 0,
                                                       ls, out_is, cst, lst, s);
            }
        }
    };
    const bool hphase = g.th != g.h, vphase = g.tw != g.w;
    phase(g.w, g.h, g.w - g.tw, g.pitch_a, g.epitch_a, 0, 0, hphase ? OUT_PLANE : OUT_ROWS);
    if (hphase) {
        if (!vphase) {  // nothing removed vertically: plain transpose into the height-phase layout
            Prof pr(c, s, KK_TRANSPOSE, 8.0 * g.tw * g.h * nimg);
            launch_transpose(rgb[cur], g.pitch_a, g.tw, g.h, rgb[cur ^ 1], g.pitch_b, nimg, pis, pis, s);
        }
        cur ^= 1;
        phase(g.h, g.tw, g.h - g.th, g.pitch_b, g.epitch_b, (g.w - g.tw) * g.h, g.w - g.tw, OUT_PACKED);
    } else if (!vphase) {  // identity carve
        Prof pr(c, s, KK_PACK, 7.0 * g.tw * g.th * nimg);
        launch_pack(c, rgb[cur], g.pitch_a, g.tw, g.th, false, d_out, nimg, pis, out_is, s);
    }
}

void ensure_carve_buffers(Ctx& c, const CarveGeometry& g, int nimg, bool cost_planes = false) {
    c.rgb[0].ensure(g.plane * 4 * nimg);
    if (g.th != g.h) c.rgb[1].ensure(g.plane * 4 * nimg);
    // cost_planes: two sets of three FP64 cost planes (forward + recompute=false)
    c.e[0].ensure(g.eplane * 8 * nimg * (cost_planes ? 3 : 1));
    if (cost_planes) c.e[1].ensure(g.eplane * 8 * nimg * 3);
    c.mbound.ensure(size_t(g.mb_istride) * 8 * nimg);
}

// ---------------------------------------------------------------------------
// bench.hpp:67-94 make_test_image (host fixture generator)

void make_test_image_host(int w, int h, uint32_t variant, uint8_t* out) {
    uint32_t s = 0x9E3779B9u ^ (uint32_t(w) * 2654435761u) ^ uint32_t(h);
    if (variant) {
        s ^= variant;
        if (!s) s = 1u;
    }
    auto next = [&s] {
        s ^= s << 13;
        s ^= s >> 17;
        s ^= s << 5;
        return s;
    };
    auto clampd = [](double v, double lo, double hi) { return std::clamp(v, lo, hi); };
    const double pi = 3.14159265358979323846;
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) {
            const double u = double(i) / std::max(1, h - 1);
            const double v = double(j) / std::max(1, w - 1);
            double base = 60.0 + 70.0 * (u + v) / 2.0 + 45.0 * std::sin(3.0 * pi * u) * std::cos(3.0 * pi * v);
            if (u > 0.33 && u < 0.66 && v > 0.25 && v < 0.75) base += (((i / 3) + (j / 3)) % 2) ? 55.0 : -55.0;
            const int n1 = int(next() % 37) - 18;
            const int n2 = int(next() % 37) - 18;
            const int n3 = int(next() % 37) - 18;
            uint8_t* p = out + (size_t(i) * w + j) * 3;
            p[0] = uint8_t(clampd(base + n1, 0.0, 255.0));
            p[1] = uint8_t(clampd(base * 0.85 + 24.0 + n2, 8.0, 255.0));
            p[2] = uint8_t(clampd(210.0 - base * 0.55 + n3, 0.0, 255.0));
        }
}

void validate_seam_host(const int32_t* seam, int n, int w, int h) {
    if (n != h) fail(CARVE_E_INVALID_SEAM, "seam length does not match image height");
    for (int i = 0; i < n; ++i) {
        if (seam[i] < 0 || seam[i] >= w) fail(CARVE_E_INVALID_SEAM, "seam column out of range");
        if (i > 0 && std::abs(seam[i] - seam[i - 1]) > 1) fail(CARVE_E_INVALID_SEAM, "seam is not connected");
    }
}

// stamps -> per-seam timings (SeamTiming, carver.hpp:23-27): a lap is 0 where its
// stamps were not written (the work is fused into another kernel)
void stamps_to_timings(const std::vector<unsigned long long>& st, int nseams, carve_seam_timing* timings) {
    auto lap = [](unsigned long long a, unsigned long long b) { return a && b > a ? double(b - a) * 1e-9 : 0.0; };
    for (int k = 0; k < nseams; ++k) {
        const unsigned long long* q = &st[size_t(k) * kStampsPerSeam];
        timings[k].energy_s = lap(q[0], q[1]);
        timings[k].solve_s = lap(q[2], q[3]);
        timings[k].remove_s = lap(q[4], q[5]);
    }
}

void launch_seams_to_original(const int* log, int count, int H, int* out, cudaStream_t s) {
    const long long n = (long long)count * H;
    if (n == 0) return;
    k_seams_to_original<<<unsigned((n + 255) / 256), 256, 0, s>>>(log, count, H, out);
    LAUNCHED("k_seams_to_original");
}

void launch_expand_rows(const uint8_t* in, int W, int H, const int* cols, int count, long long cstride, uint8_t* out,
                        cudaStream_t s) {
    constexpr int WPB = 4;
    const size_t smem = size_t(WPB) * ((W + 31) / 32) * 4;
    if (smem > 48 * 1024) {
        ck(cudaFuncSetAttribute(k_expand_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
           "cudaFuncSetAttribute(k_expand_rows)");
    }
    k_expand_rows<<<unsigned((H + WPB - 1) / WPB), WPB * 32, smem, s>>>(in, W, H, cols, count, cstride, out);
    LAUNCHED("k_expand_rows");
}

// record_seams (carver.hpp:226-262) on a packed device image: the ordinary
// device carve loop to width w - count (its output is discarded), then the
// logged seams mapped back to original coordinates. d_orig: count * h ints.
void record_device(Ctx& c, const uint8_t* d_in, int w, int h, int count, int* d_orig, unsigned long long* d_st,
                   CarveOpts o = {}) {
    if (count <= 0) return;
    const CarveGeometry g = geometry(w, h, w - count, h);
    ensure_carve_buffers(c, g, 1, o.forward && !o.recompute);
    int* d_log = static_cast<int*>(c.seams.ensure(std::max<size_t>(g.seam_ints, 1) * 4));
    uint8_t* d_scratch = static_cast<uint8_t*>(c.scratch_a.ensure(size_t(w - count) * h * 3));
    run_carve(c, d_in, d_scratch, 1, g, d_log, g.seam_ints, d_st, c.stream, o);
    launch_seams_to_original(d_log, count, h, d_orig, c.stream);
}

// packed w x h -> packed h x w (raster.hpp:73-79) through an RGBX plane
void transpose_packed(Ctx& c, const uint8_t* d_in, int w, int h, uint8_t* d_out) {
    const int pitch = int(round_up(w, 32));
    uint32_t* plane = static_cast<uint32_t*>(c.rgb[0].ensure(size_t(pitch) * h * 4));
    launch_unpack(c, d_in, w, h, plane, pitch, 1, 0, 0, c.stream);
    launch_pack(c, plane, pitch, h, w, true, d_out, 1, 0, 0, c.stream);
}

// enlarge_to_width's target checks (carver.hpp:268-270)
void check_enlarge(int w, int target) {
    if (target < w) fail(CARVE_E_INVALID_TARGET, "enlargement target is below the current width");
    if (target > 2 * w - 1) fail(CARVE_E_TARGET_TOO_LARGE, "single-pass enlargement is limited to 2*width-1");
}

// One device-resident carve as a CUDA graph: the first call for a key captures the
// launches (stream capture on the context stream, programmatic dependencies kept), later
// calls replay the instantiated graph — no per-launch host work. The key also holds the
// context's buffer addresses and the CARVE_* environment (which can change the plan);
// kernel-event profiling and CARVE_SYNC_DEBUG run uncaptured, and so does any body that
// fails to capture (e.g. a buffer growing mid-capture), retried once uncaptured.
template <class F>
void run_graphed(Ctx& c, std::vector<uintptr_t> key, F&& body) {
    if (c.prof || sync_debug() || env_int("CARVE_GRAPH", 1) == 0) {
        body();
        return;
    }
    for (const DevBuf* b : {&c.rgb[0], &c.rgb[1], &c.e[0], &c.e[1], &c.mbound, &c.glab, &c.seams})
        key.push_back(uintptr_t(b->p));
    for (char** ev = environ; *ev; ++ev)
        if (std::strncmp(*ev, "CARVE_", 6) == 0) key.push_back(std::hash<std::string>{}(*ev));
    for (auto& ge : c.graphs)
        if (ge.key == key) {
            ck(cudaGraphLaunch(ge.exec, c.stream), "cudaGraphLaunch");
            t_launches += ge.launches;
            return;
        }
    const uint64_t l0 = t_launches;
    cudaGraph_t graph = nullptr;
    ck(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    bool ok = true;
    try {
        body();
    } catch (...) {
        ok = false;
    }
    const cudaError_t ec = cudaStreamEndCapture(c.stream, &graph);
    cudaGetLastError();  // a failed capture leaves a sticky-free error behind; clear it
    cudaGraphExec_t exec = nullptr;
    if (ok && ec == cudaSuccess && graph && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
        cudaGraphDestroy(graph);
        ck(cudaGraphLaunch(exec, c.stream), "cudaGraphLaunch");
        if (c.graphs.size() >= 8) {
            cudaGraphExecDestroy(c.graphs.front().exec);
            c.graphs.erase(c.graphs.begin());
        }
        c.graphs.push_back({std::move(key), exec, t_launches - l0});
        return;
    }
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    t_launches = l0;
    body();  // uncaptured
}

void carve_one_host(Ctx& c, const uint8_t* rgb, int w, int h, int tw, int th, uint8_t* out, int32_t* seams_out,
                    carve_seam_timing* timings, CarveOpts o = {}) {
    const CarveGeometry g = geometry(w, h, tw, th);
    cudaStream_t s = c.stream;
    const size_t in_bytes = size_t(w) * h * 3, out_bytes = size_t(tw) * th * 3;
    uint8_t* d_in = static_cast<uint8_t*>(c.packed_in.ensure(in_bytes));
    uint8_t* d_out = static_cast<uint8_t*>(c.packed_out.ensure(out_bytes));
    ensure_carve_buffers(c, g, 1, o.forward && !o.recompute);
    int* d_seams = static_cast<int*>(c.seams.ensure(std::max<size_t>(g.seam_ints, 1) * 4));
    unsigned long long* d_st = nullptr;
    if (timings) {
        d_st = static_cast<unsigned long long*>(c.stamps.ensure(stamp_words(g) * 8));
        ck(cudaMemsetAsync(d_st, 0, stamp_words(g) * 8, s), "memset stamps");
    }
    ck(cudaMemcpyAsync(d_in, rgb, in_bytes, cudaMemcpyHostToDevice, s), "H2D rgb");
    run_graphed(c, {uintptr_t(w), uintptr_t(h), uintptr_t(tw), uintptr_t(th), uintptr_t(d_in), uintptr_t(d_out),
                    uintptr_t(d_seams), uintptr_t(d_st), uintptr_t(o.forward), uintptr_t(o.recompute)},
                [&] { run_carve(c, d_in, d_out, 1, g, d_seams, g.seam_ints, d_st, s, o); });
    ck(cudaMemcpyAsync(out, d_out, out_bytes, cudaMemcpyDeviceToHost, s), "D2H rgb");
    if (seams_out && g.seam_ints)
        ck(cudaMemcpyAsync(seams_out, d_seams, g.seam_ints * 4, cudaMemcpyDeviceToHost, s), "D2H seams");
    std::vector<unsigned long long> st;
    if (timings) {
        st.resize(stamp_words(g));
        ck(cudaMemcpyAsync(st.data(), d_st, st.size() * 8, cudaMemcpyDeviceToHost, s), "D2H stamps");
    }
    sync(c);
    if (timings) stamps_to_timings(st, g.nseams, timings);
}

// ---------------------------------------------------------------------------
// stream / context plumbing for the asynchronous and batch entry points

// Fork `into` from the caller's stream `s` (an event), join it back at the end.
// RAII: the fork event is destroyed on every path.
struct StreamFork {
    cudaStream_t s;
    cudaStream_t into = nullptr;
    cudaEvent_t fork = nullptr;
    explicit StreamFork(cudaStream_t s_) : s(s_) {
        ck(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "event create");
        ck(cudaEventRecord(fork, s), "record fork");
    }
    StreamFork(cudaStream_t s_, cudaStream_t into_) : StreamFork(s_) {
        into = into_;
        fork_into(into);
    }
    void fork_into(cudaStream_t x) { ck(cudaStreamWaitEvent(x, fork, 0), "wait fork"); }
    void join_from(cudaStream_t x) {
        cudaEvent_t j;
        ck(cudaEventCreateWithFlags(&j, cudaEventDisableTiming), "event create");
        const cudaError_t e1 = cudaEventRecord(j, x);
        const cudaError_t e2 = e1 == cudaSuccess ? cudaStreamWaitEvent(s, j, 0) : e1;
        cudaEventDestroy(j);
        ck(e2, "join");
    }
    void join() { join_from(into); }
    ~StreamFork() {
        if (fork) cudaEventDestroy(fork);
    }
    StreamFork(const StreamFork&) = delete;
    StreamFork& operator=(const StreamFork&) = delete;
};

// The (device, pipeline) slot contexts 0..P-1, locked for the scope (in index
// order, so concurrent callers cannot deadlock) and created on first use.
// `lane`: the position of the device in a batch call's device list, so a device
// listed twice gets two independent sets of contexts (two concurrent workers).
struct SlotSet {
    int dev;
    std::vector<std::unique_lock<std::mutex>> locks;
    std::vector<Ctx*> ctxs;
    SlotSet(int dev_, int P, int lane = 0) : dev(dev_) {
        for (int q = 0; q < P; ++q) {
            PipeSlot& slot = pipe_slot(dev, lane * CARVE_MAX_PIPELINES + q);
            locks.emplace_back(slot.m);
            if (!slot.c) {
                slot.c = std::make_unique<Ctx>(dev);
                init_kernel_attributes(*slot.c);
            }
            ctxs.push_back(slot.c.get());
        }
    }
    // make slot q the calling thread's current context (ctx() returns it)
    Ctx& use(int q) {
        t_ctx_override = ctxs[q];
        return ctx();
    }
    ~SlotSet() { t_ctx_override = nullptr; }
};

// concurrent carves the DP shape choice counts (dp2_plan), for one scope
struct ConcurrencyScope {
    explicit ConcurrencyScope(int p) { t_concurrency = p; }
    ~ConcurrencyScope() { t_concurrency = 1; }
};

// Host batch pipeline shape: P pipelines per device, chunks of `chunk` images.
// CARVE_PIPELINES / CARVE_PIPE_CHUNK override (read per call).
struct BatchPlan {
    int pipes, chunk;
};

BatchPlan batch_plan(int n, int ndev, const CarveGeometry& g) {
    const int share = (n + ndev - 1) / ndev;
    // measured on B200 (tools/share_sweep.py --grid, profiles/r02_share_grid_b.txt, batches
    // without PDL): 4 pipelines, chunks of a quarter share up to 128 images — 1024: 3.56K
    // e2e images/s (2 x 256: 3.47K), 512: 3.38K, 256 as 4 x 64: 2.92K (2 x 128: 2.85K),
    // 128 as 4 x 32: 2.46K (2 x 64: 2.32K)
    int P = std::max(1, std::min(CARVE_MAX_PIPELINES, env_int("CARVE_PIPELINES", 4)));
    // per-image device footprint (planes, energy, M rows, packed in/out double
    // buffers, seam log): the chunks in flight stay well inside 180 GB of HBM
    const size_t in_bytes = size_t(g.w) * g.h * 3, out_bytes = size_t(g.tw) * g.th * 3;
    const size_t per_img = g.plane * 8 + g.eplane * 8 + size_t(g.mb_istride) * 8 + 2 * (in_bytes + out_bytes) +
                           g.seam_ints * 4;
    const int cap = int(std::max<size_t>(1, (size_t(48) << 30) / (per_img * size_t(P))));
    int ch = env_int("CARVE_PIPE_CHUNK", 0);
    if (ch <= 0) ch = std::max(16, std::min(128, (share + 3) / 4));
    ch = std::max(1, std::min({ch, cap, share}));
    const int nchunks = (share + ch - 1) / ch;
    P = std::max(1, std::min(P, nchunks));
    return BatchPlan{P, ch};
}

}  // namespace

// ===========================================================================
extern "C" {

const char* carve_cuda_last_error(void) { return t_err.c_str(); }
const char* carve_cuda_version(void) { return "carve_cuda 0.1 (sm_100a)"; }

int carve_cuda_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

carve_status carve_cuda_set_device(int device) {
    return guarded([&] {
        const int n = carve_cuda_device_count();
        if (device < 0 || device >= n) fail(CARVE_E_CUDA, "invalid device index " + std::to_string(device));
        t_device = device;
    });
}

uint64_t carve_cuda_launch_count(void) { return t_launches; }

carve_status carve_cuda_set_kernel_events(int on) {
    return guarded([&] {
        Ctx& c = ctx();
        c.prof = on != 0;
        for (auto& r : c.prof_recs) {
            c.ev_pool.push_back(r.a);
            c.ev_pool.push_back(r.b);
        }
        c.prof_recs.clear();
    });
}

carve_status carve_cuda_kernel_event_stats(int kind, double* ms_total, uint64_t* launches, double* bytes_total) {
    return guarded([&] {
        Ctx& c = ctx();
        sync(c);
        double ms = 0.0, bytes = 0.0;
        uint64_t n = 0;
        for (auto& r : c.prof_recs)
            if (r.kind == kind) {
                float x = 0.f;
                ck(cudaEventElapsedTime(&x, r.a, r.b), "cudaEventElapsedTime");
                ms += x;
                bytes += r.bytes;
                ++n;
            }
        *ms_total = ms;
        *launches = n;
        *bytes_total = bytes;
    });
}
void carve_cuda_reset_launch_count(void) { t_launches = 0; }

carve_status carve_make_test_image(int w, int h, uint32_t variant, uint8_t* out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "PixelGrid dimensions must be >= 1");
        make_test_image_host(w, h, variant, out);
    });
}

carve_status carve_cuda_validate_seam(const int32_t* seam, int n, int w, int h) {
    return guarded([&] { validate_seam_host(seam, n, w, h); });
}

carve_status carve_cuda_to_grayscale(const uint8_t* rgb, int w, int h, double* luma_out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "PixelGrid dimensions must be >= 1");
        Ctx& c = ctx();
        const int pitch = int(round_up(w, 32));
        uint8_t* d_in = static_cast<uint8_t*>(c.packed_in.ensure(size_t(w) * h * 3));
        uint32_t* plane = static_cast<uint32_t*>(c.rgb[0].ensure(size_t(pitch) * h * 4));
        double* l = static_cast<double*>(c.scratch_a.ensure(size_t(w) * h * 8));
        ck(cudaMemcpyAsync(d_in, rgb, size_t(w) * h * 3, cudaMemcpyHostToDevice, c.stream), "H2D");
        launch_unpack(c, d_in, w, h, plane, pitch, 1, 0, 0, c.stream);
        k_luma<<<grid_for((long long)w * h, 256), 256, 0, c.stream>>>(plane, pitch, w, h, l);
        LAUNCHED("k_luma");
        ck(cudaMemcpyAsync(luma_out, l, size_t(w) * h * 8, cudaMemcpyDeviceToHost, c.stream), "D2H");
        sync(c);
    });
}

carve_status carve_cuda_energy_e1_rgb(const uint8_t* rgb, int w, int h, double* e_out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "PixelGrid dimensions must be >= 1");
        Ctx& c = ctx();
        const int pitch = int(round_up(w, 32));
        uint8_t* d_in = static_cast<uint8_t*>(c.packed_in.ensure(size_t(w) * h * 3));
        uint32_t* plane = static_cast<uint32_t*>(c.rgb[0].ensure(size_t(pitch) * h * 4));
        double* e = static_cast<double*>(c.e[0].ensure(size_t(pitch) * h * 8));
        ck(cudaMemcpyAsync(d_in, rgb, size_t(w) * h * 3, cudaMemcpyHostToDevice, c.stream), "H2D");
        launch_unpack(c, d_in, w, h, plane, pitch, 1, 0, 0, c.stream);
        launch_energy(plane, pitch, w, h, e, pitch, 1, 0, 0, c.stream);
        ck(cudaMemcpy2DAsync(e_out, size_t(w) * 8, e, size_t(pitch) * 8, size_t(w) * 8, h, cudaMemcpyDeviceToHost,
                             c.stream),
           "D2H");
        sync(c);
    });
}

carve_status carve_cuda_energy_e1_luma(const double* luma, int w, int h, double* e_out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "LumaGrid dimensions must be >= 1");
        Ctx& c = ctx();
        double* l = static_cast<double*>(c.scratch_a.ensure(size_t(w) * h * 8));
        double* e = static_cast<double*>(c.scratch_b.ensure(size_t(w) * h * 8));
        ck(cudaMemcpyAsync(l, luma, size_t(w) * h * 8, cudaMemcpyHostToDevice, c.stream), "H2D");
        k_energy_luma<<<grid_for((long long)w * h, 256), 256, 0, c.stream>>>(l, w, h, e);
        LAUNCHED("k_energy_luma");
        ck(cudaMemcpyAsync(e_out, e, size_t(w) * h * 8, cudaMemcpyDeviceToHost, c.stream), "D2H");
        sync(c);
    });
}

carve_status carve_cuda_transpose_rgb(const uint8_t* rgb, int w, int h, uint8_t* out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "PixelGrid dimensions must be >= 1");
        Ctx& c = ctx();
        const int pa = int(round_up(w, 32)), pb = int(round_up(h, 32));
        uint8_t* d_in = static_cast<uint8_t*>(c.packed_in.ensure(size_t(w) * h * 3));
        uint8_t* d_out = static_cast<uint8_t*>(c.packed_out.ensure(size_t(w) * h * 3));
        uint32_t* a = static_cast<uint32_t*>(c.rgb[0].ensure(size_t(pa) * h * 4));
        uint32_t* b = static_cast<uint32_t*>(c.rgb[1].ensure(size_t(pb) * w * 4));
        ck(cudaMemcpyAsync(d_in, rgb, size_t(w) * h * 3, cudaMemcpyHostToDevice, c.stream), "H2D");
        launch_unpack(c, d_in, w, h, a, pa, 1, 0, 0, c.stream);
        launch_transpose(a, pa, w, h, b, pb, 1, 0, 0, c.stream);
        launch_pack(c, b, pb, h, w, false, d_out, 1, 0, 0, c.stream);
        ck(cudaMemcpyAsync(out, d_out, size_t(w) * h * 3, cudaMemcpyDeviceToHost, c.stream), "D2H");
        sync(c);
    });
}

carve_status carve_cuda_dp_seam(const double* e, int w, int h, double* m_out, int32_t* b_out, int32_t* seam_out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "image is empty");
        if ((m_out == nullptr) != (b_out == nullptr)) fail(CARVE_E_USAGE_ERROR, "m_out and b_out go together");
        Ctx& c = ctx();
        const Dp2Plan pl = dp2_plan(w, h);
        const int pitch = int(round_up(w, 32));
        const int epitch = padded_epitch(w);
        double* de = static_cast<double*>(c.e[0].ensure(size_t(epitch) * (h + EPAD_B) * 8)) + EPAD_L;
        double* mb = static_cast<double*>(c.mbound.ensure(size_t(pl.nblk + 1) * pitch * 8));
        int* dseam = static_cast<int*>(c.seams.ensure(size_t(h) * 4));
        double* dm = nullptr;
        int* db = nullptr;
        if (m_out) {
            dm = static_cast<double*>(c.scratch_a.ensure(size_t(w) * h * 8));
            db = static_cast<int*>(c.scratch_b.ensure(size_t(w) * h * 4));
        }
        ck(cudaMemcpy2DAsync(de, size_t(epitch) * 8, e, size_t(w) * 8, size_t(w) * 8, h, cudaMemcpyHostToDevice,
                             c.stream),
           "H2D energy");
        launch_fill_pads(de, epitch, w, h, 1, 0, c.stream);
        Dp2Params p{};
        p.e = de;
        p.epitch = epitch;
        p.W = w;
        p.H = h;
        p.mbound = mb;
        p.mpitch = pitch;
        p.seam = dseam;
        p.m_out = dm;
        p.b_out = db;
        launch_dp2(c, pl, p, 1, c.stream);
        ck(cudaMemcpyAsync(seam_out, dseam, size_t(h) * 4, cudaMemcpyDeviceToHost, c.stream), "D2H seam");
        if (m_out) {
            ck(cudaMemcpyAsync(m_out, dm, size_t(w) * h * 8, cudaMemcpyDeviceToHost, c.stream), "D2H m");
            ck(cudaMemcpyAsync(b_out, db, size_t(w) * h * 4, cudaMemcpyDeviceToHost, c.stream), "D2H b");
        }
        sync(c);
    });
}

carve_status carve_cuda_dp_profile(const double* e, int w, int h, long long* counters, int ncounters, int* warps) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "image is empty");
        Ctx& c = ctx();
        const Dp2Plan pl = dp2_plan(w, h);
        const int pitch = int(round_up(w, 32));
        const int epitch = padded_epitch(w);
        double* de = static_cast<double*>(c.e[0].ensure(size_t(epitch) * (h + EPAD_B) * 8)) + EPAD_L;
        double* mb = static_cast<double*>(c.mbound.ensure(size_t(pl.nblk + 1) * pitch * 8));
        int* dseam = static_cast<int*>(c.seams.ensure(size_t(h) * 4));
        const int G = pl.ncl * pl.v->NW;
        long long* dprof = static_cast<long long*>(c.scratch_a.ensure(size_t(G) * 8 * 8));
        ck(cudaMemcpy2DAsync(de, size_t(epitch) * 8, e, size_t(w) * 8, size_t(w) * 8, h, cudaMemcpyHostToDevice,
                             c.stream),
           "H2D energy");
        launch_fill_pads(de, epitch, w, h, 1, 0, c.stream);
        Dp2Params p{};
        p.e = de;
        p.epitch = epitch;
        p.W = w;
        p.H = h;
        p.mbound = mb;
        p.mpitch = pitch;
        p.seam = dseam;
        p.prof = dprof;
        launch_dp2(c, pl, p, 1, c.stream);
        ck(cudaMemcpyAsync(counters, dprof, size_t(std::min(ncounters, G * 8)) * 8, cudaMemcpyDeviceToHost, c.stream),
           "D2H prof");
        sync(c);
        *warps = G;
    });
}

carve_status carve_cuda_insert_columns_rgb(const uint8_t* rgb, int w, int h, const int32_t* cols, int n,
                                           uint8_t* out) {
    return guarded([&] {
        // detail::insert_columns (carver.hpp:118-132): no connectivity requirement;
        // columns outside [0, w) would be undefined behaviour in the reference
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "PixelGrid dimensions must be >= 1");
        if (n != h) fail(CARVE_E_INVALID_SEAM, "one column per row is required");
        for (int i = 0; i < n; ++i)
            if (cols[i] < 0 || cols[i] >= w) fail(CARVE_E_INVALID_SEAM, "column out of range");
        Ctx& c = ctx();
        uint8_t* d_in = static_cast<uint8_t*>(c.packed_in.ensure(size_t(w) * h * 3));
        uint8_t* d_out = static_cast<uint8_t*>(c.packed_out.ensure(size_t(w + 1) * h * 3));
        int* ds = static_cast<int*>(c.rec.ensure(size_t(h) * 4));
        ck(cudaMemcpyAsync(d_in, rgb, size_t(w) * h * 3, cudaMemcpyHostToDevice, c.stream), "H2D");
        ck(cudaMemcpyAsync(ds, cols, size_t(h) * 4, cudaMemcpyHostToDevice, c.stream), "H2D cols");
        launch_expand_rows(d_in, w, h, ds, 1, h, d_out, c.stream);
        ck(cudaMemcpyAsync(out, d_out, size_t(w + 1) * h * 3, cudaMemcpyDeviceToHost, c.stream), "D2H");
        sync(c);
    });
}

carve_status carve_cuda_insert_seam_rgb(const uint8_t* rgb, int w, int h, const int32_t* seam, int n, uint8_t* out) {
    return guarded([&] {
        validate_seam_host(seam, n, w, h);  // carver.hpp:138
        Ctx& c = ctx();
        uint8_t* d_in = static_cast<uint8_t*>(c.packed_in.ensure(size_t(w) * h * 3));
        uint8_t* d_out = static_cast<uint8_t*>(c.packed_out.ensure(size_t(w + 1) * h * 3));
        int* ds = static_cast<int*>(c.rec.ensure(size_t(h) * 4));
        ck(cudaMemcpyAsync(d_in, rgb, size_t(w) * h * 3, cudaMemcpyHostToDevice, c.stream), "H2D");
        ck(cudaMemcpyAsync(ds, seam, size_t(h) * 4, cudaMemcpyHostToDevice, c.stream), "H2D seam");
        launch_expand_rows(d_in, w, h, ds, 1, h, d_out, c.stream);
        ck(cudaMemcpyAsync(out, d_out, size_t(w + 1) * h * 3, cudaMemcpyDeviceToHost, c.stream), "D2H");
        sync(c);
    });
}

carve_status carve_cuda_record_seams(const uint8_t* rgb, int w, int h, int count, const carve_cuda_config* cfg,
                                     int32_t* seams_out, carve_seam_timing* timings_out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "PixelGrid dimensions must be >= 1");
        if (count < 0 || count > w - 1) fail(CARVE_E_INVALID_TARGET, "cannot record more seams than width-1");
        const CarveOpts o = opts_of(cfg);
        if (count == 0) return;
        Ctx& c = ctx();
        uint8_t* d_in = static_cast<uint8_t*>(c.packed_in.ensure(size_t(w) * h * 3));
        int* d_orig = static_cast<int*>(c.rec.ensure(size_t(count) * h * 4));
        const CarveGeometry g = geometry(w, h, w - count, h);
        unsigned long long* d_st = nullptr;
        if (timings_out) {
            d_st = static_cast<unsigned long long*>(c.stamps.ensure(stamp_words(g) * 8));
            ck(cudaMemsetAsync(d_st, 0, stamp_words(g) * 8, c.stream), "memset stamps");
        }
        ck(cudaMemcpyAsync(d_in, rgb, size_t(w) * h * 3, cudaMemcpyHostToDevice, c.stream), "H2D");
        record_device(c, d_in, w, h, count, d_orig, d_st, o);
        ck(cudaMemcpyAsync(seams_out, d_orig, size_t(count) * h * 4, cudaMemcpyDeviceToHost, c.stream), "D2H seams");
        std::vector<unsigned long long> st;
        if (timings_out) {
            st.resize(stamp_words(g));
            ck(cudaMemcpyAsync(st.data(), d_st, st.size() * 8, cudaMemcpyDeviceToHost, c.stream), "D2H stamps");
        }
        sync(c);
        if (timings_out) stamps_to_timings(st, count, timings_out);
    });
}

carve_status carve_cuda_enlarge(const uint8_t* rgb, int w, int h, int target_w, int target_h,
                                const carve_cuda_config* cfg, uint8_t* rgb_out, int32_t* seams_out) {
    return carve_cuda_enlarge_timed(rgb, w, h, target_w, target_h, cfg, rgb_out, seams_out, nullptr);
}

carve_status carve_cuda_enlarge_timed(const uint8_t* rgb, int w, int h, int target_w, int target_h,
                                      const carve_cuda_config* cfg, uint8_t* rgb_out, int32_t* seams_out,
                                      carve_seam_timing* timings_out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "PixelGrid dimensions must be >= 1");
        if (target_w != w) check_enlarge(w, target_w);
        if (target_h != h) check_enlarge(h, target_h);
        const CarveOpts o = opts_of(cfg);
        Ctx& c = ctx();
        const int kw = target_w - w, kh = target_h - h;
        const size_t big = size_t(target_w) * target_h * 3;
        uint8_t* d_in = static_cast<uint8_t*>(c.packed_in.ensure(size_t(w) * h * 3));
        uint8_t* d_out = static_cast<uint8_t*>(c.packed_out.ensure(big));
        uint8_t* e0 = static_cast<uint8_t*>(c.enl[0].ensure(big));
        uint8_t* e1p = static_cast<uint8_t*>(c.enl[1].ensure(big));
        uint8_t* e2 = static_cast<uint8_t*>(c.enl[2].ensure(big));
        const size_t nrec = size_t(kw) * h + size_t(kh) * target_w;
        int* d_orig = static_cast<int*>(c.rec.ensure(std::max<size_t>(nrec, 1) * 4));
        // per-seam stamps of both recordings (the reports' per_seam, carver.hpp:299-309)
        const size_t swa = size_t(kw) * kStampsPerSeam + 4, swb = size_t(kh) * kStampsPerSeam + 4;
        unsigned long long* d_st = nullptr;
        if (timings_out && (kw > 0 || kh > 0)) {
            d_st = static_cast<unsigned long long*>(c.stamps.ensure((swa + swb) * 8));
            ck(cudaMemsetAsync(d_st, 0, (swa + swb) * 8, c.stream), "memset stamps");
        }
        ck(cudaMemcpyAsync(d_in, rgb, size_t(w) * h * 3, cudaMemcpyHostToDevice, c.stream), "H2D");
        const uint8_t* cur = d_in;
        if (kw > 0) {  // enlarge_to_width (carver.hpp:266-285)
            record_device(c, d_in, w, h, kw, d_orig, d_st, o);
            launch_expand_rows(d_in, w, h, d_orig, kw, h, e0, c.stream);
            cur = e0;
        }
        if (kh > 0) {  // the height: enlarge_to_width of the transpose (cli.hpp:271-274)
            int* d_orig_h = d_orig + size_t(kw) * h;
            transpose_packed(c, cur, target_w, h, e1p);  // h wide, target_w high
            record_device(c, e1p, h, target_w, kh, d_orig_h, d_st ? d_st + swa : nullptr, o);
            launch_expand_rows(e1p, h, target_w, d_orig_h, kh, target_w, e2, c.stream);
            transpose_packed(c, e2, target_h, target_w, d_out);
            cur = d_out;
        }
        ck(cudaMemcpyAsync(rgb_out, cur, big, cudaMemcpyDeviceToHost, c.stream), "D2H");
        if (seams_out && nrec)
            ck(cudaMemcpyAsync(seams_out, d_orig, nrec * 4, cudaMemcpyDeviceToHost, c.stream), "D2H seams");
        std::vector<unsigned long long> st;
        if (d_st) {
            st.resize(swa + swb);
            ck(cudaMemcpyAsync(st.data(), d_st, st.size() * 8, cudaMemcpyDeviceToHost, c.stream), "D2H stamps");
        }
        sync(c);
        if (d_st) {
            std::vector<unsigned long long> b(st.begin() + swa, st.end());
            stamps_to_timings(st, kw, timings_out);
            stamps_to_timings(b, kh, timings_out + kw);
        }
    });
}

carve_status carve_cuda_remove_seam_rgb(const uint8_t* rgb, int w, int h, const int32_t* seam, int n, uint8_t* out) {
    return guarded([&] {
        validate_seam_host(seam, n, w, h);  // carver.hpp:72
        if (w < 2) fail(CARVE_E_WIDTH_TOO_SMALL, "cannot remove a seam from a 1-pixel-wide image");
        Ctx& c = ctx();
        const int pitch = int(round_up(w, 32));
        uint8_t* d_in = static_cast<uint8_t*>(c.packed_in.ensure(size_t(w) * h * 3));
        uint8_t* d_out = static_cast<uint8_t*>(c.packed_out.ensure(size_t(w - 1) * h * 3));
        uint32_t* a = static_cast<uint32_t*>(c.rgb[0].ensure(size_t(pitch) * h * 4));
        uint32_t* b = static_cast<uint32_t*>(c.rgb[1].ensure(size_t(pitch) * h * 4));
        int* ds = static_cast<int*>(c.seams.ensure(size_t(h) * 4));
        ck(cudaMemcpyAsync(d_in, rgb, size_t(w) * h * 3, cudaMemcpyHostToDevice, c.stream), "H2D");
        ck(cudaMemcpyAsync(ds, seam, size_t(h) * 4, cudaMemcpyHostToDevice, c.stream), "H2D seam");
        launch_unpack(c, d_in, w, h, a, pitch, 1, 0, 0, c.stream);
        CompactParams q{};
        q.rgb_in = a;
        q.rgb_out = b;
        q.pitch = pitch;
        q.W = w;
        q.H = h;
        q.seam = ds;
        launch_compact(q, 1, c.stream);
        launch_pack(c, b, pitch, w - 1, h, false, d_out, 1, 0, 0, c.stream);
        ck(cudaMemcpyAsync(out, d_out, size_t(w - 1) * h * 3, cudaMemcpyDeviceToHost, c.stream), "D2H");
        sync(c);
    });
}

carve_status carve_cuda_carve(const uint8_t* rgb, int w, int h, int target_w, int target_h, uint8_t* rgb_out,
                              int32_t* seams_out, carve_seam_timing* timings_out) {
    return guarded([&] {
        check_targets(w, h, target_w, target_h);
        Ctx& c = ctx();
        carve_one_host(c, rgb, w, h, target_w, target_h, rgb_out, seams_out, timings_out);
    });
}

carve_status carve_cuda_carve_cfg(const uint8_t* rgb, int w, int h, int target_w, int target_h,
                                  const carve_cuda_config* cfg, uint8_t* rgb_out, int32_t* seams_out,
                                  carve_seam_timing* timings_out) {
    return guarded([&] {
        check_targets(w, h, target_w, target_h);
        const CarveOpts o = opts_of(cfg);
        Ctx& c = ctx();
        carve_one_host(c, rgb, w, h, target_w, target_h, rgb_out, seams_out, timings_out, o);
    });
}

carve_status carve_cuda_forward_costs(const double* luma, int w, int h, double* left, double* up, double* right) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "LumaGrid dimensions must be >= 1");
        Ctx& c = ctx();
        const size_t n = size_t(w) * h;
        double* l = static_cast<double*>(c.scratch_a.ensure(n * 8 * 4));
        ck(cudaMemcpyAsync(l, luma, n * 8, cudaMemcpyHostToDevice, c.stream), "H2D luma");
        k_forward_costs<<<grid_for((long long)n, 256), 256, 0, c.stream>>>(l, w, h, l + n, l + 2 * n, l + 3 * n, w);
        LAUNCHED("k_forward_costs");
        ck(cudaMemcpyAsync(left, l + n, n * 8, cudaMemcpyDeviceToHost, c.stream), "D2H left");
        ck(cudaMemcpyAsync(up, l + 2 * n, n * 8, cudaMemcpyDeviceToHost, c.stream), "D2H up");
        ck(cudaMemcpyAsync(right, l + 3 * n, n * 8, cudaMemcpyDeviceToHost, c.stream), "D2H right");
        sync(c);
    });
}

}  // extern "C"
namespace {
// dp_seam_forward (solvers.hpp:294-326) on three padded device cost planes
// (cost_left at d_costs, cost_up at + cplane, cost_right at + 2*cplane)
void dp_forward_on_planes(Ctx& c, double* d_costs, int epitch, long long cplane, int w, int h, double* m_out,
                          int32_t* b_out, int32_t* seam_out) {
    const Dp2Plan pl = dp2_plan(w, h, false, RING_COSTS);
    const int pitch = int(round_up(w, 32));
    double* mb = static_cast<double*>(c.mbound.ensure(size_t(pl.nblk + 1) * pitch * 8));
    int* dseam = static_cast<int*>(c.seams.ensure(size_t(h) * 4));
    double* dm = nullptr;
    int* db = nullptr;
    if (m_out) {
        dm = static_cast<double*>(c.scratch_a.ensure(size_t(w) * h * 8));
        db = static_cast<int*>(c.scratch_b.ensure(size_t(w) * h * 4));
    }
    Dp2Params p{};
    p.e = d_costs;
    p.cplane = cplane;
    p.epitch = epitch;
    p.W = w;
    p.H = h;
    p.mbound = mb;
    p.mpitch = pitch;
    p.seam = dseam;
    p.m_out = dm;
    p.b_out = db;
    launch_dp2(c, pl, p, 1, c.stream, false, true);
    ck(cudaMemcpyAsync(seam_out, dseam, size_t(h) * 4, cudaMemcpyDeviceToHost, c.stream), "D2H seam");
    if (m_out) {
        ck(cudaMemcpyAsync(m_out, dm, size_t(w) * h * 8, cudaMemcpyDeviceToHost, c.stream), "D2H m");
        ck(cudaMemcpyAsync(b_out, db, size_t(w) * h * 4, cudaMemcpyDeviceToHost, c.stream), "D2H b");
    }
    sync(c);
}

// three padded FP64 cost planes in c.e[0] (rows of epitch doubles, EPAD_B spare rows)
double* cost_planes(Ctx& c, int w, int h, int& epitch, long long& cplane) {
    epitch = padded_epitch(w);
    cplane = (long long)epitch * (h + EPAD_B);
    return static_cast<double*>(c.e[0].ensure(size_t(cplane) * 3 * 8)) + EPAD_L;
}
}  // namespace
extern "C" {

carve_status carve_cuda_dp_seam_forward(const double* luma, int w, int h, double* m_out, int32_t* b_out,
                                        int32_t* seam_out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "image is empty");
        if ((m_out == nullptr) != (b_out == nullptr)) fail(CARVE_E_USAGE_ERROR, "m_out and b_out go together");
        Ctx& c = ctx();
        int epitch;
        long long cplane;
        double* d = cost_planes(c, w, h, epitch, cplane);
        // forward_costs(gray) on the device, straight into the DP's padded planes
        double* dl = static_cast<double*>(c.scratch_b.ensure(size_t(w) * h * 8));
        ck(cudaMemcpyAsync(dl, luma, size_t(w) * h * 8, cudaMemcpyHostToDevice, c.stream), "H2D luma");
        k_forward_costs<<<grid_for((long long)w * h, 256), 256, 0, c.stream>>>(dl, w, h, d, d + cplane,
                                                                              d + 2 * cplane, epitch);
        LAUNCHED("k_forward_costs");
        dp_forward_on_planes(c, d, epitch, cplane, w, h, m_out, b_out, seam_out);
    });
}

carve_status carve_cuda_dp_seam_forward_costs(const double* left, const double* up, const double* right, int w,
                                              int h, double* m_out, int32_t* b_out, int32_t* seam_out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "image is empty");
        if ((m_out == nullptr) != (b_out == nullptr)) fail(CARVE_E_USAGE_ERROR, "m_out and b_out go together");
        // the device scan compares finite candidates (out-of-image neighbours are +inf);
        // the reference's best = +inf start differs from it only for non-finite costs
        const size_t n = size_t(w) * h;
        for (const double* pl : {left, up, right})
            for (size_t k = 0; k < n; ++k)
                if (!std::isfinite(pl[k]))
                    fail(CARVE_E_USAGE_ERROR, "non-finite forward costs are not supported by the B200 engine");
        Ctx& c = ctx();
        int epitch;
        long long cplane;
        double* d = cost_planes(c, w, h, epitch, cplane);
        const double* src[3] = {left, up, right};
        for (int k = 0; k < 3; ++k)
            ck(cudaMemcpy2DAsync(d + k * cplane, size_t(epitch) * 8, src[k], size_t(w) * 8, size_t(w) * 8, h,
                                 cudaMemcpyHostToDevice, c.stream),
               "H2D costs");
        dp_forward_on_planes(c, d, epitch, cplane, w, h, m_out, b_out, seam_out);
    });
}

}  // extern "C"
namespace {
// remove_seam on a scalar plane (carver.hpp:84-112): the reference does not
// validate these overloads; out-of-range columns would be undefined behaviour
// there, so they are rejected here with invalid_seam
template <typename T>
void drop_columns_device(const T* in, int w, int h, const int32_t* seam, int n, T* out) {
    if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "plane dimensions must be >= 1");
    if (n != h) fail(CARVE_E_INVALID_SEAM, "seam length does not match the plane height");
    for (int i = 0; i < n; ++i)
        if (seam[i] < 0 || seam[i] >= w) fail(CARVE_E_INVALID_SEAM, "seam column out of range");
    Ctx& c = ctx();
    const size_t nin = size_t(w) * h, nout = size_t(w - 1) * h;
    T* d_in = static_cast<T*>(c.scratch_a.ensure(nin * sizeof(T)));
    T* d_out = static_cast<T*>(c.scratch_b.ensure(std::max<size_t>(nout, 1) * sizeof(T)));
    int* ds = static_cast<int*>(c.seams.ensure(size_t(h) * 4));
    ck(cudaMemcpyAsync(d_in, in, nin * sizeof(T), cudaMemcpyHostToDevice, c.stream), "H2D plane");
    ck(cudaMemcpyAsync(ds, seam, size_t(h) * 4, cudaMemcpyHostToDevice, c.stream), "H2D seam");
    if (nout) {
        k_drop_columns<T><<<grid_for((long long)nout, 256), 256, 0, c.stream>>>(d_in, w, h, ds, d_out);
        LAUNCHED("k_drop_columns");
        ck(cudaMemcpyAsync(out, d_out, nout * sizeof(T), cudaMemcpyDeviceToHost, c.stream), "D2H plane");
    }
    sync(c);
}
}  // namespace
extern "C" {

carve_status carve_cuda_remove_seam_f64(const double* in, int w, int h, const int32_t* seam, int n, double* out) {
    return guarded([&] { drop_columns_device<double>(in, w, h, seam, n, out); });
}

carve_status carve_cuda_remove_seam_u8(const uint8_t* in, int w, int h, const int32_t* seam, int n, uint8_t* out) {
    return guarded([&] { drop_columns_device<uint8_t>(in, w, h, seam, n, out); });
}

carve_status carve_cuda_mask_from_rgb(const uint8_t* rgb, int w, int h, uint8_t* flags) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "PixelGrid dimensions must be >= 1");
        Ctx& c = ctx();
        const long long n = (long long)w * h;
        uint8_t* d_in = static_cast<uint8_t*>(c.packed_in.ensure(size_t(n) * 3));
        uint8_t* d_f = static_cast<uint8_t*>(c.packed_out.ensure(size_t(n)));
        ck(cudaMemcpyAsync(d_in, rgb, size_t(n) * 3, cudaMemcpyHostToDevice, c.stream), "H2D");
        k_mask_from_rgb<<<grid_for(n, 256), 256, 0, c.stream>>>(d_in, n, d_f);
        LAUNCHED("k_mask_from_rgb");
        ck(cudaMemcpyAsync(flags, d_f, size_t(n), cudaMemcpyDeviceToHost, c.stream), "D2H");
        sync(c);
    });
}

carve_status carve_cuda_apply_mask(const double* e, int w, int h, const uint8_t* mask, double* out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "EnergyMap dimensions must be >= 1");
        Ctx& c = ctx();
        const size_t n = size_t(w) * h;
        double* d_e = static_cast<double*>(c.scratch_a.ensure(n * 16));
        uint8_t* d_m = static_cast<uint8_t*>(c.packed_in.ensure(n));
        MaskStats* st = static_cast<MaskStats*>(c.stats.ensure(sizeof(MaskStats)));
        ck(cudaMemcpyAsync(d_e, e, n * 8, cudaMemcpyHostToDevice, c.stream), "H2D e");
        ck(cudaMemcpyAsync(d_m, mask, n, cudaMemcpyHostToDevice, c.stream), "H2D mask");
        ck(cudaMemsetAsync(st, 0, sizeof(MaskStats), c.stream), "memset stats");
        k_mask_stats<true><<<grid_for((long long)n, 256), 256, 0, c.stream>>>(d_e, w, d_m, nullptr, 0, w, h, st);
        LAUNCHED("k_mask_stats");
        k_apply_mask<true><<<grid_for((long long)n, 256), 256, 0, c.stream>>>(d_e, w, d_m, nullptr, 0, w, h, st,
                                                                              d_e + n, w, 0);
        LAUNCHED("k_apply_mask");
        ck(cudaMemcpyAsync(out, d_e + n, n * 8, cudaMemcpyDeviceToHost, c.stream), "D2H");
        sync(c);
    });
}

carve_status carve_cuda_remove_object_ex(const uint8_t* rgb, int w, int h, const uint8_t* mask,
                                         const carve_cuda_config* cfg, int restore, int orientation,
                                         uint8_t* rgb_out, int* out_w, int* out_h, int32_t* seams_out, int* nseams,
                                         carve_seam_timing* timings_out) {
    return guarded([&] {
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "PixelGrid dimensions must be >= 1");
        if (orientation < 0 || orientation > 1) fail(CARVE_E_USAGE_ERROR, "orientation must be 0 (auto) or 1");
        const CarveOpts o = opts_of(cfg);
        // mask_bounds (energy.hpp:272-283) of the caller's flags: picks the orientation
        int top = h, left = w, bottom = -1, right = -1;
        for (int i = 0; i < h; ++i)
            for (int j = 0; j < w; ++j)
                if (mask[size_t(i) * w + j]) {
                    top = std::min(top, i);
                    left = std::min(left, j);
                    bottom = std::max(bottom, i);
                    right = std::max(right, j);
                }
        // remove_object fails on an empty mask (carver.hpp:333); remove_object_vertical
        // (orientation 1) just carves nothing (its loop condition, carver.hpp:297)
        if (bottom < top && orientation == 0) fail(CARVE_E_EMPTY_MASK, "removal mask marks no pixels");
        const bool transposed = orientation == 0 && right - left + 1 > bottom - top + 1;
        Ctx& c = ctx();
        cudaStream_t s = c.stream;
        const size_t n = size_t(w) * h;
        // the vertical loop runs on a W x H view: the image itself or its transpose
        const int W = transposed ? h : w, H = transposed ? w : h;
        const int pitch = padded_epitch(W), epitch = padded_epitch(W);
        const size_t plane = size_t(pitch) * (H + EPAD_B);
        uint8_t* d_in = static_cast<uint8_t*>(c.packed_in.ensure(n * 3));
        uint8_t* d_mask = static_cast<uint8_t*>(c.enl[2].ensure(n));
        uint32_t* rgbx = static_cast<uint32_t*>(c.rgb[0].ensure(plane * 4)) + EPAD_L;
        double* e = static_cast<double*>(c.e[0].ensure(plane * 8)) + EPAD_L;
        double* eb = static_cast<double*>(c.e[1].ensure(plane * 8)) + EPAD_L;
        // the removal's seam log (c.seams belongs to the carve loop the restore runs)
        int* d_seams = static_cast<int*>(c.dir.ensure(std::max<size_t>(n, 1) * 4));
        MaskStats* st = static_cast<MaskStats*>(c.stats.ensure(sizeof(MaskStats) + 64));
        int* d_flags = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(st) + sizeof(MaskStats) + 32);  // done, count
        unsigned long long* d_st = nullptr;
        if (timings_out) {
            d_st = static_cast<unsigned long long*>(c.stamps.ensure(size_t(W) * kStampsPerSeam * 8));
            ck(cudaMemsetAsync(d_st, 0, size_t(W) * kStampsPerSeam * 8, s), "memset stamps");
        }
        const int mpitch = epitch;
        double* mb = static_cast<double*>(c.mbound.ensure(size_t((H + LBLK - 1) / LBLK + 1) * mpitch * 8));
        ck(cudaMemcpyAsync(d_in, rgb, n * 3, cudaMemcpyHostToDevice, s), "H2D rgb");
        ck(cudaMemcpyAsync(d_mask, mask, n, cudaMemcpyHostToDevice, s), "H2D mask");
        ck(cudaMemsetAsync(d_flags, 0, 8, s), "memset flags");
        if (!transposed) {
            k_unpack_masked<<<grid_for((long long)n, 256), 256, 0, s>>>(d_in, d_mask, w, h, rgbx, pitch);
            LAUNCHED("k_unpack_masked");
        } else {  // transpose(grid), transpose(mask) (carver.hpp:337-339): the mask bit travels along
            uint32_t* tmp = static_cast<uint32_t*>(c.rgb[1].ensure(size_t(round_up(w, 32)) * h * 4));
            const int tp = int(round_up(w, 32));
            k_unpack_masked<<<grid_for((long long)n, 256), 256, 0, s>>>(d_in, d_mask, w, h, tmp, tp);
            LAUNCHED("k_unpack_masked");
            launch_transpose(tmp, tp, w, h, rgbx, pitch, 1, 0, 0, s);
        }
        // e1 of the start image; +inf pads on both planes (SPEC.md:315 exclusion)
        launch_energy(rgbx, pitch, W, H, e, epitch, 1, 0, 0, s);
        launch_fill_pads(e, epitch, W, H, 1, 0, s);
        launch_fill_pads(eb, epitch, W, H, 1, 0, s);
        // remove_object_vertical (carver.hpp:291-315), one seam per iteration: stats ->
        // stop test -> biased map -> DP -> removal of image, mask and map -> fix-up.
        // The loop length is data-dependent; iterations are enqueued in batches without
        // a host round trip per seam: k_mask_decide sets a device flag once no marked
        // pixel is left, and every later kernel of the batch returns at once. The host
        // reads the flag once per batch (batch sizes start at the mask's bounding-box
        // width and double).
        int cw = W, issued = 0, ns = 0, batch = std::max(1, bottom < top ? 1 : (transposed ? bottom - top : right - left) + 1);
        int done = 0;
        const int* stop = d_flags;
        for (;;) {
            const int nb = std::min(batch, cw - 1);  // every iteration of the batch starts at width >= 2
            for (int b = 0; b < nb; ++b, ++issued, --cw) {
                unsigned long long* sk = d_st ? d_st + size_t(issued) * kStampsPerSeam : nullptr;
                ck(cudaMemsetAsync(st, 0, sizeof(MaskStats), s), "memset stats");
                k_mask_stats<false><<<grid_for((long long)cw * H, 256), 256, 0, s>>>(e, epitch, nullptr, rgbx, pitch,
                                                                                    cw, H, st, stop, sk);
                LAUNCHED("k_mask_stats");
                k_mask_decide<<<1, 1, 0, s>>>(st, d_flags, d_flags + 1);
                LAUNCHED("k_mask_decide");
                k_apply_mask<false><<<grid_for((long long)cw * H, 256), 256, 0, s>>>(
                    e, epitch, nullptr, rgbx, pitch, cw, H, st, eb, epitch, 1, stop, sk ? sk + 1 : nullptr);
                LAUNCHED("k_apply_mask");
                int* seam = d_seams + size_t(issued) * H;
                const Dp2Plan pl = dp2_plan(cw, H);
                Dp2Params q{};
                q.e = eb;
                q.epitch = epitch;
                q.W = cw;
                q.H = H;
                q.mbound = mb;
                q.mpitch = mpitch;
                q.seam = seam;
                q.stop = stop;
                q.stamps = sk;
                launch_dp2(c, pl, q, 1, s);
                CompactParams r{};
                r.rgb_in = r.rgb_out = rgbx;
                r.e_in = r.e_out = e;
                r.pitch = pitch;
                r.epitch = epitch;
                r.W = cw;
                r.H = H;
                r.seam = seam;
                r.stop = stop;
                r.stamps = sk ? sk + 4 : nullptr;
                launch_compact_inplace(r, 1, s);
                k_fixup_energy<<<grid_for(H, 256), 256, 0, s>>>(e, epitch, rgbx, pitch, cw - 1, H, seam, stop,
                                                                sk ? sk + 5 : nullptr);
                LAUNCHED("k_fixup_energy");
            }
            int hv[2];
            ck(cudaMemcpyAsync(hv, d_flags, 8, cudaMemcpyDeviceToHost, s), "D2H flags");
            sync(c);
            done = hv[0];
            ns = hv[1];
            if (done) break;
            if (cw < 2) {
                // width 1 with marked pixels left (carver.hpp:298-299), unless the last
                // batch's final seam removed them: one more stop test at width 1
                ck(cudaMemsetAsync(st, 0, sizeof(MaskStats), s), "memset stats");
                k_mask_stats<false><<<grid_for((long long)cw * H, 256), 256, 0, s>>>(e, epitch, nullptr, rgbx, pitch,
                                                                                    cw, H, st, stop, nullptr);
                LAUNCHED("k_mask_stats");
                unsigned long long marked = 0;
                ck(cudaMemcpyAsync(&marked, &st->marked, 8, cudaMemcpyDeviceToHost, s), "D2H marked");
                sync(c);
                if (marked) fail(CARVE_E_WIDTH_TOO_SMALL, "mask cannot be carved out of a 1-pixel-wide image");
                break;
            }
            batch *= 2;
        }
        cw = W - ns;  // the width after the last seam actually carved
        // restore (carver.hpp:309-313): enlarge_to_width back to the original width
        uint8_t* d_cur = static_cast<uint8_t*>(c.packed_out.ensure(n * 3));
        launch_pack(c, rgbx, pitch, cw, H, false, d_cur, 1, 0, 0, s);
        const uint8_t* res = d_cur;
        int rw = cw;
        if (restore && cw < W) {
            uint8_t* d_big = static_cast<uint8_t*>(c.enl[0].ensure(n * 3));
            int* d_orig = static_cast<int*>(c.rec.ensure(size_t(W - cw) * H * 4));
            check_enlarge(cw, W);
            record_device(c, d_cur, cw, H, W - cw, d_orig, nullptr, o);
            launch_expand_rows(d_cur, cw, H, d_orig, W - cw, H, d_big, s);
            res = d_big;
            rw = W;
        }
        if (transposed) {  // back to the caller's orientation
            uint8_t* d_t = static_cast<uint8_t*>(c.enl[1].ensure(n * 3));
            transpose_packed(c, res, rw, H, d_t);
            res = d_t;
        }
        *out_w = transposed ? w : rw;
        *out_h = transposed ? rw : h;
        ck(cudaMemcpyAsync(rgb_out, res, size_t(rw) * H * 3, cudaMemcpyDeviceToHost, s), "D2H");
        if (seams_out && ns)
            ck(cudaMemcpyAsync(seams_out, d_seams, size_t(ns) * H * 4, cudaMemcpyDeviceToHost, s), "D2H seams");
        std::vector<unsigned long long> sth;
        if (timings_out && ns) {
            sth.resize(size_t(ns) * kStampsPerSeam);
            ck(cudaMemcpyAsync(sth.data(), d_st, sth.size() * 8, cudaMemcpyDeviceToHost, s), "D2H stamps");
        }
        sync(c);
        if (timings_out && ns) stamps_to_timings(sth, ns, timings_out);
        if (nseams) *nseams = ns;
    });
}

carve_status carve_cuda_remove_object(const uint8_t* rgb, int w, int h, const uint8_t* mask,
                                      const carve_cuda_config* cfg, int restore, uint8_t* rgb_out, int* out_w,
                                      int* out_h, int32_t* seams_out, int* nseams) {
    return carve_cuda_remove_object_ex(rgb, w, h, mask, cfg, restore, 0, rgb_out, out_w, out_h, seams_out, nseams,
                                       nullptr);
}

carve_status carve_cuda_carve_device(const uint8_t* d_rgb, int w, int h, int target_w, int target_h, uint8_t* d_out,
                                     int32_t* d_seams, void* stream) {
    return guarded([&] {
        check_targets(w, h, target_w, target_h);
        Ctx& c = ctx();
        const CarveGeometry g = geometry(w, h, target_w, target_h);
        ensure_carve_buffers(c, g, 1);
        int* seams = d_seams ? d_seams : static_cast<int*>(c.seams.ensure(std::max<size_t>(g.seam_ints, 1) * 4));
        // the context's scratch is ordered on its own stream: forked from and joined back
        // into the caller's stream (NULL = the legacy default stream), so a later call on
        // any stream of this thread cannot overwrite scratch this carve still uses
        StreamFork f(static_cast<cudaStream_t>(stream), c.stream);
        const std::vector<uintptr_t> key = {uintptr_t(w), uintptr_t(h), uintptr_t(target_w), uintptr_t(target_h),
                                            uintptr_t(d_rgb), uintptr_t(d_out), uintptr_t(seams)};
        run_graphed(c, key, [&] { run_carve(c, d_rgb, d_out, 1, g, seams, g.seam_ints, nullptr, c.stream); });
        f.join();
    });
}

carve_status carve_cuda_carve_batch_device(const uint8_t* d_rgb, int n, int w, int h, int target_w, int target_h,
                                           uint8_t* d_out, void* stream) {
    return guarded([&] {
        if (n < 1) fail(CARVE_E_EMPTY_INPUT, "empty batch");
        check_targets(w, h, target_w, target_h);
        Ctx& c = ctx();
        const CarveGeometry g = geometry(w, h, target_w, target_h);
        cudaStream_t s = static_cast<cudaStream_t>(stream);  // NULL = the legacy default stream
        // Split into P concurrent sub-batches (CARVE_DEVICE_SPLIT, of at least
        // CARVE_DEVICE_SPLIT_MIN images), each on its own (device, pipeline) context and
        // stream, forked from and joined back into `s`, so one sub-batch's per-seam
        // launches fill the other's wave tails. Per-kernel event profiling (c.prof) keeps
        // the calling thread's context (one stream, serial launch timings).
        const int want = std::max(1, std::min(CARVE_MAX_PIPELINES, env_int("CARVE_DEVICE_SPLIT", 4)));
        // measured (profiles/r02_share_grid_b.txt): 128 images as 4 x 32 2.82K vs 2 x 64 2.71K
        // images/s, 512 as 4 x 128 3.78K vs 2 x 256 3.75K, 1024 as 4 or 2 sub-batches the same
        const int min_sub = std::max(1, env_int("CARVE_DEVICE_SPLIT_MIN", 32));
        const int P = c.prof ? 1 : std::max(1, std::min(want, n / min_sub));
        const size_t in_bytes = size_t(w) * h * 3, out_bytes = size_t(target_w) * target_h * 3;
        if (c.prof) {
            ensure_carve_buffers(c, g, n);
            int* seams = static_cast<int*>(c.seams.ensure(std::max<size_t>(g.seam_ints, 1) * 4 * n));
            StreamFork f(s, c.stream);
            run_carve(c, d_rgb, d_out, n, g, seams, std::max<size_t>(g.seam_ints, 1), nullptr, c.stream);
            f.join();
            return;
        }
        // every slot's buffers are ensured before any work is enqueued, so a failure
        // (e.g. an allocation) leaves nothing in flight
        SlotSet slots(c.device, P);
        for (int q = 0; q < P; ++q) {
            const int a = int((long long)n * q / P), b = int((long long)n * (q + 1) / P);
            Ctx& cq = slots.use(q);
            ensure_carve_buffers(cq, g, b - a);
            cq.seams.ensure(std::max<size_t>(g.seam_ints, 1) * 4 * (b - a));
        }
        ConcurrencyScope cs(P);
        StreamFork f(s);
        for (int q = 0; q < P; ++q) {
            const int a = int((long long)n * q / P), b = int((long long)n * (q + 1) / P);
            Ctx& cq = slots.use(q);
            f.fork_into(cq.stream);
            run_carve(cq, d_rgb + in_bytes * a, d_out + out_bytes * a, b - a, g, cq.seams.as<int>(),
                      std::max<size_t>(g.seam_ints, 1), nullptr, cq.stream);
            f.join_from(cq.stream);
        }
    });
}

carve_status carve_cuda_batch_plan(int n, int w, int h, int target_w, int target_h, int ndev, int* pipes,
                                   int* chunk) {
    return guarded([&] {
        if (n < 1) fail(CARVE_E_EMPTY_INPUT, "empty batch");
        if (ndev < 1) fail(CARVE_E_USAGE_ERROR, "ndev must be >= 1");
        if (w < 1 || h < 1) fail(CARVE_E_EMPTY_IMAGE, "PixelGrid dimensions must be >= 1");
        if (target_w < 1 || target_w > w || target_h < 1 || target_h > h)
            fail(CARVE_E_INVALID_TARGET, "target must be in [1, size]");
        const BatchPlan p = batch_plan(n, ndev, geometry(w, h, target_w, target_h));
        *pipes = p.pipes;
        *chunk = p.chunk;
    });
}

carve_status carve_cuda_carve_batch(const uint8_t* const* rgb, int n, int w, int h, int target_w, int target_h,
                                    uint8_t* const* rgb_out, const int* devices, int ndev) {
    return guarded([&] {
        if (n < 1) fail(CARVE_E_EMPTY_INPUT, "empty batch");
        check_targets(w, h, target_w, target_h);
        const int avail = carve_cuda_device_count();
        if (avail == 0) fail(CARVE_E_CUDA, "no CUDA device available");
        if (ndev <= 0) ndev = avail;
        std::vector<int> devs(ndev);
        for (int k = 0; k < ndev; ++k) {
            devs[k] = devices ? devices[k] : k;
            if (devs[k] < 0 || devs[k] >= avail) fail(CARVE_E_CUDA, "invalid device index");
        }
        const CarveGeometry g = geometry(w, h, target_w, target_h);
        const BatchPlan plan = batch_plan(n, ndev, g);
        const size_t in_bytes = size_t(w) * h * 3, out_bytes = size_t(target_w) * target_h * 3;
        // SURVEY.md §8e work queue: chunks of whole images are claimed from one atomic
        // counter by one host thread per listed device, so a faster (or less loaded)
        // device takes more chunks; there is no inter-device communication.
        std::atomic<int> next{0};
        std::vector<int> status(ndev, CARVE_OK);
        std::vector<std::string> msgs(ndev);
        auto device_worker = [&](int k) {
            t_device = devs[k];
            status[k] = guarded([&] {
                // P pipelines per device, each a (device, pipeline) context with its own
                // compute stream and buffers; the copies of all of them go through one H2D
                // and one D2H stream (slot 0's), in claim order, so the first chunk's
                // upload does not share PCIe bandwidth with later ones
                const int P = plan.pipes, ch = plan.chunk;
                SlotSet slots(devs[k], P, k);
                Ctx& c0 = slots.use(0);
                c0.ensure_pipeline();
                for (int q = 0; q < P; ++q) {  // allocate everything before enqueuing any work
                    Ctx& cq = slots.use(q);
                    cq.ensure_pipeline();
                    ensure_carve_buffers(cq, g, ch);
                    cq.seams.ensure(std::max<size_t>(g.seam_ints, 1) * 4 * ch);
                    for (int b = 0; b < 2; ++b) {
                        cq.pin_in[b].ensure(in_bytes * ch);
                        cq.pin_out[b].ensure(out_bytes * ch);
                    }
                }
                enum { H2D = 0, COMP = 1, D2H = 2 };
                struct Reset {
                    ~Reset() { t_concurrency = 1; }
                } reset;
                for (int t = 0;; ++t) {
                    const int b0 = next.fetch_add(ch);
                    if (b0 >= n) break;
                    const int m = std::min(ch, n - b0), q = t % P, b = (t / P) & 1;
                    Ctx& cq = slots.use(q);
                    // flow control: at most 2P chunks in flight per device; the buffer pair
                    // (q, b) is reused only after its previous chunk has fully drained
                    if (t >= 2 * P) ck(cudaEventSynchronize(cq.pipe_ev[D2H][b]), "wait d2h");
                    uint8_t* d_in = cq.pin_in[b].as<uint8_t>();
                    uint8_t* d_out = cq.pin_out[b].as<uint8_t>();
                    // one copy per run of images that are contiguous in host memory
                    for (int i = 0; i < m;) {
                        int j = i + 1;
                        while (j < m && rgb[b0 + j] == rgb[b0 + j - 1] + in_bytes) ++j;
                        ck(cudaMemcpyAsync(d_in + in_bytes * i, rgb[b0 + i], in_bytes * (j - i),
                                           cudaMemcpyHostToDevice, c0.h2d),
                           "H2D");
                        i = j;
                    }
                    ck(cudaEventRecord(cq.pipe_ev[H2D][b], c0.h2d), "record h2d");
                    ck(cudaStreamWaitEvent(cq.stream, cq.pipe_ev[H2D][b], 0), "wait h2d");
                    // the DP shape counts the other pipelines' carves (they fill the SMs
                    // alongside this one) unless the whole share is this one chunk
                    t_concurrency = (t == 0 && b0 + m >= n) ? 1 : P;
                    run_carve(cq, d_in, d_out, m, g, cq.seams.as<int>(), std::max<size_t>(g.seam_ints, 1), nullptr,
                              cq.stream);
                    ck(cudaEventRecord(cq.pipe_ev[COMP][b], cq.stream), "record comp");
                    ck(cudaStreamWaitEvent(c0.d2h, cq.pipe_ev[COMP][b], 0), "wait comp");
                    for (int i = 0; i < m;) {
                        int j = i + 1;
                        while (j < m && rgb_out[b0 + j] == rgb_out[b0 + j - 1] + out_bytes) ++j;
                        ck(cudaMemcpyAsync(rgb_out[b0 + i], d_out + out_bytes * i, out_bytes * (j - i),
                                           cudaMemcpyDeviceToHost, c0.d2h),
                           "D2H");
                        i = j;
                    }
                    ck(cudaEventRecord(cq.pipe_ev[D2H][b], c0.d2h), "record d2h");
                }
                ck(cudaStreamSynchronize(c0.d2h), "sync d2h");
                for (int q = 0; q < P; ++q) sync(slots.use(q));
            });
            if (status[k]) msgs[k] = t_err;
        };
        std::vector<std::thread> pool;
        for (int k = 1; k < ndev; ++k) pool.emplace_back(device_worker, k);
        const int saved = t_device;
        device_worker(0);
        t_device = saved;
        for (auto& th : pool) th.join();
        for (int k = 0; k < ndev; ++k)
            if (status[k]) fail(status[k], msgs[k]);
    });
}

}  // extern "C"
