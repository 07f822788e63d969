// ecsr_b200.cu -- libecsr_b200.so: packer, launchers and the C-ABI of include/ecsr_b200.h.
//
// Host responsibilities:
//   * validate a container once (executor.py:50-77, storage.py:312-329) instead of per call;
//   * convert values to fp16 (IEEE RNE) and build the tiled, block-major device arena the
//     fast kernel streams with bulk async copies; byte-balance tiles over a persistent grid;
//   * build the slot tables of the ordered (bitwise-reproducible) y reduction;
//   * keep the cold section (pad_mask, set descriptors) on the host for exact unpack;
//   * expose the reference backend-protocol call spmv_set (_speedups.pyx:55-78).
#include <cuda.h>  // driver API types only (entry points via cudaGetDriverEntryPoint)
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ecsr_b200.h"
#include "ecsr_kernels.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define ECSR_CUDA(expr)                                                                  \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(ECSR_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// bytes of whole records per tile: 16 KB with two CTAs per SM, 32 KB with one. The
// product library has no runtime knobs; a tuning build (-DECSR_B200_TUNING, scripts/
// build_exp.sh, never the shipped .so) reads ECSR_B200_TILE / _PRE / _RECCAP / _RECMAX
// and can record a per-CTA timeline (ECSR_B200_TRACE).
int g_tile_default = 16384;
thread_local int t_tile_override = 0;  // ECSR_PACK_TILE_KB(n) of the pack in progress
#ifdef ECSR_B200_TUNING
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}
int tile_target() {
    const int v = env_int("ECSR_B200_TILE", 0);
    return t_tile_override ? t_tile_override : v ? std::max(1024, v) : g_tile_default;
}
int pre_tiles() { return std::max(0, env_int("ECSR_B200_PRE", 2)); }
bool trace_enabled() { return env_int("ECSR_B200_TRACE", 0) != 0; }
bool trace_caller_resets() { return env_int("ECSR_B200_TRACE", 0) == 2; }
bool coop_launch() { return env_int("ECSR_B200_COOP", 0) != 0; }
bool group_force_cps1() { return env_int("ECSR_B200_GROUP_CPS1", 0) != 0; }
bool pack_ffd() { return env_int("ECSR_B200_FFD", 1) != 0; }
bool pack_mixed() { return env_int("ECSR_B200_MIXED", 1) != 0; }
bool force_full() { return env_int("ECSR_B200_FULL", 0) != 0; }
#else
constexpr bool force_full() { return false; }
constexpr bool coop_launch() { return false; }
constexpr bool group_force_cps1() { return false; }
constexpr bool pack_ffd() { return true; }
constexpr bool pack_mixed() { return true; }
int tile_target() { return t_tile_override ? t_tile_override : g_tile_default; }
int pre_tiles() { return 2; }  // tiles streamed before griddepcontrol.wait and the x copy
constexpr bool trace_enabled() { return false; }
constexpr bool trace_caller_resets() { return false; }
#endif
constexpr int kMaxStageBytes = 65536;   // largest tile a ring slot may hold
#ifndef ECSR_SMEM_RESERVE
#define ECSR_SMEM_RESERVE 4096
#endif
constexpr int64_t kSmemReserve = ECSR_SMEM_RESERVE;  // static shared memory (~1 KB) + margin
constexpr int kMaxStages = 16;
constexpr int kPackInternal = 1 << 30;  // spmv_set: unbounded u32 deltas (validated by range)
constexpr double kQueueShare = 0.05;       // cost share of each CTA's range drawn from the tail
                                           // queue: a single matrix's launch
constexpr double kGroupQueueShare = 0.40;  // the same for a grouped launch (one tail per step,
                                           // members' CTAs sharing SMs: measured best 0.35-0.45)
#ifdef ECSR_B200_TUNING
double group_queue_share() { return env_int("ECSR_B200_GROUP_QPCT", 40) / 100.0; }
#else
double group_queue_share() { return kGroupQueueShare; }
#endif

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// IEEE-754 binary64 -> binary16, round to nearest even (also exact for f32 inputs).
uint16_t f64_to_f16(double d) {
    uint64_t bits;
    std::memcpy(&bits, &d, 8);
    const uint16_t sign = static_cast<uint16_t>((bits >> 48) & 0x8000u);
    if (std::isnan(d)) return sign | 0x7e00u;
    const double a = std::fabs(d);
    if (a >= 65520.0) return sign | 0x7c00u;  // 65520 ties to even -> inf
    if (a < 6.103515625e-05) {                 // below 2^-14: subnormal grid of 2^-24
        const double q = std::nearbyint(a * 16777216.0);  // exact scaling, RNE
        return sign | static_cast<uint16_t>(q);          // q == 1024 encodes 2^-14
    }
    int ex;
    std::frexp(a, &ex);  // a = f * 2^ex, f in [0.5, 1)
    int e = ex - 1;      // a in [2^e, 2^(e+1))
    double m = std::nearbyint(std::ldexp(a, 10 - e));  // in [1024, 2048]
    if (m >= 2048.0) {
        m = 1024.0;
        ++e;
    }
    if (e + 15 >= 31) return sign | 0x7c00u;
    return sign | static_cast<uint16_t>(((e + 15) << 10) | (static_cast<int>(m) - 1024));
}

float f16_to_f32(uint16_t h) {
    const uint32_t s = (h & 0x8000u) << 16;
    const uint32_t e = (h >> 10) & 0x1fu;
    const uint32_t m = h & 0x3ffu;
    float out;
    if (e == 0) {
        out = std::ldexp(static_cast<float>(m), -24);
        uint32_t b;
        std::memcpy(&b, &out, 4);
        b |= s;
        std::memcpy(&out, &b, 4);
        return out;
    }
    uint32_t b;
    if (e == 31)
        b = s | 0x7f800000u | (m << 13);
    else
        b = s | ((e + 112) << 23) | (m << 13);
    std::memcpy(&out, &b, 4);
    return out;
}

double host_value(const void* vals, int dtype, int64_t i) {
    if (dtype == ECSR_F64) return static_cast<const double*>(vals)[i];
    if (dtype == ECSR_F32) return static_cast<const float*>(vals)[i];
    return f16_to_f32(static_cast<const uint16_t*>(vals)[i]);
}

int elem_size(int dtype) { return dtype == ECSR_F64 ? 8 : dtype == ECSR_F32 ? 4 : 2; }

// Per-tile work features (cost-model calibration, ecsr_b200_debug_ctafeat).
struct TileFeat {
    double rec[4] = {0, 0, 0, 0};    // records with g = 1, 2, 4, >= 8
    double steps[4] = {0, 0, 0, 0};  // block-chunk steps (sum over blocks of chunks)
    double bytes = 0;
};
inline int gclass(int g) { return g == 1 ? 0 : g == 2 ? 1 : g == 4 ? 2 : 3; }

struct SetDesc {
    int32_t g = 0, v = 0;
    int64_t nb = 0, stored = 0, real = 0;
    int64_t slot0 = 0;    // global slot of (block 0, row 0)
    int64_t row_off = 0;  // offset into concatenated row_indices (== slot0)
    int64_t base_off = 0, indptr_off = 0, col_off = 0, val_off = 0;
};

// Contiguous tile ranges [cta[c], cta[c+1]) of ~equal summed cost (a tile goes to the
// range holding its cost midpoint).
std::vector<uint32_t> balanced_ranges(const std::vector<double>& tcost, int grid) {
    const int64_t ntiles = static_cast<int64_t>(tcost.size());
    std::vector<uint32_t> cta(grid + 1, 0);
    std::vector<double> cum(ntiles + 1, 0.0);
    for (int64_t t = 0; t < ntiles; ++t) cum[t + 1] = cum[t] + tcost[t];
    const double total_cost = cum[ntiles];
    int c = 1;
    for (int64_t t = 0; t < ntiles && c < grid; ++t) {
        const double mid = 0.5 * (cum[t] + cum[t + 1]);
        while (c < grid && mid >= total_cost * c / grid) cta[c++] = static_cast<uint32_t>(t);
    }
    while (c < grid) cta[c++] = static_cast<uint32_t>(ntiles);
    cta[grid] = static_cast<uint32_t>(ntiles);
    for (int i = 1; i <= grid; ++i) cta[i] = std::max(cta[i], cta[i - 1]);
    return cta;
}

// Block b's range index: co-resident CTAs of one SM are blocks b and b + grid/2 (the
// block scheduler fills every SM once before doubling up). Contiguous ranges would give
// both the same relative position in row-stacked matrices (q|k|v, gate|up) and so the
// same set type; the second slot walks the ranges in reverse instead, so each SM pairs
// complementary work.
int range_of_block(int b, int grid, int ctas_per_sm) {
    return (ctas_per_sm == 2 && b >= grid / 2) ? grid - 1 - (b - grid / 2) : b;
}

template <typename T>
T* dalloc_copy(const std::vector<T>& h, int64_t* total, cudaError_t* err) {
    T* d = nullptr;
    const size_t bytes = std::max<size_t>(h.size() * sizeof(T), 16);
    *err = cudaMalloc(&d, bytes);
    if (*err != cudaSuccess) return nullptr;
    *total += static_cast<int64_t>(bytes);
    if (!h.empty()) *err = cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
    return d;
}

}  // namespace

namespace ecsr_internal {  // other translation units (ecsr_loader.cpp) report errors here
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace ecsr_internal

struct ecsr_dev {
    int device = 0;
    int64_t M = 0, K = 0;
    int32_t W = 0, B = 0, vbits = 16, dtype = ECSR_F16, layout = 2;
    std::vector<SetDesc> sets;
    std::vector<uint8_t> pad_mask;  // cold section, concatenated per set
    int64_t nslots = 0;
    // tiled layout
    uint8_t* d_arena = nullptr;
    int64_t arena_bytes = 0;
    uint32_t* d_tile_start16 = nullptr;
    int64_t ntiles = 0;
    uint4* d_cta_work = nullptr;           // [grid] {member 0, tile lo, tile hi, slice} of each CTA
    double total_cost = 0;                 // summed tile cost (group CTA split)
    uint32_t* d_tile_meta = nullptr;       // [2 * ntiles] {start16, nrec | bytes16 << 16}
    uint32_t* d_queue_meta = nullptr;      // [2 * nqueue] the tail queue's tile metadata
    uint32_t nqueue = 0;                   // tail-queue tiles of a launch of this handle alone
    std::vector<uint32_t> tile_meta_h;     // host copy of d_tile_meta
    std::vector<double> tile_cost_h;       // per tile (arena order): fitted consumer cost
    bool lean = false;                     // every run uses a lean-kernel record variant
    bool gate_ok = true;                   // the whole grid can be resident (zero-y gate)
    int ctas_per_sm = 2;                   // co-resident CTAs per SM (9 or 18 consumer warps)
    std::vector<TileFeat> tile_feat;       // per tile (cost-model calibration)
    std::vector<uint32_t> cta_tile_h;      // host copy of the CTA tile boundaries
    std::vector<uint32_t> cta_range_h;     // per block [lo, hi) (launch order)
    unsigned long long* d_trace = nullptr; // tuning builds: per-CTA timeline
    int grid = 0, stage_bytes = 0, nstages = 0, wide = 0, smem_bytes = 0;
    // Per-stream launch workspaces: the zero-y gate's generation counter and the
    // ordered mode's block partials are written by a launch, so two launches of one
    // handle may overlap only if they use different ones. A handle binds up to
    // kStreamSlots streams (first come) to its own workspace each; launches issued on
    // (or captured from) one stream are stream-ordered, so they never share one
    // concurrently. Allocated at pack time: nothing is allocated on the launch path
    // (safe under CUDA graph capture).
    struct Workspace {
        unsigned long long* gate = nullptr;  // zero-y gate words (ecsr_kernels.cuh: kGate*)
        uint32_t* queue = nullptr;           // tail queue {next tile, CTAs done} (own 128-B line)
        void* partials = nullptr;            // [nslots] ordered-mode block partials
    };
    static constexpr int kStreamSlots = 4;
    Workspace ws[kStreamSlots];
    mutable cudaStream_t ws_stream[kStreamSlots] = {};
    mutable int ws_bound = 0;
    mutable std::mutex ws_mu;

    // The workspace of `stream` (bound on first use), or null when kStreamSlots other
    // streams already hold one.
    const Workspace* workspace(cudaStream_t stream) const {
        std::lock_guard<std::mutex> lock(ws_mu);
        for (int i = 0; i < ws_bound; ++i)
            if (ws_stream[i] == stream) return &ws[i];
        if (ws_bound == kStreamSlots) return nullptr;
        ws_stream[ws_bound] = stream;
        return &ws[ws_bound++];
    }
    // ordered reduction
    uint32_t* d_row_ptr = nullptr;
    uint32_t* d_row_slots = nullptr;
    // generic layout
    uint32_t* d_bases = nullptr;
    int64_t* d_indptr = nullptr;
    uint32_t* d_deltas = nullptr;
    void* d_values = nullptr;
    uint32_t* d_rows = nullptr;
    ecsr_bytes bytes{};
    std::vector<void*> allocs;

    ~ecsr_dev() {
        for (void* p : allocs) cudaFree(p);
    }
};

namespace {

// Structural + range validation (executor.py:50-77; storage.py:312-329), plus row
// ids < num_rows (the reference leaves that to unchecked C; a device write must not).
// B == 32 is internal (spmv_set): the reference's in-RAM u32 deltas carry no bit bound.
int validate(const ecsr_host_set* sets, int nsets, int64_t M, int64_t K, int W, int B) {
    if (W < 1 || W > 32) return fail(ECSR_ERR_VALUE, "warp_size must be in [1, 32]");
    if (B != 4 && B != 8 && B != 16 && B != 32)
        return fail(ECSR_ERR_VALUE, "delta_bits must be 4, 8 or 16");
    if (M < 0 || K < 0) return fail(ECSR_ERR_VALUE, "negative matrix shape");
    const uint64_t limit = B == 32 ? (1ull << 32) : (1ull << B);
    for (int si = 0; si < nsets; ++si) {
        const ecsr_host_set& s = sets[si];
        if (s.granularity < 1 || s.vector_size < 1)
            return fail(ECSR_ERR_CONTAINER, "set granularity and vector size must be positive");
        if (s.num_blocks < 0 || s.stored_cols < 0)
            return fail(ECSR_ERR_CONTAINER, "negative set size");
        const int64_t nb = s.num_blocks, g = s.granularity, v = s.vector_size;
        if (nb > 0 && (!s.block_indptr || !s.row_indices || !s.base_indices))
            return fail(ECSR_ERR_VALUE, "null set array");
        if (s.stored_cols > 0 && (!s.delta_indices || !s.block_values))
            return fail(ECSR_ERR_VALUE, "null set array");
        if (nb == 0) {
            if (s.stored_cols != 0)
                return fail(ECSR_ERR_CONTAINER, "block_indptr does not cover stored columns");
            continue;
        }
        if (s.block_indptr[0] != 0)
            return fail(ECSR_ERR_CONTAINER, "block_indptr must start at 0 and be non-decreasing");
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t w = s.block_indptr[b + 1] - s.block_indptr[b];
            if (w < 0)
                return fail(ECSR_ERR_CONTAINER, "block_indptr must start at 0 and be non-decreasing");
            if (w % (static_cast<int64_t>(W) * v))
                return fail(ECSR_ERR_CONTAINER,
                            "block widths must be multiples of warp_size * vector_size");
        }
        if (s.block_indptr[nb] != s.stored_cols)
            return fail(ECSR_ERR_CONTAINER, "block_indptr does not cover stored columns");
        for (int64_t i = 0; i < s.stored_cols; ++i)
            if (s.delta_indices[i] >= limit)
                return fail(ECSR_ERR_CONTAINER, "delta " + std::to_string(s.delta_indices[i]) +
                                                    " exceeds " + std::to_string(B) + "-bit range");
        for (int64_t i = 0; i < nb * W; ++i)
            if (s.base_indices[i] >= static_cast<uint64_t>(std::max<int64_t>(K, 1)))
                return fail(ECSR_ERR_CONTAINER, "base index out of range");
        for (int64_t i = 0; i < nb * g; ++i)
            if (s.row_indices[i] >= static_cast<uint64_t>(std::max<int64_t>(M, 1)))
                return fail(ECSR_ERR_CONTAINER, "row index out of range");
        std::vector<int64_t> top(W);
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t start = s.block_indptr[b], n = s.block_indptr[b + 1] - start;
            if (n == 0) continue;
            for (int t = 0; t < W; ++t) top[t] = s.base_indices[b * W + t];
            const int64_t chunk = static_cast<int64_t>(W) * v;
            for (int64_t i = 0; i < n; ++i) top[(i % chunk) / v] += s.delta_indices[start + i];
            for (int t = 0; t < W; ++t)
                if (top[t] >= K)
                    return fail(ECSR_ERR_CONTAINER, "decoded column " + std::to_string(top[t]) +
                                                        " out of range " + std::to_string(K));
        }
    }
    return ECSR_OK;
}

bool pow2_le32(int g) { return g == 1 || g == 2 || g == 4 || g == 8 || g == 16 || g == 32; }

struct DeviceLimits {
    int sms = 148;
    int smem_optin = 232448;
    int smem_per_sm = 233472;
};

// SMs the current context may keep busy at once: the device's, reduced to a green
// context's SM partition (cuCtxGetDevResource) and to the MPS active-thread percentage
// (CUDA_MPS_ACTIVE_THREAD_PERCENTAGE). The zero-y gate needs the whole grid resident.
int usable_sms(int device_sms) {
    using GetCurrent = CUresult (*)(CUcontext*);
    using GetResource = CUresult (*)(CUcontext, CUdevResource*, CUdevResourceType);
    static GetCurrent get_current = nullptr;
    static GetResource get_resource = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            get_current = reinterpret_cast<GetCurrent>(f);
        if (cudaGetDriverEntryPoint("cuCtxGetDevResource", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            get_resource = reinterpret_cast<GetResource>(f);
        cudaGetLastError();
    });
    int sms = device_sms;
    CUcontext ctx = nullptr;
    if (get_current && get_resource && get_current(&ctx) == CUDA_SUCCESS && ctx) {
        CUdevResource r{};
        if (get_resource(ctx, &r, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS && r.sm.smCount > 0)
            sms = std::min<int>(sms, static_cast<int>(r.sm.smCount));
    }
    if (const char* e = std::getenv("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE")) {
        const double pct = std::atof(e);
        if (pct > 0 && pct < 100) sms = std::min(sms, std::max(1, static_cast<int>(sms * pct / 100.0)));
    }
    return sms;
}

int query_limits(int device, DeviceLimits* lim) {
    ECSR_CUDA(cudaDeviceGetAttribute(&lim->sms, cudaDevAttrMultiProcessorCount, device));
    ECSR_CUDA(cudaDeviceGetAttribute(&lim->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    ECSR_CUDA(cudaDeviceGetAttribute(&lim->smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device));
    return ECSR_OK;
}

// ---------------------------------------------------------------------------------
// Tiled device layout (read by ecsr_tiled_kernel; constants in ecsr_kernels.cuh).
//
// Blocks are grouped, in container order, into group records of P = 8 / g consecutive
// blocks of one (g, v) run (P = 1 for g >= 8), so that one warp carries 8 row
// accumulators and walks the P blocks' chunk streams interleaved with one pointer:
//   [0, 32)  u32 slot[8]      ordered-mode partial slot of each block's row 0
//   [32, 48) u16 ntail[8]     chunks beyond nmin, per block
//   [48, 54) u16 nmin | u8 g | u8 v | u8 nblk | u8 present (bit b: block b has chunks)
//   [64, ..) u32 rows[P][g]   | pad 16
//   bases    per lane P entries (u16; u32 when K > 65535)
//   nmin x [deltas_0..P-1 (32v each) | values_0..P-1 (64vg each)]
//   tails    block 0's ntail[0] x [32v | 64vg], then block 1's, ...
// Every 32v / 64vg span is exactly one chunk of the reference's chunk-permuted streams
// (storage.py:147-181), so unpack restores the reference arrays bit-exactly. Missing
// blocks of a short last record get zero chunks in the interleaved part (never emitted).
// Records are packed into tiles of one (g, v) run:
//   u32 nrec | u16 (g << 8 | v) | u16 0 | u16 rec_off16[nrec] | pad 16 | records
// ---------------------------------------------------------------------------------
struct GroupPlan {
    std::vector<std::pair<int, int64_t>> blocks;  // (set, block), container order
    int P = 1;                                    // block slots of the record (>= blocks)
};

// A record of P blocks must fit a ring stage next to x: runs of very wide blocks
// (large K) get fewer blocks per record.
constexpr int64_t kRecordCap = 24 * 1024;
// A ring stage holds whole records, so records much larger than a tile leave consumer
// warps without work (fewer resident records than warps): a run's AVERAGE record is
// also held to ~rec_cap() = half a tile (ECSR_B200_RECCAP overrides, for tuning).
#ifdef ECSR_B200_TUNING
int64_t rec_max() {
    return std::max(512, env_int("ECSR_B200_RECMAX", static_cast<int>(std::min<int64_t>(kRecordCap, tile_target() - 16))));
}
int64_t rec_cap() { return std::max(512, env_int("ECSR_B200_RECCAP", tile_target() / 2)); }
#else
// A record wider than the tile target would get a tile of its own and stretch every
// stage of the pool to its size (fewer, emptier stages): P halves until it fits.
int64_t rec_max() { return std::min<int64_t>(kRecordCap, tile_target() - 16); }
int64_t rec_cap() { return tile_target() / 2; }
#endif

int group_p(int g) { return g > 8 ? 1 : ecsr::group_blocks(g); }

int64_t block_chunks(const ecsr_host_set& s, int64_t b) {
    return (s.block_indptr[b + 1] - s.block_indptr[b]) / (32 * s.vector_size);
}

int64_t group_record_bytes(const ecsr_host_set* sets, const GroupPlan& gp, bool wide) {
    const ecsr_host_set& s0 = sets[gp.blocks[0].first];
    const int g = s0.granularity, v = s0.vector_size, P = gp.P;
    int64_t nmin = INT64_MAX, total = 0;
    for (auto& sb : gp.blocks) {
        const int64_t n = block_chunks(sets[sb.first], sb.second);
        nmin = std::min(nmin, n);
        total += n;
    }
    const int64_t chunk = 32 * v + 64 * v * g;
    const int64_t tails = total - nmin * static_cast<int64_t>(gp.blocks.size());
    return ecsr::group_header_bytes(g, P) + (wide ? 128 : 64) * P + chunk * (nmin * P + tails);
}

// Consumer-time estimate of one record (tile balancing), fitted to measured per-CTA
// times of the bench layer (scripts/calibrate_cost.py, ECSR_CAL_DUMP; median error 3 %):
// ~151 CTA cycles per record (dispatch, stage lookup, header, reduce-scatter, emit),
// ~8 per block-chunk step and ~0.057 per byte. The per-record term is as large as the
// byte term for the small g = 2 / g = 4 records, so tiles of many small records
// weigh more than their bytes.
double group_record_cost(const ecsr_host_set* sets, const GroupPlan& gp, bool wide) {
    double steps = 0;
    for (auto& sb : gp.blocks) steps += static_cast<double>(block_chunks(sets[sb.first], sb.second));
    return 151.0 + 8.0 * steps + 0.057 * static_cast<double>(group_record_bytes(sets, gp, wide));
}

void write_group_record(const ecsr_host_set* sets, const std::vector<SetDesc>& desc, const GroupPlan& gp,
                        int host_dtype, bool wide, uint8_t* r) {
    const ecsr_host_set& s0 = sets[gp.blocks[0].first];
    const int g = s0.granularity, v = s0.vector_size, P = gp.P;
    const int nb = static_cast<int>(gp.blocks.size());
    std::vector<int64_t> nch(nb), st(nb);
    int64_t nmin = INT64_MAX;
    uint8_t present = 0;
    for (int b = 0; b < nb; ++b) {
        const ecsr_host_set& s = sets[gp.blocks[b].first];
        nch[b] = block_chunks(s, gp.blocks[b].second);
        st[b] = s.block_indptr[gp.blocks[b].second];
        nmin = std::min(nmin, nch[b]);
        if (nch[b] > 0) present |= static_cast<uint8_t>(1u << b);
        const uint32_t slot = static_cast<uint32_t>(desc[gp.blocks[b].first].slot0 + gp.blocks[b].second * g);
        std::memcpy(r + 4 * b, &slot, 4);
    }
    for (int b = 0; b < nb; ++b) {
        const uint16_t t16 = static_cast<uint16_t>(nch[b] - nmin);
        std::memcpy(r + 32 + 2 * b, &t16, 2);
    }
    const uint16_t nmin16 = static_cast<uint16_t>(nmin);
    std::memcpy(r + 48, &nmin16, 2);
    r[50] = static_cast<uint8_t>(g);
    r[51] = static_cast<uint8_t>(v);
    r[52] = static_cast<uint8_t>(nb);
    r[53] = present;
    r[54] = static_cast<uint8_t>(P);
    uint8_t has_tail = 0;
    for (int b = 0; b < nb; ++b) has_tail |= nch[b] > nmin ? 1 : 0;
    r[55] = has_tail;  // the kernel skips all tail loops at once when no block has one
    for (int b = 0; b < nb; ++b)
        std::memcpy(r + 64 + 4 * g * b, sets[gp.blocks[b].first].row_indices + gp.blocks[b].second * g, 4 * g);
    uint8_t* q = r + ecsr::group_header_bytes(g, P);
    const int esz = wide ? 4 : 2;
    for (int t = 0; t < 32; ++t)
        for (int b = 0; b < nb; ++b) {
            const uint32_t bv = sets[gp.blocks[b].first].base_indices[gp.blocks[b].second * 32 + t];
            if (wide) std::memcpy(q + (t * P + b) * esz, &bv, 4);
            else {
                const uint16_t b16 = static_cast<uint16_t>(bv);
                std::memcpy(q + (t * P + b) * esz, &b16, 2);
            }
        }
    q += 32 * P * esz;
    const int64_t dch = 32 * v, vch = 32 * v * g;  // per chunk: deltas (bytes), values (elements)
    auto put_deltas = [&](int b, int64_t c) {
        const ecsr_host_set& s = sets[gp.blocks[b].first];
        for (int64_t i = 0; i < dch; ++i) q[i] = static_cast<uint8_t>(s.delta_indices[st[b] + c * dch + i]);
        q += dch;
    };
    auto put_values = [&](int b, int64_t c) {
        const ecsr_host_set& s = sets[gp.blocks[b].first];
        uint16_t* hv = reinterpret_cast<uint16_t*>(q);
        const int64_t v0 = (st[b] + c * dch) * g;
        for (int64_t i = 0; i < vch; ++i) hv[i] = f64_to_f16(host_value(s.block_values, host_dtype, v0 + i));
        q += 2 * vch;
    };
    for (int64_t c = 0; c < nmin; ++c) {
        for (int b = 0; b < P; ++b) {
            if (b < nb) put_deltas(b, c);
            else q += dch;  // missing block: zero chunk
        }
        for (int b = 0; b < P; ++b) {
            if (b < nb) put_values(b, c);
            else q += 2 * vch;
        }
    }
    for (int b = 0; b < nb; ++b)
        for (int64_t c = nmin; c < nch[b]; ++c) {
            put_deltas(b, c);
            put_values(b, c);
        }
}

// Build the tiled arena: group records in container order, tiles of one (g, v) run.
void build_tiled_arena(const ecsr_host_set* sets, int nsets, const std::vector<SetDesc>& desc,
                       int host_dtype, bool wide, std::vector<uint8_t>* arena,
                       std::vector<uint32_t>* tile_start16, std::vector<uint32_t>* tile_rec_start,
                       std::vector<double>* tile_cost, std::vector<TileFeat>* tile_feat,
                       int64_t* max_tile) {
    arena->clear();
    tile_start16->clear();
    tile_rec_start->assign(1, 0u);
    tile_cost->clear();
    tile_feat->clear();
    *max_tile = 0;
    // 1. plan records: P consecutive blocks of a (g, v) run; P halves while the run's
    //    widest block would make a record exceed kRecordCap
    std::vector<std::vector<GroupPlan>> runs;
    std::vector<int> run_p;
    for (int si = 0; si < nsets;) {
        int se = si + 1;
        while (se < nsets && sets[se].granularity == sets[si].granularity &&
               sets[se].vector_size == sets[si].vector_size)
            ++se;
        const int g = sets[si].granularity, v = sets[si].vector_size;
        int64_t widest = 0, nblk = 0, sum_chunks = 0;
        for (int k = si; k < se; ++k)
            for (int64_t b = 0; b < sets[k].num_blocks; ++b) {
                widest = std::max(widest, block_chunks(sets[k], b));
                sum_chunks += block_chunks(sets[k], b);
                ++nblk;
            }
        const int64_t chunk = 32 * v + 64 * v * g;
        const double mean = nblk ? static_cast<double>(sum_chunks) / static_cast<double>(nblk) : 0.0;
        int P = group_p(g);
        auto hdr_p = [&](int q) { return ecsr::group_header_bytes(g, q) + (wide ? 128 : 64) * q; };
        while (v == 4 && P > 1 &&  // the kernel has reduced-P variants for v = 4 only
               (hdr_p(P) + P * widest * chunk > rec_max() ||
                static_cast<double>(hdr_p(P)) + P * mean * static_cast<double>(chunk) > static_cast<double>(rec_cap())))
            P /= 2;
        runs.emplace_back();
        for (int k = si; k < se; ++k)
            for (int64_t b = 0; b < sets[k].num_blocks; ++b) {
                auto& run = runs.back();
                if (run.empty() || static_cast<int>(run.back().blocks.size()) == P) {
                    run.emplace_back();
                    run.back().P = P;
                }
                run.back().blocks.emplace_back(k, b);
            }
        si = se;
    }
    // 2. pack the records into tiles of <= tile_target() bytes, first-fit decreasing
    //    over ALL runs (a tile may mix (g, v, P): the kernel dispatches on each record's
    //    header): records keep whole-record granularity, so sequential per-run packing
    //    left a stage ~22 % empty on average (two 5.5 KB records in a 17 KB stage); FFD
    //    over mixed runs fills ~95 % (a record's place is free: blocks are identified by
    //    their slot).
    auto hdr_of = [](size_t n) { return round_up(8 + 2 * static_cast<int64_t>(n), 16); };
    if (pack_mixed()) {  // one pool of every run's records: tiles may mix (g, v, P)
        std::vector<GroupPlan> all;
        for (const auto& run : runs) all.insert(all.end(), run.begin(), run.end());
        runs.assign(1, all);
    }
    for (const auto& run : runs) {
        std::vector<int64_t> rb(run.size());
        for (size_t i = 0; i < run.size(); ++i) rb[i] = round_up(group_record_bytes(sets, run[i], wide), 16);
        std::vector<std::vector<size_t>> bins;
        std::vector<int64_t> bin_bytes;
        if (pack_ffd()) {
            std::vector<size_t> order(run.size());
            for (size_t i = 0; i < order.size(); ++i) order[i] = i;
            std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) { return rb[x] > rb[y]; });
            size_t first_open = 0;  // bins before it cannot take even the smallest record
            const int64_t smallest = run.empty() ? 0 : *std::min_element(rb.begin(), rb.end());
            for (size_t i : order) {
                size_t bi = first_open;
                for (; bi < bins.size(); ++bi)
                    if (hdr_of(bins[bi].size() + 1) + bin_bytes[bi] + rb[i] <= tile_target()) break;
                if (bi == bins.size()) {
                    bins.emplace_back();
                    bin_bytes.push_back(0);
                }
                bins[bi].push_back(i);
                bin_bytes[bi] += rb[i];
                while (first_open < bins.size() &&
                       hdr_of(bins[first_open].size() + 1) + bin_bytes[first_open] + smallest > tile_target())
                    ++first_open;
            }
        } else {  // sequential (container order)
            for (size_t i = 0; i < run.size(); ++i) {
                if (bins.empty() || hdr_of(bins.back().size() + 1) + bin_bytes.back() + rb[i] > tile_target()) {
                    bins.emplace_back();
                    bin_bytes.push_back(0);
                }
                bins.back().push_back(i);
                bin_bytes.back() += rb[i];
            }
        }
        for (size_t bi = 0; bi < bins.size(); ++bi) {
            const std::vector<size_t>& recs = bins[bi];
            const size_t n = recs.size();
            const int64_t bytes = bin_bytes[bi];
            const int64_t start = static_cast<int64_t>(arena->size());
            const int64_t hdr = hdr_of(n);
            arena->resize(start + hdr + bytes, 0);
            uint8_t* base = arena->data() + start;
            const uint32_t nrec = static_cast<uint32_t>(n);
            std::memcpy(base, &nrec, 4);
            const ecsr_host_set& s0 = sets[run[recs[0]].blocks[0].first];
            const uint16_t gv = static_cast<uint16_t>((s0.granularity << 8) | s0.vector_size);
            std::memcpy(base + 4, &gv, 2);
            const uint16_t p16 = static_cast<uint16_t>(run[recs[0]].P);
            std::memcpy(base + 6, &p16, 2);
            int64_t off = hdr;
            double cost = 0;
            TileFeat tf;
            for (size_t k = 0; k < n; ++k) {
                const GroupPlan& gp = run[recs[k]];
                const int gc = gclass(sets[gp.blocks[0].first].granularity);
                tf.rec[gc] += 1;
                for (auto& sb : gp.blocks) tf.steps[gc] += static_cast<double>(block_chunks(sets[sb.first], sb.second));
                tf.bytes += static_cast<double>(group_record_bytes(sets, gp, wide));
                const uint16_t off16 = static_cast<uint16_t>(off / 16);
                std::memcpy(base + 8 + 2 * k, &off16, 2);
                write_group_record(sets, desc, gp, host_dtype, wide, base + off);
                off += rb[recs[k]];
                cost += group_record_cost(sets, gp, wide);
            }
            tile_start16->push_back(static_cast<uint32_t>(start / 16));
            tile_rec_start->push_back(tile_rec_start->back() + static_cast<uint32_t>(n));
            tile_cost->push_back(cost);
            tile_feat->push_back(tf);
            *max_tile = std::max<int64_t>(*max_tile, hdr + bytes);
        }
    }
    tile_start16->push_back(static_cast<uint32_t>(arena->size() / 16));
}

// Tail queue of a launch: in every job's LPT-ordered static range [lo, hi) of handle d,
// the cheapest suffix worth `share` of the range's cost moves to the queue (job.z
// shrinks), drawn most expensive tile first by whichever CTAs of the member run ahead.
// qmeta: the queue's {start16, info} pairs in draw order.
void split_tail_queue(const ecsr_dev* d, std::vector<uint4>* jobs, double share, std::vector<uint32_t>* qmeta) {
    std::vector<uint32_t> q;
    for (uint4& j : *jobs) {
        double rcost = 0, moved = 0;
        for (uint32_t t = j.y; t < j.z; ++t) rcost += d->tile_cost_h[t];
        uint32_t keep = j.z;
        while (keep > j.y + 1 && moved + d->tile_cost_h[keep - 1] <= share * rcost) moved += d->tile_cost_h[--keep];
        for (uint32_t t = keep; t < j.z; ++t) q.push_back(t);
        j.z = keep;
    }
    std::stable_sort(q.begin(), q.end(), [&](uint32_t a, uint32_t b) { return d->tile_cost_h[a] > d->tile_cost_h[b]; });
    qmeta->clear();
    for (uint32_t t : q) {
        qmeta->push_back(d->tile_meta_h[2 * t]);
        qmeta->push_back(d->tile_meta_h[2 * t + 1]);
    }
}

// Zero-y gate words of a launch (one counter on its own 128-B line).
size_t gate_bytes(int) { return 8 * ecsr::kGateWords; }

int build_slots(ecsr_dev* d, const ecsr_host_set* sets, int nsets, int64_t* total) {
    std::vector<uint32_t> cnt(d->M + 1, 0);
    for (int si = 0; si < nsets; ++si) {
        const ecsr_host_set& s = sets[si];
        for (int64_t b = 0; b < s.num_blocks; ++b) {
            if (s.block_indptr[b + 1] == s.block_indptr[b]) continue;  // skipped by the kernel
            for (int k = 0; k < s.granularity; ++k) cnt[s.row_indices[b * s.granularity + k] + 1]++;
        }
    }
    std::vector<uint32_t> row_ptr(d->M + 1, 0);
    for (int64_t r = 0; r < d->M; ++r) row_ptr[r + 1] = row_ptr[r] + cnt[r + 1];
    std::vector<uint32_t> fill(row_ptr.begin(), row_ptr.begin() + d->M);
    std::vector<uint32_t> slots(row_ptr[d->M]);
    for (int si = 0; si < nsets; ++si) {
        const ecsr_host_set& s = sets[si];
        for (int64_t b = 0; b < s.num_blocks; ++b) {
            if (s.block_indptr[b + 1] == s.block_indptr[b]) continue;
            for (int k = 0; k < s.granularity; ++k) {
                const uint32_t r = s.row_indices[b * s.granularity + k];
                slots[fill[r]++] = static_cast<uint32_t>(d->sets[si].slot0 + b * s.granularity + k);
            }
        }
    }
    cudaError_t err = cudaSuccess;
    d->d_row_ptr = dalloc_copy(row_ptr, total, &err);
    if (d->d_row_ptr) d->allocs.push_back(d->d_row_ptr);
    ECSR_CUDA(err);
    d->d_row_slots = dalloc_copy(slots, total, &err);
    if (d->d_row_slots) d->allocs.push_back(d->d_row_slots);
    ECSR_CUDA(err);
    const size_t pbytes = round_up(std::max<int64_t>(16, d->nslots * (d->dtype == ECSR_F64 ? 8 : 4)), 256);
    uint8_t* part = nullptr;
    ECSR_CUDA(cudaMalloc(&part, pbytes * ecsr_dev::kStreamSlots));
    d->allocs.push_back(part);
    const size_t wbytes = gate_bytes(d->grid) + 128;  // gate words, then the queue's own line
    uint8_t* sync = nullptr;
    ECSR_CUDA(cudaMalloc(&sync, wbytes * ecsr_dev::kStreamSlots));
    d->allocs.push_back(sync);
    ECSR_CUDA(cudaMemset(sync, 0, wbytes * ecsr_dev::kStreamSlots));
    for (int i = 0; i < ecsr_dev::kStreamSlots; ++i) {
        d->ws[i].partials = part + pbytes * i;
        d->ws[i].gate = reinterpret_cast<unsigned long long*>(sync + wbytes * i);
        d->ws[i].queue = reinterpret_cast<uint32_t*>(sync + wbytes * i + gate_bytes(d->grid));
    }
    *total += static_cast<int64_t>((pbytes + wbytes) * ecsr_dev::kStreamSlots);
    return ECSR_OK;
}

template <typename VT>
void convert_values(const ecsr_host_set& s, int host_dtype, std::vector<VT>* out);
template <>
void convert_values<uint16_t>(const ecsr_host_set& s, int host_dtype, std::vector<uint16_t>* out) {
    for (int64_t i = 0; i < s.stored_cols * s.granularity; ++i)
        out->push_back(f64_to_f16(host_value(s.block_values, host_dtype, i)));
}
template <>
void convert_values<float>(const ecsr_host_set& s, int host_dtype, std::vector<float>* out) {
    for (int64_t i = 0; i < s.stored_cols * s.granularity; ++i)
        out->push_back(static_cast<float>(host_value(s.block_values, host_dtype, i)));
}
template <>
void convert_values<double>(const ecsr_host_set& s, int host_dtype, std::vector<double>* out) {
    for (int64_t i = 0; i < s.stored_cols * s.granularity; ++i)
        out->push_back(host_value(s.block_values, host_dtype, i));
}

template <typename VT>
int build_generic(ecsr_dev* d, const ecsr_host_set* sets, int nsets, int host_dtype, int64_t* total) {
    std::vector<uint32_t> bases, deltas, rows;
    std::vector<int64_t> indptr;
    std::vector<VT> vals;
    for (int si = 0; si < nsets; ++si) {
        const ecsr_host_set& s = sets[si];
        SetDesc& sd = d->sets[si];
        sd.base_off = static_cast<int64_t>(bases.size());
        sd.indptr_off = static_cast<int64_t>(indptr.size());
        sd.col_off = static_cast<int64_t>(deltas.size());
        sd.val_off = static_cast<int64_t>(vals.size());
        bases.insert(bases.end(), s.base_indices, s.base_indices + s.num_blocks * d->W);
        if (s.num_blocks > 0) indptr.insert(indptr.end(), s.block_indptr, s.block_indptr + s.num_blocks + 1);
        else indptr.push_back(0);
        deltas.insert(deltas.end(), s.delta_indices, s.delta_indices + s.stored_cols);
        rows.insert(rows.end(), s.row_indices, s.row_indices + s.num_blocks * s.granularity);
        convert_values<VT>(s, host_dtype, &vals);
    }
    cudaError_t err = cudaSuccess;
    d->d_bases = dalloc_copy(bases, total, &err);
    if (d->d_bases) d->allocs.push_back(d->d_bases);
    ECSR_CUDA(err);
    d->d_indptr = dalloc_copy(indptr, total, &err);
    if (d->d_indptr) d->allocs.push_back(d->d_indptr);
    ECSR_CUDA(err);
    d->d_deltas = dalloc_copy(deltas, total, &err);
    if (d->d_deltas) d->allocs.push_back(d->d_deltas);
    ECSR_CUDA(err);
    d->d_rows = dalloc_copy(rows, total, &err);
    if (d->d_rows) d->allocs.push_back(d->d_rows);
    ECSR_CUDA(err);
    VT* dv = dalloc_copy(vals, total, &err);
    d->d_values = dv;
    if (dv) d->allocs.push_back(dv);
    ECSR_CUDA(err);
    return ECSR_OK;
}

void fill_model_bytes(ecsr_dev* d, const ecsr_host_set* sets, int nsets) {
    ecsr_bytes& b = d->bytes;
    b.desc = 30 + 32 * static_cast<int64_t>(nsets);  // _HEADER_BYTES + _DESC_BYTES (storage.py:575-576)
    for (int si = 0; si < nsets; ++si) {
        const ecsr_host_set& s = sets[si];
        b.row_indices += 4 * s.num_blocks * s.granularity;
        b.block_indptr += 8 * (s.num_blocks + 1);
        b.base_indices += 4 * s.num_blocks * d->W;
        b.delta_indices += d->B == 4 ? (s.stored_cols + 1) / 2 : s.stored_cols * (d->B / 8);
        b.pad_mask += (s.stored_cols + 7) / 8;
        b.block_values += s.stored_cols * s.granularity * 16 / 8;
    }
    b.model_kernel_bytes = b.row_indices + b.block_indptr + b.base_indices + b.delta_indices +
                           b.block_values + 2 * d->K + 4 * d->M;
}

// The dynamic shared-memory opt-in is a per-device (per-context) function attribute:
// track the configured size per device index.
int configure_tiled_kernels(int device, int smem) {
    static std::mutex mu;
    static std::vector<int> configured;
    std::lock_guard<std::mutex> lock(mu);
    if (device >= static_cast<int>(configured.size())) configured.resize(device + 1, 0);
    if (configured[device] >= smem) return ECSR_OK;
    constexpr int kHalf = ecsr::kConsumerWarpsPerSm / 2, kAll = ecsr::kConsumerWarpsPerSm;
    ECSR_CUDA(cudaFuncSetAttribute(ecsr::ecsr_tiled_kernel<true, kHalf>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    ECSR_CUDA(cudaFuncSetAttribute(ecsr::ecsr_tiled_kernel<false, kHalf>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    ECSR_CUDA(cudaFuncSetAttribute(ecsr::ecsr_tiled_kernel<true, kAll>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    ECSR_CUDA(cudaFuncSetAttribute(ecsr::ecsr_tiled_kernel<false, kAll>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured[device] = smem;
    return ECSR_OK;
}

// Makes `device` current for the scope of a call and restores the caller's device.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int device) {
        err = cudaGetDevice(&prev);
        if (err == cudaSuccess && prev != device) err = cudaSetDevice(device);
        else if (err == cudaSuccess) prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

template <typename K, typename... Args>
cudaError_t launch_ex(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, bool coop,
                      Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = coop ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}
template <typename K, typename... Args>
cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args... args) {
    return launch_ex(kernel, grid, block, smem, stream, false, args...);
}

// One launch of the tiled kernel over `n` members (a single handle, or a group).
struct MemberLaunch {
    const ecsr_dev* d;
    const void* x;
    void* y;
    uint32_t* queue;   // the member's tail-queue words in the launch's workspace
    void* partials;    // ordered mode
    int ctas;          // CTAs of the launch working on this member
    int nstages;       // stage-pool depth of its CTAs (the handle's, or a group's)
    const uint32_t* queue_meta;  // the launch's tail queue of this member
    uint32_t nqueue;
};

cudaError_t launch_tiled(const MemberLaunch* m, int n, const uint4* cta_work, int grid, int nc, bool lean,
                         int smem, unsigned long long* gate, bool ordered, bool zero_y,
                         unsigned long long* trace, cudaStream_t st) {
    ecsr::TiledParams p{};
    int pre = pre_tiles();
    for (int i = 0; i < n; ++i) {
        const ecsr_dev* d = m[i].d;
        ecsr::TiledMember& t = p.mem[i];
        t.arena = d->d_arena;
        t.tile_meta = reinterpret_cast<const uint2*>(d->d_tile_meta);
        t.x = static_cast<const __half*>(m[i].x);
        t.y = static_cast<float*>(m[i].y);
        t.partials = static_cast<float*>(m[i].partials);
        t.queue = m[i].queue;
        t.M = d->M;
        t.queue_meta = reinterpret_cast<const uint2*>(m[i].queue_meta);
        t.nqueue = m[i].nqueue;
        t.K = static_cast<int32_t>(d->K);
        t.stage_bytes = d->stage_bytes;
        t.nstages = m[i].nstages;
        t.x_vec16 = (reinterpret_cast<uintptr_t>(m[i].x) % 16) == 0;
        t.ctas = m[i].ctas;
        pre = std::min(pre, std::max(1, m[i].nstages - 1));
    }
    p.cta_work = cta_work;
    p.gate = gate;
    p.nmem = n;
    p.wide = m[0].d->wide;
    p.ordered = ordered ? 1 : 0;
    p.zero_y = zero_y ? 1 : 0;
    p.pre_tiles = pre;
    p.trace = trace;
    const bool coop = coop_launch();
    const dim3 blk(ecsr::tiled_threads(nc)), grd(grid);
    constexpr int kHalf = ecsr::kConsumerWarpsPerSm / 2, kAll = ecsr::kConsumerWarpsPerSm;
    if (nc == kHalf)
        return lean ? launch_ex(ecsr::ecsr_tiled_kernel<false, kHalf>, grd, blk, smem, st, coop, p)
                    : launch_ex(ecsr::ecsr_tiled_kernel<true, kHalf>, grd, blk, smem, st, coop, p);
    return lean ? launch_ex(ecsr::ecsr_tiled_kernel<false, kAll>, grd, blk, smem, st, coop, p)
                : launch_ex(ecsr::ecsr_tiled_kernel<true, kAll>, grd, blk, smem, st, coop, p);
}

template <typename T, typename VT, typename XT>
cudaError_t launch_generic_set(const ecsr_dev* d, const SetDesc& sd, const void* x, void* partials,
                               cudaStream_t st) {
    ecsr::GenericSet gs;
    gs.base_indices = d->d_bases + sd.base_off;
    gs.block_indptr = d->d_indptr + sd.indptr_off;
    gs.delta_indices = d->d_deltas + sd.col_off;
    gs.block_values = static_cast<const VT*>(d->d_values) + sd.val_off;
    gs.num_blocks = sd.nb;
    gs.slot0 = sd.slot0;
    gs.g = sd.g;
    gs.warp = d->W;
    gs.v = sd.v;
    int p2 = 1;
    while (p2 < d->W) p2 <<= 1;
    gs.lanes_p2 = p2;
    const int warps_per_cta = 8;
    int64_t ctas = (sd.nb + warps_per_cta - 1) / warps_per_cta;
    ctas = std::max<int64_t>(1, std::min<int64_t>(ctas, 148 * 16));
    T* part = static_cast<T*>(partials);
    const XT* xx = static_cast<const XT*>(x);
    dim3 grid(static_cast<unsigned>(ctas)), block(32 * warps_per_cta);
    if (sd.g <= 1) return launch_pdl(ecsr::ecsr_generic_kernel<T, VT, XT, 1>, grid, block, 0, st, gs, xx, part);
    if (sd.g <= 2) return launch_pdl(ecsr::ecsr_generic_kernel<T, VT, XT, 2>, grid, block, 0, st, gs, xx, part);
    if (sd.g <= 4) return launch_pdl(ecsr::ecsr_generic_kernel<T, VT, XT, 4>, grid, block, 0, st, gs, xx, part);
    if (sd.g <= 8) return launch_pdl(ecsr::ecsr_generic_kernel<T, VT, XT, 8>, grid, block, 0, st, gs, xx, part);
    return launch_pdl(ecsr::ecsr_generic_kernel<T, VT, XT, 16>, grid, block, 0, st, gs, xx, part);
}

template <typename T>
cudaError_t launch_finish(const ecsr_dev* d, void* y, int accumulate, const void* partials, cudaStream_t st) {
    const int threads = 256;
    int64_t ctas = (d->M + threads - 1) / threads;
    ctas = std::max<int64_t>(1, std::min<int64_t>(ctas, 148 * 8));
    return launch_pdl(ecsr::ecsr_finish_rows<T>, dim3(static_cast<unsigned>(ctas)), dim3(threads), 0,
                      st, static_cast<const uint32_t*>(d->d_row_ptr),
                      static_cast<const uint32_t*>(d->d_row_slots),
                      static_cast<const T*>(partials), static_cast<T*>(y), d->M, accumulate);
}

}  // namespace

extern "C" {

const char* ecsr_b200_last_error(void) { return g_last_error.c_str(); }

const char* ecsr_b200_version(void) { return "ecsr_b200 0.1.0 (sm_100a)"; }

int ecsr_b200_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int ecsr_b200_to_f16(const void* src, int32_t src_dtype, uint16_t* dst, int64_t n) {
    if (src_dtype != ECSR_F32 && src_dtype != ECSR_F64) return fail(ECSR_ERR_VALUE, "src dtype");
    for (int64_t i = 0; i < n; ++i) dst[i] = f64_to_f16(host_value(src, src_dtype, i));
    return ECSR_OK;
}

int ecsr_b200_pack(const ecsr_host_set* sets, int32_t nsets, int64_t num_rows, int64_t num_cols,
                   int32_t warp_size, int32_t delta_bits, int32_t value_bits,
                   int32_t host_value_dtype, int32_t device_dtype, int32_t flags, ecsr_dev** out) {
    if (!out) return fail(ECSR_ERR_VALUE, "out is null");
    *out = nullptr;
    if (nsets < 0 || (nsets > 0 && !sets)) return fail(ECSR_ERR_VALUE, "bad set list");
    if (host_value_dtype != ECSR_F32 && host_value_dtype != ECSR_F64 && host_value_dtype != ECSR_F16)
        return fail(ECSR_ERR_VALUE, "host values must be f16, f32 or f64");
    if (device_dtype != ECSR_F16 && device_dtype != ECSR_F32 && device_dtype != ECSR_F64)
        return fail(ECSR_ERR_VALUE, "device dtype must be f16, f32 or f64");
    if (delta_bits == 32 && !(flags & kPackInternal)) return fail(ECSR_ERR_VALUE, "delta_bits must be 4, 8 or 16");
    int rc = validate(sets, nsets, num_rows, num_cols, warp_size, delta_bits);
    if (rc) return rc;

    int64_t nslots = 0;
    for (int si = 0; si < nsets; ++si) nslots += sets[si].num_blocks * sets[si].granularity;
    if (nslots >= (1ll << 32) || num_rows >= (1ll << 32) - 1)
        return fail(ECSR_ERR_VALUE, "container too large for 32-bit slot tables");

    int dev = 0;
    ECSR_CUDA(cudaGetDevice(&dev));
    DeviceLimits lim;
    rc = query_limits(dev, &lim);
    if (rc) return rc;

    auto* d = new ecsr_dev();
    d->device = dev;
    d->M = num_rows;
    d->K = num_cols;
    d->W = warp_size;
    d->B = delta_bits;
    d->vbits = value_bits;
    d->dtype = device_dtype;
    d->nslots = nslots;
    d->sets.resize(nsets);
    int64_t slot = 0;
    for (int si = 0; si < nsets; ++si) {
        SetDesc& sd = d->sets[si];
        sd.g = sets[si].granularity;
        sd.v = sets[si].vector_size;
        sd.nb = sets[si].num_blocks;
        sd.stored = sets[si].stored_cols;
        sd.real = sets[si].real_nnz;
        sd.slot0 = slot;
        sd.row_off = slot;
        slot += sd.nb * sd.g;
        if (sets[si].pad_mask)
            d->pad_mask.insert(d->pad_mask.end(), sets[si].pad_mask, sets[si].pad_mask + sd.stored);
        else
            d->pad_mask.insert(d->pad_mask.end(), sd.stored, 0);
    }
    fill_model_bytes(d, sets, nsets);
    int64_t total = 0;

    // Tiled fast layout: fp16 values, W = 32, deltas <= 8 bits, supported (g, v), x fits smem.
    bool tiled = device_dtype == ECSR_F16 && !(flags & ECSR_PACK_FORCE_GENERIC) && warp_size == 32 &&
                 delta_bits <= 8;
    for (int si = 0; si < nsets && tiled; ++si) {
        const int g = sets[si].granularity, v = sets[si].vector_size;
        if (!pow2_le32(g) || !(v == 1 || v == 4)) tiled = false;  // kernel variants: v in {1, 4}
        for (int64_t b = 0; b < sets[si].num_blocks && tiled; ++b)
            if ((sets[si].block_indptr[b + 1] - sets[si].block_indptr[b]) / (32 * v) > 65535) tiled = false;
    }
    const bool wide = num_cols > 65535;
    // Two co-resident CTAs per SM (9 consumer warps each; consecutive launches overlap)
    // while x is small; one CTA of 18 consumer warps when two copies of x would crowd
    // out the stage pool.
    const int64_t xbytes = round_up(2 * std::max<int64_t>(num_cols, 1), 16);
    const int ctas_per_sm = xbytes <= 32768 ? 2 : 1;
    if (tiled) {
        static std::mutex tile_mu;  // the packer is host code; serialise the tile default
        std::lock_guard<std::mutex> lock(tile_mu);
        t_tile_override = ((flags >> 8) & 0xff) * 1024;  // 0: the default
        // The stage pool fills the CTA's shared memory: stages of ~16 KB (2 CTAs/SM) or
        // ~32 KB (1 CTA), stretched so that a whole number of them uses all of it
        // (more bytes in flight per SM; e.g. 5 x 18.3 KB instead of 5 x 16 KB at K = 8192).
        const int64_t cta_smem = ctas_per_sm == 1 ? lim.smem_optin : (lim.smem_per_sm / ctas_per_sm) - 1024;
        const int64_t avail = cta_smem - kSmemReserve - 16 * kMaxStages - xbytes;  // static smem + barriers
        {
            const int64_t base = ctas_per_sm == 2 ? 16384 : 32768;
            const int64_t n0 = std::min<int64_t>(kMaxStages, std::max<int64_t>(2, avail / base));
            g_tile_default = static_cast<int>(std::max<int64_t>(4096, (avail / n0) / 128 * 128));
        }
        std::vector<uint8_t> arena;
        std::vector<uint32_t> tstart, trec;
        std::vector<double> tcost;
        int64_t max_tile = 0;
        build_tiled_arena(sets, nsets, d->sets, host_value_dtype, wide, &arena, &tstart, &trec, &tcost,
                          &d->tile_feat, &max_tile);
        // the lean kernel covers v = 4 runs with the default blocks-per-record (or half
        // of it for g = 2, down to a quarter for g = 1) and g <= 8, and v = 1 runs of g = 1 (the reference's short set)
        d->lean = !force_full();  // every record's (g, v, P) has a lean-kernel variant
        for (int64_t t = 0; t + 1 < static_cast<int64_t>(tstart.size()) && d->lean; ++t) {
            const uint8_t* th = arena.data() + 16ull * tstart[t];
            uint32_t nrec;
            std::memcpy(&nrec, th, 4);
            for (uint32_t jr = 0; jr < nrec; ++jr) {
                uint16_t off16;
                std::memcpy(&off16, th + 8 + 2 * jr, 2);
                const uint8_t* rh = th + 16 * off16;
                const int g = rh[50], v = rh[51], pp = rh[54];
                const bool ok = (v == 4 && g <= 8 &&
                                 (pp == group_p(g) || (g <= 2 && 2 * pp == group_p(g)) ||
                                  (g == 1 && 4 * pp == group_p(g)))) ||
                                (v == 1 && g == 1);
                if (!ok) d->lean = false;
            }
        }
        const int64_t stage = round_up(std::max<int64_t>(max_tile, tile_target()), 128);
        d->ctas_per_sm = ctas_per_sm;  // CTAs share the SM's 228 KB (1 KB reserved each)
        const int64_t nst = std::min<int64_t>(kMaxStages, avail / std::max<int64_t>(stage, 1));
        if (stage > kMaxStageBytes || nst < 2 || arena.size() / 16 >= (1ull << 32)) tiled = false;
        if (tiled) {
            d->layout = 1;
            d->wide = wide;
            d->stage_bytes = static_cast<int>(stage);
            d->nstages = static_cast<int>(nst);
            d->smem_bytes = static_cast<int>(round_up(8 * nst + 8, 128) + nst * stage + xbytes);
            const int64_t ntiles = static_cast<int64_t>(tstart.size()) - 1;
            d->ntiles = ntiles;
            const int grid =
                static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(int64_t{lim.sms} * ctas_per_sm, ntiles)));
            d->grid = grid;
            // cost-balanced contiguous tile ranges (fitted consumer-time model)
            const std::vector<uint32_t> cta = balanced_ranges(tcost, grid);
            // Within each CTA's range, tiles go longest record first (LPT): records are
            // handed to warps in issue order, so the last ones of a CTA are short. The
            // cheapest end of every range (cost share `qshare`) moves to the launch's tail
            // queue, most expensive tile first, drawn by whichever CTAs run ahead of the
            // cost model. Unpack identifies blocks by slot, not position.
            const double qshare = (flags & (0x80 << 16)) ? ((flags >> 16) & 0x7f) / 100.0 : kQueueShare;
            std::vector<uint32_t> order, scta(grid + 1, 0);
            order.reserve(ntiles);
            for (int c2 = 0; c2 < grid; ++c2) {
                std::vector<uint32_t> ts;
                for (uint32_t t = cta[c2]; t < cta[c2 + 1]; ++t) ts.push_back(t);
                std::stable_sort(ts.begin(), ts.end(), [&](uint32_t x, uint32_t y) {
                    const double cx = tcost[x] / std::max<uint32_t>(1, trec[x + 1] - trec[x]);
                    const double cy = tcost[y] / std::max<uint32_t>(1, trec[y + 1] - trec[y]);
                    return cx > cy;
                });
                scta[c2] = static_cast<uint32_t>(order.size());
                order.insert(order.end(), ts.begin(), ts.end());
            }
            scta[grid] = static_cast<uint32_t>(order.size());
            {
                std::vector<uint8_t> na;
                na.reserve(arena.size());
                std::vector<uint32_t> nts(ntiles + 1), ntr(ntiles + 1, 0);
                std::vector<double> ntc(ntiles);
                std::vector<TileFeat> ntf(ntiles);
                for (int64_t i = 0; i < ntiles; ++i) {
                    const uint32_t t = order[i];
                    nts[i] = static_cast<uint32_t>(na.size() / 16);
                    na.insert(na.end(), arena.begin() + 16ull * tstart[t], arena.begin() + 16ull * tstart[t + 1]);
                    ntr[i + 1] = ntr[i] + (trec[t + 1] - trec[t]);
                    ntc[i] = tcost[t];
                    ntf[i] = d->tile_feat[t];
                }
                nts[ntiles] = static_cast<uint32_t>(na.size() / 16);
                arena.swap(na);
                tstart.swap(nts);
                trec.swap(ntr);
                tcost.swap(ntc);
                d->tile_feat.swap(ntf);
            }
            // per tile {start16, nrec | bytes16 << 16} (a tile is at most 64 KB)
            std::vector<uint32_t> meta(2 * std::max<int64_t>(ntiles, 1), 0u);
            for (int64_t t = 0; t < ntiles; ++t) {
                meta[2 * t] = tstart[t];
                meta[2 * t + 1] = (trec[t + 1] - trec[t]) | ((tstart[t + 1] - tstart[t]) << 16);
            }
            cudaError_t err = cudaSuccess;
            d->arena_bytes = static_cast<int64_t>(arena.size());
            d->d_arena = dalloc_copy(arena, &total, &err);
            if (d->d_arena) d->allocs.push_back(d->d_arena);
            if (err == cudaSuccess) {
                d->d_tile_start16 = dalloc_copy(tstart, &total, &err);
                if (d->d_tile_start16) d->allocs.push_back(d->d_tile_start16);
            }
            if (err == cudaSuccess) {
                d->d_tile_meta = dalloc_copy(meta, &total, &err);
                if (d->d_tile_meta) d->allocs.push_back(d->d_tile_meta);
            }
            d->cta_tile_h = scta;
            d->tile_meta_h = meta;
            d->tile_cost_h = tcost;
            d->gate_ok = grid <= usable_sms(lim.sms) * ctas_per_sm;
            for (double c : tcost) d->total_cost += c;
            std::vector<uint4> jobs(grid), work(grid);
            for (int r = 0; r < grid; ++r) jobs[r] = make_uint4(0u, scta[r], scta[r + 1], static_cast<uint32_t>(r));
            std::vector<uint32_t> qmeta;
            split_tail_queue(d, &jobs, qshare, &qmeta);
            d->nqueue = static_cast<uint32_t>(qmeta.size() / 2);
            std::vector<uint32_t> ranges(2 * grid);
            for (int b = 0; b < grid; ++b) {
                work[b] = jobs[range_of_block(b, grid, ctas_per_sm)];
                ranges[2 * b] = work[b].y;
                ranges[2 * b + 1] = work[b].z;
            }
            d->cta_range_h = ranges;
            if (err == cudaSuccess) {
                d->d_cta_work = dalloc_copy(work, &total, &err);
                if (d->d_cta_work) d->allocs.push_back(d->d_cta_work);
            }
            if (err == cudaSuccess) {
                d->d_queue_meta = dalloc_copy(qmeta, &total, &err);
                if (d->d_queue_meta) d->allocs.push_back(d->d_queue_meta);
            }
            if (err != cudaSuccess) {
                delete d;
                return fail(ECSR_ERR_CUDA, std::string("tiled upload: ") + cudaGetErrorString(err));
            }
            rc = configure_tiled_kernels(dev, d->smem_bytes);
            if (rc) {
                delete d;
                return rc;
            }
        }
    }
    if (!tiled) {
        d->layout = 2;
        if (device_dtype == ECSR_F16) rc = build_generic<uint16_t>(d, sets, nsets, host_value_dtype, &total);
        else if (device_dtype == ECSR_F32) rc = build_generic<float>(d, sets, nsets, host_value_dtype, &total);
        else rc = build_generic<double>(d, sets, nsets, host_value_dtype, &total);
        if (rc) {
            delete d;
            return rc;
        }
    }
    t_tile_override = 0;
    rc = build_slots(d, sets, nsets, &total);
    if (rc) {
        delete d;
        return rc;
    }
    d->bytes.device_arena_bytes = d->layout == 1 ? d->arena_bytes : total;
    d->bytes.device_total_bytes = total;
    d->bytes.layout = d->layout;
    d->bytes.grid = d->grid;
    d->bytes.stages = d->nstages;
    d->bytes.stage_bytes = d->stage_bytes;
    d->bytes.tiles = d->ntiles;
    d->bytes.queue_tiles = d->nqueue;
    *out = d;
    return ECSR_OK;
}

int ecsr_b200_spmv(const ecsr_dev* d, const void* x, void* y, int32_t mode, void* stream) {
    if (!d) return fail(ECSR_ERR_VALUE, "null handle");
    if ((!x && d->K > 0) || (!y && d->M > 0)) return fail(ECSR_ERR_VALUE, "null x or y");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int accumulate = mode & ECSR_SPMV_ACCUMULATE;
    const bool ordered = (mode & ECSR_SPMV_ORDERED) != 0 || d->layout == 2;
    if (d->M == 0) return ECSR_OK;
    const ecsr_dev::Workspace* ws = d->workspace(st);
    if (!ws)
        return fail(ECSR_ERR_VALUE, "handle already used from " + std::to_string(ecsr_dev::kStreamSlots) +
                                        " other streams (one workspace per stream)");
    DeviceGuard guard(d->device);  // the handle's device, whatever the caller's current one
    ECSR_CUDA(guard.err);
    if (d->layout == 1) {
        unsigned long long* trace = nullptr;
        if (trace_enabled()) {  // tuning builds only
            ecsr_dev* dm = const_cast<ecsr_dev*>(d);
            if (!dm->d_trace) {
                ECSR_CUDA(cudaMalloc(&dm->d_trace, 8 * 16 * d->grid));
                dm->allocs.push_back(dm->d_trace);
            }
            if (!trace_caller_resets()) {
                std::vector<unsigned long long> init(16 * d->grid, 0ull);
                for (int c = 0; c < d->grid; ++c) init[16 * c + 7] = ~0ull;
                ECSR_CUDA(cudaMemcpyAsync(dm->d_trace, init.data(), 8 * init.size(), cudaMemcpyHostToDevice, st));
                ECSR_CUDA(cudaStreamSynchronize(st));
            }
            trace = dm->d_trace;
        }
        // overwrite: zero y inside the kernel (gate) when the whole grid can be resident,
        // else (or on request) a memset first and an ungated launch
        const bool memset_y = !ordered && !accumulate && (!d->gate_ok || (mode & ECSR_SPMV_MEMSET_Y));
        if (memset_y) ECSR_CUDA(cudaMemsetAsync(y, 0, 4 * d->M, st));
        const MemberLaunch m{d, x, y, ws->queue, ws->partials, d->grid, d->nstages, d->d_queue_meta, d->nqueue};
        ECSR_CUDA(launch_tiled(&m, 1, d->d_cta_work, d->grid, ecsr::kConsumerWarpsPerSm / d->ctas_per_sm, d->lean,
                               d->smem_bytes, ws->gate, ordered, !ordered && !accumulate && !memset_y, trace, st));
        if (ordered) ECSR_CUDA(launch_finish<float>(d, y, accumulate, ws->partials, st));
        return ECSR_OK;
    }
    for (const SetDesc& sd : d->sets) {
        if (sd.nb == 0) continue;
        cudaError_t e;
        if (d->dtype == ECSR_F16) e = launch_generic_set<float, __half, __half>(d, sd, x, ws->partials, st);
        else if (d->dtype == ECSR_F32) e = launch_generic_set<float, float, float>(d, sd, x, ws->partials, st);
        else e = launch_generic_set<double, double, double>(d, sd, x, ws->partials, st);
        ECSR_CUDA(e);
    }
    if (d->dtype == ECSR_F64) ECSR_CUDA(launch_finish<double>(d, y, accumulate, ws->partials, st));
    else ECSR_CUDA(launch_finish<float>(d, y, accumulate, ws->partials, st));
    return ECSR_OK;
}

// ---------------------------------------------------------------------------------
// Grouped launch: several independent products y_i = A_i x_i in ONE tiled launch. Each
// CTA works on one member (its x, a contiguous run of the member's own cost-balanced
// tile ranges, its tail queue); members get CTAs in proportion to their tile cost, and
// co-resident CTAs pair a member's first ranges with another's last. One launch ramp,
// one x-load latency and one tail are paid for the whole group instead of per matrix.
// ---------------------------------------------------------------------------------
struct ecsr_group {
    // Members packed for two CTAs per SM run in one launch, members packed for one CTA
    // per SM (x > 32 KB) in a second one (a "part" each), issued back to back.
    struct Part {
        std::vector<int> idx;   // members of this launch (group order)
        std::vector<int> ctas;  // CTAs per member
        std::vector<int> nst;   // stage-pool depth per member in this launch
        std::vector<uint32_t*> qmeta;  // per member: this launch's tail queue (device)
        std::vector<uint32_t> nqueue;
        int grid = 0, nc = 8, smem = 0, cps = 2;
        bool lean = true, gate_ok = true;
        uint4* d_cta_work = nullptr;
        size_t gate_off = 0;    // gate words in each workspace
    };
    int device = 0;
    std::vector<const ecsr_dev*> mats;
    std::vector<Part> parts;
    size_t queue_off = 0, ws_bytes = 0;  // member i's queue: queue_off + 128 * i
    static constexpr int kStreamSlots = 4;
    uint8_t* ws_base = nullptr;          // kStreamSlots workspaces of ws_bytes
    unsigned long long* d_trace = nullptr;  // tuning builds: per-CTA timeline of part 0
    mutable cudaStream_t ws_stream[kStreamSlots] = {};
    mutable int ws_bound = 0;
    mutable std::mutex ws_mu;
    std::vector<void*> allocs;
    uint8_t* workspace(cudaStream_t stream) const {
        std::lock_guard<std::mutex> lock(ws_mu);
        for (int i = 0; i < ws_bound; ++i)
            if (ws_stream[i] == stream) return ws_base + ws_bytes * i;
        if (ws_bound == kStreamSlots) return nullptr;
        ws_stream[ws_bound] = stream;
        return ws_base + ws_bytes * ws_bound++;
    }
    ~ecsr_group() {
        for (void* p : allocs) cudaFree(p);
    }
};

namespace {

// Plan one launch over members `idx` at `cps` CTAs per SM: CTAs per member in proportion
// to tile cost (at least 1, at most the member's static range count), member i's j-th
// CTA merging its static ranges [j R / c, (j + 1) R / c) (contiguous in the arena, equal
// cost each); co-resident CTAs pair one member's first ranges with another's last.
int plan_part(const std::vector<const ecsr_dev*>& mats, const DeviceLimits& lim, ecsr_group::Part* pt,
              std::vector<uint4>* work, std::vector<std::vector<uint32_t>>* qmetas) {
    const int n = static_cast<int>(pt->idx.size());
    pt->nc = ecsr::kConsumerWarpsPerSm / pt->cps;
    int64_t cap = 0;
    double total = 0;
    for (int i : pt->idx) {
        const ecsr_dev* d = mats[i];
        int nst = d->nstages, smem = d->smem_bytes;
        if (d->ctas_per_sm != pt->cps) {  // a two-CTA member in a one-CTA launch: deepen its pool
            const int64_t xbytes = round_up(2 * std::max<int64_t>(d->K, 1), 16);
            const int64_t avail = lim.smem_optin - kSmemReserve - 16 * kMaxStages - xbytes;
            nst = static_cast<int>(std::min<int64_t>(kMaxStages, avail / std::max(d->stage_bytes, 1)));
            smem = static_cast<int>(round_up(8 * nst + 8, 128) + int64_t{nst} * d->stage_bytes + xbytes);
        }
        pt->nst.push_back(nst);
        pt->smem = std::max(pt->smem, smem);
        pt->lean = pt->lean && d->lean;
        cap += d->grid;
        total += d->total_cost;
    }
    const int grid = static_cast<int>(std::min<int64_t>(int64_t{lim.sms} * pt->cps, cap));
    std::vector<int> c(n, 1);
    int used = n;
    while (used < grid) {
        int best = -1;
        double deficit = -1e300;
        for (int k = 0; k < n; ++k) {
            const ecsr_dev* d = mats[pt->idx[k]];
            if (c[k] >= d->grid) continue;
            const double want = grid * d->total_cost / std::max(total, 1e-30);
            if (want - c[k] > deficit) {
                deficit = want - c[k];
                best = k;
            }
        }
        if (best < 0) break;
        ++c[best];
        ++used;
    }
    pt->grid = used;
    pt->ctas = c;
    pt->gate_ok = pt->grid <= usable_sms(lim.sms) * pt->cps;
    std::vector<uint4> jobs;
    qmetas->assign(n, {});
    for (int k = 0; k < n; ++k) {
        const ecsr_dev* d = mats[pt->idx[k]];
        const int R = d->grid;
        std::vector<uint4> mj;
        for (int j = 0; j < c[k]; ++j) {
            const int r0 = static_cast<int>(static_cast<int64_t>(j) * R / c[k]);
            const int r1 = static_cast<int>(static_cast<int64_t>(j + 1) * R / c[k]);
            mj.push_back(make_uint4(static_cast<uint32_t>(k), d->cta_tile_h[r0], d->cta_tile_h[r1],
                                    static_cast<uint32_t>(j)));
        }
        split_tail_queue(d, &mj, group_queue_share(), &(*qmetas)[k]);
        jobs.insert(jobs.end(), mj.begin(), mj.end());
    }
    work->assign(pt->grid, make_uint4(0, 0, 0, 0));
    for (int b = 0; b < pt->grid; ++b) (*work)[b] = jobs[range_of_block(b, pt->grid, pt->cps)];
    return ECSR_OK;
}

}  // namespace

int ecsr_b200_group_create(const ecsr_dev* const* mats, int32_t n, ecsr_group** out) {
    if (!out) return fail(ECSR_ERR_VALUE, "out is null");
    *out = nullptr;
    if (!mats || n < 1 || n > ecsr::kMaxMembers)
        return fail(ECSR_ERR_VALUE, "a group holds 1 to " + std::to_string(ecsr::kMaxMembers) + " matrices");
    for (int i = 0; i < n; ++i) {
        const ecsr_dev* d = mats[i];
        if (!d) return fail(ECSR_ERR_VALUE, "null handle in group");
        if (d->layout != 1 || d->M == 0 || d->grid == 0)
            return fail(ECSR_ERR_VALUE, "group members must use the tiled layout (fp16, W = 32, B <= 8)");
        if (d->device != mats[0]->device) return fail(ECSR_ERR_VALUE, "group members on different devices");
        if (d->wide != mats[0]->wide)
            return fail(ECSR_ERR_VALUE, "group members must all have K <= 65535 or all K > 65535");
    }
    DeviceLimits lim;
    int rc = query_limits(mats[0]->device, &lim);
    if (rc) return rc;
    auto* g = new ecsr_group();
    g->device = mats[0]->device;
    g->mats.assign(mats, mats + n);
    for (int cps : {2, 1}) {
        ecsr_group::Part pt;
        pt.cps = cps;
        for (int i = 0; i < n; ++i)
            if ((group_force_cps1() ? 1 : mats[i]->ctas_per_sm) == cps) pt.idx.push_back(i);
        if (!pt.idx.empty()) g->parts.push_back(pt);
    }
    DeviceGuard guard(g->device);
    if (guard.err != cudaSuccess) {
        delete g;
        return fail(ECSR_ERR_CUDA, cudaGetErrorString(guard.err));
    }
    size_t off = 0;
    for (auto& pt : g->parts) {
        std::vector<uint4> work;
        std::vector<std::vector<uint32_t>> qmetas;
        plan_part(g->mats, lim, &pt, &work, &qmetas);
        int64_t total_bytes = 0;
        cudaError_t err = cudaSuccess;
        pt.d_cta_work = dalloc_copy(work, &total_bytes, &err);
        if (pt.d_cta_work) g->allocs.push_back(pt.d_cta_work);
        for (auto& q : qmetas) {
            uint32_t* dq = err == cudaSuccess ? dalloc_copy(q, &total_bytes, &err) : nullptr;
            if (dq) g->allocs.push_back(dq);
            pt.qmeta.push_back(dq);
            pt.nqueue.push_back(static_cast<uint32_t>(q.size() / 2));
        }
        if (err == cudaSuccess) rc = configure_tiled_kernels(g->device, pt.smem);
        else rc = fail(ECSR_ERR_CUDA, std::string("group schedule: ") + cudaGetErrorString(err));
        if (rc) {
            delete g;
            return rc;
        }
        pt.gate_off = off;
        off += gate_bytes(pt.grid);
    }
    g->queue_off = off;
    g->ws_bytes = off + 128 * static_cast<size_t>(n);
    cudaError_t err = cudaMalloc(&g->ws_base, g->ws_bytes * ecsr_group::kStreamSlots);
    if (g->ws_base) g->allocs.push_back(g->ws_base);
    if (err == cudaSuccess) err = cudaMemset(g->ws_base, 0, g->ws_bytes * ecsr_group::kStreamSlots);
    if (err != cudaSuccess) {
        delete g;
        return fail(ECSR_ERR_CUDA, std::string("group workspace: ") + cudaGetErrorString(err));
    }
    *out = g;
    return ECSR_OK;
}

int ecsr_b200_group_spmv(const ecsr_group* g, const void* const* xs, void* const* ys, int32_t mode,
                         void* stream) {
    if (!g || !xs || !ys) return fail(ECSR_ERR_VALUE, "null argument");
    const int n = static_cast<int>(g->mats.size());
    for (int i = 0; i < n; ++i)
        if (!xs[i] || !ys[i]) return fail(ECSR_ERR_VALUE, "null x or y");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (mode & ECSR_SPMV_ORDERED) {  // bitwise mode: the members one after another
        for (int i = 0; i < n; ++i) {
            const int rc = ecsr_b200_spmv(g->mats[i], xs[i], ys[i], mode, stream);
            if (rc) return rc;
        }
        return ECSR_OK;
    }
    uint8_t* ws = g->workspace(st);
    if (!ws)
        return fail(ECSR_ERR_VALUE, "group already used from " + std::to_string(ecsr_group::kStreamSlots) +
                                        " other streams (one workspace per stream)");
    DeviceGuard guard(g->device);
    ECSR_CUDA(guard.err);
    for (const auto& pt : g->parts) {
        MemberLaunch m[ecsr::kMaxMembers];
        const int k = static_cast<int>(pt.idx.size());
        for (int j = 0; j < k; ++j) {
            const int i = pt.idx[j];
            m[j] = MemberLaunch{g->mats[i], xs[i], ys[i], reinterpret_cast<uint32_t*>(ws + g->queue_off + 128 * i),
                                nullptr, pt.ctas[j], pt.nst[j], pt.qmeta[j], pt.nqueue[j]};
        }
        const bool overwrite = (mode & ECSR_SPMV_ACCUMULATE) == 0;
        const bool memset_y = overwrite && (!pt.gate_ok || (mode & ECSR_SPMV_MEMSET_Y));
        if (memset_y)
            for (int j = 0; j < k; ++j) ECSR_CUDA(cudaMemsetAsync(m[j].y, 0, 4 * m[j].d->M, st));
        unsigned long long* trace = nullptr;
        if (trace_enabled() && &pt == &g->parts[0]) {  // tuning builds only (caller resets)
            ecsr_group* gm = const_cast<ecsr_group*>(g);
            if (!gm->d_trace) {
                ECSR_CUDA(cudaMalloc(&gm->d_trace, 8 * 16 * pt.grid));
                ECSR_CUDA(cudaMemset(gm->d_trace, 0, 8 * 16 * pt.grid));
                gm->allocs.push_back(gm->d_trace);
            }
            trace = gm->d_trace;
        }
        ECSR_CUDA(launch_tiled(m, k, pt.d_cta_work, pt.grid, pt.nc, pt.lean, pt.smem,
                               reinterpret_cast<unsigned long long*>(ws + pt.gate_off), false,
                               overwrite && !memset_y, trace, st));
    }
    return ECSR_OK;
}

int ecsr_b200_group_info(const ecsr_group* g, int32_t* launches, int32_t* grid, int32_t* ctas, int32_t n) {
    if (!g) return fail(ECSR_ERR_VALUE, "null group");
    if (launches) *launches = static_cast<int32_t>(g->parts.size());
    if (grid) *grid = 0;
    for (const auto& pt : g->parts) {
        if (grid) *grid += pt.grid;
        for (size_t j = 0; j < pt.idx.size(); ++j)
            if (ctas && pt.idx[j] < n) ctas[pt.idx[j]] = pt.ctas[j];
    }
    return ECSR_OK;
}

void ecsr_b200_group_free(ecsr_group* g) { delete g; }

// Internal tuning aid: the per-CTA timeline of a group's first launch (16 u64 per CTA;
// reset = zero it, with slot 7 = ~0).
int ecsr_b200_debug_group_trace(ecsr_group* g, unsigned long long* out, int64_t n, int32_t reset) {
    if (!g || g->parts.empty()) return fail(ECSR_ERR_VALUE, "no group");
    const int grid = g->parts[0].grid;
    if (!g->d_trace) return fail(ECSR_ERR_VALUE, "no trace recorded");
    if (reset) {
        std::vector<unsigned long long> init(16 * grid, 0ull);
        for (int c = 0; c < grid; ++c) init[16 * c + 7] = ~0ull;
        ECSR_CUDA(cudaMemcpy(g->d_trace, init.data(), 8 * init.size(), cudaMemcpyHostToDevice));
        return ECSR_OK;
    }
    ECSR_CUDA(cudaMemcpy(out, g->d_trace, 8 * std::min<int64_t>(n, 16 * grid), cudaMemcpyDeviceToHost));
    return ECSR_OK;
}

int ecsr_b200_info(const ecsr_dev* d, int64_t* num_rows, int64_t* num_cols, int32_t* nsets,
                   int32_t* warp_size, int32_t* delta_bits, int32_t* value_bits, int32_t* device_dtype) {
    if (!d) return fail(ECSR_ERR_VALUE, "null handle");
    if (num_rows) *num_rows = d->M;
    if (num_cols) *num_cols = d->K;
    if (nsets) *nsets = static_cast<int32_t>(d->sets.size());
    if (warp_size) *warp_size = d->W;
    if (delta_bits) *delta_bits = d->B;
    if (value_bits) *value_bits = d->vbits;
    if (device_dtype) *device_dtype = d->dtype;
    return ECSR_OK;
}

int ecsr_b200_set_info(const ecsr_dev* d, int32_t set, ecsr_set_info* info) {
    if (!d || !info) return fail(ECSR_ERR_VALUE, "null argument");
    if (set < 0 || set >= static_cast<int32_t>(d->sets.size())) return fail(ECSR_ERR_VALUE, "set index");
    const SetDesc& s = d->sets[set];
    info->granularity = s.g;
    info->vector_size = s.v;
    info->num_blocks = s.nb;
    info->stored_cols = s.stored;
    info->real_nnz = s.real;
    return ECSR_OK;
}

static void store_value(void* dst, int dtype, int64_t i, double v) {
    if (dtype == ECSR_F64) static_cast<double*>(dst)[i] = v;
    else if (dtype == ECSR_F32) static_cast<float*>(dst)[i] = static_cast<float>(v);
    else static_cast<uint16_t*>(dst)[i] = f64_to_f16(v);
}

int ecsr_b200_unpack(const ecsr_dev* d, ecsr_out_set* out, int32_t nsets, int32_t out_value_dtype) {
    if (!d || (!out && nsets > 0)) return fail(ECSR_ERR_VALUE, "null argument");
    if (nsets != static_cast<int32_t>(d->sets.size())) return fail(ECSR_ERR_VALUE, "set count mismatch");
    if (out_value_dtype != ECSR_F16 && out_value_dtype != ECSR_F32 && out_value_dtype != ECSR_F64)
        return fail(ECSR_ERR_VALUE, "bad output dtype");
    // cold section: pad_mask
    int64_t moff = 0;
    for (int si = 0; si < nsets; ++si) {
        std::memcpy(out[si].pad_mask, d->pad_mask.data() + moff, d->sets[si].stored);
        moff += d->sets[si].stored;
    }
    if (d->layout == 1) {
        std::vector<uint8_t> arena(d->arena_bytes);
        std::vector<uint32_t> tstart(d->ntiles + 1);
        ECSR_CUDA(cudaMemcpy(arena.data(), d->d_arena, d->arena_bytes, cudaMemcpyDeviceToHost));
        ECSR_CUDA(cudaMemcpy(tstart.data(), d->d_tile_start16, 4 * (d->ntiles + 1), cudaMemcpyDeviceToHost));
        // Records may sit in any order (the packer orders each CTA's tiles longest
        // record first); every block is identified by its ordered-mode slot, which is
        // unique: slot = set.slot0 + block * g. Pass 1 finds every block's record and
        // chunk count, pass 2 restores the reference arrays.
        struct Ref {
            const uint8_t* rec = nullptr;
            int bk = 0;
            int64_t nch = -1;
        };
        std::vector<std::vector<Ref>> refs(nsets);
        for (int si = 0; si < nsets; ++si) refs[si].resize(d->sets[si].nb);
        auto set_of_slot = [&](uint32_t slot) -> int {
            int lo = 0, hi = nsets - 1, ans = -1;
            while (lo <= hi) {  // last set with slot0 <= slot (sets are in slot order)
                const int mid = (lo + hi) / 2;
                if (d->sets[mid].slot0 <= slot) {
                    ans = mid;
                    lo = mid + 1;
                } else {
                    hi = mid - 1;
                }
            }
            while (ans >= 0 && d->sets[ans].nb == 0) --ans;  // empty sets own no slots
            return ans;
        };
        for (int64_t t = 0; t < d->ntiles; ++t) {
            const uint8_t* tile = arena.data() + 16ull * tstart[t];
            uint32_t nrec;
            std::memcpy(&nrec, tile, 4);
            for (uint32_t jr = 0; jr < nrec; ++jr) {
                uint16_t off16;
                std::memcpy(&off16, tile + 8 + 2 * jr, 2);
                const uint8_t* r = tile + 16 * off16;
                uint16_t nmin;
                std::memcpy(&nmin, r + 48, 2);
                const int g = r[50], v = r[51], nb = r[52];
                for (int bk = 0; bk < nb; ++bk) {
                    uint32_t slot;
                    std::memcpy(&slot, r + 4 * bk, 4);
                    const int si = set_of_slot(slot);
                    if (si < 0) return fail(ECSR_ERR_CONTAINER, "record slot outside every set");
                    const SetDesc& sd = d->sets[si];
                    if (g != sd.g || v != sd.v) return fail(ECSR_ERR_CONTAINER, "arena/set descriptor mismatch");
                    const int64_t blk = (static_cast<int64_t>(slot) - sd.slot0) / g;
                    if (blk >= sd.nb || refs[si][blk].nch >= 0)
                        return fail(ECSR_ERR_CONTAINER, "record slot out of range or repeated");
                    uint16_t nt;
                    std::memcpy(&nt, r + 32 + 2 * bk, 2);
                    refs[si][blk] = Ref{r, bk, static_cast<int64_t>(nmin) + nt};
                }
            }
        }
        const int esz = d->wide ? 4 : 2;
        for (int si = 0; si < nsets; ++si) {
            const SetDesc& sd = d->sets[si];
            ecsr_out_set& o = out[si];
            o.block_indptr[0] = 0;
            for (int64_t b = 0; b < sd.nb; ++b) {
                const Ref& rf = refs[si][b];
                if (rf.nch < 0) return fail(ECSR_ERR_CONTAINER, "arena holds fewer blocks than sets");
                const uint8_t* r = rf.rec;
                const int g = r[50], v = r[51], P = r[54], bk = rf.bk;
                uint16_t nmin;
                std::memcpy(&nmin, r + 48, 2);
                const uint8_t* q = r + ecsr::group_header_bytes(g, P);
                const uint8_t* body = q + 32 * P * esz;
                const int64_t dch = 32 * v, vch = 32 * v * g;
                const int64_t S = P * (dch + 2 * vch);
                const uint8_t* tail = body + nmin * S;  // block bk's tail follows blocks < bk
                for (int pb = 0; pb < bk; ++pb) {
                    uint16_t nt;
                    std::memcpy(&nt, r + 32 + 2 * pb, 2);
                    tail += static_cast<int64_t>(nt) * (dch + 2 * vch);
                }
                const int64_t nch = rf.nch;
                o.block_indptr[b + 1] = o.block_indptr[b] + nch * dch;
                std::memcpy(o.row_indices + b * g, r + 64 + 4 * g * bk, 4 * g);
                for (int l = 0; l < 32; ++l) {
                    uint32_t bv = 0;
                    std::memcpy(&bv, q + (l * P + bk) * esz, esz);
                    o.base_indices[b * 32 + l] = bv;
                }
                const int64_t st0 = o.block_indptr[b];
                for (int64_t c = 0; c < nch; ++c) {
                    const uint8_t* dp;
                    const uint8_t* vp;
                    if (c < nmin) {
                        dp = body + c * S + bk * dch;
                        vp = body + c * S + P * dch + bk * 2 * vch;
                    } else {
                        dp = tail;
                        vp = tail + dch;
                        tail += dch + 2 * vch;
                    }
                    for (int64_t i = 0; i < dch; ++i) o.delta_indices[st0 + c * dch + i] = dp[i];
                    for (int64_t i = 0; i < vch; ++i) {
                        uint16_t h;
                        std::memcpy(&h, vp + 2 * i, 2);
                        const int64_t at = (st0 + c * dch) * g + i;
                        if (out_value_dtype == ECSR_F16) static_cast<uint16_t*>(o.block_values)[at] = h;
                        else store_value(o.block_values, out_value_dtype, at, f16_to_f32(h));
                    }
                }
            }
        }
        return ECSR_OK;
    }
    // generic layout: copy the reference arrays back
    int64_t voff = 0;
    const int esz = elem_size(d->dtype);
    for (int si = 0; si < nsets; ++si) {
        const SetDesc& sd = d->sets[si];
        ecsr_out_set& o = out[si];
        ECSR_CUDA(cudaMemcpy(o.block_indptr, d->d_indptr + sd.indptr_off, 8 * (sd.nb + 1), cudaMemcpyDeviceToHost));
        if (sd.nb) {
            ECSR_CUDA(cudaMemcpy(o.base_indices, d->d_bases + sd.base_off, 4 * sd.nb * d->W, cudaMemcpyDeviceToHost));
            ECSR_CUDA(cudaMemcpy(o.row_indices, d->d_rows + sd.row_off, 4 * sd.nb * sd.g, cudaMemcpyDeviceToHost));
        }
        if (sd.stored) {
            ECSR_CUDA(cudaMemcpy(o.delta_indices, d->d_deltas + sd.col_off, 4 * sd.stored, cudaMemcpyDeviceToHost));
            std::vector<uint8_t> raw(sd.stored * sd.g * esz);
            ECSR_CUDA(cudaMemcpy(raw.data(), static_cast<const uint8_t*>(d->d_values) + voff * esz, raw.size(),
                                 cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < sd.stored * sd.g; ++i) {
                if (out_value_dtype == d->dtype) {
                    std::memcpy(static_cast<uint8_t*>(o.block_values) + i * esz, raw.data() + i * esz, esz);
                } else {
                    store_value(o.block_values, out_value_dtype, i, host_value(raw.data(), d->dtype, i));
                }
            }
        }
        voff += sd.stored * sd.g;
    }
    return ECSR_OK;
}

// Access trace of the device layout (the reference's
// spmv_ec_traced + check_coalescing, executor.py:106-221): one entry per block, warp
// step and array, in the order the kernel issues the shared-memory reads, each mapped
// back to the reference array span it carries. The tiled walk replays the kernel's
// own pointer arithmetic (tiled_group_record / tiled_wide_record in ecsr_kernels.cuh),
// not unpack's, so the audit checks the addresses the kernel really reads.
int ecsr_b200_trace(const ecsr_dev* d, ecsr_trace_rec* out, int64_t cap, int64_t* count) {
    if (!d || !count) return fail(ECSR_ERR_VALUE, "null argument");
    const int nsets = static_cast<int>(d->sets.size());
    std::vector<int64_t> warp0(nsets + 1, 0);
    for (int si = 0; si < nsets; ++si) warp0[si + 1] = warp0[si] + d->sets[si].nb;
    int64_t n = 0;
    auto emit = [&](int64_t warp, int32_t step, int32_t array, int32_t set, int32_t lane_bytes, int64_t start,
                    int64_t span, int64_t dev_offset, int64_t dev_bytes) {
        if (out && n < cap)
            out[n] = ecsr_trace_rec{warp, step, array, set, lane_bytes, start, span, dev_offset, dev_bytes};
        ++n;
    };
    if (d->layout == 2) {  // generic kernel: the reference arrays, element loads per lane
        const int esz = elem_size(d->dtype);
        for (int si = 0; si < nsets; ++si) {
            const SetDesc& sd = d->sets[si];
            std::vector<int64_t> indptr(sd.nb + 1);
            ECSR_CUDA(cudaMemcpy(indptr.data(), d->d_indptr + sd.indptr_off, 8 * (sd.nb + 1), cudaMemcpyDeviceToHost));
            const int64_t chunk = static_cast<int64_t>(d->W) * sd.v;
            for (int64_t b = 0; b < sd.nb; ++b)
                for (int64_t c = 0; c < (indptr[b + 1] - indptr[b]) / chunk; ++c) {
                    const int64_t st = indptr[b] + c * chunk;
                    emit(warp0[si] + b, static_cast<int32_t>(c), 0, si, 4, st, chunk, 4 * (sd.col_off + st), 4 * chunk);
                    emit(warp0[si] + b, static_cast<int32_t>(c), 1, si, esz, st * sd.g, chunk * sd.g,
                         esz * (sd.val_off + st * sd.g), esz * chunk * sd.g);
                }
        }
        *count = n;
        return ECSR_OK;
    }
    std::vector<uint8_t> arena(d->arena_bytes);
    std::vector<uint32_t> tstart(d->ntiles + 1);
    ECSR_CUDA(cudaMemcpy(arena.data(), d->d_arena, d->arena_bytes, cudaMemcpyDeviceToHost));
    ECSR_CUDA(cudaMemcpy(tstart.data(), d->d_tile_start16, 4 * (d->ntiles + 1), cudaMemcpyDeviceToHost));
    // pass 1: chunk count of every block -> the reference's block_indptr (in chunks)
    std::vector<std::vector<int64_t>> nch(nsets);
    for (int si = 0; si < nsets; ++si) nch[si].assign(d->sets[si].nb, -1);
    auto locate = [&](uint32_t slot, int g, int* set, int64_t* blk) -> bool {
        for (int si = nsets - 1; si >= 0; --si) {
            const SetDesc& sd = d->sets[si];
            if (sd.nb == 0 || sd.slot0 > slot) continue;
            if (sd.g != g) return false;
            *set = si;
            *blk = (static_cast<int64_t>(slot) - sd.slot0) / g;
            return *blk < sd.nb;
        }
        return false;
    };
    for (int64_t t = 0; t < d->ntiles; ++t) {
        const uint8_t* tile = arena.data() + 16ull * tstart[t];
        uint32_t nrec;
        std::memcpy(&nrec, tile, 4);
        for (uint32_t jr = 0; jr < nrec; ++jr) {
            uint16_t off16, nmin;
            std::memcpy(&off16, tile + 8 + 2 * jr, 2);
            const uint8_t* r = tile + 16 * off16;
            std::memcpy(&nmin, r + 48, 2);
            for (int bk = 0; bk < r[52]; ++bk) {
                uint32_t slot;
                uint16_t nt;
                std::memcpy(&slot, r + 4 * bk, 4);
                std::memcpy(&nt, r + 32 + 2 * bk, 2);
                int si;
                int64_t blk;
                if (!locate(slot, r[50], &si, &blk) || nch[si][blk] >= 0)
                    return fail(ECSR_ERR_CONTAINER, "record slot outside every set or repeated");
                nch[si][blk] = static_cast<int64_t>(nmin) + nt;
            }
        }
    }
    std::vector<std::vector<int64_t>> first(nsets);  // stored column of each block's chunk 0
    for (int si = 0; si < nsets; ++si) {
        const SetDesc& sd = d->sets[si];
        first[si].assign(sd.nb, 0);
        int64_t acc = 0;
        for (int64_t b = 0; b < sd.nb; ++b) {
            if (nch[si][b] < 0) return fail(ECSR_ERR_CONTAINER, "arena holds fewer blocks than sets");
            first[si][b] = acc;
            acc += nch[si][b] * 32 * sd.v;
        }
    }
    // pass 2: the kernel's walk
    const int64_t bases = d->wide ? 128 : 64;  // lane bases per block, bytes
    for (int64_t t = 0; t < d->ntiles; ++t) {
        const int64_t tile = 16ll * tstart[t];
        uint32_t nrec;
        std::memcpy(&nrec, arena.data() + tile, 4);
        for (uint32_t jr = 0; jr < nrec; ++jr) {
            uint16_t off16, nmin;
            std::memcpy(&off16, arena.data() + tile + 8 + 2 * jr, 2);
            const int64_t r = tile + 16 * off16;
            const uint8_t* rh = arena.data() + r;
            std::memcpy(&nmin, rh + 48, 2);
            const int g = rh[50], v = rh[51], nb = rh[52], P = rh[54];
            int sb[8];
            int64_t bb[8];
            for (int bk = 0; bk < nb; ++bk) {
                uint32_t slot;
                std::memcpy(&slot, rh + 4 * bk, 4);
                locate(slot, g, &sb[bk], &bb[bk]);
            }
            const int64_t dch = 32 * v;
            auto chunk = [&](int bk, int64_t c, int64_t dptr, int64_t vptr, int64_t vbytes) {
                const int si = sb[bk];
                const int64_t st = first[si][bb[bk]] + c * dch;
                emit(warp0[si] + bb[bk], static_cast<int32_t>(c), 0, si, v, st, dch, dptr, dch);
                emit(warp0[si] + bb[bk], static_cast<int32_t>(c), 1, si, g > 8 ? 16 : 2 * v * g, st * g, dch * g,
                     vptr, vbytes);
            };
            if (g <= 8) {  // tiled_group_record<G, V, P>
                const int64_t vch = 64 * v * g;
                int64_t ptr = r + ecsr::group_header_bytes(g, P) + bases * P;
                for (int64_t c = 0; c < nmin; ++c, ptr += P * (dch + vch))
                    for (int bk = 0; bk < nb; ++bk) chunk(bk, c, ptr + bk * dch, ptr + P * dch + bk * vch, vch);
                for (int bk = 0; bk < nb; ++bk) {
                    uint16_t nt;
                    std::memcpy(&nt, rh + 32 + 2 * bk, 2);
                    for (int64_t c = 0; c < nt; ++c, ptr += dch + vch) chunk(bk, nmin + c, ptr, ptr + dch, vch);
                }
            } else {  // tiled_wide_record<V>: one block, g / 8 passes over the same spans
                const int64_t vch = 64ll * v * g;
                int64_t ptr = r + ecsr::group_header_bytes(g, 1) + bases;
                for (int64_t c = 0; c < nmin; ++c, ptr += dch + vch) chunk(0, c, ptr, ptr + dch, vch);
            }
        }
    }
    *count = n;
    return ECSR_OK;
}

int ecsr_b200_bytes(const ecsr_dev* d, ecsr_bytes* out) {
    if (!d || !out) return fail(ECSR_ERR_VALUE, "null argument");
    *out = d->bytes;
    return ECSR_OK;
}

void ecsr_b200_free(ecsr_dev* d) { delete d; }

// Internal tuning aid (not part of the public header): the last traced launch's
// per-CTA timeline, 8 u64 globaltimer stamps per CTA (ECSR_B200_DEBUG & 4).
int ecsr_b200_debug_trace(const ecsr_dev* d, unsigned long long* out, int64_t n) {
    if (!d || !d->d_trace) return fail(ECSR_ERR_VALUE, "no trace recorded");
    ECSR_CUDA(cudaMemcpy(out, d->d_trace, 8 * std::min<int64_t>(n, 16 * d->grid), cudaMemcpyDeviceToHost));
    return ECSR_OK;
}

// Internal tuning aid: clear the trace buffer (after one traced launch allocated it).
int ecsr_b200_debug_trace_reset(ecsr_dev* d) {
    if (!d || d->layout != 1) return fail(ECSR_ERR_VALUE, "no tiled layout");
    if (!d->d_trace) {
        ECSR_CUDA(cudaMalloc(&d->d_trace, 8 * 16 * d->grid));
        d->allocs.push_back(d->d_trace);
    }
    std::vector<unsigned long long> init(16 * d->grid, 0ull);
    for (int c = 0; c < d->grid; ++c) init[16 * c + 7] = ~0ull;
    ECSR_CUDA(cudaMemcpy(d->d_trace, init.data(), 8 * init.size(), cudaMemcpyHostToDevice));
    return ECSR_OK;
}

// Internal tuning aid: per CTA 9 doubles -- records and block-chunk steps for g = 1, 2,
// 4, >= 8 (interleaved rec, steps) and record bytes -- of its static tile range.
int ecsr_b200_debug_ctafeat(const ecsr_dev* d, double* out, int64_t n) {
    if (!d || d->layout != 1) return fail(ECSR_ERR_VALUE, "no tiled layout");
    for (int c = 0; c < d->grid && 9 * (c + 1) <= n; ++c) {
        double f[9] = {0};
        for (uint32_t t = d->cta_range_h[2 * c]; t < d->cta_range_h[2 * c + 1]; ++t) {
            const TileFeat& tf = d->tile_feat[t];
            for (int k = 0; k < 4; ++k) {
                f[2 * k] += tf.rec[k];
                f[2 * k + 1] += tf.steps[k];
            }
            f[8] += tf.bytes;
        }
        std::memcpy(out + 9 * c, f, sizeof f);
    }
    return ECSR_OK;
}

int ecsr_b200_spmv_set(int32_t g, int32_t warp_size, int32_t vector_size, int64_t num_blocks,
                       const uint32_t* row_ids, const int64_t* block_indptr,
                       const uint32_t* base_indices, const uint32_t* delta_indices,
                       const void* block_values, const void* x, int64_t x_len, void* y,
                       int64_t y_len, int32_t y_dtype) {
    if (y_dtype != ECSR_F32 && y_dtype != ECSR_F64) return fail(ECSR_ERR_VALUE, "y must be f32 or f64");
    if (num_blocks < 0) return fail(ECSR_ERR_VALUE, "negative block count");
    ecsr_host_set s{};
    s.granularity = g;
    s.vector_size = vector_size;
    s.num_blocks = num_blocks;
    s.stored_cols = num_blocks > 0 ? block_indptr[num_blocks] : 0;
    s.real_nnz = 0;
    s.row_indices = row_ids;
    s.block_indptr = block_indptr;
    s.base_indices = base_indices;
    s.delta_indices = delta_indices;
    s.pad_mask = nullptr;
    s.block_values = block_values;
    // The reference kernel takes deltas as u32 and never range-checks them; accept any
    // width up to 16 bits here and let validate() bound every decoded column.
    ecsr_dev* d = nullptr;
    int rc = ecsr_b200_pack(&s, 1, y_len, x_len, warp_size, 32, 16, y_dtype, y_dtype,
                            ECSR_PACK_FORCE_GENERIC | kPackInternal, &d);
    if (rc) return rc;
    const size_t esz = y_dtype == ECSR_F64 ? 8 : 4;
    void* dx = nullptr;
    void* dy = nullptr;
    int out = ECSR_OK;
    cudaError_t e = cudaMalloc(&dx, std::max<size_t>(16, x_len * esz));
    if (e == cudaSuccess) e = cudaMalloc(&dy, std::max<size_t>(16, y_len * esz));
    if (e == cudaSuccess && x_len) e = cudaMemcpy(dx, x, x_len * esz, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && y_len) e = cudaMemcpy(dy, y, y_len * esz, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        out = ecsr_b200_spmv(d, dx, dy, ECSR_SPMV_ACCUMULATE | ECSR_SPMV_ORDERED, nullptr);
        if (out == ECSR_OK) e = cudaDeviceSynchronize();
        if (out == ECSR_OK && e == cudaSuccess && y_len) e = cudaMemcpy(y, dy, y_len * esz, cudaMemcpyDeviceToHost);
    }
    if (dx) cudaFree(dx);
    if (dy) cudaFree(dy);
    ecsr_b200_free(d);
    if (out) return out;
    if (e != cudaSuccess) return fail(ECSR_ERR_CUDA, std::string("spmv_set: ") + cudaGetErrorString(e));
    return ECSR_OK;
}

}  // extern "C"
