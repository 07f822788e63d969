// ecsr_xchg.cu -- the row-sharded path's y exchange over NVLink peer memory
// (SURVEY.md §8(e), §8(f) #4): push-with-signal, PDL-chained after the shard SpMV.
//
// Every rank owns one device buffer (CUDA IPC, mapped by every peer):
//   [ y_full (all ranks' rows, final layout) | pad | arrival flags: world x 128 B |
//     ready flags: world x 128 B | local words: step, done ]
// One exchange = ONE kernel launched right behind the rank's SpMV launch (PDL: its CTAs
// are resident while the SpMV drains and start copying the moment it completes):
//   CTAs (q, part) copy a slice of this rank's segments of y (its shard rows of every
//           matrix, from the SpMV's output) into rank q's y_full at their final offsets
//           -- plain stores through the peer mapping (NVLink / NVSwitch for q != rank),
//           32 / world CTAs per destination -- then fence (system scope) and bump
//           flag[rank] in rank q's buffer (release);
//   then    each waits until this rank's own flag[q] counts all of rank q's slices of
//           the step (rank q's push into us landed, acquire), so when the kernel
//           completes y_full holds every rank's rows and everything stream-ordered after
//           it may read them.
// It replaces the NCCL all-gather + index assembly of the sharded step (one exchange
// per step, whatever the number of matrices). Steps are counted on the device (the last
// CTA of an exchange advances the rank's step word), so graph replays stay in sync.
// No push overwrites a y_full its owner still reads: before pushing step s into rank q,
// a CTA waits for q's `ready` word (in its own buffer) to reach s; rank q sets it when
// its own exchange s passes griddepcontrol.wait, i.e. once everything stream-ordered
// before that exchange on q -- every reader of q's y_full of step s-1 -- has completed.
// A y_full therefore stays valid until its owner's next exchange call, however far
// another rank runs ahead (tests/test_gpu_exchange.py: a lagging peer).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ecsr_b200.h"

namespace ecsr_internal {
int set_error(int code, const std::string& msg);
}

namespace {

constexpr int kMaxRanks = 16;
constexpr int kMaxSegs = 64;  // segments ride in the kernel parameters (no dependent loads)
constexpr int kLine = 128;

struct XchgParams {
    const uint8_t* src;                 // this rank's SpMV output (device)
    ecsr_xchg_seg segs[kMaxSegs];
    int32_t nsegs;
    int32_t rank, world;
    int32_t parts;                      // CTAs per destination rank
    uint8_t* peer_base[kMaxRanks];      // every rank's buffer (own included), mapped here
    int64_t flags_off;                  // byte offset of the flags area in every buffer
    unsigned long long* step_word;      // local: exchanges completed
    unsigned int* done_word;            // local: CTAs finished in the current exchange
};

__global__ void __launch_bounds__(256) ecsr_xchg_kernel(const __grid_constant__ XchgParams p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the SpMV's y is complete
    const int q = blockIdx.x % p.world, part = blockIdx.x / p.world;  // destination, slice
    unsigned long long step;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(step) : "l"(p.step_word) : "memory");
    ++step;
    uint8_t* dst = p.peer_base[q];
#ifndef ECSR_XCHG_NO_READY  // (experiment builds only: shows the race the handshake closes)
    if (threadIdx.x == 0) {
        // Past griddepcontrol.wait everything before this exchange on our stream has
        // completed, the readers of our y_full's previous step included: tell rank q
        // (ready[rank] in q's buffer) that it may push this step into us. Then wait for
        // q to say the same before pushing into its y_full.
        if (part == 0) {
            unsigned long long* ready = reinterpret_cast<unsigned long long*>(
                dst + p.flags_off + static_cast<int64_t>(p.world + p.rank) * kLine);
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(ready), "l"(step) : "memory");
        }
        const unsigned long long* qready = reinterpret_cast<const unsigned long long*>(
            p.peer_base[p.rank] + p.flags_off + static_cast<int64_t>(p.world + q) * kLine);
        unsigned long long v;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(qready) : "memory");
        } while (v < step);
    }
    __syncthreads();
#endif
    const int64_t stride = static_cast<int64_t>(p.parts) * blockDim.x;
    for (int s = 0; s < p.nsegs; ++s) {
        const ecsr_xchg_seg sg = p.segs[s];
        const uint8_t* a = p.src + sg.src_off;
        uint8_t* b = dst + sg.dst_off;
        const int64_t first = static_cast<int64_t>(part) * blockDim.x + threadIdx.x;
        const bool vec = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | sg.bytes) & 15) == 0;
        if (vec) {
            const int64_t n = sg.bytes / 16;
            for (int64_t i = first; i < n; i += stride)
                reinterpret_cast<uint4*>(b)[i] = reinterpret_cast<const uint4*>(a)[i];
        } else {
            const int64_t n = sg.bytes / 4;
            for (int64_t i = first; i < n; i += stride)
                reinterpret_cast<uint32_t*>(b)[i] = reinterpret_cast<const uint32_t*>(a)[i];
        }
    }
    // every thread's stores, then one system-scope fence for the CTA (the pattern of
    // cooperative groups' grid sync: bar.sync, then thread 0 fences and signals)
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
    if (threadIdx.x == 0) {
        unsigned long long* flag =
            reinterpret_cast<unsigned long long*>(dst + p.flags_off + static_cast<int64_t>(p.rank) * kLine);
#ifdef ECSR_XCHG_GPU_SCOPE
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(flag) : "memory");
#else
        asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(flag) : "memory");
#endif
        // wait for rank q's push into this rank (its flag slot in our own buffer)
        const unsigned long long* mine = reinterpret_cast<const unsigned long long*>(
            p.peer_base[p.rank] + p.flags_off + static_cast<int64_t>(q) * kLine);
        unsigned long long v;
#ifndef ECSR_XCHG_NO_WAIT
        do {
#ifdef ECSR_XCHG_GPU_SCOPE
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
#else
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
#endif
        } while (v < step * static_cast<unsigned long long>(p.parts));  // all of rank q's slices
#endif
        // the last CTA of the exchange advances the step (the next exchange on this
        // stream reads it after its griddepcontrol.wait, i.e. after this grid completed)
        if (atomicAdd(p.done_word, 1u) == gridDim.x - 1u) {
            *p.done_word = 0u;
            *p.step_word = step;
        }
    }
}

int fail(int code, const std::string& msg) { return ecsr_internal::set_error(code, msg); }

}  // namespace

struct ecsr_xchg {
    int device = 0, rank = 0, world = 1;
    int64_t y_bytes = 0, flags_off = 0, bytes = 0;
    uint8_t* buf = nullptr;                     // own buffer
    std::vector<uint8_t*> peer;                 // mapped peer buffers (own at [rank])
    std::vector<bool> opened;                   // cudaIpcOpenMemHandle'd (to close)
    std::vector<ecsr_xchg_seg> segs;            // the planned segments
    ~ecsr_xchg() {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (size_t i = 0; i < peer.size(); ++i)
            if (opened[i] && peer[i]) cudaIpcCloseMemHandle(peer[i]);
        if (buf) cudaFree(buf);
        if (prev >= 0) cudaSetDevice(prev);
    }
};

extern "C" {

int ecsr_b200_xchg_create(int64_t y_bytes, int32_t rank, int32_t world, ecsr_xchg** out) {
    if (!out) return fail(ECSR_ERR_VALUE, "out is null");
    *out = nullptr;
    if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world || y_bytes < 0)
        return fail(ECSR_ERR_VALUE, "bad rank / world (world <= 16) / size");
    auto* x = new ecsr_xchg();
    cudaGetDevice(&x->device);
    x->rank = rank;
    x->world = world;
    x->y_bytes = y_bytes;
    x->flags_off = (y_bytes + kLine - 1) / kLine * kLine;
    x->bytes = x->flags_off + static_cast<int64_t>(2 * world + 2) * kLine;  // arrival, ready, step, done
    cudaError_t e = cudaMalloc(&x->buf, x->bytes);
    if (e == cudaSuccess) e = cudaMemset(x->buf, 0, x->bytes);
    if (e != cudaSuccess) {
        delete x;
        return fail(ECSR_ERR_CUDA, std::string("xchg buffer: ") + cudaGetErrorString(e));
    }
    x->peer.assign(world, nullptr);
    x->opened.assign(world, false);
    x->peer[rank] = x->buf;
    *out = x;
    return ECSR_OK;
}

int ecsr_b200_xchg_handle(const ecsr_xchg* x, void* handle64) {
    if (!x || !handle64) return fail(ECSR_ERR_VALUE, "null argument");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, x->buf);
    if (e != cudaSuccess) return fail(ECSR_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle64, &h, 64);
    return ECSR_OK;
}

int ecsr_b200_xchg_open(ecsr_xchg* x, const void* handles) {
    if (!x || (!handles && x->world > 1)) return fail(ECSR_ERR_VALUE, "null argument");
    for (int r = 0; r < x->world; ++r) {
        if (r == x->rank || x->peer[r]) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const uint8_t*>(handles) + 64 * r, 64);
        void* p = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess)
            return fail(ECSR_ERR_CUDA, "cudaIpcOpenMemHandle(rank " + std::to_string(r) + "): " + cudaGetErrorString(e));
        x->peer[r] = static_cast<uint8_t*>(p);
        x->opened[r] = true;
    }
    return ECSR_OK;
}

void* ecsr_b200_xchg_y(const ecsr_xchg* x) { return x ? x->buf : nullptr; }

int ecsr_b200_xchg_plan(ecsr_xchg* x, const ecsr_xchg_seg* segs, int32_t nsegs) {
    if (!x || (!segs && nsegs > 0) || nsegs < 0) return fail(ECSR_ERR_VALUE, "null argument");
    if (nsegs > kMaxSegs) return fail(ECSR_ERR_VALUE, "at most " + std::to_string(kMaxSegs) + " segments");
    for (int i = 0; i < nsegs; ++i)
        if (segs[i].src_off < 0 || segs[i].bytes < 0 || (segs[i].bytes & 3) || (segs[i].src_off & 3) ||
            (segs[i].dst_off & 3) || segs[i].dst_off < 0 || segs[i].dst_off + segs[i].bytes > x->y_bytes)
            return fail(ECSR_ERR_VALUE, "segment outside y_full or not 4-byte aligned");
    x->segs.assign(segs, segs + nsegs);
    return ECSR_OK;
}

int ecsr_b200_xchg_run(const ecsr_xchg* x, const void* src, void* stream) {
    if (!x || (!src && !x->segs.empty())) return fail(ECSR_ERR_VALUE, "null argument");
    for (int r = 0; r < x->world; ++r)
        if (!x->peer[r]) return fail(ECSR_ERR_VALUE, "peer buffers not opened (ecsr_b200_xchg_open)");
    XchgParams p{};
    p.src = static_cast<const uint8_t*>(src);
    for (size_t i = 0; i < x->segs.size(); ++i) p.segs[i] = x->segs[i];
    p.nsegs = static_cast<int32_t>(x->segs.size());
    p.rank = x->rank;
    p.world = x->world;
    p.parts = std::max(1, 32 / x->world);  // >= 32 CTAs push, each destination gets 32/world
    for (int r = 0; r < x->world; ++r) p.peer_base[r] = x->peer[r];
    p.flags_off = x->flags_off;
    p.step_word = reinterpret_cast<unsigned long long*>(x->buf + x->flags_off + static_cast<int64_t>(2 * x->world) * kLine);
    p.done_word = reinterpret_cast<unsigned int*>(x->buf + x->flags_off + static_cast<int64_t>(2 * x->world + 1) * kLine);
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != x->device) cudaSetDevice(x->device);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(x->world * p.parts);
    cfg.blockDim = dim3(256);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, ecsr_xchg_kernel, p);
    if (prev >= 0 && prev != x->device) cudaSetDevice(prev);
    if (e != cudaSuccess) return fail(ECSR_ERR_CUDA, std::string("xchg launch: ") + cudaGetErrorString(e));
    return ECSR_OK;
}

void ecsr_b200_xchg_free(ecsr_xchg* x) { delete x; }

}  // extern "C"
