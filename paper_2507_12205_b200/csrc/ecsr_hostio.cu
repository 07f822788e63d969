// ecsr_hostio.cu -- a step's host traffic as one small PDL-chained kernel (SURVEY.md §8(d),
// the end-to-end leg: x in from pinned host memory, the result out to pinned host memory).
//
// Why a kernel and not cudaMemcpyAsync on a copy stream: in a graph of steps, a launch
// that waits on a copy node (a cross-stream event) loses its programmatic (PDL) edge to
// the previous launch, so it can no longer be resident and ramp while its predecessor
// drains -- measured +5 us per step on the headline layer (scripts/e2e_probe.py), more
// than the copies themselves. This kernel moves the bytes with plain 16-B loads/stores
// through the UVA mapping of pinned host memory and sits in the launch chain:
//
//   ... SpMV(i-1) -> io(i): x(i) host->dev, y(i-2) dev->host -> SpMV(i) -> ...
//
// It triggers its dependents at once and (by default) calls griddepcontrol.wait only
// AFTER its copies: the copies overlap the predecessor, and the kernel completes right
// behind it, so the next SpMV's own griddepcontrol.wait still orders it after the
// previous SpMV. 128 threads and <= 32 registers per CTA: it co-resides with the SpMV's
// two 96-register CTAs per SM. ECSR_IO_AFTER_PREDECESSOR makes it wait first (the last
// step's y, read right after the launch that wrote it).
//
// The caller owns the hazards of the pipeline (bench.py's e2e leg, device.host_io):
// a span must not be written by the launch this kernel overlaps.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "../../include/ecsr_b200.h"

namespace ecsr_internal {
int set_error(int code, const std::string& msg);
}

namespace {

constexpr int kMaxSpans = ECSR_IO_MAX_SPANS;
constexpr int kThreads = 128;
constexpr int kUnroll = 2;

struct IoParams {
    const uint4* src[kMaxSpans];
    uint4* dst[kMaxSpans];
    long long end[kMaxSpans];  // inclusive prefix sum of the spans' 16-B chunks
    int tail[kMaxSpans];       // bytes past the span's last whole 16-B chunk (0..15)
    int n;
    int wait_first;
};

__device__ __forceinline__ uint4 ld_cg(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kThreads, 16) ecsr_host_io_kernel(const __grid_constant__ IoParams p) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (p.wait_first) asm volatile("griddepcontrol.wait;" ::: "memory");
    const long long total = p.end[p.n - 1];
    const long long stride = static_cast<long long>(gridDim.x) * kThreads;
    for (long long i = static_cast<long long>(blockIdx.x) * kThreads + threadIdx.x; i < total;
         i += kUnroll * stride) {
        uint4 v[kUnroll];
        uint4* d[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {  // every load in flight before the stores
            const long long j = i + u * stride;
            d[u] = nullptr;
            if (j < total) {
                int s = 0;
                while (j >= p.end[s]) ++s;
                const long long k = j - (s ? p.end[s - 1] : 0);
                v[u] = ld_cg(p.src[s] + k);
                d[u] = p.dst[s] + k;
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (d[u]) *d[u] = v[u];
    }
    if (blockIdx.x == 0 && threadIdx.x < p.n && p.tail[threadIdx.x]) {  // ragged ends, byte by byte
        const int s = threadIdx.x;
        const long long whole = p.end[s] - (s ? p.end[s - 1] : 0);
        const uint8_t* a = reinterpret_cast<const uint8_t*>(p.src[s] + whole);
        uint8_t* b = reinterpret_cast<uint8_t*>(p.dst[s] + whole);
        for (int k = 0; k < p.tail[s]; ++k) b[k] = a[k];
    }
    if (!p.wait_first) asm volatile("griddepcontrol.wait;" ::: "memory");
}

int fail(int code, const std::string& msg) { return ecsr_internal::set_error(code, msg); }

bool mapped(const void* ptr, int device) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (a.type == cudaMemoryTypeHost) return a.devicePointer == ptr;  // pinned, UVA-mapped
    if (a.type == cudaMemoryTypeDevice) return a.device == device;
    return a.type == cudaMemoryTypeManaged;
}

}  // namespace

extern "C" {

int ecsr_b200_host_io(const ecsr_io_span* spans, int32_t nspans, int32_t flags, void* stream) {
    if (nspans < 0 || nspans > kMaxSpans || (nspans && !spans))
        return fail(ECSR_ERR_VALUE, "spans: 0.." + std::to_string(kMaxSpans) + " entries");
    if (flags & ~ECSR_IO_AFTER_PREDECESSOR) return fail(ECSR_ERR_VALUE, "unknown flags");
    int device = 0;
    cudaGetDevice(&device);
    IoParams p{};
    long long chunks = 0;
    for (int i = 0; i < nspans; ++i) {
        const ecsr_io_span& s = spans[i];
        if (s.bytes < 0 || ((reinterpret_cast<uintptr_t>(s.src) | reinterpret_cast<uintptr_t>(s.dst)) & 15))
            return fail(ECSR_ERR_VALUE, "span " + std::to_string(i) + ": src and dst must be 16-B aligned");
        if (s.bytes && (!s.src || !s.dst)) return fail(ECSR_ERR_VALUE, "span " + std::to_string(i) + ": null pointer");
        if (s.bytes && (!mapped(s.src, device) || !mapped(s.dst, device)))
            return fail(ECSR_ERR_VALUE, "span " + std::to_string(i) +
                                            ": src and dst must be device memory of the current device or "
                                            "pinned (mapped) host memory");
        if (!s.bytes) continue;
        p.src[p.n] = static_cast<const uint4*>(s.src);
        p.dst[p.n] = static_cast<uint4*>(s.dst);
        chunks += s.bytes / 16;
        p.tail[p.n] = static_cast<int>(s.bytes & 15);
        p.end[p.n++] = chunks;
    }
    p.wait_first = (flags & ECSR_IO_AFTER_PREDECESSOR) ? 1 : 0;
    if (p.n == 0) {  // keep the chain's ordering (a dependent may rely on the wait)
        p.src[0] = nullptr;
        p.end[0] = 0;
        p.n = 1;
    }
    // about 2 KB per CTA keeps every load of a thread in flight at once (PCIe latency)
    const long long per_cta = static_cast<long long>(kThreads) * kUnroll;
    const int grid = static_cast<int>(std::max(1LL, std::min(1024LL, (chunks + per_cta - 1) / per_cta)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, ecsr_host_io_kernel, p);
    if (e != cudaSuccess) return fail(ECSR_ERR_CUDA, std::string("host io launch: ") + cudaGetErrorString(e));
    return ECSR_OK;
}

}  // extern "C"
