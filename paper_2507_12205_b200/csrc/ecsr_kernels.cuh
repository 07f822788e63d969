// ecsr_kernels.cuh -- sm_100a device code for the EC-CSR SpMV hot path.
//
// Two kernels compute y = A x over an EC-CSR container (pkg/src/ecsr/storage.py:50-96):
//
//  * ecsr_tiled_kernel -- the product. Persistent grid (one CTA per SM). The packer
//    lays every block out block-major in one arena, grouped into <= ~8 KB tiles of
//    whole blocks; each CTA owns a contiguous, byte-balanced tile range. One producer
//    thread streams tiles HBM -> shared memory with cp.async.bulk (TMA bulk copies,
//    SASS UBLKCP) into an mbarrier-guarded ring; NCONS consumer warps stage x (fp16)
//    in shared memory once, then each decodes whole blocks: per-lane delta decode in
//    registers, x gathered from shared memory, g FP32 FMAs per column, butterfly
//    reduce-scatter over lanes, then red.global.add.f32 into y (or one partial per
//    block row for the ordered, bitwise-reproducible mode).
//
//  * ecsr_generic_kernel -- the reference's arithmetic for ANY container
//    (W <= 32, any v, g, B in {4, 8, 16}; f16/f32/f64), one warp per block straight
//    from the reference arrays, unfused multiply/add like the reference's
//    -ffp-contract=off build (pkg/setup.py:25-26). Used by the per-set backend
//    protocol (ecsr_b200_spmv_set) and for containers the tiled layout cannot hold.
//
// Arithmetic parity with pkg/src/ecsr/_speedups.pyx:81-129:
//  - lane t walks its own segment: idx = base[t]; idx += delta; acc[k] += val * x[idx]
//    (:110-119). With fp16 values and x the product is exact in fp32, so fmaf equals
//    the reference's unfused a + v*x;
//  - lanes combine in the fixed binary tree res[t] += res[t + m/2] (:120-127). The
//    xor butterfly below produces bit-identical sums (IEEE addition is commutative),
//    and the reduce-scatter variant hands row k to lane k*(32/g);
//  - ordered mode sums each row's block partials in container order starting from
//    0 (executor.py:89, _speedups.pyx:128-129).
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

namespace ecsr {

constexpr int kNumConsumerWarps = 12;
constexpr int kThreadsTiled = 32 * (kNumConsumerWarps + 1);
constexpr int kProducerWarp = kNumConsumerWarps;

struct TiledParams {
    const uint8_t* arena;          // block-major tiles, 16-B aligned
    const uint32_t* tile_start16;  // [ntiles + 1] tile offsets in 16-B units
    const uint32_t* cta_tile;      // [grid + 1] first tile of each CTA
    const __half* x;               // [K]
    float* y;                      // [M]
    float* partials;               // [nslots] (ordered mode)
    int32_t K;
    int32_t ordered;
    int32_t stage_bytes;
    int32_t nstages;
    int32_t x_vec16;               // x is 16-B aligned
};

// ---------------------------------------------------------------------------------
// PTX wrappers: mbarrier, bulk async copy (TMA), programmatic dependent launch.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// 1-D bulk copy global -> shared, completion signalled on `bar` (complete_tx::bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void consumer_bar_sync() {
    asm volatile("bar.sync 1, %0;" ::"r"(kNumConsumerWarps * 32) : "memory");
}

// ---------------------------------------------------------------------------------
// Butterfly reduce-scatter of G per-lane accumulators over the 32 lanes.
// After it, lane k*(32/G) holds the full sum of accumulator k, bit-identical to the
// reference's tree res[t] += res[t + m/2] with m = 32 (_speedups.pyx:120-127).
// ---------------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ float warp_reduce_scatter(float (&acc)[G], int lane) {
#pragma unroll
    for (int lvl = 0; lvl < 5; ++lvl) {
        const int off = 16 >> lvl;
        const int n = G >> lvl;  // accumulators still held by each lane
        if (n >= 2) {
            const bool upper = (lane & off) != 0;
#pragma unroll
            for (int i = 0; i < n / 2; ++i) {
                const float send = upper ? acc[i] : acc[i + n / 2];
                const float keep = upper ? acc[i + n / 2] : acc[i];
                acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
        } else {
            acc[0] = acc[0] + __shfl_xor_sync(0xffffffffu, acc[0], off);
        }
    }
    return acc[0];
}

// Load `Bytes` (power of two, >= 2) from 16-B-aligned-enough shared memory into regs.
template <int Bytes>
__device__ __forceinline__ void lds_bytes(const uint8_t* p, uint32_t* r) {
    if constexpr (Bytes >= 16) {
#pragma unroll
        for (int i = 0; i < Bytes / 16; ++i) {
            const uint4 v = reinterpret_cast<const uint4*>(p)[i];
            r[4 * i + 0] = v.x;
            r[4 * i + 1] = v.y;
            r[4 * i + 2] = v.z;
            r[4 * i + 3] = v.w;
        }
    } else if constexpr (Bytes == 8) {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        r[0] = v.x;
        r[1] = v.y;
    } else if constexpr (Bytes == 4) {
        r[0] = *reinterpret_cast<const uint32_t*>(p);
    } else if constexpr (Bytes == 2) {
        r[0] = *reinterpret_cast<const uint16_t*>(p);
    } else {
        r[0] = *p;
    }
}

__device__ __forceinline__ float half_lo(uint32_t w) {
    return __half2float(__ushort_as_half(static_cast<unsigned short>(w & 0xffffu)));
}
__device__ __forceinline__ float half_hi(uint32_t w) {
    return __half2float(__ushort_as_half(static_cast<unsigned short>(w >> 16)));
}
template <int N>
__device__ __forceinline__ float half_at(const uint32_t (&r)[N], int i) {
    return (i & 1) ? half_hi(r[i >> 1]) : half_lo(r[i >> 1]);
}

// Block record (packer: ecsr_b200.cu, build_tiled_layout):
//   u32 slot0 | u16 nchunk | u8 g | u8 v | u32 rows[g] | pad to 16
//   | bases[32] (u16, or u32 when WIDE) | u8 deltas[n] | f16 values[g*n]
// deltas and values keep the reference's chunk permutation (storage.py:147-181):
// chunk c holds, per lane t, v deltas at c*32*v + t*v and v*g values at
// (c*32*v + t*v)*g, so every warp step reads one contiguous span.
template <int G>
__host__ __device__ constexpr int header_bytes() {
    return (8 + 4 * G + 15) & ~15;
}

template <int G, int V, bool WIDE>
__device__ __forceinline__ void tiled_block(const uint8_t* __restrict__ blk,
                                            const __half* __restrict__ xs, int lane,
                                            const TiledParams& p) {
    const uint32_t slot0 = *reinterpret_cast<const uint32_t*>(blk);
    const uint32_t nchunk = *reinterpret_cast<const uint16_t*>(blk + 4);
    const uint32_t* rows = reinterpret_cast<const uint32_t*>(blk + 8);
    const uint8_t* q = blk + header_bytes<G>();
    uint32_t idx = WIDE ? reinterpret_cast<const uint32_t*>(q)[lane]
                        : static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(q)[lane]);
    q += WIDE ? 128 : 64;
    const uint8_t* dl = q + lane * V;
    const uint8_t* vl = q + nchunk * (32 * V) + lane * (2 * V * G);
    const unsigned short* xsu = reinterpret_cast<const unsigned short*>(xs);

    float acc[G];
#pragma unroll
    for (int k = 0; k < G; ++k) acc[k] = 0.0f;

    constexpr int kValBytes = 2 * V * G;       // per lane per chunk
    constexpr bool kWhole = kValBytes <= 64;   // load a lane's chunk at once
#pragma unroll 2
    for (uint32_t c = 0; c < nchunk; ++c) {
        uint32_t d[(V + 3) / 4];
        lds_bytes<V>(dl + c * (32 * V), d);
        if constexpr (kWhole) {
            uint32_t w[(kValBytes + 3) / 4];
            lds_bytes<kValBytes>(vl + c * (32 * kValBytes), w);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                idx += (d[j >> 2] >> (8 * (j & 3))) & 0xffu;
                const float xv = __half2float(__ushort_as_half(xsu[idx]));
#pragma unroll
                for (int k = 0; k < G; ++k) acc[k] = fmaf(half_at(w, j * G + k), xv, acc[k]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < V; ++j) {
                idx += (d[j >> 2] >> (8 * (j & 3))) & 0xffu;
                const float xv = __half2float(__ushort_as_half(xsu[idx]));
                uint32_t w[G / 2];
                lds_bytes<2 * G>(vl + c * (32 * kValBytes) + j * 2 * G, w);
#pragma unroll
                for (int k = 0; k < G; ++k) acc[k] = fmaf(half_at(w, k), xv, acc[k]);
            }
        }
    }
    if (nchunk == 0) return;  // zero-width blocks contribute nothing (_speedups.pyx:105-106)
    const float sum = warp_reduce_scatter<G>(acc, lane);
    constexpr int kStride = 32 / G;
    if ((lane & (kStride - 1)) == 0) {
        const int k = lane / kStride;
        if (p.ordered) {
            p.partials[slot0 + k] = sum;
        } else {
            atomicAdd(p.y + rows[k], sum);  // RED.E.ADD.F32 (result unused)
        }
    }
}

template <bool WIDE>
__device__ __forceinline__ void tiled_dispatch(const uint8_t* blk, const __half* xs, int lane,
                                               const TiledParams& p) {
    const uint32_t g = blk[6], v = blk[7];
#define ECSR_CASE(GG, VV)                          \
    case (GG << 4) | VV:                           \
        tiled_block<GG, VV, WIDE>(blk, xs, lane, p); \
        break;
    switch ((g << 4) | v) {
        ECSR_CASE(1, 4)
        ECSR_CASE(2, 4)
        ECSR_CASE(4, 4)
        ECSR_CASE(8, 4)
        ECSR_CASE(16, 4)
        ECSR_CASE(1, 1)
        ECSR_CASE(2, 1)
        ECSR_CASE(4, 1)
        ECSR_CASE(8, 1)
        ECSR_CASE(16, 1)
        ECSR_CASE(1, 2)
        ECSR_CASE(2, 2)
        ECSR_CASE(4, 2)
        ECSR_CASE(8, 2)
        ECSR_CASE(16, 2)
        ECSR_CASE(1, 8)
        ECSR_CASE(2, 8)
        ECSR_CASE(4, 8)
        ECSR_CASE(8, 8)
        ECSR_CASE(16, 8)
        ECSR_CASE(32, 1)
        ECSR_CASE(32, 2)
        ECSR_CASE(32, 4)
        ECSR_CASE(32, 8)
        default:
            break;  // packer guarantees a supported (g, v)
    }
#undef ECSR_CASE
}

template <bool WIDE>
__global__ void __launch_bounds__(kThreadsTiled, 1) ecsr_tiled_kernel(const TiledParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + p.nstages;
    uint8_t* stages = smem + ((16 * p.nstages + 127) & ~127);
    __half* xs = reinterpret_cast<__half*>(stages + p.nstages * p.stage_bytes);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t t0 = p.cta_tile[blockIdx.x];
    const uint32_t t1 = p.cta_tile[blockIdx.x + 1];

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.nstages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNumConsumerWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_trigger();

    if (warp == kProducerWarp) {
        // Weights do not depend on the previous kernel: stream them before pdl_wait.
        if (lane == 0) {
            const uint64_t policy = l2_evict_first_policy();
            int stage = 0;
            uint32_t phase = 0;
            for (uint32_t t = t0; t < t1; ++t) {
                mbar_wait(&empty[stage], phase ^ 1u);
                const uint32_t a = p.tile_start16[t], b = p.tile_start16[t + 1];
                const uint32_t bytes = (b - a) * 16u;
                mbar_arrive_expect_tx(&full[stage], bytes);
                bulk_g2s(stages + stage * p.stage_bytes, p.arena + static_cast<size_t>(a) * 16u,
                         bytes, &full[stage], policy);
                if (++stage == p.nstages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
        return;
    }

    // Consumers: x (the previous kernel's output) -> shared memory, once per CTA.
    pdl_wait();
    {
        const int tid = threadIdx.x;
        const int nthr = kNumConsumerWarps * 32;
        if (p.x_vec16) {
            const int nvec = p.K >> 3;
            const uint4* src = reinterpret_cast<const uint4*>(p.x);
            uint4* dst = reinterpret_cast<uint4*>(xs);
            for (int i = tid; i < nvec; i += nthr) dst[i] = __ldg(src + i);
            for (int i = (nvec << 3) + tid; i < p.K; i += nthr) xs[i] = p.x[i];
        } else {
            for (int i = tid; i < p.K; i += nthr) xs[i] = p.x[i];
        }
    }
    consumer_bar_sync();

    int stage = 0;
    uint32_t phase = 0;
    uint32_t j = static_cast<uint32_t>(warp);  // round-robin block index across the CTA range
    for (uint32_t t = t0; t < t1; ++t) {
        mbar_wait(&full[stage], phase);
        const uint8_t* tile = stages + stage * p.stage_bytes;
        const uint32_t nblk = *reinterpret_cast<const uint32_t*>(tile);
        const uint16_t* offs = reinterpret_cast<const uint16_t*>(tile + 4);
        for (; j < nblk; j += kNumConsumerWarps) tiled_dispatch<WIDE>(tile + offs[j] * 16u, xs, lane, p);
        j -= nblk;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == p.nstages) {
            stage = 0;
            phase ^= 1u;
        }
    }
}

// Ordered finish: y[r] = (accumulate ? y[r] : 0) + sum of the row's block partials in
// container order (executor.py:89 then _speedups.pyx:128-129, block after block).
template <typename T>
__global__ void ecsr_finish_rows(const uint32_t* __restrict__ row_ptr,
                                 const uint32_t* __restrict__ row_slots,
                                 const T* __restrict__ partials, T* __restrict__ y, int64_t M,
                                 int accumulate) {
    pdl_wait();
    pdl_trigger();
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < M;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        T acc = accumulate ? y[r] : T(0);
        const uint32_t a = row_ptr[r], b = row_ptr[r + 1];
        for (uint32_t i = a; i < b; ++i) acc = acc + partials[row_slots[i]];
        y[r] = acc;
    }
}

// ---------------------------------------------------------------------------------
// Generic kernel: the reference arrays as-is, any W <= 32, v, g; one warp per block.
// ---------------------------------------------------------------------------------
struct GenericSet {
    const uint32_t* base_indices;  // [W * nb]
    const int64_t* block_indptr;   // [nb + 1] (set-local)
    const uint32_t* delta_indices; // set-local
    const void* block_values;      // set-local, value type VT
    int64_t num_blocks;
    int64_t slot0;                 // global slot of (block 0, row 0)
    int32_t g, warp, v, lanes_p2;
};

template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__device__ __forceinline__ T to_acc(__half v) { return static_cast<T>(__half2float(v)); }
template <typename T>
__device__ __forceinline__ T to_acc(float v) { return static_cast<T>(v); }
template <typename T>
__device__ __forceinline__ T to_acc(double v) { return static_cast<T>(v); }

template <typename T, typename VT, typename XT, int GM>
__global__ void __launch_bounds__(256) ecsr_generic_kernel(const GenericSet s,
                                                          const XT* __restrict__ x,
                                                          T* __restrict__ partials) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t warps_total = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const VT* vals = static_cast<const VT*>(s.block_values);
    for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
         b < s.num_blocks; b += warps_total) {
        const int64_t start = s.block_indptr[b];
        const int64_t n = s.block_indptr[b + 1] - start;
        if (n == 0) continue;
        const int64_t chunk = static_cast<int64_t>(s.warp) * s.v;
        const int64_t iters = n / chunk;
        for (int kc = 0; kc < s.g; kc += GM) {
            T acc[GM];
#pragma unroll
            for (int k = 0; k < GM; ++k) acc[k] = T(0);
            if (lane < s.warp) {
                int64_t idx = s.base_indices[b * s.warp + lane];
                for (int64_t i = 0; i < iters; ++i) {
                    const int64_t off = start + i * chunk + static_cast<int64_t>(lane) * s.v;
                    for (int j = 0; j < s.v; ++j) {
                        idx += s.delta_indices[off + j];
                        const T xv = to_acc<T>(x[idx]);
                        const VT* vp = vals + (off + j) * s.g + kc;
#pragma unroll
                        for (int k = 0; k < GM; ++k)
                            if (kc + k < s.g) acc[k] = add_rn<T>(acc[k], mul_rn<T>(to_acc<T>(vp[k]), xv));
                    }
                }
            }
            // tree over lanes padded to lanes_p2 (_speedups.pyx:120-127)
            for (int off = s.lanes_p2 >> 1; off >= 1; off >>= 1) {
#pragma unroll
                for (int k = 0; k < GM; ++k) acc[k] = add_rn<T>(acc[k], __shfl_xor_sync(0xffffffffu, acc[k], off));
            }
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < GM; ++k)
                    if (kc + k < s.g) partials[s.slot0 + b * s.g + kc + k] = acc[k];
            }
        }
    }
    pdl_trigger();
}

}  // namespace ecsr
