// ecsr_kernels.cuh -- sm_100a device code for the EC-CSR SpMV hot path.
//
// Two kernels compute y = A x over an EC-CSR container (pkg/src/ecsr/storage.py:50-96):
//
//  * ecsr_tiled_kernel -- the product. Persistent grid: two co-resident CTAs per SM
//    (9 consumer warps each) while x fits twice, else one (18 consumer warps). The
//    packer lays the container out as group records (P blocks of one set whose chunk
//    streams are interleaved: P*g row accumulators per warp) packed into tiles that
//    fill the CTA's stage pool; each CTA owns a contiguous, cost-balanced tile range.
//    A producer warp streams tiles HBM -> shared memory with cp.async.bulk (TMA bulk
//    copies, SASS UBLKCP) into an mbarrier-guarded stage pool; consumer warps take
//    records from a shared counter: per-lane delta decode (IDP.4A), x (fp16) gathered
//    from shared memory, FHFMA (f16 x f16 + f32), butterfly reduce-scatter over lanes,
//    then red.global.add.f32 into y (or one partial per block row for the ordered,
//    bitwise-reproducible mode).
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

// 18 consumer warps per SM: either 2 co-resident CTAs of 9 (consecutive launches
// overlap; x fits twice) or 1 CTA of 18 (large K: x would not leave room for stages).
// Measured 1 % faster than 16 on the grouped layer step; 20 is slower (register cap 80).
#ifndef ECSR_CONSUMER_WARPS_PER_SM
#define ECSR_CONSUMER_WARPS_PER_SM 18
#endif
constexpr int kConsumerWarpsPerSm = ECSR_CONSUMER_WARPS_PER_SM;
__host__ __device__ constexpr int tiled_threads(int nc) { return 32 * (nc + 1); }
constexpr int kMaxRingStages = 16;
#ifndef ECSR_TICKETS
#define ECSR_TICKETS 3
#endif
constexpr int kTickets = ECSR_TICKETS;  // tail-queue tickets a producer keeps in flight
// Back-off of the producer's stage-pool poll and of a consumer waiting for its record's
// tile to be issued (tuning builds may override them).
#ifndef ECSR_PRODUCER_POLL_NS
#define ECSR_PRODUCER_POLL_NS 20
#endif
#ifndef ECSR_CONSUMER_POLL_NS
#define ECSR_CONSUMER_POLL_NS 64
#endif
constexpr unsigned kProducerPollNs = ECSR_PRODUCER_POLL_NS, kConsumerPollNs = ECSR_CONSUMER_POLL_NS;
// Chunk-loop unroll of a group record (1: one chunk of every block per iteration).
#ifndef ECSR_CHUNK_UNROLL
#define ECSR_CHUNK_UNROLL 1
#endif
constexpr int kChunkUnroll = ECSR_CHUNK_UNROLL;
#ifndef ECSR_GATE_LANE
#define ECSR_GATE_LANE 0
#endif
constexpr int kGateLane = ECSR_GATE_LANE;  // producer lane that counts the CTA's zeroed slice
constexpr int kMaxMembers = 8;  // matrices of one grouped launch

// One matrix of a (grouped) launch: its packed arena and this launch's x and y.
struct TiledMember {
    const uint8_t* arena;          // tiles, 16-B aligned
    const uint2* tile_meta;        // [ntiles] {start16, nrec | bytes16 << 16}
    const __half* x;               // [K]
    float* y;                      // [M]
    float* partials;               // [nslots] (ordered mode)
    uint32_t* queue;               // [2] tail queue {next tile, CTAs done} (per-stream workspace)
    int64_t M;
    const uint2* queue_meta;       // [nqueue] the launch's tail queue (tile metadata, draw order)
    uint32_t nqueue;
    int32_t K;
    int32_t stage_bytes;
    int32_t nstages;
    int32_t x_vec16;               // x is 16-B aligned
    int32_t ctas;                  // CTAs of the launch working on this matrix
};

// Zero-y gate workspace (per stream): one 64-bit counter of zeroed slices, on its own
// 128-B line. A launch of `grid` CTAs adds exactly `grid` to it.
constexpr int kGateWords = 16;

struct TiledParams {
    TiledMember mem[kMaxMembers];
    const uint4* cta_work;         // [grid] {member, tile lo, tile hi, slice index in member}
    unsigned long long* gate;      // zero-y gate workspace (zero_y mode)
    int32_t nmem;
    int32_t ordered;
    int32_t wide;                  // K > 65535 (every member): u32 bases (else u16)
    int32_t zero_y;                // overwrite: the kernel zeroes y itself (no memset launch)
    int32_t pre_tiles;             // tiles streamed before griddepcontrol.wait / x
    unsigned long long* trace;     // tuning builds: per-CTA timeline [grid][16] or null
};

// What a record needs: its member's outputs (registers) and the launch-wide flags,
// read from the kernel parameters so they stay uniform (uniform branches).
struct RecCtx {
    float* y;
    float* partials;
    const TiledParams* tp;
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
// Returns 0 through an asm output: add it to addresses of data the wait guards.
__device__ __forceinline__ uint32_t mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t token;
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t"
        "mov.u32 %0, 0;\n\t}"
        : "=r"(token)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return token;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
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
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define ECSR_TRACE(slot, cond)                                                       \
    do {                                                                             \
        if (p.trace && (cond)) p.trace[blockIdx.x * 16 + (slot)] = gtimer();        \
    } while (0)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <int NC>
__device__ __forceinline__ void consumer_bar_sync() {
    asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
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

// Load `Bytes` (power of two) from shared memory (32-bit shared address) into regs.
// These asm statements have no memory operands the compiler can see, so nothing but
// data dependences orders them: every address into a stage or into x is derived from
// the token of the mbarrier wait that completes its fill (mbar_wait returns 0 through
// an asm output), so no load can be scheduled above that wait.
template <int Bytes>
__device__ __forceinline__ void lds_bytes(uint32_t addr, uint32_t* r) {
    if constexpr (Bytes >= 16) {
#pragma unroll
        for (int i = 0; i < Bytes / 16; ++i)
            asm("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(r[4 * i]), "=r"(r[4 * i + 1]), "=r"(r[4 * i + 2]), "=r"(r[4 * i + 3])
                         : "r"(addr + 16 * i));
    } else if constexpr (Bytes == 8) {
        asm("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
    } else if constexpr (Bytes == 4) {
        asm("ld.shared.u32 %0, [%1];" : "=r"(r[0]) : "r"(addr));
    } else if constexpr (Bytes == 2) {
        asm("ld.shared.u16 %0, [%1];" : "=r"(r[0]) : "r"(addr));
    } else {
        asm("ld.shared.u8 %0, [%1];" : "=r"(r[0]) : "r"(addr));
    }
}

__device__ __forceinline__ unsigned short lds_h(uint32_t addr) {
    unsigned short h;
    asm("ld.shared.b16 %0, [%1];" : "=h"(h) : "r"(addr));
    return h;
}

// Mixed-precision FMA (sm_100a FHFMA): acc + a*b with f16 a, b and f32 acc, rounded
// once. An f16 x f16 product is exact in f32, so this equals the reference's unfused
// `res += val * x` in f32 (_speedups.pyx:119 under -ffp-contract=off, pkg/setup.py:26).
__device__ __forceinline__ float fhfma(unsigned short a, unsigned short b, float acc) {
    asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(a), "h"(b));
    return acc;
}

template <int N>
__device__ __forceinline__ unsigned short half_at(const uint32_t (&r)[N], int i) {
    unsigned short lo, hi;
    asm("mov.b32 {%0,%1}, %2;" : "=h"(lo), "=h"(hi) : "r"(r[i >> 1]));
    return (i & 1) ? hi : lo;
}

// Tile (packer: ecsr_b200.cu, build_tiled_arena), 16-B aligned, homogeneous in (g, v):
//   u32 nblk | u8 g | u8 v | u16 0 | u16 block_off16[nblk] | pad to 16 | records
// Block record:
//   u32 slot0 | u16 nchunk | u8 g | u8 v | u32 rows[g] | pad to 16
//   | bases[32] (u16, or u32 when WIDE) | u8 deltas[n] | f16 values[g*n]
// deltas and values keep the reference's chunk permutation (storage.py:147-181):
// chunk c holds, per lane t, v deltas at c*32*v + t*v and v*g values at
// (c*32*v + t*v)*g, so every warp step reads one contiguous span.
template <int G>
__host__ __device__ constexpr int header_bytes() {
    return (8 + 4 * G + 15) & ~15;
}

// Zero-y gate (overwrite mode without a memset launch): every slice of y -- one per CTA
// of the launch: rows [M*i/ctas, M*(i+1)/ctas) of the CTA's member -- must be zeroed
// before any red.global.add into y. Each CTA's producer zeroes its slice after
// griddepcontrol.wait and adds 1 to the gate counter (release); the counter's old value
// gives the launch's target (the next multiple of the grid). The first consumer warp of
// a CTA to reach the gate polls the counter (acquire) and opens the gate for the others
// (a CTA-scope release/acquire flag; atomics, so racecheck sees synchronised accesses).
// Every CTA of the grid must be able to be resident at once: the launcher checks that
// against the SMs this context may use (green-context SM partitions, the MPS active
// thread percentage) and otherwise clears y with a memset and launches without the gate.
// Measured alternative (round 2): per-slice claims that let resident CTAs zero absent
// CTAs' slices cost an extra atomic round trip per CTA near launch start, where atomics
// queue behind the bulk tile copies (~1-5 us), i.e. 3-10 % of the step.
__device__ __forceinline__ uint32_t atom_load_cta(const uint32_t* a) {
    uint32_t v;
    asm volatile("atom.acquire.cta.shared.or.b32 %0, [%1], 0;" : "=r"(v) : "r"(smem_addr(a)) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long atom_load_cta64(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("atom.acquire.cta.shared.or.b64 %0, [%1], 0;" : "=l"(v) : "r"(smem_addr(a)) : "memory");
    return v;
}
__device__ __forceinline__ void atom_store_cta64(unsigned long long* a, unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.release.cta.shared.exch.b64 %0, [%1], %2;" : "=l"(old) : "r"(smem_addr(a)), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long shfl64(unsigned long long v, int src) {
    const uint32_t lo = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v), src);
    const uint32_t hi = __shfl_sync(0xffffffffu, static_cast<uint32_t>(v >> 32), src);
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}

// Zero the slice of y that CTA work item `w` owns, with `n` lanes starting at `l`.
__device__ __forceinline__ void zero_slice(const TiledParams& p, const uint4& w, int l, int n) {
    const TiledMember& m = p.mem[w.x];
    const int64_t r0 = m.M * w.w / m.ctas, r1 = m.M * (w.w + 1) / m.ctas;
    for (int64_t r = r0 + l; r < r1; r += n) m.y[r] = 0.0f;
}

// The closed-gate path: out of line, so the ~20 record variants that inline pass() stay
// small (instruction cache).
__device__ __noinline__ void ygate_wait(const TiledParams* p, unsigned long long* target_smem, uint32_t* state,
                                        int lane);

struct YGate {
    const TiledParams* p;
    unsigned long long* target_smem;  // counter target + 1, published by the producer
    uint32_t* state;                  // 0 closed, 1 a warp polls, 2 open
    bool open;
    __device__ __forceinline__ void pass(int lane) {
#ifdef ECSR_EXP_NO_GATE  // timing experiment only: y is NOT correct
        return;
#endif
        if (open) return;
        ygate_wait(p, target_smem, state, lane);
        open = true;
    }
};

__device__ __noinline__ void ygate_wait(const TiledParams* p, unsigned long long* target_smem, uint32_t* state,
                                        int lane) {
    {
        uint32_t st = 0;
        if (lane == 0) st = atomicCAS(state, 0u, 1u);
        st = __shfl_sync(0xffffffffu, st, 0);
        if (st == 0) {  // this warp polls the grid counter for the CTA
            unsigned long long tgt = 0;  // target + 1, once the producer published it
            if (lane == 0)
                do {
                    tgt = atom_load_cta64(target_smem);
                } while (tgt == 0);
            if (lane == 0) {
                --tgt;
                unsigned long long v;
                do {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p->gate) : "memory");
                } while (static_cast<long long>(v - tgt) < 0);
            }
            __syncwarp();
            if (lane == 0) {
                uint32_t old;
                asm volatile("atom.release.cta.shared.exch.b32 %0, [%1], 2;" : "=r"(old) : "r"(smem_addr(state)) : "memory");
                if (p->trace) p->trace[blockIdx.x * 16 + 14] = gtimer();  // tuning builds: gate open
            }
        } else if (lane == 0) {
            while (st != 2u) {
                __nanosleep(32);
                st = atom_load_cta(state);
            }
        }
        __syncwarp();
    }
}

// Group records (packer: ecsr_b200.cu, build_tiled_arena / write_group_record): P = 8/g
// consecutive blocks (P = 1 for g >= 8) whose chunk streams are interleaved, so a warp
// carries 8 row accumulators and P independent column walks.
#ifndef ECSR_ACC
#define ECSR_ACC 8
#endif
constexpr int kAccPerWarp = ECSR_ACC;  // row accumulators per warp in a group record
__host__ __device__ constexpr int group_blocks(int g) { return g >= kAccPerWarp ? 1 : kAccPerWarp / g; }
__host__ __device__ constexpr int group_header_bytes(int g, int P) { return 64 + ((4 * g * P + 15) & ~15); }

template <int V>
__device__ __forceinline__ void load_deltas(uint32_t addr, uint32_t (&d)[(V + 3) / 4]) {
    lds_bytes<V>(addr, d);
}

// One chunk of one block on one lane: V columns, G rows each. Lane t's running column
// index advances by its deltas exactly like _speedups.pyx:112-119; products go into
// the block's G accumulators in the reference order.
// x byte addresses of a lane's columns in one chunk: column j sits at
// xa + 2 * (d_0 + ... + d_j). One IDP.4A per column (dot product of the delta bytes
// with 2 * [1, .., 1, 0, ..]) replaces a byte extract + add, and the V addresses no
// longer form a dependency chain.
template <int V>
__device__ __forceinline__ void chunk_addrs(const uint32_t (&d)[(V + 3) / 4], uint32_t& xa,
                                            uint32_t (&a)[V]) {
    constexpr uint32_t kSel[4] = {0x02u, 0x0202u, 0x020202u, 0x02020202u};
#pragma unroll
    for (int w = 0; w < (V + 3) / 4; ++w) {
#pragma unroll
        for (int j = 0; j < 4 && 4 * w + j < V; ++j) a[4 * w + j] = __dp4a(d[w], kSel[j], xa);
        xa = a[(4 * w + 3 < V) ? 4 * w + 3 : V - 1];
    }
}

#ifdef ECSR_EXP_NOGATHER
__device__ uint32_t g_xs_dbg;
#endif
template <int G, int V, int NW>
__device__ __forceinline__ void chunk_fma(const uint32_t (&d)[(V + 3) / 4], const uint32_t (&w)[NW],
                                          uint32_t& xa, float* acc) {
#ifdef ECSR_EXP_NOGATHER
    const uint32_t xs_dbg = 0;  // shared window offset 0: the barrier area (benign reads)
#endif
    uint32_t a[V];
    chunk_addrs<V>(d, xa, a);
#pragma unroll
    for (int j = 0; j < V; ++j) {
#ifdef ECSR_EXP_NOGATHER
        const unsigned short xh = lds_h(xs_dbg + ((a[j] >> 31) << 1));  // broadcast
#else
        const unsigned short xh = lds_h(a[j]);
#endif
#pragma unroll
        for (int k = 0; k < G; ++k) acc[k] = fhfma(half_at(w, j * G + k), xh, acc[k]);
    }
}

// Emit one row sum: red.global.add.f32 into y (fast) or the block's partial slot
// (ordered; summed per row in container order by ecsr_finish_rows).
__device__ __forceinline__ void emit_row(uint32_t r, int g, int P, int blk, int k, float sum,
                                         const RecCtx& p) {
    if (p.tp->ordered) {
        uint32_t slot;
        lds_bytes<4>(r + 4 * blk, &slot);
        asm volatile("st.global.f32 [%0], %1;" ::"l"(p.partials + slot + k), "f"(sum) : "memory");
    } else {
        uint32_t row;
        lds_bytes<4>(r + 64 + 4 * (blk * g + k), &row);
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p.y + row), "f"(sum) : "memory");
    }
}

// One group record, g = G <= 8: P = 8/G blocks walked together. Per block, lane t
// accumulates its segment sequentially (reference order); the 8 accumulators then
// share one butterfly reduce-scatter whose per-accumulator association is the
// reference's lane tree (_speedups.pyx:120-127).
// `next` runs once per record, right before the lane reduction: the consumer loop claims
// its next record there, so the claim's round trip overlaps the shuffles.
template <int G, int V, int P, class Next>
__device__ __forceinline__ void tiled_group_record(uint32_t r, const uint32_t (&m)[2], uint32_t xs, int lane,
                                                   const RecCtx& p, YGate& gate, Next&& next) {
    constexpr int NACC = P * G;
    constexpr int kStride = 32 / NACC;
    const int a = lane / kStride;  // accumulator a after the reduce-scatter: block a / G, row a % G
    const int blk = a / G, k = a % G;
    // header, lane bases and the lane's output row (or partial slot) are independent
    // shared loads: issue them together so their latencies overlap
    const uint32_t q = r + group_header_bytes(G, P);
    uint32_t out_idx;
    lds_bytes<4>(p.tp->ordered ? r + 4 * blk : r + 64 + 4 * (blk * G + k), &out_idx);
    uint32_t xa[P];
    if (p.tp->wide) {
        uint32_t bb[P];
        lds_bytes<4 * P>(q + lane * 4 * P, bb);
#pragma unroll
        for (int b = 0; b < P; ++b) xa[b] = xs + 2u * bb[b];
    } else {
        uint32_t bb[(P + 1) / 2];
        lds_bytes<2 * P>(q + lane * 2 * P, bb);
#pragma unroll
        for (int b = 0; b < P; ++b) xa[b] = xs + 2u * ((bb[b >> 1] >> (16 * (b & 1))) & 0xffffu);
    }
    const uint32_t nmin = m[0] & 0xffffu, present = (m[1] >> 8) & 0xffu;
    if (!present) {  // zero-width blocks only (_speedups.pyx:105-106)
        next();
        return;
    }
    const bool has_tail = (m[1] >> 24) != 0;  // header byte 55
    constexpr uint32_t DCH = 32 * V, VCH = 64 * V * G, LV = 2 * V * G;  // bytes
    constexpr int NW = (LV + 3) / 4;
    uint32_t ptr = q + (p.tp->wide ? 128u : 64u) * P;
    float acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0f;
#pragma unroll kChunkUnroll
    for (uint32_t c = 0; c < nmin; ++c, ptr += P * (DCH + VCH)) {
        uint32_t d[P][(V + 3) / 4], w[P][NW];
#ifdef ECSR_EXP_NOWEIGHTLDS
#pragma unroll
        for (int b = 0; b < P; ++b) {
            for (int i = 0; i < (V + 3) / 4; ++i) d[b][i] = 0x01010101u + (c & 1);
            for (int i = 0; i < NW; ++i) w[b][i] = 0x3c003c00u ^ (c << 3);
        }
#else
#pragma unroll
        for (int b = 0; b < P; ++b) load_deltas<V>(ptr + b * DCH + lane * V, d[b]);
#pragma unroll
        for (int b = 0; b < P; ++b) lds_bytes<LV>(ptr + P * DCH + b * VCH + lane * LV, w[b]);
#endif
#pragma unroll
        for (int b = 0; b < P; ++b) chunk_fma<G, V, NW>(d[b], w[b], xa[b], acc + b * G);
    }
    if (has_tail) {  // blocks of a record are near-equal (sorted by nnz): usually none
        uint32_t tl[(P + 1) / 2];
        lds_bytes<2 * P>(r + 32, tl);  // ntail[P]
#pragma unroll
        for (int b = 0; b < P; ++b) {  // tails: chunks beyond nmin, block after block
            const uint32_t nt = (tl[b >> 1] >> (16 * (b & 1))) & 0xffffu;
#pragma unroll 1
            for (uint32_t c = 0; c < nt; ++c, ptr += DCH + VCH) {
                uint32_t d[(V + 3) / 4], w[NW];
                load_deltas<V>(ptr + lane * V, d);
                lds_bytes<LV>(ptr + DCH + lane * LV, w);
                chunk_fma<G, V, NW>(d, w, xa[b], acc + b * G);
            }
        }
    }
    next();
    const float sum = warp_reduce_scatter<NACC>(acc, lane);
    if (!p.tp->ordered) gate.pass(lane);
    if ((lane & (kStride - 1)) == 0 && ((present >> blk) & 1u)) {
        if (p.tp->ordered)
            asm volatile("st.global.f32 [%0], %1;" ::"l"(p.partials + out_idx + k), "f"(sum) : "memory");
        else
            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p.y + out_idx), "f"(sum) : "memory");
    }
}

// A single-block record of g = 8 * passes rows (g in {16, 32}): one walk per pass of
// 8 rows; a column's g values are contiguous, so a pass reads one 16-byte slice.
template <int V, class Next>
__device__ __forceinline__ void tiled_wide_record(uint32_t r, const uint32_t (&m)[2], int g, uint32_t xs, int lane,
                                                  const RecCtx& p, YGate& gate, Next&& next) {
    constexpr int G = 8;
    next();
    const uint32_t nch = m[0] & 0xffffu, present = (m[1] >> 8) & 0xffu;
    if (!present) return;
    const uint32_t q = r + group_header_bytes(g, 1);
    uint32_t base;
    if (p.tp->wide) lds_bytes<4>(q + lane * 4, &base);
    else {
        lds_bytes<2>(q + lane * 2, &base);
        base &= 0xffffu;
    }
    constexpr uint32_t DCH = 32 * V;
    const uint32_t vch = 64u * V * g;
    const uint32_t body = q + (p.tp->wide ? 128u : 64u);
    for (int pass = 0; pass < g / G; ++pass) {
        uint32_t xa = xs + 2u * base;
        float acc[G];
#pragma unroll
        for (int k = 0; k < G; ++k) acc[k] = 0.0f;
        uint32_t ptr = body;
#pragma unroll 1
        for (uint32_t c = 0; c < nch; ++c, ptr += DCH + vch) {
            uint32_t d[(V + 3) / 4], xaddr[V];
            load_deltas<V>(ptr + lane * V, d);
            chunk_addrs<V>(d, xa, xaddr);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const unsigned short xh = lds_h(xaddr[j]);
                uint32_t w[4];
                lds_bytes<16>(ptr + DCH + (lane * V + j) * 2u * g + 16u * pass, w);
#pragma unroll
                for (int k = 0; k < G; ++k) acc[k] = fhfma(half_at(w, k), xh, acc[k]);
            }
        }
        const float sum = warp_reduce_scatter<G>(acc, lane);
        if (!p.tp->ordered) gate.pass(lane);
        if ((lane & 3) == 0) emit_row(r, g, 1, 0, (lane >> 2) + G * pass, sum, p);
    }
}

// kFull: every (g, v, P) record variant; otherwise only the common ones (v = 4 with
// the default P, or half of it for g = 2, or down to a quarter for g = 1; v = 1 with g = 1) -- a smaller kernel body keeps the instruction
// cache warm; the packer picks the lean kernel when the container needs nothing else.
// Dispatch on the record's own (g, v, P) (header bytes 50, 51, 54): a tile may mix runs.
template <bool kFull, class Next>
__device__ __forceinline__ void tiled_record(uint32_t r, const uint32_t (&m)[2], uint32_t xs, int lane,
                                             const RecCtx& p, YGate& gate, Next&& next) {
    const uint32_t gv = ((m[0] >> 8) & 0xff00u) | (m[0] >> 24);  // g << 8 | v
    const uint32_t P = (m[1] >> 16) & 0xffu;
    const int g = static_cast<int>(gv >> 8);
    const bool v4 = (gv & 0xffu) == 4;
    if constexpr (!kFull) {
        if (!v4) {
            tiled_group_record<1, 1, group_blocks(1)>(r, m, xs, lane, p, gate, next);
            return;
        }
        switch (g) {
            case 1:
                if (P == group_blocks(1)) tiled_group_record<1, 4, group_blocks(1)>(r, m, xs, lane, p, gate, next);
                else if (P == group_blocks(1) / 2) tiled_group_record<1, 4, group_blocks(1) / 2>(r, m, xs, lane, p, gate, next);
                else tiled_group_record<1, 4, group_blocks(1) / 4>(r, m, xs, lane, p, gate, next);
                break;
            case 2:
                if (P == group_blocks(2)) tiled_group_record<2, 4, group_blocks(2)>(r, m, xs, lane, p, gate, next);
                else tiled_group_record<2, 4, group_blocks(2) / 2>(r, m, xs, lane, p, gate, next);
                break;
            case 4: tiled_group_record<4, 4, group_blocks(4)>(r, m, xs, lane, p, gate, next); break;
            default: tiled_group_record<8, 4, 1>(r, m, xs, lane, p, gate, next); break;
        }
        return;
    }
    if (!v4) {  // short 1-grained sets (v = 1, storage.py:99-122) and other narrow blocks
        if (g == 1) tiled_group_record<1, 1, group_blocks(1)>(r, m, xs, lane, p, gate, next);
        else if (g == 2) tiled_group_record<2, 1, group_blocks(2)>(r, m, xs, lane, p, gate, next);
        else if (g == 4) tiled_group_record<4, 1, group_blocks(4)>(r, m, xs, lane, p, gate, next);
        else if (g == 8) tiled_group_record<8, 1, 1>(r, m, xs, lane, p, gate, next);
        else tiled_wide_record<1>(r, m, g, xs, lane, p, gate, next);
        return;
    }
    switch ((g << 4) | P) {  // (g, blocks per record) of this run (packer: kRecordCap)
        case (1 << 4) | 8: tiled_group_record<1, 4, 8>(r, m, xs, lane, p, gate, next); break;
        case (1 << 4) | 4: tiled_group_record<1, 4, 4>(r, m, xs, lane, p, gate, next); break;
        case (1 << 4) | 2: tiled_group_record<1, 4, 2>(r, m, xs, lane, p, gate, next); break;
        case (1 << 4) | 1: tiled_group_record<1, 4, 1>(r, m, xs, lane, p, gate, next); break;
        case (2 << 4) | 4: tiled_group_record<2, 4, 4>(r, m, xs, lane, p, gate, next); break;
        case (2 << 4) | 2: tiled_group_record<2, 4, 2>(r, m, xs, lane, p, gate, next); break;
        case (2 << 4) | 1: tiled_group_record<2, 4, 1>(r, m, xs, lane, p, gate, next); break;
        case (4 << 4) | 2: tiled_group_record<4, 4, 2>(r, m, xs, lane, p, gate, next); break;
        case (4 << 4) | 1: tiled_group_record<4, 4, 1>(r, m, xs, lane, p, gate, next); break;
        case (8 << 4) | 1: tiled_group_record<8, 4, 1>(r, m, xs, lane, p, gate, next); break;
        default: tiled_wide_record<4>(r, m, g, xs, lane, p, gate, next); break;  // g = 16, 32
    }
}

// Persistent grid (1 or 2 CTAs per SM, kConsumerWarpsPerSm above), warp-specialised.
// A launch covers one matrix or a group of independent products (TiledMember each):
// CTA b works on member cta_work[b].x only -- its x, its static tile range, its tail
// queue -- so a group pays one launch ramp and one tail for all of its matrices.
//   * producer warp: streams this CTA's tiles HBM -> shared memory with cp.async.bulk
//     into the stage pool, L2 evict_first: first its static tile range (the first tiles
//     before griddepcontrol.wait -- the weights never depend on the previous kernel, so
//     they stream under the predecessor's tail), then tiles from its member's tail queue
//     until it is empty. The queue (the cheapest ~5 % of the work, most expensive
//     first) goes to whichever CTAs run ahead, so the CTAs finish together: the static
//     split alone leaves a +-12 % spread of per-CTA times (HBM and SM variation a cost
//     model cannot see), i.e. a ~3 us tail per launch;
//   * consumer warps: wait for the predecessor (x producer) and for x in shared
//     memory, then take records in issue order from a shared counter.
// Overwrite without a memset launch (zero_y): see YGate. A member's queue counter is
// reset by its last CTA once every CTA of the member has drawn its last (failing)
// ticket; the next launch on the stream draws only after its griddepcontrol.wait, i.e.
// after that reset.
template <bool kFull, int NC>
__global__ void __launch_bounds__(tiled_threads(NC), kConsumerWarpsPerSm / NC)
    ecsr_tiled_kernel(const __grid_constant__ TiledParams p) {
    constexpr int kProducerWarp = NC;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ unsigned long long gate_target;
    __shared__ uint32_t gate_state;                 // 0 closed, 1 a warp polls, 2 open
    __shared__ uint32_t rec_next;                   // record claim counter
    __shared__ uint32_t final_rec;                  // records of all issued tiles, once final
    __shared__ uint32_t stage_done[kMaxRingStages];  // finished records per stage
    // The stages form a pool, not an in-order ring: the producer refills whichever stage
    // was released (a long record then holds one stage, not the whole pool). At issue it
    // publishes, for the CTA's li-th tile, the records of tiles [0, li] and then (li,
    // stage, parity of this fill of the stage's full barrier); consumers find the tile
    // of their record there and wait on that parity. A ring of 32 > kMaxRingStages
    // entries: a tile's entry is reused only after 16 later tiles were fully consumed.
    // entry: low word (li << 6 | stage << 1 | parity), high word records of tiles [0, li];
    // one 64-bit store / load, so a consumer never sees half an entry
    __shared__ unsigned long long tile_stage[32];

    const uint4 work = p.cta_work[blockIdx.x];  // {member, [t0, t1) static tiles, slice}
    const TiledMember& me = p.mem[work.x];
    const uint32_t t0 = work.y, t1 = work.z;
    const int nstages = me.nstages, stage_bytes = me.stage_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* xbar = full + nstages;  // x staged (bulk copy or consumer copy)
    uint8_t* stages = smem + ((8 * nstages + 8 + 127) & ~127);
    __half* xs = reinterpret_cast<__half*>(stages + nstages * stage_bytes);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // x by one bulk copy when it is 16-B aligned and a multiple of 16 bytes
    const bool x_bulk = me.x_vec16 && (me.K & 7) == 0 && me.K > 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) {
            mbar_init(&full[s], 1);
            stage_done[s] = 0;
        }
        for (int i = 0; i < 32; ++i) tile_stage[i] = 0xffffffffull;
        mbar_init(xbar, 1);
        rec_next = 0;
        final_rec = 0xffffffffu;
        gate_target = 0;
        gate_state = 0;
        fence_mbar_init();
    }
    __syncthreads();
    ECSR_TRACE(0, threadIdx.x == 0);
    if (p.trace && threadIdx.x == 0) {
        uint32_t smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[blockIdx.x * 16 + 12] = smid;
    }

    if (warp == kProducerWarp) {
        // The whole warp runs the producer loop: lanes < nstages poll the stage pool in
        // parallel (ballot), lane 0 issues the copies. `pre_tiles` tiles go out before
        // x; the rest waits until x has landed, so the x request is not queued behind
        // this SM's whole weight stream.
        if (!p.zero_y) pdl_trigger();
        const uint64_t policy = l2_evict_first_policy();
        uint32_t fill_parity = 0;  // bit s: parity of the next fill of stage s
        uint32_t li = 0;           // tiles issued by this CTA (static, then queue tiles)
        uint32_t rec_end = 0;      // records of the issued tiles
        // lane s < nstages: records of the tile in stage s. A stage is free once the
        // consumers' done count (a shared red, no return value on their side) reaches it.
        uint32_t expect = 0;
        auto issue_tile = [&](uint32_t a16, uint32_t info) {  // info: nrec | bytes16 << 16
            uint32_t freeset;
            while (true) {
                uint32_t f = 0;
                if (lane < nstages) {
                    uint32_t done;
                    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(done) : "r"(smem_addr(&stage_done[lane])) : "memory");
                    f = done == expect;
                }
                freeset = __ballot_sync(0xffffffffu, f != 0);
                if (freeset) break;
                __nanosleep(kProducerPollNs);
            }
            const int stage = __ffs(freeset) - 1;
            const uint32_t nrec = info & 0xffffu;
            if (lane == stage) expect = nrec;
            rec_end += nrec;
            if (lane == 0) {
                stage_done[stage] = 0;
                // generic-proxy reads of the old tile are complete (their values were
                // consumed); order them before the async-proxy overwrite
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const uint32_t par = (fill_parity >> stage) & 1u;
                const uint32_t bytes = (info >> 16) * 16u;
                asm volatile("st.volatile.shared.v2.u32 [%0], {%1, %2};" ::"r"(smem_addr(&tile_stage[li & 31u])),
                             "r"((li << 6) | (static_cast<uint32_t>(stage) << 1) | par), "r"(rec_end)
                             : "memory");
                mbar_arrive_expect_tx(&full[stage], bytes);
                bulk_g2s(stages + stage * stage_bytes, me.arena + static_cast<size_t>(a16) * 16u, bytes,
                         &full[stage], policy);
            }
            fill_parity ^= 1u << stage;
            ++li;
            __syncwarp();
        };
        // static tiles: their metadata rides in the lanes, 32 tiles per coalesced load
        uint32_t t = t0, win_base = t0;
        uint2 win = t0 + lane < t1 ? me.tile_meta[t0 + lane] : make_uint2(0u, 0u);
        auto issue_static = [&]() {
            if (t - win_base >= 32u) {  // warp-uniform window slide
                win_base = t;
                win = t + lane < t1 ? me.tile_meta[t + lane] : make_uint2(0u, 0u);
            }
            const uint32_t a16 = __shfl_sync(0xffffffffu, win.x, t - win_base);
            const uint32_t info = __shfl_sync(0xffffffffu, win.y, t - win_base);
            issue_tile(a16, info);
            ++t;
        };
        for (int k = 0; k < p.pre_tiles && t < t1; ++k) issue_static();
        if (x_bulk || me.nqueue || p.zero_y) pdl_wait();
        if (x_bulk && lane == 0) {
            const uint32_t xbytes = static_cast<uint32_t>(me.K) * 2u;
            mbar_arrive_expect_tx(xbar, xbytes);
            bulk_g2s(xs, me.x, xbytes, xbar, l2_evict_last_policy());
        }
        if (p.zero_y) {
            // Zero-y gate (after the predecessor: y may alias its inputs): zero this CTA's
            // slice, count it (release), publish the target; PDL dependents are released
            // only after the arrival, so launches on one workspace never mix generations.
            zero_slice(p, work, lane, 32);
            __syncwarp();
            if (lane == kGateLane) {  // (ECSR_GATE_LANE: a lane that issued no bulk copies)
                unsigned long long old;
                asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(p.gate) : "memory");
                atom_store_cta64(&gate_target, old - old % gridDim.x + gridDim.x + 1);
                pdl_trigger();
            }
            __syncwarp();
        }
        mbar_wait(xbar, 0);
        while (t < t1) issue_static();
        if (me.nqueue) {
            // Tail queue: lanes 0..kTickets-1 each hold one drawn ticket and its tile's
            // metadata, so ticket and metadata latencies (~1 us each) overlap each other
            // and the wait for free stages; an exhausted lane stops drawing.
            uint32_t tk = 0xffffffffu;
            uint2 meta = make_uint2(0u, 0u);
            if (lane < kTickets) {
                tk = atomicAdd(me.queue, 1u);
                if (tk < me.nqueue) meta = me.queue_meta[tk];
            }
            int head = 0;
            while (true) {
                const uint32_t valid = __ballot_sync(0xffffffffu, tk < me.nqueue);
                if (!valid) break;
                // the next valid lane at or after head (round robin)
                const uint32_t rot = (valid >> head) | (valid << ((32 - head) & 31));
                const int src = (head + __ffs(rot) - 1) & 31;
                issue_tile(__shfl_sync(0xffffffffu, meta.x, src), __shfl_sync(0xffffffffu, meta.y, src));
                if (lane == src) {
                    tk = atomicAdd(me.queue, 1u);
                    if (tk < me.nqueue) meta = me.queue_meta[tk];
                }
                head = (src + 1) % kTickets;
            }
            // every ticket this CTA drew has landed (its value was used): check out; the
            // member's last CTA out resets its queue for the next launch on this workspace
            if (lane == 0) {
                const uint32_t out = atomicAdd(me.queue + 1, 1u);
                if (out == static_cast<uint32_t>(me.ctas) - 1u) {
                    me.queue[0] = 0u;
                    me.queue[1] = 0u;
                }
            }
        }
        if (lane == 0)  // after the last tile's entry: consumers past it may exit
            asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(smem_addr(&final_rec)), "r"(rec_end) : "memory");
        ECSR_TRACE(5, lane == 0);
        return;
    }

    // Consumers: wait for the predecessor (x producer; y may alias its inputs), then x.
    const int tid = threadIdx.x;
    constexpr int nthr = NC * 32;
    pdl_wait();
    ECSR_TRACE(1, threadIdx.x == 0);
    if (!x_bulk) {
        for (int i = tid; i < me.K; i += nthr) xs[i] = me.x[i];
        consumer_bar_sync<NC>();
        if (tid == 0) mbar_arrive(xbar);
    }
    const RecCtx rc{me.y, me.partials, &p};
    YGate gate{&p, &gate_target, &gate_state, !p.zero_y};
    const uint32_t xs_addr = smem_addr(xs) + mbar_wait(xbar, 0);  // x gathers after x landed
    ECSR_TRACE(2, threadIdx.x == 0);

    const uint32_t stages_addr = smem_addr(stages);
    // Warps claim records in issue order from a shared counter (balances unequal
    // records); the last record of a tile to finish releases its stage to the producer.
    uint32_t ti = 0;          // this warp's tile cursor (issue order)
    uint32_t tile_begin = 0;  // records of tiles [0, ti)
#ifdef ECSR_TRACE_CYCLES
    unsigned long long cyc_wait = 0, cyc_work = 0, nwork = 0, cyc_unissued = 0;
#endif
    // Each warp claims a record when it starts it. (ECSR_EXP_EARLY_CLAIM: claim the next
    // one before the current one's lane reduction instead; measured slower, 1-4 %.)
#ifdef ECSR_EXP_EARLY_CLAIM
    uint32_t k_next = 0;
    if (lane == 0) k_next = atomicAdd(&rec_next, 1u);
    auto claim_next = [&]() {
        if (lane == 0) k_next = atomicAdd(&rec_next, 1u);
    };
#else
    auto claim_next = []() {};
#endif
    while (true) {
#ifdef ECSR_EXP_EARLY_CLAIM
        const uint32_t k = __shfl_sync(0xffffffffu, k_next, 0);
#else
        uint32_t k = 0;
        if (lane == 0) k = atomicAdd(&rec_next, 1u);
        k = __shfl_sync(0xffffffffu, k, 0);
#endif
#ifdef ECSR_TRACE_CYCLES
        const unsigned long long c0 = clock64();
#endif
        uint32_t stage = 0, par = 0;
        bool have = false;
        while (true) {  // the tile holding record k: walk the issued tiles' entries
            uint32_t e, end;
            asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(e), "=r"(end)
                         : "r"(smem_addr(&tile_stage[ti & 31u])) : "memory");
            if ((e >> 6) == ti && e != 0xffffffffu) {
                if (k < end) {
                    stage = (e >> 1) & 31u;
                    par = e & 1u;
                    have = true;
                    break;
                }
                tile_begin = end;
                ++ti;
                continue;
            }
            uint32_t fin;  // not issued (yet): past the CTA's last record?
            asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(fin) : "r"(smem_addr(&final_rec)) : "memory");
            if (k >= fin) break;
            __nanosleep(kConsumerPollNs);
        }
        if (!have) break;
#ifdef ECSR_TRACE_CYCLES
        cyc_unissued += clock64() - c0;  // the tile was not issued yet (no free stage)
#endif
        const uint32_t tok = mbar_wait(&full[stage], par);
#ifdef ECSR_TRACE_CYCLES
        const unsigned long long c1 = clock64();
        cyc_wait += c1 - c0;
#endif
        ECSR_TRACE(3, threadIdx.x == 0 && ti == 0);
        const uint32_t tile = stages_addr + stage * stage_bytes + tok;  // reads after the fill
        uint32_t off16;
        lds_bytes<2>(tile + 8 + 2 * (k - tile_begin), &off16);
        const uint32_t r = tile + 16u * (off16 & 0xffffu);
        uint32_t m[2];
        lds_bytes<8>(r + 48, m);  // nmin | g | v ; nblk | present | P | has_tail
        tiled_record<kFull>(r, m, xs_addr, lane, rc, gate, claim_next);
#ifdef ECSR_TRACE_CYCLES
        cyc_work += clock64() - c1;
        ++nwork;
#endif
        __syncwarp();
        if (lane == 0)  // record done (its stage reads were consumed by the FMAs above):
                        // the producer refills the stage once all of its records are
            asm volatile("red.relaxed.cta.shared.add.u32 [%0], 1;" ::"r"(smem_addr(&stage_done[stage])) : "memory");
    }
    ECSR_TRACE(4, threadIdx.x == 0);
    if (p.trace && lane == 0) {
        atomicMax(p.trace + blockIdx.x * 16 + 6, gtimer());
        atomicMin(p.trace + blockIdx.x * 16 + 7, gtimer());
#ifdef ECSR_TRACE_CYCLES
        atomicAdd(p.trace + blockIdx.x * 16 + 8, cyc_wait);
        atomicAdd(p.trace + blockIdx.x * 16 + 9, cyc_work);
        atomicAdd(p.trace + blockIdx.x * 16 + 10, nwork);
        atomicAdd(p.trace + blockIdx.x * 16 + 13, cyc_unissued);
#endif
        atomicAdd(p.trace + blockIdx.x * 16 + 11, static_cast<unsigned long long>(t1 - t0));
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
