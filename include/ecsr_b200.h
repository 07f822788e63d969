/*
 * ecsr_b200.h -- C-ABI of libecsr_b200.so, the B200-native EC-CSR SpMV hot path.
 *
 * The reference's drop-in boundary for this path is the kernel-backend module
 * protocol of `pkg/src/ecsr/_kernels.py:17-71`: a module exposing NAME,
 * overlap_counts(...) and spmv_set(...), selected with use_backend(name).
 * Its compiled implementation is `pkg/src/ecsr/_speedups.pyx:55-129`.
 *
 *   ecsr_b200_spmv_set   replaces _speedups.spmv_set          (_speedups.pyx:55-78)
 *                        -- same arguments, host arrays, y accumulated in place,
 *                        precision chosen by y's dtype, canonical arithmetic order
 *                        (_speedups.pyx:81-129).
 *   ecsr_b200_pack       replaces the per-call validate_container + set loop of
 *                        executor.spmv_ec (executor.py:50-96): validates ONCE
 *                        and uploads a device-resident, TMA-tiled layout.
 *   ecsr_b200_spmv       replaces executor.spmv_ec(ec, x, validate=False)
 *                        (executor.py:80-96) on device buffers, stream-ordered.
 *   ecsr_b200_unpack     inverse of pack: reproduces the reference set arrays
 *                        (storage.py:50-62) from device memory, for the
 *                        bit-exact encoding check.
 *   ecsr_b200_bytes      byte model of storage_report (storage.py:579-649) plus
 *                        the device layout's actual bytes (roofline numerator).
 *
 * Return codes map onto ecsr.errors (errors.py:4-16) in the Python shim:
 *   0 OK, 1 ContainerError, 2 ValueError (shape/dtype/argument), 3 CUDA error.
 * Every failing call sets a thread-local message, read with ecsr_b200_last_error().
 * No entry point synchronises the device except ecsr_b200_spmv_set and
 * ecsr_b200_unpack (which return host data).
 */
#ifndef ECSR_B200_H
#define ECSR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ECSR_OK 0
#define ECSR_ERR_CONTAINER 1
#define ECSR_ERR_VALUE 2
#define ECSR_ERR_CUDA 3

/* element types (host values, device values, x and y) */
#define ECSR_F16 1
#define ECSR_F32 2
#define ECSR_F64 3

/* ecsr_b200_pack flags */
#define ECSR_PACK_DEFAULT 0
#define ECSR_PACK_FORCE_GENERIC 1 /* skip the tiled fast layout (parity/debug) */
/* tiled layout: tile (stage) size override in KB, 1..64 (tests: many tiles per CTA) */
#define ECSR_PACK_TILE_KB(kb) (((kb) & 0xff) << 8)
/* tiled layout: cost share (percent, 0..100) of each CTA's tiles handed out through the
 * launch's tail queue instead of its static range (default 5) */
#define ECSR_PACK_QUEUE_PCT(pct) (((((pct) & 0x7f) | 0x80)) << 16)

/* ecsr_b200_spmv modes */
#define ECSR_SPMV_OVERWRITE 0   /* y  = A x */
#define ECSR_SPMV_ACCUMULATE 1  /* y += A x */
#define ECSR_SPMV_ORDERED 2     /* OR-flag: per-block partials + ordered per-row sum;
                                   bitwise-reproducible, reference order
                                   (executor.py:89 + _speedups.pyx:128-129) */
#define ECSR_SPMV_MEMSET_Y 4    /* OR-flag: overwrite through a memset of y and a launch
                                   without the in-kernel zero-y gate (the path taken
                                   automatically when the whole grid cannot be resident:
                                   green-context SM partitions, MPS thread percentage) */

/* One block set, exactly the arrays of ecsr.storage.EcCsrSet (storage.py:50-62). */
typedef struct ecsr_host_set {
    int32_t granularity;           /* g rows per block */
    int32_t vector_size;           /* v columns per lane per warp step */
    int64_t num_blocks;
    int64_t stored_cols;           /* block_indptr[num_blocks] */
    int64_t real_nnz;
    const uint32_t* row_indices;   /* [g * num_blocks] */
    const int64_t* block_indptr;   /* [num_blocks + 1] */
    const uint32_t* base_indices;  /* [warp * num_blocks] */
    const uint32_t* delta_indices; /* [stored_cols], chunk-permuted */
    const uint8_t* pad_mask;       /* [stored_cols] bool bytes (cold: never read by kernels) */
    const void* block_values;      /* [g * stored_cols], chunk-permuted, value_dtype */
} ecsr_host_set;

/* Output of ecsr_b200_unpack: caller-allocated arrays sized from ecsr_b200_set_info. */
typedef struct ecsr_out_set {
    uint32_t* row_indices;
    int64_t* block_indptr;
    uint32_t* base_indices;
    uint32_t* delta_indices;
    uint8_t* pad_mask;
    void* block_values;            /* written in `out_value_dtype` */
} ecsr_out_set;

typedef struct ecsr_set_info {
    int32_t granularity;
    int32_t vector_size;
    int64_t num_blocks;
    int64_t stored_cols;
    int64_t real_nnz;
} ecsr_set_info;

typedef struct ecsr_bytes {
    /* storage_report(value_bits=16) components (storage.py:592-613) */
    int64_t row_indices, block_indptr, base_indices, delta_indices, pad_mask, block_values, desc;
    int64_t model_kernel_bytes; /* components - pad_mask - desc + 2K (x f16) + 4M (y f32) */
    int64_t device_arena_bytes; /* bytes the fast kernel streams from HBM per SpMV */
    int64_t device_total_bytes; /* every device allocation owned by the handle */
    int32_t layout;             /* 1 = tiled fast layout, 2 = generic */
    int32_t grid;               /* CTAs of the fast kernel */
    int32_t stages;             /* smem ring depth */
    int32_t stage_bytes;
    int64_t tiles;
    int64_t queue_tiles;        /* tiles drawn from the launch's tail queue */
} ecsr_bytes;

/* Opaque handle. The packed layout is read-only after pack; each launch also writes a
 * small workspace (zero-y grid-gate counter, ordered-mode block partials), one per
 * CUDA stream: a handle binds up to 4 streams on first use, so launches issued on (or
 * captured from) different streams may run concurrently, and launches on one stream
 * are stream-ordered. A 5th stream gets ECSR_ERR_VALUE. Launches run on the device the
 * handle was packed on, whatever the caller's current device. */
typedef struct ecsr_dev ecsr_dev;

/* Validate + pack + upload. device_dtype: ECSR_F16 (the product: fp16 values and x,
 * fp32 accumulate and y), ECSR_F32 or ECSR_F64 (generic kernel, container precision). */
int ecsr_b200_pack(const ecsr_host_set* sets, int32_t nsets, int64_t num_rows, int64_t num_cols,
                   int32_t warp_size, int32_t delta_bits, int32_t value_bits,
                   int32_t host_value_dtype, int32_t device_dtype, int32_t flags,
                   ecsr_dev** out);

/* y = A x (or y += A x). x: device [num_cols] of the handle's x type (f16 for an
 * ECSR_F16 handle), y: device [num_rows] (f32 for ECSR_F16/F32, f64 for F64).
 * Asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream). */
int ecsr_b200_spmv(const ecsr_dev* dev, const void* x, void* y, int32_t mode, void* stream);

/* Grouped launch: k <= 8 independent products y_i = A_i x_i in one launch of the tiled
 * kernel -- two when the members mix x sizes on both sides of 32 KB (one launch per
 * CTAs-per-SM class). Every member must use the tiled layout, on one device, all with
 * K <= 65535 or all above. The members' CTAs run side by side, so the group pays one
 * launch ramp and one tail instead of k (e.g. the projections of a decoder layer whose
 * inputs are all ready). The handles must outlive the group. xs / ys: host arrays of k
 * device pointers, read at call time (graph capture records them). Modes as
 * ecsr_b200_spmv; ORDERED runs the members one after another (bitwise reproducible).
 * Like a handle, a group keeps one launch workspace per stream (up to 4 streams).
 * ecsr_b200_group_info: launches per call, total CTAs, CTAs per member (ctas[k]). */
typedef struct ecsr_group ecsr_group;
int ecsr_b200_group_create(const ecsr_dev* const* mats, int32_t k, ecsr_group** out);
int ecsr_b200_group_spmv(const ecsr_group* group, const void* const* xs, void* const* ys,
                         int32_t mode, void* stream);
int ecsr_b200_group_info(const ecsr_group* group, int32_t* launches, int32_t* grid, int32_t* ctas,
                         int32_t k);
void ecsr_b200_group_free(ecsr_group* group);
/* Row-sharded y exchange over NVLink peer memory: every
 * rank owns a y_full buffer (all ranks' rows in their final layout) that its peers map
 * through CUDA IPC. ecsr_b200_xchg_run launches ONE kernel (PDL-chained behind the
 * rank's shard SpMV) that stores this rank's segments of its SpMV output into every
 * rank's y_full, signals each peer (system-scope release on a per-source flag) and
 * waits until every peer's push into this rank landed -- the NCCL all-gather + index
 * assembly of the sharded step in one launch. Setup: create (y_full bytes, rank,
 * world <= 16), export handle (64 B) -> all-gather the handles (host) -> open, plan the
 * segments once (<= 64; src/dst byte offsets, multiples of 4). ecsr_b200_xchg_y: the local
 * y_full. Steps are counted on the device, so the run can be graph-captured. */
typedef struct ecsr_xchg ecsr_xchg;
typedef struct ecsr_xchg_seg {
    int64_t src_off;  /* bytes into the SpMV output passed to ecsr_b200_xchg_run */
    int64_t dst_off;  /* bytes into every rank's y_full */
    int64_t bytes;
} ecsr_xchg_seg;
int ecsr_b200_xchg_create(int64_t y_full_bytes, int32_t rank, int32_t world, ecsr_xchg** out);
int ecsr_b200_xchg_handle(const ecsr_xchg* xchg, void* handle64);
int ecsr_b200_xchg_open(ecsr_xchg* xchg, const void* handles /* world x 64 B */);
int ecsr_b200_xchg_plan(ecsr_xchg* xchg, const ecsr_xchg_seg* segs, int32_t nsegs);
int ecsr_b200_xchg_run(const ecsr_xchg* xchg, const void* src, void* stream);
void* ecsr_b200_xchg_y(const ecsr_xchg* xchg);
void ecsr_b200_xchg_free(ecsr_xchg* xchg);
/* A step's host traffic as one PDL-chained kernel (end-to-end leg):
 * copies each span (src -> dst; device memory of the current device or pinned host
 * memory, which the GPU reaches through its UVA mapping; src and dst 16-B aligned, any
 * byte count) with plain loads/stores, in the stream's launch chain instead of on a copy
 * stream, so the next SpMV keeps its programmatic edge (csrc/ecsr_hostio.cu). Default:
 * the copies overlap the preceding launch and the kernel completes after it (the spans
 * must not be written by that launch); ECSR_IO_AFTER_PREDECESSOR: wait for it first
 * (read a result the preceding launch wrote). */
#define ECSR_IO_MAX_SPANS 16
#define ECSR_IO_AFTER_PREDECESSOR 1
typedef struct ecsr_io_span {
    const void* src;
    void* dst;
    int64_t bytes;
} ecsr_io_span;
int ecsr_b200_host_io(const ecsr_io_span* spans, int32_t nspans, int32_t flags, void* stream);
/* .ecsr wire format (storage.py:389-483) straight to a device handle, no numpy round trip
 * (SURVEY.md §8(f) #3). ecsr_b200_parse parses and shape-checks a blob on the host only,
 * rejecting corruption with the reference's ContainerError (code 1) and message: bad
 * magic, version, value width / precision tag, delta width, warp, g/v, truncation,
 * array-shape mismatch, trailing bytes (storage.py:431-483, 312-329). ecsr_b200_load
 * parses the same way and then packs like ecsr_b200_pack (values in the blob's f32/f64). */
typedef struct ecsr_blob_info {
    int64_t num_rows;
    int64_t num_cols;
    int32_t nsets;
    int32_t warp_size;
    int32_t delta_bits;
    int32_t value_bits;     /* precision tag of the header */
    int32_t value_bytes;    /* 4 (f32) or 8 (f64) on the wire */
    int64_t num_blocks;     /* over all sets */
    int64_t stored_cols;
    int64_t real_nnz;
} ecsr_blob_info;

int ecsr_b200_parse(const uint8_t* blob, int64_t len, ecsr_blob_info* info);
int ecsr_b200_load(const uint8_t* blob, int64_t len, int32_t device_dtype, int32_t flags,
                   ecsr_dev** out);

/* Host-side (de)serialization of the wire format, the reference's storage.serialize /
 * deserialize (storage.py:389-483): ecsr_b200_blob_open parses and shape-checks like
 * ecsr_b200_parse and keeps the sets on the host; _set_info sizes the caller's arrays and
 * _copy_set fills them (values in the blob's f32/f64). ecsr_b200_serialize writes a
 * container byte-identical to storage.serialize (call with out = NULL to size it). */
typedef struct ecsr_blob ecsr_blob;
int ecsr_b200_blob_open(const uint8_t* blob, int64_t len, ecsr_blob** out);
int ecsr_b200_blob_header(const ecsr_blob* blob, ecsr_blob_info* info);
int ecsr_b200_blob_set_info(const ecsr_blob* blob, int32_t set, ecsr_set_info* info);
int ecsr_b200_blob_copy_set(const ecsr_blob* blob, int32_t set, ecsr_out_set* out);
void ecsr_b200_blob_free(ecsr_blob* blob);
int ecsr_b200_serialize(const ecsr_host_set* sets, int32_t nsets, int64_t num_rows, int64_t num_cols,
                        int32_t warp_size, int32_t delta_bits, int32_t value_bits, int32_t value_dtype,
                        uint8_t* out, int64_t cap, int64_t* len);
int ecsr_b200_info(const ecsr_dev* dev, int64_t* num_rows, int64_t* num_cols, int32_t* nsets,
                   int32_t* warp_size, int32_t* delta_bits, int32_t* value_bits,
                   int32_t* device_dtype);
int ecsr_b200_set_info(const ecsr_dev* dev, int32_t set, ecsr_set_info* info);
int ecsr_b200_unpack(const ecsr_dev* dev, ecsr_out_set* out, int32_t nsets,
                     int32_t out_value_dtype);
int ecsr_b200_bytes(const ecsr_dev* dev, ecsr_bytes* out);
void ecsr_b200_free(ecsr_dev* dev);

/* Access trace of the device layout (the reference's
 * spmv_ec_traced + check_coalescing, executor.py:106-221): one entry per block, warp
 * step and array (0 = deltas, 1 = values) in the order the kernel reads them, mapped
 * back to the reference span it carries (`warp` = the block's index in container order,
 * `start`/`span` in elements of the set's delta_indices / block_values) and located in
 * device memory (`dev_offset`/`dev_bytes`: bytes into the tiled arena, or into the
 * generic layout's u32 delta / value arrays; `lane_bytes`: width of each lane's load).
 * Writes min(cap, count) entries; `count` gets the total (call with cap 0 to size). */
typedef struct ecsr_trace_rec {
    int64_t warp;
    int32_t step;
    int32_t array;
    int32_t set_index;
    int32_t lane_bytes;
    int64_t start;
    int64_t span;
    int64_t dev_offset;
    int64_t dev_bytes;
} ecsr_trace_rec;
int ecsr_b200_trace(const ecsr_dev* dev, ecsr_trace_rec* out, int64_t cap, int64_t* count);
/* The reference backend protocol entry (_speedups.pyx:55-78): host arrays, one set,
 * y (host, y_dtype ECSR_F32 or ECSR_F64) accumulated in place in the canonical
 * order. values/x are given in y's precision (the shim coerces like
 * np.ascontiguousarray(dtype=...) does). Synchronous. */
int ecsr_b200_spmv_set(int32_t g, int32_t warp_size, int32_t vector_size, int64_t num_blocks,
                       const uint32_t* row_ids, const int64_t* block_indptr,
                       const uint32_t* base_indices, const uint32_t* delta_indices,
                       const void* block_values, const void* x, int64_t x_len, void* y,
                       int64_t y_len, int32_t y_dtype);

/* ---- Native encoder (host, OpenMP): bit-exact with the reference's offline pipeline
 * storage.convert_csr (storage.py:700-708 -> extraction.py:153-356, balance.py:10-55,
 * storage.py:99-251). Replaces the reference's O(M^2 K)-per-round numpy encoder.
 * Input: CSR with strictly increasing columns per row (core.py:24-57); values f32/f64.
 * max_levels < 0 = None, clip_limit < 0 = None (automatic threshold), threads <= 0 =
 * OpenMP default. Output sets are read with ecsr_b200_enc_set_info / _copy_set (the
 * same arrays as ecsr.storage.EcCsrSet; ecsr_out_set buffers sized from the info). */
typedef struct ecsr_enc ecsr_enc;
int ecsr_b200_encode(int64_t num_rows, int64_t num_cols, const int64_t* row_ptr,
                     const int64_t* col_idx, const void* values, int32_t value_dtype,
                     int32_t warp_size, int32_t vector_size, int32_t delta_bits,
                     int32_t max_levels, int64_t clip_limit, int32_t threads, ecsr_enc** out);
int ecsr_b200_enc_nsets(const ecsr_enc* enc);
int ecsr_b200_enc_set_info(const ecsr_enc* enc, int32_t set, ecsr_set_info* info);
int ecsr_b200_enc_copy_set(const ecsr_enc* enc, int32_t set, ecsr_out_set* out,
                           int32_t out_value_dtype);
void ecsr_b200_enc_free(ecsr_enc* enc);
const char* ecsr_b200_enc_last_error(void);

/* IEEE round-to-nearest-even conversion used by pack (exposed for tests). */
int ecsr_b200_to_f16(const void* src, int32_t src_dtype, uint16_t* dst, int64_t n);

const char* ecsr_b200_last_error(void);
const char* ecsr_b200_version(void);
int ecsr_b200_device_count(void);

#ifdef __cplusplus
}
#endif

#endif /* ECSR_B200_H */
