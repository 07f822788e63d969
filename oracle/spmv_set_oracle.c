/*
 * spmv_set_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference's canonical EC-CSR SpMV arithmetic,
 * `_spmv_set_impl` in pkg/src/ecsr/_speedups.pyx:81-129, built with
 * -ffp-contract=off exactly like pkg/setup.py:25-26 so every multiply and add
 * rounds separately. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg load it (oracle/liboracle.so).
 *
 * Pinned against the reference: tests/test_oracle.py checks it bit-for-bit
 * against the reference's compiled backend (this container) and against the
 * committed golden vectors in tests/golden/ (generated from the reference by
 * tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DEFINE_SPMV_SET(NAME, T)                                                            \
    int NAME(int g, int warp_size, int vector_size, int64_t num_blocks,                     \
             const uint32_t* row_ids, const int64_t* block_indptr,                          \
             const uint32_t* base_indices, const uint32_t* delta_indices,                   \
             const T* block_values, const T* x, T* y) {                                     \
        /* _speedups.pyx:97-100: lanes padded to a power of two */                          \
        int lanes_p2 = 1;                                                                   \
        while (lanes_p2 < warp_size) lanes_p2 *= 2;                                         \
        const int64_t chunk = (int64_t)warp_size * vector_size;                             \
        T* res = (T*)calloc((size_t)lanes_p2 * (size_t)g, sizeof(T));                       \
        if (!res) return 1;                                                                 \
        for (int64_t b = 0; b < num_blocks; ++b) {               /* :102 */                 \
            const int64_t start = block_indptr[b];                                          \
            const int64_t n = block_indptr[b + 1] - start;                                  \
            if (n == 0) continue;                                 /* :105-106 */            \
            const int64_t iters = n / chunk;                                                \
            memset(res, 0, (size_t)lanes_p2 * (size_t)g * sizeof(T));                       \
            for (int t = 0; t < warp_size; ++t) {                 /* :110 */                \
                int64_t idx = base_indices[b * warp_size + t];    /* :111 */                \
                for (int64_t i = 0; i < iters; ++i) {             /* :112 */                \
                    const int64_t off = start + i * chunk + (int64_t)t * vector_size;       \
                    for (int j = 0; j < vector_size; ++j) {       /* :113-116 */            \
                        idx += delta_indices[off + j];                                      \
                        const T xv = x[idx];                      /* :117 */                \
                        for (int k = 0; k < g; ++k)               /* :118-119 */            \
                            res[t * g + k] += block_values[(off + j) * g + k] * xv;         \
                    }                                                                       \
                }                                                                           \
            }                                                                               \
            for (int m = lanes_p2; m > 1; m /= 2) {               /* :120-127 */            \
                const int half = m / 2;                                                     \
                for (int t = 0; t < half; ++t)                                              \
                    for (int k = 0; k < g; ++k)                                             \
                        res[t * g + k] = res[t * g + k] + res[(t + half) * g + k];          \
            }                                                                               \
            for (int k = 0; k < g; ++k) y[row_ids[b * g + k]] += res[k]; /* :128-129 */     \
        }                                                                                   \
        free(res);                                                                          \
        return 0;                                                                           \
    }

DEFINE_SPMV_SET(oracle_spmv_set_f32, float)
DEFINE_SPMV_SET(oracle_spmv_set_f64, double)
