// ecsr_loader.cpp -- `.ecsr` blob -> device handle without the numpy round trip
// (SURVEY.md §8(f) #3).
//
// Parses the reference's wire format (pkg/src/ecsr/storage.py:389-483: magic "ECSR",
// header <BBBBHQQL, per set a <LLQQQ descriptor and u64-length-prefixed arrays; deltas
// packed 4-bit low nibble first / u8 / u16le; pad_mask packbits little-endian; values
// f32/f64 le) and rejects corruption with the reference's ContainerError messages
// (storage.py:431-483 and _check_set_shapes, storage.py:312-329): bad magic, version,
// value width / precision tag, delta width, warp, g/v, truncation (with the field and
// offset), array-shape mismatches, trailing bytes. The parsed host sets then go through
// ecsr_b200_pack (which validates the decode ranges once, executor.py:50-77).
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ecsr_b200.h"

namespace ecsr_internal {
int set_error(int code, const std::string& msg);  // ecsr_b200.cu: ecsr_b200_last_error
}

namespace {

using ecsr_internal::set_error;

struct Reader {
    const uint8_t* data;
    int64_t size;
    int64_t pos = 0;
    // storage.py:_Reader.take -- "truncated container: needed N bytes for WHAT at offset P"
    int take(int64_t n, const char* what, const uint8_t** out) {
        if (n < 0 || pos + n > size)
            return set_error(ECSR_ERR_CONTAINER, "truncated container: needed " + std::to_string(n) +
                                                     " bytes for " + what + " at offset " + std::to_string(pos));
        *out = data + pos;
        pos += n;
        return ECSR_OK;
    }
    template <typename T>
    int scalar(const char* what, T* v) {
        const uint8_t* p;
        if (int rc = take(sizeof(T), what, &p)) return rc;
        std::memcpy(v, p, sizeof(T));  // little-endian host (x86-64 / aarch64)
        return ECSR_OK;
    }
    // u64 count, then count * sizeof(T) bytes
    template <typename T>
    int array(const char* what, std::vector<T>* out) {
        uint64_t count;
        const std::string lw = std::string(what) + " length";
        if (int rc = scalar(lw.c_str(), &count)) return rc;
        if (count > static_cast<uint64_t>(size)) {  // cannot fit: report as truncation
            return set_error(ECSR_ERR_CONTAINER, "truncated container: needed " +
                                                     std::to_string(count * sizeof(T)) + " bytes for " + what +
                                                     " at offset " + std::to_string(pos));
        }
        const uint8_t* p;
        if (int rc = take(static_cast<int64_t>(count * sizeof(T)), what, &p)) return rc;
        out->resize(count);
        if (count) std::memcpy(out->data(), p, count * sizeof(T));
        return ECSR_OK;
    }
};

struct ParsedSet {
    uint32_t g = 0, v = 0;
    uint64_t nb = 0, stored = 0, real = 0;
    std::vector<uint32_t> rows;
    std::vector<int64_t> indptr;
    std::vector<uint32_t> bases, deltas;
    std::vector<uint8_t> mask;
    std::vector<float> vf;
    std::vector<double> vd;
};

struct Parsed {
    uint8_t version = 0, vsize = 0, vbits = 0, dbits = 0;
    uint16_t warp = 0;
    uint64_t rows = 0, cols = 0;
    uint32_t nsets = 0;
    std::vector<ParsedSet> sets;
};

int64_t delta_bytes(uint64_t count, int bits) {  // storage.py:_delta_bytes
    if (bits == 4) return static_cast<int64_t>((count + 1) / 2);
    return static_cast<int64_t>(count * (bits / 8));
}

// storage.py:_check_set_shapes
int check_shapes(const ParsedSet& s, uint16_t warp) {
    auto bad = [](const char* m) { return set_error(ECSR_ERR_CONTAINER, m); };
    if (s.indptr.size() != s.nb + 1) return bad("block_indptr length mismatch");
    if (s.indptr[0] != 0) return bad("block_indptr must start at 0 and be non-decreasing");
    for (size_t i = 1; i < s.indptr.size(); ++i)
        if (s.indptr[i] < s.indptr[i - 1]) return bad("block_indptr must start at 0 and be non-decreasing");
    if (static_cast<uint64_t>(s.indptr.back()) != s.stored) return bad("block_indptr does not cover stored columns");
    if (s.deltas.size() != s.stored || s.mask.size() != s.stored) return bad("delta or mask array length mismatch");
    const size_t nv = s.vf.empty() ? s.vd.size() : s.vf.size();
    if (nv != s.stored * s.g) return bad("block_values length mismatch");
    if (s.rows.size() != s.nb * s.g) return bad("row_indices length mismatch");
    if (s.bases.size() != s.nb * warp) return bad("base_indices length mismatch");
    const int64_t chunk = static_cast<int64_t>(warp) * s.v;
    for (size_t i = 1; i < s.indptr.size(); ++i)
        if ((s.indptr[i] - s.indptr[i - 1]) % chunk) return bad("block widths must be multiples of warp_size * vector_size");
    return ECSR_OK;
}

int parse(const uint8_t* data, int64_t len, Parsed* out) {
    if (!data && len) return set_error(ECSR_ERR_VALUE, "null blob");
    if (len < 0) return set_error(ECSR_ERR_VALUE, "negative blob length");
    Reader rd{data, len};
    const uint8_t* magic;
    if (int rc = rd.take(4, "magic", &magic)) return rc;
    if (std::memcmp(magic, "ECSR", 4) != 0) return set_error(ECSR_ERR_CONTAINER, "bad magic: not an ECSR container");
    Parsed& P = *out;
    // header <BBBBHQQL (storage.py:436-438): 26 bytes, unpacked as one field
    const uint8_t* h;
    if (int rc = rd.take(26, "header", &h)) return rc;
    P.version = h[0];
    P.vsize = h[1];
    P.vbits = h[2];
    P.dbits = h[3];
    std::memcpy(&P.warp, h + 4, 2);
    std::memcpy(&P.rows, h + 6, 8);
    std::memcpy(&P.cols, h + 14, 8);
    std::memcpy(&P.nsets, h + 22, 4);
    if (P.version != 1) return set_error(ECSR_ERR_CONTAINER, "unsupported container version " + std::to_string(P.version));
    if (P.vsize != 4 && P.vsize != 8)
        return set_error(ECSR_ERR_CONTAINER, "unsupported value width " + std::to_string(P.vsize));
    if (P.vbits != 16 && P.vbits != 32 && P.vbits != 64)
        return set_error(ECSR_ERR_CONTAINER, "unsupported value precision tag " + std::to_string(P.vbits));
    if (P.dbits != 4 && P.dbits != 8 && P.dbits != 16)
        return set_error(ECSR_ERR_CONTAINER, "unsupported delta precision " + std::to_string(P.dbits));
    if (P.warp < 1) return set_error(ECSR_ERR_CONTAINER, "warp size must be positive");
    P.sets.clear();
    for (uint32_t si = 0; si < P.nsets; ++si) {
        ParsedSet s;
        const uint8_t* d;
        if (int rc = rd.take(32, "set descriptor", &d)) return rc;  // <LLQQQ
        std::memcpy(&s.g, d, 4);
        std::memcpy(&s.v, d + 4, 4);
        std::memcpy(&s.nb, d + 8, 8);
        std::memcpy(&s.stored, d + 16, 8);
        std::memcpy(&s.real, d + 24, 8);
        if (s.g < 1 || s.v < 1) return set_error(ECSR_ERR_CONTAINER, "set granularity and vector size must be positive");
        if (int rc = rd.array("row_indices", &s.rows)) return rc;
        std::vector<uint64_t> ip;
        if (int rc = rd.array("block_indptr", &ip)) return rc;
        s.indptr.assign(ip.begin(), ip.end());
        if (int rc = rd.array("base_indices", &s.bases)) return rc;
        uint64_t dcount;
        if (int rc = rd.scalar("delta_indices length", &dcount)) return rc;
        if (dcount > static_cast<uint64_t>(len) * 2)
            return set_error(ECSR_ERR_CONTAINER, "truncated container: needed " +
                                                     std::to_string(delta_bytes(dcount, P.dbits)) +
                                                     " bytes for delta_indices at offset " + std::to_string(rd.pos));
        const uint8_t* dp;
        if (int rc = rd.take(delta_bytes(dcount, P.dbits), "delta_indices", &dp)) return rc;
        s.deltas.resize(dcount);
        for (uint64_t i = 0; i < dcount; ++i) {
            if (P.dbits == 4) s.deltas[i] = (dp[i / 2] >> (4 * (i & 1))) & 0xFu;
            else if (P.dbits == 8) s.deltas[i] = dp[i];
            else s.deltas[i] = static_cast<uint32_t>(dp[2 * i]) | (static_cast<uint32_t>(dp[2 * i + 1]) << 8);
        }
        uint64_t mcount;
        if (int rc = rd.scalar("pad_mask length", &mcount)) return rc;
        if (mcount > static_cast<uint64_t>(len) * 8)
            return set_error(ECSR_ERR_CONTAINER, "truncated container: needed " + std::to_string((mcount + 7) / 8) +
                                                     " bytes for pad_mask at offset " + std::to_string(rd.pos));
        const uint8_t* mp;
        if (int rc = rd.take(static_cast<int64_t>((mcount + 7) / 8), "pad_mask", &mp)) return rc;
        s.mask.resize(mcount);
        for (uint64_t i = 0; i < mcount; ++i) s.mask[i] = (mp[i / 8] >> (i % 8)) & 1u;
        if (P.vsize == 4) {
            if (int rc = rd.array("block_values", &s.vf)) return rc;
        } else {
            if (int rc = rd.array("block_values", &s.vd)) return rc;
        }
        if (int rc = check_shapes(s, P.warp)) return rc;
        P.sets.push_back(std::move(s));
    }
    if (rd.pos != len)
        return set_error(ECSR_ERR_CONTAINER, std::to_string(len - rd.pos) + " trailing bytes after container");
    return ECSR_OK;
}

}  // namespace

extern "C" {

int ecsr_b200_parse(const uint8_t* blob, int64_t len, ecsr_blob_info* info) {
    Parsed P;
    if (int rc = parse(blob, len, &P)) return rc;
    if (info) {
        info->num_rows = static_cast<int64_t>(P.rows);
        info->num_cols = static_cast<int64_t>(P.cols);
        info->nsets = static_cast<int32_t>(P.nsets);
        info->warp_size = P.warp;
        info->delta_bits = P.dbits;
        info->value_bits = P.vbits;
        info->value_bytes = P.vsize;
        int64_t stored = 0, blocks = 0, real = 0;
        for (const auto& s : P.sets) {
            stored += static_cast<int64_t>(s.stored);
            blocks += static_cast<int64_t>(s.nb);
            real += static_cast<int64_t>(s.real);
        }
        info->stored_cols = stored;
        info->num_blocks = blocks;
        info->real_nnz = real;
    }
    return ECSR_OK;
}

int ecsr_b200_load(const uint8_t* blob, int64_t len, int32_t device_dtype, int32_t flags, ecsr_dev** out) {
    if (!out) return set_error(ECSR_ERR_VALUE, "null output handle");
    Parsed P;
    if (int rc = parse(blob, len, &P)) return rc;
    std::vector<ecsr_host_set> hs(P.sets.size());
    for (size_t i = 0; i < P.sets.size(); ++i) {
        const ParsedSet& s = P.sets[i];
        ecsr_host_set& h = hs[i];
        h.granularity = static_cast<int32_t>(s.g);
        h.vector_size = static_cast<int32_t>(s.v);
        h.num_blocks = static_cast<int64_t>(s.nb);
        h.stored_cols = static_cast<int64_t>(s.stored);
        h.real_nnz = static_cast<int64_t>(s.real);
        h.row_indices = s.rows.data();
        h.block_indptr = s.indptr.data();
        h.base_indices = s.bases.data();
        h.delta_indices = s.deltas.data();
        h.pad_mask = s.mask.data();
        h.block_values = P.vsize == 4 ? static_cast<const void*>(s.vf.data()) : static_cast<const void*>(s.vd.data());
    }
    return ecsr_b200_pack(hs.data(), static_cast<int32_t>(hs.size()), static_cast<int64_t>(P.rows),
                          static_cast<int64_t>(P.cols), P.warp, P.dbits, P.vbits, P.vsize == 4 ? ECSR_F32 : ECSR_F64,
                          device_dtype, flags, out);
}

// A parsed blob held on the host: the sets as the reference arrays (deserialize).
struct ecsr_blob {
    Parsed P;
};

int ecsr_b200_blob_open(const uint8_t* blob, int64_t len, ecsr_blob** out) {
    if (!out) return set_error(ECSR_ERR_VALUE, "null output handle");
    *out = nullptr;
    auto* b = new ecsr_blob();
    if (int rc = parse(blob, len, &b->P)) {
        delete b;
        return rc;
    }
    *out = b;
    return ECSR_OK;
}

int ecsr_b200_blob_header(const ecsr_blob* b, ecsr_blob_info* info) {
    if (!b || !info) return set_error(ECSR_ERR_VALUE, "null argument");
    const Parsed& P = b->P;
    *info = ecsr_blob_info{};
    info->num_rows = static_cast<int64_t>(P.rows);
    info->num_cols = static_cast<int64_t>(P.cols);
    info->nsets = static_cast<int32_t>(P.nsets);
    info->warp_size = P.warp;
    info->delta_bits = P.dbits;
    info->value_bits = P.vbits;
    info->value_bytes = P.vsize;
    for (const auto& s : P.sets) {
        info->stored_cols += static_cast<int64_t>(s.stored);
        info->num_blocks += static_cast<int64_t>(s.nb);
        info->real_nnz += static_cast<int64_t>(s.real);
    }
    return ECSR_OK;
}

int ecsr_b200_blob_set_info(const ecsr_blob* b, int32_t set, ecsr_set_info* info) {
    if (!b || !info) return set_error(ECSR_ERR_VALUE, "null argument");
    if (set < 0 || set >= static_cast<int32_t>(b->P.sets.size())) return set_error(ECSR_ERR_VALUE, "set index");
    const ParsedSet& s = b->P.sets[set];
    info->granularity = static_cast<int32_t>(s.g);
    info->vector_size = static_cast<int32_t>(s.v);
    info->num_blocks = static_cast<int64_t>(s.nb);
    info->stored_cols = static_cast<int64_t>(s.stored);
    info->real_nnz = static_cast<int64_t>(s.real);
    return ECSR_OK;
}

int ecsr_b200_blob_copy_set(const ecsr_blob* b, int32_t set, ecsr_out_set* out) {
    if (!b || !out) return set_error(ECSR_ERR_VALUE, "null argument");
    if (set < 0 || set >= static_cast<int32_t>(b->P.sets.size())) return set_error(ECSR_ERR_VALUE, "set index");
    const ParsedSet& s = b->P.sets[set];
    auto put = [](void* dst, const void* src, size_t bytes) {
        if (bytes) std::memcpy(dst, src, bytes);
    };
    put(out->row_indices, s.rows.data(), 4 * s.rows.size());
    put(out->block_indptr, s.indptr.data(), 8 * s.indptr.size());
    put(out->base_indices, s.bases.data(), 4 * s.bases.size());
    put(out->delta_indices, s.deltas.data(), 4 * s.deltas.size());
    put(out->pad_mask, s.mask.data(), s.mask.size());
    if (b->P.vsize == 4) put(out->block_values, s.vf.data(), 4 * s.vf.size());
    else put(out->block_values, s.vd.data(), 8 * s.vd.size());
    return ECSR_OK;
}

void ecsr_b200_blob_free(ecsr_blob* b) { delete b; }

// storage.serialize (storage.py:389-428): header <BBBBHQQL, per set <LLQQQ and
// u64-length-prefixed arrays; deltas 4-bit (low nibble first) / u8 / u16le; pad_mask
// packbits little-endian; values f32/f64 le. out == NULL (or cap too small) sizes.
int ecsr_b200_serialize(const ecsr_host_set* sets, int32_t nsets, int64_t num_rows, int64_t num_cols,
                        int32_t warp_size, int32_t delta_bits, int32_t value_bits, int32_t value_dtype,
                        uint8_t* out, int64_t cap, int64_t* len) {
    if (!len || (nsets > 0 && !sets) || nsets < 0) return set_error(ECSR_ERR_VALUE, "null argument");
    if (value_dtype != ECSR_F32 && value_dtype != ECSR_F64) return set_error(ECSR_ERR_VALUE, "values must be f32 or f64");
    if (delta_bits != 4 && delta_bits != 8 && delta_bits != 16)
        return set_error(ECSR_ERR_VALUE, "delta_bits must be 4, 8 or 16");
    const int vsize = value_dtype == ECSR_F32 ? 4 : 8;
    std::vector<uint8_t> buf;
    auto raw = [&](const void* p, size_t n) {
        const uint8_t* b = static_cast<const uint8_t*>(p);
        buf.insert(buf.end(), b, b + n);
    };
    auto u64 = [&](uint64_t v) { raw(&v, 8); };
    raw("ECSR", 4);
    const uint8_t hb[4] = {1, static_cast<uint8_t>(vsize), static_cast<uint8_t>(value_bits),
                           static_cast<uint8_t>(delta_bits)};
    raw(hb, 4);
    const uint16_t w16 = static_cast<uint16_t>(warp_size);
    raw(&w16, 2);
    u64(static_cast<uint64_t>(num_rows));
    u64(static_cast<uint64_t>(num_cols));
    const uint32_t ns = static_cast<uint32_t>(nsets);
    raw(&ns, 4);
    const uint64_t limit = 1ull << delta_bits;
    for (int si = 0; si < nsets; ++si) {
        const ecsr_host_set& s = sets[si];
        const uint32_t gv[2] = {static_cast<uint32_t>(s.granularity), static_cast<uint32_t>(s.vector_size)};
        raw(gv, 8);
        u64(static_cast<uint64_t>(s.num_blocks));
        u64(static_cast<uint64_t>(s.stored_cols));
        u64(static_cast<uint64_t>(s.real_nnz));
        const int64_t nr = s.num_blocks * s.granularity, ni = s.num_blocks > 0 ? s.num_blocks + 1 : 1;
        u64(static_cast<uint64_t>(nr));
        raw(s.row_indices, 4 * nr);
        u64(static_cast<uint64_t>(ni));
        if (s.num_blocks > 0) raw(s.block_indptr, 8 * ni);
        else u64(0);
        u64(static_cast<uint64_t>(s.num_blocks * warp_size));
        raw(s.base_indices, 4 * s.num_blocks * warp_size);
        u64(static_cast<uint64_t>(s.stored_cols));
        for (int64_t i = 0; i < s.stored_cols; ++i)
            if (s.delta_indices[i] >= limit)
                return set_error(ECSR_ERR_CONTAINER, "delta exceeds " + std::to_string(delta_bits) + "-bit range");
        if (delta_bits == 4) {
            for (int64_t i = 0; i < s.stored_cols; i += 2) {
                const uint8_t lo = static_cast<uint8_t>(s.delta_indices[i]);
                const uint8_t hi = i + 1 < s.stored_cols ? static_cast<uint8_t>(s.delta_indices[i + 1]) : 0;
                buf.push_back(static_cast<uint8_t>(lo | (hi << 4)));
            }
        } else if (delta_bits == 8) {
            for (int64_t i = 0; i < s.stored_cols; ++i) buf.push_back(static_cast<uint8_t>(s.delta_indices[i]));
        } else {
            for (int64_t i = 0; i < s.stored_cols; ++i) {
                const uint16_t d = static_cast<uint16_t>(s.delta_indices[i]);
                raw(&d, 2);
            }
        }
        u64(static_cast<uint64_t>(s.stored_cols));
        for (int64_t i = 0; i < s.stored_cols; i += 8) {
            uint8_t byte = 0;
            for (int k = 0; k < 8 && i + k < s.stored_cols; ++k)
                if (s.pad_mask && s.pad_mask[i + k]) byte |= static_cast<uint8_t>(1u << k);
            buf.push_back(byte);
        }
        u64(static_cast<uint64_t>(s.stored_cols * s.granularity));
        raw(s.block_values, static_cast<size_t>(vsize) * s.stored_cols * s.granularity);
    }
    *len = static_cast<int64_t>(buf.size());
    if (out && cap >= *len) std::memcpy(out, buf.data(), buf.size());
    return ECSR_OK;
}

}  // extern "C"
