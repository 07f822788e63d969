// ecsr_encoder.cpp -- native EC-CSR encoder (host C++, OpenMP), bit-exact with the
// reference pipeline `storage.convert_csr` (pkg/src/ecsr/storage.py:700-708):
//
//   extract_blocks      extraction.py:341-356   (level loop)
//     multi_round_extract extraction.py:251-261 (rounds until nothing is extracted)
//       row_matching      extraction.py:153-178 (greedy pairing, ties -> smallest row)
//       extract_round     extraction.py:218-248 (intersect, run selection, units)
//     encode_units        extraction.py:264-286
//     decode_residual     extraction.py:317-338 (+ _bridge_gaps 289-314)
//   clip_blocks         balance.py:20-44        (threshold balance.py:10-17)
//   reorder_sets        balance.py:47-55        (stable sorts)
//   split_one_grained   storage.py:99-122
//   encode_ec_csr       storage.py:207-251      (_stored_arrays 184-204, compress 125-144,
//                                                 chunk permutation 147-181)
//
// The reference computes the pairwise shared-column counts as a dense M x M matrix
// (O(M^2 K) per round: 11 min for 8192^2, hours for 28672 x 8192).
// Here the greedy matching computes, for the row being visited only, its exact
// overlap with every still-available row from per-row column bitsets (AND + popcount,
// OpenMP over candidates), and skips candidates whose nonzero count is below the
// W*V bar (they can never be chosen: the reference pairs only at overlap >= bar).
// The choices are therefore the reference's: rows visited in ascending order,
// argmax over available rows with ties to the smallest index.
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/ecsr_b200.h"

namespace ecsr_enc_impl {

struct Level {  // EncodedMatrix (extraction.py:100-134)
    int level = 0;
    int64_t rows = 0;
    std::vector<int64_t> row_ptr;
    std::vector<int32_t> col;
    std::vector<double> payload;  // nnz x g, row-major
    std::vector<int64_t> row_map;  // rows x g
    int g() const { return 1 << level; }
};

struct Block {  // extraction.Block: g rows sharing nnc increasing columns
    int g = 1;
    std::vector<int64_t> row_ids;
    std::vector<int32_t> cols;
    std::vector<double> vals;    // g x nnc, row-major (values[k, :] is row row_ids[k])
    std::vector<uint8_t> ins;    // gap-bridging zero columns
    int64_t nnc() const { return static_cast<int64_t>(cols.size()); }
    int64_t real_nnz() const {
        int64_t r = 0;
        for (uint8_t v : ins) r += v ? 0 : 1;
        return g * r;
    }
};

struct BlockSet {
    int g = 1;
    int v = 1;
    std::vector<Block> blocks;
};

struct Cfg {
    int warp = 32, vector = 4, delta_bits = 8;
    int max_levels = -1;
    int64_t clip_limit = -1;
    int64_t chunk() const { return static_cast<int64_t>(warp) * vector; }
    int64_t limit() const { return (int64_t{1} << delta_bits) - 1; }
};

// --- row_matching (extraction.py:153-178) -------------------------------------------
// Rounds of one level re-match every row, but a round only changes the rows it paired
// (their shared columns leave). MatchCache keeps, per level, the candidates' column
// bitsets and their pairwise overlaps (upper triangle, uint16: overlaps <= K < 65536);
// a round recomputes only the rows the previous one changed. Without room for the
// triangle (or K >= 65536) every overlap is computed on the fly, pruned by the nnz bound.
constexpr int64_t kMaxCacheBytes = int64_t{1} << 30;

struct MatchCache {
    bool built = false, tri_ok = false;
    int64_t words = 0;
    std::vector<int64_t> cand, cidx;  // candidate rows (nnz >= bar when built), inverse map
    std::vector<uint64_t> bits;       // cand x words
    std::vector<uint16_t> tri;        // overlap(c1 < c2) at tidx(c1, c2)
    std::vector<int64_t> dirty;       // rows changed since the cache was brought up to date
    int64_t tidx(int64_t a, int64_t b) const {  // a < b
        const int64_t n = static_cast<int64_t>(cand.size());
        return a * n - a * (a + 1) / 2 + (b - a - 1);
    }
};

int64_t popand(const uint64_t* a, const uint64_t* b, int64_t words) {
    int64_t cnt = 0;
    for (int64_t w = 0; w < words; ++w) cnt += __builtin_popcountll(a[w] & b[w]);
    return cnt;
}

void set_bits(const Level& L, int64_t r, uint64_t* b, int64_t words) {
    std::memset(b, 0, words * sizeof(uint64_t));
    for (int64_t p = L.row_ptr[r]; p < L.row_ptr[r + 1]; ++p) b[L.col[p] >> 6] |= uint64_t{1} << (L.col[p] & 63);
}

void refresh_cache(const Level& L, int64_t K, int64_t bar, MatchCache* mc) {
    const int64_t M = L.rows;
    if (!mc->built) {
        mc->words = (K + 63) / 64;
        mc->cand.clear();
        for (int64_t r = 0; r < M; ++r)
            if (L.row_ptr[r + 1] - L.row_ptr[r] >= bar) mc->cand.push_back(r);
        const int64_t nc = static_cast<int64_t>(mc->cand.size());
        mc->cidx.assign(M, -1);
        for (int64_t c = 0; c < nc; ++c) mc->cidx[mc->cand[c]] = c;
        mc->bits.assign(nc * mc->words, 0);
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < nc; ++c) set_bits(L, mc->cand[c], mc->bits.data() + c * mc->words, mc->words);
        mc->tri_ok = K < 65536 && nc * (nc - 1) / 2 * 2 <= kMaxCacheBytes;
        if (mc->tri_ok) {
            mc->tri.assign(nc * (nc - 1) / 2, 0);
#pragma omp parallel for schedule(dynamic, 16)
            for (int64_t a = 0; a < nc; ++a) {
                const uint64_t* ba = mc->bits.data() + a * mc->words;
                uint16_t* out = mc->tri.data() + mc->tidx(a, a + 1);
                for (int64_t b = a + 1; b < nc; ++b)
                    out[b - a - 1] = static_cast<uint16_t>(popand(ba, mc->bits.data() + b * mc->words, mc->words));
            }
        }
        mc->built = true;
        mc->dirty.clear();
        return;
    }
    // rows changed by the last round: new bitsets, then their overlaps with every candidate
    std::vector<int64_t> dc;
    for (int64_t r : mc->dirty)
        if (mc->cidx[r] >= 0) dc.push_back(mc->cidx[r]);
    std::sort(dc.begin(), dc.end());
    dc.erase(std::unique(dc.begin(), dc.end()), dc.end());
    mc->dirty.clear();
    const int64_t nd = static_cast<int64_t>(dc.size());
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nd; ++k) set_bits(L, mc->cand[dc[k]], mc->bits.data() + dc[k] * mc->words, mc->words);
    if (!mc->tri_ok || nd == 0) return;
    const int64_t nc = static_cast<int64_t>(mc->cand.size());
    std::vector<uint8_t> isd(nc, 0);
    for (int64_t c : dc) isd[c] = 1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k = 0; k < nd; ++k) {
        const int64_t d = dc[k];
        const uint64_t* bd = mc->bits.data() + d * mc->words;
        for (int64_t c = 0; c < nc; ++c) {
            if (c == d || (isd[c] && c < d)) continue;  // a pair of changed rows: the smaller writes
            const uint16_t v = static_cast<uint16_t>(popand(bd, mc->bits.data() + c * mc->words, mc->words));
            mc->tri[c < d ? mc->tidx(c, d) : mc->tidx(d, c)] = v;
        }
    }
}

std::vector<std::pair<int64_t, int64_t>> row_matching(const Level& L, int64_t K, const Cfg& cfg, MatchCache* mc) {
    const int64_t M = L.rows;
    const int64_t bar = cfg.chunk();
    refresh_cache(L, K, bar, mc);
    const int64_t words = mc->words;
    std::vector<int64_t> nnz(M);
    for (int64_t r = 0; r < M; ++r) nnz[r] = L.row_ptr[r + 1] - L.row_ptr[r];
    // only rows that can reach the bar are ever chosen as partners (nnz only shrinks
    // within a level, so the candidates of the cache's first round cover them)
    const std::vector<int64_t>& cand = mc->cand;
    const std::vector<int64_t>& cidx = mc->cidx;
    const int64_t nc = static_cast<int64_t>(cand.size());
    std::vector<uint8_t> avail(M, 0);
    for (int64_t r = 0; r < M; ++r) avail[r] = nnz[r] > 0;
    std::vector<uint8_t> cavail(nc, 1);
    std::vector<std::pair<int64_t, int64_t>> pairs;
    const int nth = omp_get_max_threads();
    std::vector<int64_t> tbest(nth, -1), tidx(nth, -1);
    // A candidate sharing ALL of row i's columns cannot be beaten, and ties go to the
    // smaller row: once one is found, no candidate above it can be chosen (planted blocks
    // make such rows common).
    std::atomic<int64_t> full_at{nc};
    // One parallel region for the whole greedy pass: every thread walks the rows in
    // order and scans its index range of row i's candidates; one thread then takes the
    // argmax and marks the partner (a row is visited once, and only candidates above it
    // are scanned, so nothing else needs updating).
#pragma omp parallel num_threads(nth)
    {
        const int t = omp_get_thread_num();
        const int nt = omp_get_num_threads();
        for (int64_t i = 0; i < M; ++i) {
            // empty rows are never visited; taken rows are skipped; a row below the bar
            // stays unmatched (its best overlap is below it)
            if (!avail[i] || nnz[i] < bar) continue;
            const int64_t ci = cidx[i];
            const uint64_t* bi = mc->bits.data() + ci * words;
            const uint16_t* trow = mc->tri_ok ? mc->tri.data() + mc->tidx(ci, ci + 1) - (ci + 1) : nullptr;
            const int64_t c0 = ci + 1;  // available candidates all lie above row i
            const int64_t per = (nc - c0 + nt - 1) / nt;  // thread t: the t-th index range
            const int64_t lo = c0 + t * per, hi = std::min(nc, lo + per);
            int64_t best = -1, bidx = -1;
            for (int64_t c = lo; c < hi; ++c) {
                if (c > full_at.load(std::memory_order_relaxed)) break;
                if (!cavail[c]) continue;
                const int64_t up = std::min(nnz[i], nnz[cand[c]]);
                if (up < bar || up <= best) continue;  // cannot win (ties keep the smaller row)
                const int64_t cnt = trow ? static_cast<int64_t>(trow[c]) : popand(bi, mc->bits.data() + c * words, words);
                if (cnt > best) {
                    best = cnt;
                    bidx = c;
                    if (cnt == nnz[i]) {
                        int64_t cur = full_at.load(std::memory_order_relaxed);
                        while (c < cur && !full_at.compare_exchange_weak(cur, c, std::memory_order_relaxed)) {
                        }
                        break;
                    }
                }
            }
            tbest[t] = best;
            tidx[t] = bidx;
#pragma omp barrier
#pragma omp single
            {
                int64_t b = -1, bx = -1;
                for (int k = 0; k < nt; ++k)  // thread k holds a lower index range than k + 1
                    if (tbest[k] > b) {
                        b = tbest[k];
                        bx = tidx[k];
                    }
                if (b >= bar) {
                    pairs.emplace_back(i, cand[bx]);
                    avail[cand[bx]] = 0;
                    cavail[bx] = 0;
                }
                full_at.store(nc, std::memory_order_relaxed);
            }  // implicit barrier: every thread sees the update before row i + 1
        }
    }
    return pairs;
}

// --- extract_round (extraction.py:181-248) ------------------------------------------
struct Unit {
    std::vector<int32_t> cols;
    std::vector<double> payload;  // n x 2g
    std::vector<int64_t> row_ids; // 2g
};

bool extract_round(Level& L, const std::vector<std::pair<int64_t, int64_t>>& pairs, const Cfg& cfg,
                   std::vector<Unit>* units, std::vector<int64_t>* changed) {
    const int g = L.g();
    const int64_t nnz = L.row_ptr[L.rows];
    std::vector<uint8_t> keep(nnz, 1);
    const int64_t np = static_cast<int64_t>(pairs.size());
    std::vector<Unit> made(np);
    std::vector<uint8_t> has(np, 0);
    // the pairs of a matching are disjoint rows: each one's intersection and its `keep`
    // marks are independent of the others'
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t q = 0; q < np; ++q) {
        const int64_t i = pairs[q].first, j = pairs[q].second;
        std::vector<int32_t> shared;
        std::vector<int64_t> pi, pj;
        int64_t a = L.row_ptr[i], ae = L.row_ptr[i + 1], b = L.row_ptr[j], be = L.row_ptr[j + 1];
        while (a < ae && b < be) {  // np.intersect1d(assume_unique, return_indices)
            if (L.col[a] < L.col[b]) ++a;
            else if (L.col[a] > L.col[b]) ++b;
            else {
                shared.push_back(L.col[a]);
                pi.push_back(a);
                pj.push_back(b);
                ++a;
                ++b;
            }
        }
        // _select_run_columns: maximal runs with gaps <= delta_limit, leading chunk multiple
        std::vector<int64_t> take;
        const int64_t n = static_cast<int64_t>(shared.size());
        int64_t s = 0;
        while (s < n) {
            int64_t e = s + 1;
            while (e < n && static_cast<int64_t>(shared[e]) - shared[e - 1] <= cfg.limit()) ++e;
            const int64_t usable = ((e - s) / cfg.chunk()) * cfg.chunk();
            for (int64_t k = s; k < s + usable; ++k) take.push_back(k);
            s = e;
        }
        if (take.empty()) continue;
        Unit& u = made[q];
        has[q] = 1;
        u.cols.reserve(take.size());
        u.payload.reserve(take.size() * 2 * g);
        for (int64_t k : take) {
            u.cols.push_back(shared[k]);
            const double* pa = L.payload.data() + pi[k] * g;
            const double* pb = L.payload.data() + pj[k] * g;
            u.payload.insert(u.payload.end(), pa, pa + g);
            u.payload.insert(u.payload.end(), pb, pb + g);
            keep[pi[k]] = 0;
            keep[pj[k]] = 0;
        }
        u.row_ids.insert(u.row_ids.end(), L.row_map.begin() + i * g, L.row_map.begin() + (i + 1) * g);
        u.row_ids.insert(u.row_ids.end(), L.row_map.begin() + j * g, L.row_map.begin() + (j + 1) * g);
    }
    size_t before = units->size();
    for (int64_t q = 0; q < np; ++q) {  // units in the matching's order
        if (!has[q]) continue;
        if (changed) {
            changed->push_back(pairs[q].first);
            changed->push_back(pairs[q].second);
        }
        units->push_back(std::move(made[q]));
    }
    if (units->size() == before) return false;
    // _filter_entries (extraction.py:202-215)
    Level R;
    R.level = L.level;
    R.rows = L.rows;
    R.row_map = std::move(L.row_map);
    R.row_ptr.assign(L.rows + 1, 0);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < L.rows; ++r) {
        int64_t c = 0;
        for (int64_t p = L.row_ptr[r]; p < L.row_ptr[r + 1]; ++p) c += keep[p];
        R.row_ptr[r + 1] = c;
    }
    for (int64_t r = 0; r < L.rows; ++r) R.row_ptr[r + 1] += R.row_ptr[r];
    R.col.resize(R.row_ptr[L.rows]);
    R.payload.resize(R.row_ptr[L.rows] * g);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < L.rows; ++r) {
        int64_t o = R.row_ptr[r];
        for (int64_t p = L.row_ptr[r]; p < L.row_ptr[r + 1]; ++p)
            if (keep[p]) {
                R.col[o] = L.col[p];
                std::memcpy(R.payload.data() + o * g, L.payload.data() + p * g, g * sizeof(double));
                ++o;
            }
    }
    L = std::move(R);
    return true;
}

// --- decode_residual + _bridge_gaps (extraction.py:289-338) --------------------------
BlockSet decode_residual(const Level& L, const Cfg& cfg) {
    BlockSet bs;
    bs.g = L.g();
    bs.v = cfg.vector;
    const int g = L.g();
    const int64_t limit = cfg.limit();
    for (int64_t r = 0; r < L.rows; ++r) {
        const int64_t a = L.row_ptr[r], e = L.row_ptr[r + 1];
        if (a == e) continue;
        Block b;
        b.g = g;
        b.row_ids.assign(L.row_map.begin() + r * g, L.row_map.begin() + (r + 1) * g);
        std::vector<int32_t> cols;
        std::vector<int64_t> src;  // payload entry or -1 for an inserted zero column
        for (int64_t p = a; p < e; ++p) {
            if (p > a) {
                const int64_t gap = static_cast<int64_t>(L.col[p]) - L.col[p - 1];
                if (gap > limit) {
                    const int64_t fill = (gap - 1) / limit;
                    for (int64_t m = 1; m <= fill; ++m) {
                        cols.push_back(static_cast<int32_t>(L.col[p - 1] + limit * m));
                        src.push_back(-1);
                    }
                }
            }
            cols.push_back(L.col[p]);
            src.push_back(p);
        }
        const int64_t n = static_cast<int64_t>(cols.size());
        b.cols = std::move(cols);
        b.vals.assign(g * n, 0.0);
        b.ins.assign(n, 0);
        for (int64_t c = 0; c < n; ++c) {
            if (src[c] < 0) {
                b.ins[c] = 1;
                continue;
            }
            for (int k = 0; k < g; ++k) b.vals[k * n + c] = L.payload[src[c] * g + k];
        }
        bs.blocks.push_back(std::move(b));
    }
    return bs;
}

// --- encode_units (extraction.py:264-286) -------------------------------------------
Level encode_units(const std::vector<Unit>& units, const Level& prior) {
    Level N;
    N.level = prior.level + 1;
    N.rows = static_cast<int64_t>(units.size());
    N.row_ptr.assign(N.rows + 1, 0);
    for (int64_t u = 0; u < N.rows; ++u) N.row_ptr[u + 1] = N.row_ptr[u] + static_cast<int64_t>(units[u].cols.size());
    N.col.reserve(N.row_ptr[N.rows]);
    N.payload.reserve(N.row_ptr[N.rows] * N.g());
    N.row_map.reserve(N.rows * N.g());
    for (const Unit& u : units) {
        N.col.insert(N.col.end(), u.cols.begin(), u.cols.end());
        N.payload.insert(N.payload.end(), u.payload.begin(), u.payload.end());
        N.row_map.insert(N.row_map.end(), u.row_ids.begin(), u.row_ids.end());
    }
    return N;
}

// --- extract_blocks (extraction.py:341-356) -----------------------------------------
std::vector<BlockSet> extract_blocks(Level enc, int64_t K, const Cfg& cfg) {
    std::vector<BlockSet> sets;
    while (true) {
        if (cfg.max_levels >= 0 && enc.level >= cfg.max_levels) {
            sets.push_back(decode_residual(enc, cfg));
            break;
        }
        std::vector<Unit> units;
        MatchCache cache;  // this level's rows
        while (true) {  // multi_round_extract
            auto pairs = row_matching(enc, K, cfg, &cache);
            if (!extract_round(enc, pairs, cfg, &units, &cache.dirty)) break;
        }
        sets.push_back(decode_residual(enc, cfg));
        if (units.empty()) break;
        enc = encode_units(units, enc);
    }
    std::vector<BlockSet> out;
    for (auto& s : sets)
        if (!s.blocks.empty()) out.push_back(std::move(s));
    return out;
}

// --- balance (balance.py:10-55) -----------------------------------------------------
BlockSet clip_blocks(BlockSet bs, const Cfg& cfg) {
    const int64_t chunk = cfg.chunk();
    int64_t limit;
    if (cfg.clip_limit < 0) {
        if (bs.blocks.empty()) {
            limit = chunk;
        } else {
            double sum = 0;
            for (auto& b : bs.blocks) sum += static_cast<double>(b.nnc());
            const double mean = sum / static_cast<double>(bs.blocks.size());
            limit = std::max<int64_t>(chunk, static_cast<int64_t>(std::ceil(2.0 * mean / chunk)) * chunk);
        }
    } else {
        limit = std::max<int64_t>(
            chunk, static_cast<int64_t>(std::ceil(static_cast<double>(cfg.clip_limit) / chunk)) * chunk);
    }
    BlockSet out;
    out.g = bs.g;
    out.v = bs.v;
    for (auto& b : bs.blocks) {
        const int64_t n = b.nnc();
        if (n <= limit) {
            out.blocks.push_back(std::move(b));
            continue;
        }
        for (int64_t s = 0; s < n; s += limit) {
            const int64_t e = std::min(s + limit, n), m = e - s;
            Block c;
            c.g = b.g;
            c.row_ids = b.row_ids;
            c.cols.assign(b.cols.begin() + s, b.cols.begin() + e);
            c.ins.assign(b.ins.begin() + s, b.ins.begin() + e);
            c.vals.resize(b.g * m);
            for (int k = 0; k < b.g; ++k)
                std::copy(b.vals.begin() + k * n + s, b.vals.begin() + k * n + e, c.vals.begin() + k * m);
            out.blocks.push_back(std::move(c));
        }
    }
    return out;
}

void reorder_sets(std::vector<BlockSet>* sets) {
    for (auto& s : *sets) {
        std::vector<int64_t> key(s.blocks.size());
        for (size_t i = 0; i < s.blocks.size(); ++i) key[i] = s.blocks[i].real_nnz();
        std::vector<size_t> idx(s.blocks.size());
        std::iota(idx.begin(), idx.end(), 0);
        std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return key[a] > key[b]; });
        std::vector<Block> sorted;
        sorted.reserve(idx.size());
        for (size_t i : idx) sorted.push_back(std::move(s.blocks[i]));
        s.blocks = std::move(sorted);
    }
    std::stable_sort(sets->begin(), sets->end(), [](const BlockSet& a, const BlockSet& b) { return a.g > b.g; });
}

// split_one_grained (storage.py:99-122)
void split_one_grained(BlockSet& bs, const Cfg& cfg, BlockSet* lng, BlockSet* shrt) {
    const int64_t chunk = cfg.chunk();
    lng->g = shrt->g = 1;
    lng->v = cfg.vector;
    shrt->v = 1;
    for (auto& b : bs.blocks) {
        const int64_t n = b.nnc(), cut = (n / chunk) * chunk;
        auto piece = [&](int64_t s, int64_t e) {
            Block c;
            c.g = 1;
            c.row_ids = b.row_ids;
            c.cols.assign(b.cols.begin() + s, b.cols.begin() + e);
            c.vals.assign(b.vals.begin() + s, b.vals.begin() + e);
            c.ins.assign(b.ins.begin() + s, b.ins.begin() + e);
            return c;
        };
        if (cut) lng->blocks.push_back(piece(0, cut));
        if (cut < n) shrt->blocks.push_back(piece(cut, n));
    }
}

std::vector<BlockSet> pipeline_sets(Level enc, int64_t K, const Cfg& cfg) {
    std::vector<BlockSet> sets;
    for (auto& s : extract_blocks(std::move(enc), K, cfg)) sets.push_back(clip_blocks(std::move(s), cfg));
    reorder_sets(&sets);
    std::vector<BlockSet> fin;
    for (auto& s : sets) {
        if (s.g == 1) {
            BlockSet l, sh;
            split_one_grained(s, cfg, &l, &sh);
            if (!l.blocks.empty()) fin.push_back(std::move(l));
            if (!sh.blocks.empty()) fin.push_back(std::move(sh));
        } else {
            fin.push_back(std::move(s));
        }
    }
    reorder_sets(&fin);
    return fin;
}

// --- encode_ec_csr (storage.py:184-251) ---------------------------------------------
struct OutSet {
    int32_t g = 1, v = 1;
    int64_t nb = 0, stored = 0, real = 0;
    std::vector<uint32_t> rows, bases, deltas;
    std::vector<int64_t> indptr;
    std::vector<uint8_t> mask;
    std::vector<double> vals;  // chunk-permuted, g per stored column
};

int encode_set(const BlockSet& bs, const Cfg& cfg, OutSet* o, std::string* err) {
    const int W = cfg.warp, v = bs.v, g = bs.g;
    o->g = g;
    o->v = v;
    o->nb = static_cast<int64_t>(bs.blocks.size());
    o->indptr.assign(o->nb + 1, 0);
    for (int64_t bi = 0; bi < o->nb; ++bi) {
        const Block& b = bs.blocks[bi];
        const int64_t n = b.nnc(), wv = static_cast<int64_t>(W) * v;
        const int64_t total = (n + wv - 1) / wv * wv, seg = total / W, chunks = seg / v;
        std::vector<int64_t> cols(total, 0);
        std::vector<uint8_t> mask(total, 1);
        for (int64_t c = 0; c < n; ++c) {
            cols[c] = b.cols[c];
            mask[c] = b.ins[c];
        }
        for (int64_t p = n; p < total; ++p)
            if ((p / seg) * seg < n) cols[p] = b.cols[n - 1];  // partial segment: repeat last column
        for (int t = 0; t < W; ++t) {
            o->bases.push_back(static_cast<uint32_t>(cols[t * seg]));
            for (int64_t m = 1; m < seg; ++m) {
                const int64_t d = cols[t * seg + m] - cols[t * seg + m - 1];
                if (d > cfg.limit()) {
                    *err = "gap " + std::to_string(d) + " exceeds the " + std::to_string(cfg.limit()) + " delta range";
                    return ECSR_ERR_CONTAINER;
                }
                if (d < 0) {
                    *err = "columns must be non-decreasing within each lane segment";
                    return ECSR_ERR_VALUE;
                }
            }
        }
        const size_t d0 = o->deltas.size(), v0 = o->vals.size();
        o->deltas.resize(d0 + total);
        o->mask.resize(d0 + total);
        o->vals.resize(v0 + total * g);
        for (int t = 0; t < W; ++t)
            for (int64_t i = 0; i < chunks; ++i)
                for (int j = 0; j < v; ++j) {
                    const int64_t src = t * seg + i * v + j;
                    const int64_t dst = i * wv + static_cast<int64_t>(t) * v + j;
                    o->deltas[d0 + dst] =
                        static_cast<uint32_t>(src % seg == 0 ? 0 : cols[src] - cols[src - 1]);
                    o->mask[d0 + dst] = mask[src];
                    for (int k = 0; k < g; ++k)
                        o->vals[v0 + dst * g + k] = src < n ? b.vals[k * n + src] : 0.0;
                }
        for (int64_t c = 0; c < total; ++c) o->real += mask[c] ? 0 : g;
        o->rows.insert(o->rows.end(), b.row_ids.begin(), b.row_ids.end());
        o->indptr[bi + 1] = o->indptr[bi] + total;
    }
    o->stored = o->indptr[o->nb];
    return ECSR_OK;
}

}  // namespace ecsr_enc_impl

struct ecsr_enc {
    int64_t rows = 0, cols = 0;
    int32_t warp = 32, delta_bits = 8;
    std::vector<ecsr_enc_impl::OutSet> sets;
};

namespace {
thread_local std::string g_enc_error;
}

extern "C" {

const char* ecsr_b200_enc_last_error(void) { return g_enc_error.c_str(); }

int ecsr_b200_encode(int64_t num_rows, int64_t num_cols, const int64_t* row_ptr, const int64_t* col_idx,
                     const void* values, int32_t value_dtype, int32_t warp_size, int32_t vector_size,
                     int32_t delta_bits, int32_t max_levels, int64_t clip_limit, int32_t threads,
                     ecsr_enc** out) {
    using namespace ecsr_enc_impl;
    if (!out) return ECSR_ERR_VALUE;
    *out = nullptr;
    if (warp_size < 1 || vector_size < 1) {
        g_enc_error = "warp_size and vector_size must be >= 1";
        return ECSR_ERR_VALUE;
    }
    if (delta_bits != 4 && delta_bits != 8 && delta_bits != 16) {
        g_enc_error = "delta_bits must be one of 4, 8, 16";
        return ECSR_ERR_VALUE;
    }
    if (num_rows < 0 || num_cols < 0 || num_cols > INT32_MAX || (num_rows > 0 && !row_ptr)) {
        g_enc_error = "bad matrix shape";
        return ECSR_ERR_VALUE;
    }
    if (value_dtype != ECSR_F32 && value_dtype != ECSR_F64) {
        g_enc_error = "values must be float32 or float64";
        return ECSR_ERR_VALUE;
    }
    if (threads > 0) omp_set_num_threads(threads);
    Cfg cfg;
    cfg.warp = warp_size;
    cfg.vector = vector_size;
    cfg.delta_bits = delta_bits;
    cfg.max_levels = max_levels;
    cfg.clip_limit = clip_limit;
    // EncodedMatrix.from_csr: payload cast to float64 (extraction.py:122-131)
    Level L;
    L.rows = num_rows;
    L.row_ptr.assign(row_ptr, row_ptr + num_rows + 1);
    const int64_t nnz = num_rows > 0 ? row_ptr[num_rows] : 0;
    L.col.resize(nnz);
    L.payload.resize(nnz);
    for (int64_t p = 0; p < nnz; ++p) {
        if (col_idx[p] < 0 || col_idx[p] >= num_cols) {
            g_enc_error = "column index out of range";
            return ECSR_ERR_VALUE;
        }
        L.col[p] = static_cast<int32_t>(col_idx[p]);
        L.payload[p] = value_dtype == ECSR_F64 ? static_cast<const double*>(values)[p]
                                               : static_cast<double>(static_cast<const float*>(values)[p]);
    }
    for (int64_t r = 0; r < num_rows; ++r)
        for (int64_t p = row_ptr[r] + 1; p < row_ptr[r + 1]; ++p)
            if (col_idx[p] <= col_idx[p - 1]) {
                g_enc_error = "column indices must be strictly increasing within each row";
                return ECSR_ERR_VALUE;
            }
    L.row_map.resize(num_rows);
    std::iota(L.row_map.begin(), L.row_map.end(), 0);
    auto* e = new ecsr_enc();
    e->rows = num_rows;
    e->cols = num_cols;
    e->warp = warp_size;
    e->delta_bits = delta_bits;
    std::vector<BlockSet> sets = pipeline_sets(std::move(L), num_cols, cfg);
    e->sets.resize(sets.size());
    for (size_t i = 0; i < sets.size(); ++i) {
        std::string err;
        const int rc = encode_set(sets[i], cfg, &e->sets[i], &err);
        if (rc) {
            g_enc_error = err;
            delete e;
            return rc;
        }
    }
    *out = e;
    return ECSR_OK;
}

int ecsr_b200_enc_nsets(const ecsr_enc* e) { return e ? static_cast<int>(e->sets.size()) : -1; }

int ecsr_b200_enc_set_info(const ecsr_enc* e, int32_t set, ecsr_set_info* info) {
    if (!e || !info || set < 0 || set >= static_cast<int32_t>(e->sets.size())) return ECSR_ERR_VALUE;
    const auto& s = e->sets[set];
    info->granularity = s.g;
    info->vector_size = s.v;
    info->num_blocks = s.nb;
    info->stored_cols = s.stored;
    info->real_nnz = s.real;
    return ECSR_OK;
}

int ecsr_b200_enc_copy_set(const ecsr_enc* e, int32_t set, ecsr_out_set* o, int32_t out_value_dtype) {
    if (!e || !o || set < 0 || set >= static_cast<int32_t>(e->sets.size())) return ECSR_ERR_VALUE;
    if (out_value_dtype != ECSR_F32 && out_value_dtype != ECSR_F64) return ECSR_ERR_VALUE;
    const auto& s = e->sets[set];
    std::memcpy(o->row_indices, s.rows.data(), 4 * s.rows.size());
    std::memcpy(o->block_indptr, s.indptr.data(), 8 * s.indptr.size());
    std::memcpy(o->base_indices, s.bases.data(), 4 * s.bases.size());
    std::memcpy(o->delta_indices, s.deltas.data(), 4 * s.deltas.size());
    std::memcpy(o->pad_mask, s.mask.data(), s.mask.size());
    if (out_value_dtype == ECSR_F64) {
        std::memcpy(o->block_values, s.vals.data(), 8 * s.vals.size());
    } else {
        float* dst = static_cast<float*>(o->block_values);
        for (size_t i = 0; i < s.vals.size(); ++i) dst[i] = static_cast<float>(s.vals[i]);
    }
    return ECSR_OK;
}

void ecsr_b200_enc_free(ecsr_enc* e) { delete e; }

}  // extern "C"
