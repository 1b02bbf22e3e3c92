/* oracle/pms8_oracle.c — TEST INFRASTRUCTURE ONLY (see pms8_oracle.h).
 *
 * A CPU restatement of the reference algorithm, function by function, each
 * citing the reference file:line it follows (paths relative to
 * /root/reference/proj). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library, and only as the checker.
 *
 * Parity pinned against the reference itself: tests/golden/ holds motif sets
 * and known-answer values produced by oracle/_ref (the reference sources
 * compiled by oracle/Makefile), see tests/golden/make_golden.py.
 */
#include "pms8_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- mt19937_64 (the std::mt19937_64 engine used by src/instance.cpp:31) ---- */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

static uint64_t mt64_next(mt64* r) {
    static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= A;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* bounded_draw, src/instance.cpp:12-20: rejection below 2^64 mod bound */
static uint64_t bounded_draw(mt64* r, uint64_t bound) {
    const uint64_t threshold = (~bound + 1) % bound;
    for (;;) {
        const uint64_t x = mt64_next(r);
        if (x >= threshold) return x % bound;
    }
}

/* generate_planted_instance, src/instance.cpp:22-73 */
int pms8o_generate(int n, int m, int l, int d, int sigma, uint64_t seed, int exact, uint8_t* codes_out,
                   uint8_t* motif_out, int32_t* positions_out) {
    if (l < 1 || l > m || d < 0 || d > l || n < 1) return -1;
    if (exact && sigma < 2) return -1;
    mt64 r;
    mt64_seed(&r, seed);
    for (int p = 0; p < l; ++p) motif_out[p] = (uint8_t)bounded_draw(&r, (uint64_t)sigma);
    int* columns = (int*)malloc(sizeof(int) * (size_t)l);
    uint8_t* occ = (uint8_t*)malloc((size_t)l);
    for (int i = 0; i < n; ++i) {
        uint8_t* seq = codes_out + (size_t)i * m;
        for (int j = 0; j < m; ++j) seq[j] = (uint8_t)bounded_draw(&r, (uint64_t)sigma);
        const int pos = (int)bounded_draw(&r, (uint64_t)(m - l + 1));
        memcpy(occ, motif_out, (size_t)l);
        for (int j = 0; j < l; ++j) columns[j] = j; /* partial Fisher-Yates, :53-67 */
        for (int j = 0; j < d; ++j) {
            const int pick = j + (int)bounded_draw(&r, (uint64_t)(l - j));
            const int tmp = columns[j];
            columns[j] = columns[pick];
            columns[pick] = tmp;
            const int col = columns[j];
            if (!exact) {
                occ[col] = (uint8_t)bounded_draw(&r, (uint64_t)sigma);
            } else {
                const int old = occ[col];
                uint64_t c = bounded_draw(&r, (uint64_t)(sigma - 1));
                if (c >= (uint64_t)old) ++c;
                occ[col] = (uint8_t)c;
            }
        }
        memcpy(seq + pos, occ, (size_t)l);
        positions_out[i] = pos;
    }
    free(columns);
    free(occ);
    return 0;
}

/* ---- statistics + threshold ---- */

/* neighborhood_size, src/instance.cpp:75-87: sum_{i<=d} C(l,i)(sigma-1)^i */
static unsigned __int128 nsize(int l, int d, int sigma) {
    unsigned __int128 total = 0, binom = 1, power = 1;
    for (int i = 0; i <= d; ++i) {
        total += binom * power;
        binom = binom * (unsigned)(l - i) / (unsigned)(i + 1);
        power *= (unsigned)(sigma - 1);
    }
    return total;
}

int pms8o_neighborhood_size(int l, int d, int sigma, char* buf, int buflen) {
    if (l < 0 || d < 0 || d > l || sigma < 2 || buflen < 2) return -1;
    unsigned __int128 v = nsize(l, d, sigma);
    char tmp[64];
    int k = 0;
    if (v == 0) tmp[k++] = '0';
    while (v) {
        tmp[k++] = (char)('0' + (int)(v % 10));
        v /= 10;
    }
    if (k + 1 > buflen) return -1;
    for (int i = 0; i < k; ++i) buf[i] = tmp[k - 1 - i];
    buf[k] = 0;
    return 0;
}

static double log_nsize(int l, int d, int sigma) { return (double)logl((long double)nsize(l, d, sigma)); }

/* threshold_curve + estimate_threshold, src/solver.cpp:75-117 */
int pms8o_estimate_threshold(int n, int m, int l, int d, int sigma) {
    if (n < 2) return n;
    if (m == l) return n;
    int best_t = 2;
    double best = INFINITY;
    if (m <= l) return best_t;
    const double log_nd = log_nsize(l, d, sigma);
    const double log_n2d = log_nsize(l, 2 * d < l ? 2 * d : l, sigma);
    const double log_p = log_n2d - l * log((double)sigma);
    const double log_q = log_nd - log_n2d;
    const double log_w = log((double)(m - l + 1));
    double* terms = (double*)malloc(sizeof(double) * (size_t)n);
    for (int k = 1; k <= n; ++k) terms[k - 1] = k * log_w + 0.5 * k * (k - 1) * log_p;
    for (int t = 2; t <= n; ++t) {
        double mx = terms[0];
        for (int k = 1; k < t; ++k)
            if (terms[k] > mx) mx = terms[k];
        double sum = 0;
        for (int k = 0; k < t; ++k) sum += exp(terms[k] - mx);
        const double ls = log((double)n) + log((double)l) + mx + log(sum);
        const double lp = terms[t - 1] + log_nd + (t - 1) * log_q + log((double)l);
        const double v = ls > lp ? ls : lp;
        if (v < best - 1e-12) {
            best = v;
            best_t = t;
        }
    }
    free(terms);
    return best_t;
}

/* ---- string-level predicates (src/pruning.cpp) ---- */

/* column_profile3 + triple_common_neighbor_exists, src/pruning.cpp:50-75 */
int pms8o_triple_ok(const uint8_t* a, const uint8_t* b, const uint8_t* c, int l, int d1, int d2, int d3) {
    int n1 = 0, n2 = 0, n3 = 0, n4 = 0;
    for (int i = 0; i < l; ++i) {
        const int ab = a[i] == b[i], ac = a[i] == c[i], bc = b[i] == c[i];
        if (ab && ac) continue;
        if (bc) ++n1;
        else if (ac) ++n2;
        else if (ab) ++n3;
        else ++n4;
    }
    if (n1 + n2 + n4 > d1 + d2) return 0;
    if (n1 + n3 + n4 > d1 + d3) return 0;
    if (n2 + n3 + n4 > d2 + d3) return 0;
    return n1 + n2 + n3 + 2 * n4 <= d1 + d2 + d3;
}

/* consensus_total_distance, src/pruning.cpp:27-43 */
int pms8o_consensus_distance(const uint8_t* tuple, int k, int l) {
    int total = 0;
    for (int col = 0; col < l; ++col) {
        int freq[256] = {0}, best = 0;
        for (int i = 0; i < k; ++i) {
            const int f = ++freq[tuple[(size_t)i * l + col]];
            if (f > best) best = f;
        }
        total += k - best;
    }
    return total;
}

/* ---- common d-neighbourhood enumerator (src/neighborhood.cpp:164-270) ----
 * tuples of at most PMS8O_MAX_K members (C(8,2)=28 pairs, C(8,3)=56 triples) */
#define PMS8O_MAX_K 8
typedef struct {
    int sigma, k, l, level;
    const uint8_t* codes; /* k x l */
    int budget[64];
    uint8_t cand[64];
    int np, nt;
    int pi[64], pj[64];                 /* pairs_ */
    int ti[64], tj[64], th[64];         /* triples_ */
    int tpij[64], tpih[64], tpjh[64];
    int tof_cnt[64], tof[64][64];       /* triples_of_ */
    int* pair_suffix;                   /* (l+1) x np */
    int* triple_n4;                     /* (l+1) x nt */
    int* cons_suffix;                   /* l+1 */
    int64_t visited;
    uint8_t* out;
    int64_t cap;
    /* optional leaf hook for the search (verify + emit) */
    void (*leaf)(void* ctx, const uint8_t* cand);
    void* leaf_ctx;
} enumr;

/* prepare, src/neighborhood.cpp:164-226 */
static void en_prepare(enumr* e, const uint8_t* tuple, int k, int l, int sigma, int d, int level) {
    e->sigma = sigma;
    e->k = k;
    e->l = l;
    e->level = level;
    e->codes = tuple;
    for (int i = 0; i < k; ++i) e->budget[i] = d;
    int pidx[64][64];
    e->np = 0;
    for (int i = 0; i < k; ++i)
        for (int j = i + 1; j < k; ++j) {
            pidx[i][j] = e->np;
            e->pi[e->np] = i;
            e->pj[e->np] = j;
            e->np++;
        }
    e->nt = 0;
    for (int i = 0; i < k; ++i) e->tof_cnt[i] = 0;
    for (int i = 0; i < k; ++i)
        for (int j = i + 1; j < k; ++j)
            for (int h = j + 1; h < k; ++h) {
                const int idx = e->nt++;
                e->ti[idx] = i;
                e->tj[idx] = j;
                e->th[idx] = h;
                e->tpij[idx] = pidx[i][j];
                e->tpih[idx] = pidx[i][h];
                e->tpjh[idx] = pidx[j][h];
                e->tof[i][e->tof_cnt[i]++] = idx;
                e->tof[j][e->tof_cnt[j]++] = idx;
                e->tof[h][e->tof_cnt[h]++] = idx;
            }
    const int np = e->np, nt = e->nt;
    e->pair_suffix = (int*)calloc((size_t)(l + 1) * (size_t)(np ? np : 1), sizeof(int));
    e->triple_n4 = (int*)calloc((size_t)(l + 1) * (size_t)(nt ? nt : 1), sizeof(int));
    e->cons_suffix = (int*)calloc((size_t)(l + 1), sizeof(int));
    for (int p = l - 1; p >= 0; --p) {
        for (int x = 0; x < np; ++x)
            e->pair_suffix[p * np + x] =
                e->pair_suffix[(p + 1) * np + x] + (tuple[e->pi[x] * l + p] != tuple[e->pj[x] * l + p]);
        for (int x = 0; x < nt; ++x) {
            const uint8_t a = tuple[e->ti[x] * l + p], b = tuple[e->tj[x] * l + p], c = tuple[e->th[x] * l + p];
            e->triple_n4[p * nt + x] = e->triple_n4[(p + 1) * nt + x] + (a != b && a != c && b != c);
        }
        int freq[256] = {0}, best = 0;
        for (int i = 0; i < k; ++i) {
            const int f = ++freq[tuple[i * l + p]];
            if (f > best) best = f;
        }
        e->cons_suffix[p] = e->cons_suffix[p + 1] + (k - best);
    }
}

static void en_free(enumr* e) {
    free(e->pair_suffix);
    free(e->triple_n4);
    free(e->cons_suffix);
}

/* prune, src/neighborhood.cpp:228-270 */
static int en_prune(const enumr* e, int p, int rep) {
    for (int i = 0; i < e->k; ++i)
        if (e->budget[i] < 0) return 1;
    const int np = e->np, nt = e->nt;
    for (int x = 0; x < np; ++x)
        if (e->pair_suffix[p * np + x] > e->budget[e->pi[x]] + e->budget[e->pj[x]]) return 1;
    if (e->level == 1) return 0;
    if (e->k >= 3) {
#define VIOL(idx)                                                                                              \
    ((e->pair_suffix[p * np + e->tpij[idx]] + e->pair_suffix[p * np + e->tpih[idx]] +                          \
      e->pair_suffix[p * np + e->tpjh[idx]] + e->triple_n4[p * nt + (idx)]) /                                  \
         2 >                                                                                                   \
     e->budget[e->ti[idx]] + e->budget[e->tj[idx]] + e->budget[e->th[idx]])
        if (e->k == 3 || rep < 0) {
            for (int x = 0; x < nt; ++x)
                if (VIOL(x)) return 1;
        } else {
            for (int q = 0; q < e->tof_cnt[rep]; ++q)
                if (VIOL(e->tof[rep][q])) return 1;
        }
#undef VIOL
    }
    if (e->k >= 2) {
        int total = 0;
        for (int i = 0; i < e->k; ++i) total += e->budget[i];
        if (e->cons_suffix[p] > total) return 1;
    }
    return 0;
}

/* descend, include/pms8/neighborhood.hpp:63-88 */
static void en_descend(enumr* e, int p, int spent_in, int rep) {
    if (p == e->l) {
        for (int i = 0; i < e->k; ++i)
            if (e->budget[i] < 0) return;
        if (e->out && e->visited < e->cap) memcpy(e->out + (size_t)e->visited * e->l, e->cand, (size_t)e->l);
        ++e->visited;
        if (e->leaf) e->leaf(e->leaf_ctx, e->cand);
        return;
    }
    if (spent_in && e->level != 0 && en_prune(e, p, rep)) return;
    for (int a = 0; a < e->sigma; ++a) {
        e->cand[p] = (uint8_t)a;
        int spent = 0, next_rep = -1;
        for (int i = 0; i < e->k; ++i)
            if (e->codes[i * e->l + p] != a) {
                const int r = --e->budget[i];
                spent = 1;
                if (next_rep < 0 || r < e->budget[next_rep]) next_rep = i;
            }
        en_descend(e, p + 1, spent, next_rep);
        for (int i = 0; i < e->k; ++i)
            if (e->codes[i * e->l + p] != a) ++e->budget[i];
    }
}

int64_t pms8o_common_neighborhood(const uint8_t* tuple, int k, int l, int sigma, int d, int level, uint8_t* out,
                                  int64_t cap) {
    if (k < 1 || k > PMS8O_MAX_K || l < 1 || l > 64 || d < 0) return -1;
    enumr e;
    memset(&e, 0, sizeof e);
    en_prepare(&e, tuple, k, l, sigma, d, level);
    e.out = out;
    e.cap = out ? cap : 0;
    en_descend(&e, 0, 1, -1);
    en_free(&e);
    return e.visited;
}

/* ---- packed l-mers: 5 bit planes of one 64-bit word (l <= 64, codes < 32):
 *      bit p of plane k = bit k of the code at position p. Hamming distance is
 *      popcount(OR_k plane_k(a) ^ plane_k(b)), for DNA exactly the reference's
 *      group-folded 2-bit distance (hamming64_*, include/pms8/packed_seq.hpp:
 *      127-170) and for b-bit alphabets its b-bit groups
 *      (src/alphabet.cpp:41). `words` is always 1 here. ---- */
typedef struct {
    uint64_t pl[5];
} pk;

static inline uint64_t pk_fold(const pk* a, const pk* b, int i) {
    (void)i;
    return (a->pl[0] ^ b->pl[0]) | (a->pl[1] ^ b->pl[1]) | (a->pl[2] ^ b->pl[2]) | (a->pl[3] ^ b->pl[3]) |
           (a->pl[4] ^ b->pl[4]);
}

static inline int pk_dist(const pk* a, const pk* b, int words) {
    (void)words;
    return __builtin_popcountll(pk_fold(a, b, 0));
}

static void pk_pack(const uint8_t* codes, int l, pk* out) {
    for (int k = 0; k < 5; ++k) out->pl[k] = 0;
    for (int p = 0; p < l; ++p)
        for (int k = 0; k < 5; ++k) out->pl[k] |= (uint64_t)((codes[p] >> k) & 1u) << p;
}

/* ---- the search: RowMatrix + MotifSearch (src/solver.cpp:156-432) ---- */
typedef struct {
    int n, m, l, d, sigma, t, w, words;
    int64_t K;
    const uint8_t* codes;
    pk* lmers;        /* K packed l-mers, id = seq*w + offset (packed_seq.hpp:62-64) */
    uint32_t* storage; /* n x w ids, row-major (RowMatrix::storage_) */
    int* live;
    int* order;
    int* frames; /* (n+1) x 2n */
    int nframes;
    uint32_t* stack;
    int depth;
    uint16_t* dist_to_stack; /* t x K */
    uint32_t** snapshot;
    uint8_t* tuple_codes;
    /* raw emitted motifs */
    uint8_t* raw;
    int64_t nraw, capraw;
    int64_t ctr[6];
} search_t;

/* RowMatrix::reset_full, src/solver.cpp:167-176 */
static void rows_reset(search_t* s) {
    for (int r = 0; r < s->n; ++r) {
        for (int j = 0; j < s->w; ++j) s->storage[(size_t)r * s->w + j] = (uint32_t)(r * s->w + j);
        s->live[r] = s->w;
        s->order[r] = r;
    }
    s->nframes = 0;
}

/* RowMatrix::sort_rows_by_size, src/solver.cpp:205-217 (stable insertion) */
static void rows_sort(search_t* s, int from) {
    for (int i = from + 1; i < s->n; ++i) {
        const int row = s->order[i], size = s->live[row];
        int j = i - 1;
        while (j >= from && s->live[s->order[j]] > size) {
            s->order[j + 1] = s->order[j];
            --j;
        }
        s->order[j + 1] = row;
    }
}

/* MotifSearch::push, src/solver.cpp:245-337 */
static int push(search_t* s, uint32_t u) {
    const int p = s->depth, n = s->n, d = s->d, words = s->words;
    const int64_t K = s->K;
    /* push_frame, :189-195 */
    int* f = s->frames + (size_t)s->nframes * 2 * n;
    memcpy(f, s->live, sizeof(int) * (size_t)n);
    memcpy(f + n, s->order, sizeof(int) * (size_t)n);
    s->nframes++;
    s->stack[s->depth++] = u;
    s->ctr[0]++;
    const pk* top = &s->lmers[u];
    int hsu[64];
    uint64_t fsu[64][2];
    for (int i = 0; i < p; ++i) {
        const pk* si = &s->lmers[s->stack[i]];
        hsu[i] = pk_dist(si, top, words);
        for (int x = 0; x < words; ++x) fsu[i][x] = pk_fold(si, top, x);
    }
    int viable = 1;
    for (int q = p; q < n; ++q) {
        const int row = s->order[q];
        uint32_t* ids = s->storage + (size_t)row * s->w;
        const int count = s->live[row];
        const size_t base = (size_t)row * s->w;
        int kept = 0;
        s->ctr[4] += count;
        for (int j = 0; j < count; ++j) {
            const uint32_t v = ids[j];
            const pk* vp = &s->lmers[v];
            uint64_t fvu[2];
            int hvu = 0;
            for (int x = 0; x < words; ++x) {
                fvu[x] = pk_fold(vp, top, x);
                hvu += __builtin_popcountll(fvu[x]);
            }
            if (hvu > 2 * d) continue; /* pair bit, :291 (all-ones when 2d >= l) */
            int ok = 1;
            for (int i = 0; i < p && ok; ++i) { /* Theorem 1 with budgets d,d,d, :302-319 */
                const int hvi = s->dist_to_stack[(size_t)i * K + base + j];
                const int sum = hvi + hvu + hsu[i];
                int mn = hvi < hvu ? hvi : hvu;
                if (hsu[i] < mn) mn = hsu[i];
                if (sum > 6 * d) {
                    ok = 0;
                } else if (sum + mn > 6 * d) {
                    const pk* si = &s->lmers[s->stack[i]];
                    int n4 = 0;
                    for (int x = 0; x < words; ++x)
                        n4 += __builtin_popcountll(pk_fold(vp, si, x) & fvu[x] & fsu[i][x]);
                    ok = sum + n4 <= 6 * d;
                }
            }
            if (!ok) continue;
            uint32_t tmp = ids[kept];
            ids[kept] = ids[j];
            ids[j] = tmp;
            for (int i = 0; i < p; ++i) {
                uint16_t* a = &s->dist_to_stack[(size_t)i * K + base + kept];
                uint16_t* b = &s->dist_to_stack[(size_t)i * K + base + j];
                const uint16_t t2 = *a;
                *a = *b;
                *b = t2;
            }
            s->dist_to_stack[(size_t)p * K + base + kept] = (uint16_t)hvu;
            ++kept;
        }
        s->live[row] = kept;
        if (kept == 0 && q > p) {
            viable = 0;
            break;
        }
    }
    return viable;
}

/* MotifSearch::pop, src/solver.cpp:339-342 */
static void pop(search_t* s) {
    s->nframes--;
    const int* f = s->frames + (size_t)s->nframes * 2 * s->n;
    memcpy(s->live, f, sizeof(int) * (size_t)s->n);
    memcpy(s->order, f + s->n, sizeof(int) * (size_t)s->n);
    s->depth--;
}

/* verify_candidate, src/solver.cpp:344-362 */
static int verify(search_t* s, const uint8_t* cand) {
    pk c;
    pk_pack(cand, s->l, &c);
    for (int q = s->depth; q < s->n; ++q) {
        const int row = s->order[q];
        const uint32_t* ids = s->storage + (size_t)row * s->w;
        int hit = 0;
        for (int j = 0; j < s->live[row]; ++j) {
            s->ctr[5]++;
            if (pk_dist(&c, &s->lmers[ids[j]], s->words) <= s->d) {
                hit = 1;
                break;
            }
        }
        if (!hit) return 0;
    }
    return 1;
}

/* emit, src/solver.cpp:364-385 (no cap, no reverify) */
static void leaf_cb(void* ctx, const uint8_t* cand) {
    search_t* s = (search_t*)ctx;
    if (!verify(s, cand)) return;
    if (s->nraw == s->capraw) {
        s->capraw = s->capraw ? 2 * s->capraw : 1024;
        s->raw = (uint8_t*)realloc(s->raw, (size_t)s->capraw * s->l);
    }
    memcpy(s->raw + (size_t)s->nraw * s->l, cand, (size_t)s->l);
    s->nraw++;
    s->ctr[3]++;
}

/* enumerate_and_collect, src/solver.cpp:387-404 */
static void enumerate_and_collect(search_t* s) {
    const int k = s->depth, l = s->l;
    for (int i = 0; i < k; ++i) {
        const uint32_t id = s->stack[i];
        const int seq = (int)(id / (uint32_t)s->w), off = (int)(id % (uint32_t)s->w);
        memcpy(s->tuple_codes + (size_t)i * l, s->codes + (size_t)seq * s->m + off, (size_t)l);
    }
    enumr e;
    memset(&e, 0, sizeof e);
    en_prepare(&e, s->tuple_codes, k, l, s->sigma, s->d, 2);
    e.leaf = leaf_cb;
    e.leaf_ctx = s;
    en_descend(&e, 0, 1, -1);
    en_free(&e);
    s->ctr[1]++;
    s->ctr[2] += e.visited;
}

/* recurse, src/solver.cpp:406-419 */
static void recurse(search_t* s) {
    const int p = s->depth;
    const int row = s->order[p];
    const int cnt = s->live[row];
    uint32_t* snap = s->snapshot[p];
    memcpy(snap, s->storage + (size_t)row * s->w, sizeof(uint32_t) * (size_t)cnt);
    for (int j = 0; j < cnt; ++j) {
        if (push(s, snap[j])) {
            rows_sort(s, s->depth);
            if (s->depth == s->t) enumerate_and_collect(s);
            else recurse(s);
        }
        pop(s);
    }
}

static int cmp_l;
static int cmp_codes(const void* a, const void* b) { return memcmp(a, b, (size_t)cmp_l); }

/* canonical_motif_set, src/solver.cpp:16-21 */
static int64_t canonical(uint8_t* raw, int64_t nraw, int l) {
    if (nraw == 0) return 0;
    cmp_l = l;
    qsort(raw, (size_t)nraw, (size_t)l, cmp_codes);
    int64_t u = 1;
    for (int64_t i = 1; i < nraw; ++i)
        if (memcmp(raw + (size_t)i * l, raw + (size_t)(u - 1) * l, (size_t)l) != 0) {
            if (u != i) memcpy(raw + (size_t)u * l, raw + (size_t)i * l, (size_t)l);
            ++u;
        }
    return u;
}

int64_t pms8o_solve(const uint8_t* codes, int n, int m, int l, int d, int sigma, int t, const int32_t* anchors,
                    int nanchors, uint8_t* out, int64_t cap, int64_t* counters) {
    if (n < 1 || l < 1 || l > m || d < 0 || d > l || l > 64 || sigma < 2 || sigma > 32) return -1;
    search_t s;
    memset(&s, 0, sizeof s);
    s.n = n;
    s.m = m;
    s.l = l;
    s.d = d;
    s.sigma = sigma;
    s.t = t > 0 ? t : pms8o_estimate_threshold(n, m, l, d, sigma);
    if (s.t < 1 || s.t > n || s.t > PMS8O_MAX_K) return -1;
    s.w = m - l + 1;
    s.K = (int64_t)n * s.w;
    s.words = 1; /* one 64-bit word per bit plane */
    s.codes = codes;
    s.lmers = (pk*)malloc(sizeof(pk) * (size_t)s.K);
    for (int r = 0; r < n; ++r)
        for (int j = 0; j < s.w; ++j) pk_pack(codes + (size_t)r * m + j, l, &s.lmers[r * s.w + j]);
    s.storage = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)s.K);
    s.live = (int*)malloc(sizeof(int) * (size_t)n);
    s.order = (int*)malloc(sizeof(int) * (size_t)n);
    s.frames = (int*)malloc(sizeof(int) * (size_t)(n + 1) * 2 * (size_t)n);
    s.stack = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(s.t + 1));
    s.dist_to_stack = (uint16_t*)calloc((size_t)s.t * (size_t)s.K, sizeof(uint16_t));
    s.snapshot = (uint32_t**)malloc(sizeof(uint32_t*) * (size_t)s.t);
    for (int i = 0; i < s.t; ++i) s.snapshot[i] = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)s.w);
    s.tuple_codes = (uint8_t*)malloc((size_t)s.t * (size_t)l);
    const int jobs = s.w; /* split_subproblems, src/parallel.cpp:14-20 */
    const int na = anchors ? nanchors : jobs;
    for (int a = 0; a < na; ++a) {
        const int off = anchors ? anchors[a] : a;
        if (off < 0 || off >= jobs) continue;
        /* run_anchored, src/solver.cpp:427-432 */
        rows_reset(&s);
        s.depth = 0;
        s.storage[0] = (uint32_t)off; /* restrict_row(0, lmer_id(0, off)) */
        s.live[0] = 1;
        rows_sort(&s, 0);
        recurse(&s);
    }
    const int64_t u = canonical(s.raw, s.nraw, l);
    if (out) memcpy(out, s.raw, (size_t)(u < cap ? u : cap) * (size_t)l);
    if (counters) memcpy(counters, s.ctr, sizeof s.ctr);
    for (int i = 0; i < s.t; ++i) free(s.snapshot[i]);
    free(s.snapshot);
    free(s.lmers);
    free(s.storage);
    free(s.live);
    free(s.order);
    free(s.frames);
    free(s.stack);
    free(s.dist_to_stack);
    free(s.tuple_codes);
    free(s.raw);
    return u;
}

/* naive_is_motif, src/oracle.cpp:16-37 */
int pms8o_is_motif(const uint8_t* codes, int n, int m, int l, int d, const uint8_t* motif) {
    for (int r = 0; r < n; ++r) {
        const uint8_t* seq = codes + (size_t)r * m;
        int found = 0;
        for (int j = 0; j + l <= m && !found; ++j) {
            int mm = 0;
            for (int p = 0; p < l && mm <= d; ++p) mm += seq[j + p] != motif[p];
            found = mm <= d;
        }
        if (!found) return 0;
    }
    return 1;
}

/* brute_force_solve, src/oracle.cpp:65-75: odometer over Sigma^l in code order */
int64_t pms8o_brute_force(const uint8_t* codes, int n, int m, int l, int d, int sigma, uint8_t* out, int64_t cap) {
    if (l < 1 || l > 24) return -1;
    uint8_t word[24] = {0};
    int64_t cnt = 0;
    for (;;) {
        if (pms8o_is_motif(codes, n, m, l, d, word)) {
            if (out && cnt < cap) memcpy(out + (size_t)cnt * l, word, (size_t)l);
            ++cnt;
        }
        int i = l - 1;
        for (; i >= 0; --i) {
            if (word[i] + 1 < sigma) {
                word[i]++;
                break;
            }
            word[i] = 0;
        }
        if (i < 0) break;
    }
    return cnt;
}
