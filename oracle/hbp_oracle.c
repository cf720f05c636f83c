/*
 * hbp_oracle.c — TEST INFRASTRUCTURE ONLY (see oracle.h). Never linked into
 * the product; the product fails loudly without its CUDA library.
 *
 * A sequential plain-C restatement of the reference planner
 * (/root/reference/proj/src, cited per function as file:line). Semantics are
 * the reference's, including tie-breaks, error texts and quirks. Two data
 * structures differ from the reference where it uses an O(N^2) scan or
 * std::multiset; they return exactly the element the reference scan returns:
 *   - first_fit (packing.cpp:86-103) finds "the first pack with room" with a
 *     max-residual segment tree instead of a linear scan;
 *   - greedy_fill (balance.cpp:62-101) replaces the ordered multiset by
 *     per-length FIFO queues of ascending ids plus a predecessor bitmap over
 *     lengths (largest length <= residual, lowest id first).
 * Parity of this restatement against the compiled reference is pinned by
 * tests/test_oracle.py (oracle/_ref) and by tests/golden/ fixtures.
 */
#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* ------------------------------------------------------------------------ */
/* errors                                                                    */
/* ------------------------------------------------------------------------ */

enum { OK = 0, EVAL = 2, EINF = 3 };

typedef struct errbuf {
    char* buf;
    int len;
} errbuf;

static int fail(errbuf* e, int code, const char* fmt, ...) {
    if (e && e->buf && e->len > 0) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(e->buf, (size_t)e->len, fmt, ap);
        va_end(ap);
    }
    return code;
}

static void* xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) {
        fprintf(stderr, "hbp_oracle: out of memory\n");
        abort();
    }
    return p;
}
static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s ? s : 1);
    if (!p) {
        fprintf(stderr, "hbp_oracle: out of memory\n");
        abort();
    }
    return p;
}
static void* xrealloc(void* p, size_t n) {
    p = realloc(p, n ? n : 1);
    if (!p) {
        fprintf(stderr, "hbp_oracle: out of memory\n");
        abort();
    }
    return p;
}

/* ------------------------------------------------------------------------ */
/* RNG: SplitMix64 stream, rng.hpp:14-95                                     */
/* ------------------------------------------------------------------------ */

typedef struct rng {
    uint64_t state;
    int have_spare;
    double spare;
} rng;

static rng rng_make(uint64_t seed) {
    rng r = {seed, 0, 0.0};
    return r;
}

static uint64_t rng_next(rng* r) { /* rng.hpp:18-23 */
    uint64_t z = (r->state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static double rng_double(rng* r) { /* rng.hpp:26-28 */
    return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}

static int64_t rng_uniform(rng* r, int64_t lo, int64_t hi) { /* rng.hpp:32-41 */
    const uint64_t span = (uint64_t)(hi - lo) + 1;
    if (span == 0) return (int64_t)rng_next(r);
    const uint64_t limit = UINT64_MAX - UINT64_MAX % span;
    uint64_t v;
    do {
        v = rng_next(r);
    } while (v >= limit);
    return lo + (int64_t)(v % span);
}

static double rng_normal(rng* r) { /* rng.hpp:44-58, Box-Muller with spare */
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1, u2;
    do {
        u1 = rng_double(r);
    } while (u1 <= 0.0);
    u2 = rng_double(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double theta = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(theta);
    r->have_spare = 1;
    return rad * cos(theta);
}

/* Fisher-Yates over `n` elements of `size` bytes, rng.hpp:61-68. */
static void rng_shuffle(rng* r, void* base, int64_t n, size_t size) {
    unsigned char tmp[64];
    unsigned char* v = (unsigned char*)base;
    for (int64_t i = n; i > 1; --i) {
        const int64_t j = rng_uniform(r, 0, i - 1);
        if (j != i - 1) {
            memcpy(tmp, v + (size_t)(i - 1) * size, size);
            memcpy(v + (size_t)(i - 1) * size, v + (size_t)j * size, size);
            memcpy(v + (size_t)j * size, tmp, size);
        }
    }
}

static uint64_t derive_seed(uint64_t seed, const char* tag) { /* rng.hpp:80-89 */
    uint64_t h = 0xcbf29ce484222325ULL ^ seed;
    for (const unsigned char* c = (const unsigned char*)tag; *c; ++c) {
        h ^= *c;
        h *= 0x100000001b3ULL;
    }
    h = (h ^ (h >> 30)) * 0xbf58476d1ce4e5b9ULL;
    h = (h ^ (h >> 27)) * 0x94d049bb133111ebULL;
    return h ^ (h >> 31);
}

static uint64_t derive_seed_i(uint64_t seed, const char* tag, uint64_t index) {
    return derive_seed(seed ^ (0x9e3779b97f4a7c15ULL * (index + 1)), tag); /* rng.hpp:91-94 */
}

/* ------------------------------------------------------------------------ */
/* samples, packs, pack lists                                                */
/* ------------------------------------------------------------------------ */

typedef struct sample {
    int64_t id;
    int64_t length;
} sample;

typedef struct svec {
    sample* v;
    int64_t n, cap;
} svec;

static void sv_push(svec* s, sample x) {
    if (s->n == s->cap) {
        s->cap = s->cap ? s->cap * 2 : 4;
        s->v = (sample*)xrealloc(s->v, sizeof(sample) * (size_t)s->cap);
    }
    s->v[s->n++] = x;
}
static void sv_free(svec* s) {
    free(s->v);
    s->v = NULL;
    s->n = s->cap = 0;
}

typedef struct pack { /* metrics.hpp:16-35 */
    svec samples;
    int64_t capacity, total, attention;
} pack;

static pack pack_make(int64_t capacity) {
    pack p;
    memset(&p, 0, sizeof p);
    p.capacity = capacity;
    return p;
}
static void pack_add(pack* p, sample s) {
    sv_push(&p->samples, s);
    p->total += s.length;
    p->attention += s.length * s.length;
}
static int64_t pack_residual(const pack* p) { return p->capacity - p->total; }

typedef struct plist {
    pack* v;
    int64_t n, cap;
} plist;

static void pl_push(plist* l, pack p) {
    if (l->n == l->cap) {
        l->cap = l->cap ? l->cap * 2 : 16;
        l->v = (pack*)xrealloc(l->v, sizeof(pack) * (size_t)l->cap);
    }
    l->v[l->n++] = p;
}
static void pl_free(plist* l) {
    for (int64_t i = 0; i < l->n; ++i) sv_free(&l->v[i].samples);
    free(l->v);
    l->v = NULL;
    l->n = l->cap = 0;
}

/* device batch / iteration (balance.hpp:18-22, metrics.hpp:26-35) */
typedef struct dbatch {
    int32_t device_index;
    plist packs;
    int64_t tokens, comm_tokens, attention;
} dbatch;

static dbatch dbatch_build(int32_t d, plist packs, int sp_comm) { /* metrics.cpp:9-20 */
    dbatch b;
    b.device_index = d;
    b.packs = packs;
    b.tokens = 0;
    b.attention = 0;
    for (int64_t i = 0; i < packs.n; ++i) {
        b.tokens += packs.v[i].total;
        b.attention += packs.v[i].attention;
    }
    b.comm_tokens = sp_comm ? b.tokens : 0;
    return b;
}

typedef struct iteration {
    int32_t group_index;
    int32_t n_devices;
    dbatch* devices;
} iteration;

typedef struct ilist {
    iteration* v;
    int64_t n, cap;
} ilist;

static void il_push(ilist* l, iteration it) {
    if (l->n == l->cap) {
        l->cap = l->cap ? l->cap * 2 : 16;
        l->v = (iteration*)xrealloc(l->v, sizeof(iteration) * (size_t)l->cap);
    }
    l->v[l->n++] = it;
}
static void il_free(ilist* l) {
    for (int64_t i = 0; i < l->n; ++i) {
        for (int32_t d = 0; d < l->v[i].n_devices; ++d) pl_free(&l->v[i].devices[d].packs);
        free(l->v[i].devices);
    }
    free(l->v);
    l->v = NULL;
    l->n = l->cap = 0;
}

/* ------------------------------------------------------------------------ */
/* flat <-> structured                                                       */
/* ------------------------------------------------------------------------ */

typedef struct flat {
    int32_t* ig;
    int64_t *ido, ni;
    int32_t* di;
    int64_t *dpo, nd;
    int64_t *cap, *tot, *att, *mo, np;
    int64_t *mid, *mlen, nm;
    int64_t ci, cd, cp, cm;
} flat;

#define GROW(arr, n, c, T)                                             \
    do {                                                               \
        if ((n) >= (c)) {                                              \
            (c) = (c) ? (c) * 2 : 64;                                  \
            (arr) = (T*)xrealloc((arr), sizeof(T) * (size_t)((c) + 1)); \
        }                                                              \
    } while (0)

static void flat_init(flat* f) {
    memset(f, 0, sizeof *f);
    f->ido = (int64_t*)xcalloc(1, sizeof(int64_t));
    f->dpo = (int64_t*)xcalloc(1, sizeof(int64_t));
    f->mo = (int64_t*)xcalloc(1, sizeof(int64_t));
}

static void flat_pack(flat* f, const pack* p) {
    if (f->np + 1 >= f->cp) {
        f->cp = f->cp ? f->cp * 2 : 64;
        f->cap = (int64_t*)xrealloc(f->cap, sizeof(int64_t) * (size_t)(f->cp + 1));
        f->tot = (int64_t*)xrealloc(f->tot, sizeof(int64_t) * (size_t)(f->cp + 1));
        f->att = (int64_t*)xrealloc(f->att, sizeof(int64_t) * (size_t)(f->cp + 1));
        f->mo = (int64_t*)xrealloc(f->mo, sizeof(int64_t) * (size_t)(f->cp + 2));
    }
    f->cap[f->np] = p->capacity;
    f->tot[f->np] = p->total;
    f->att[f->np] = p->attention;
    for (int64_t k = 0; k < p->samples.n; ++k) {
        if (f->nm + 1 >= f->cm) {
            f->cm = f->cm ? f->cm * 2 : 256;
            f->mid = (int64_t*)xrealloc(f->mid, sizeof(int64_t) * (size_t)(f->cm + 1));
            f->mlen = (int64_t*)xrealloc(f->mlen, sizeof(int64_t) * (size_t)(f->cm + 1));
        }
        f->mid[f->nm] = p->samples.v[k].id;
        f->mlen[f->nm] = p->samples.v[k].length;
        f->nm++;
    }
    f->np++;
    f->mo[f->np] = f->nm;
}

static void flat_iteration(flat* f, const iteration* it) {
    if (f->ni + 1 >= f->ci) {
        f->ci = f->ci ? f->ci * 2 : 64;
        f->ig = (int32_t*)xrealloc(f->ig, sizeof(int32_t) * (size_t)(f->ci + 1));
        f->ido = (int64_t*)xrealloc(f->ido, sizeof(int64_t) * (size_t)(f->ci + 2));
    }
    f->ig[f->ni] = it->group_index;
    for (int32_t d = 0; d < it->n_devices; ++d) {
        if (f->nd + 1 >= f->cd) {
            f->cd = f->cd ? f->cd * 2 : 64;
            f->di = (int32_t*)xrealloc(f->di, sizeof(int32_t) * (size_t)(f->cd + 1));
            f->dpo = (int64_t*)xrealloc(f->dpo, sizeof(int64_t) * (size_t)(f->cd + 2));
        }
        f->di[f->nd] = it->devices[d].device_index;
        for (int64_t p = 0; p < it->devices[d].packs.n; ++p) flat_pack(f, &it->devices[d].packs.v[p]);
        f->nd++;
        f->dpo[f->nd] = f->np;
    }
    f->ni++;
    f->ido[f->ni] = f->nd;
}

static oracle_plan* flat_finish(flat* f, int32_t device_count, uint64_t seed) {
    oracle_plan* o = (oracle_plan*)xcalloc(1, sizeof(oracle_plan));
    o->device_count = device_count;
    o->seed = seed;
    o->n_iterations = f->ni;
    o->n_devices = f->nd;
    o->n_packs = f->np;
    o->n_members = f->nm;
#define ENSURE(p, T) \
    if (!(p)) (p) = (T*)xcalloc(1, sizeof(T))
    ENSURE(f->ig, int32_t);
    ENSURE(f->di, int32_t);
    ENSURE(f->cap, int64_t);
    ENSURE(f->tot, int64_t);
    ENSURE(f->att, int64_t);
    ENSURE(f->mid, int64_t);
    ENSURE(f->mlen, int64_t);
#undef ENSURE
    o->iter_group = f->ig;
    o->iter_dev_offsets = f->ido;
    o->dev_index = f->di;
    o->dev_pack_offsets = f->dpo;
    o->pack_capacity = f->cap;
    o->pack_total = f->tot;
    o->pack_attention = f->att;
    o->pack_member_offsets = f->mo;
    o->member_id = f->mid;
    o->member_length = f->mlen;
    return o;
}

static plist plist_from_flat(const oracle_plan* o) {
    plist l;
    memset(&l, 0, sizeof l);
    for (int64_t p = 0; p < o->n_packs; ++p) {
        pack pk = pack_make(o->pack_capacity[p]);
        for (int64_t k = o->pack_member_offsets[p]; k < o->pack_member_offsets[p + 1]; ++k) {
            sample s = {o->member_id[k], o->member_length[k]};
            pack_add(&pk, s);
        }
        pl_push(&l, pk);
    }
    return l;
}

/* ------------------------------------------------------------------------ */
/* validation: types.cpp:8-24 and autoselect.cpp:18-33                        */
/* ------------------------------------------------------------------------ */

/* open-addressing hash set of int64 ids */
typedef struct idset {
    int64_t* keys;
    unsigned char* used;
    uint64_t mask;
} idset;

static idset idset_make(int64_t n) {
    uint64_t cap = 16;
    while (cap < (uint64_t)n * 2) cap <<= 1;
    idset s;
    s.keys = (int64_t*)xmalloc(sizeof(int64_t) * cap);
    s.used = (unsigned char*)xcalloc(cap, 1);
    s.mask = cap - 1;
    return s;
}
static int idset_insert(idset* s, int64_t k) { /* 1 if newly inserted */
    uint64_t h = (uint64_t)k * 0x9e3779b97f4a7c15ULL;
    h ^= h >> 29;
    for (uint64_t i = h & s->mask;; i = (i + 1) & s->mask) {
        if (!s->used[i]) {
            s->used[i] = 1;
            s->keys[i] = k;
            return 1;
        }
        if (s->keys[i] == k) return 0;
    }
}
static void idset_free(idset* s) {
    free(s->keys);
    free(s->used);
}

static int validate_samples(const sample* v, int64_t n, errbuf* e) {
    if (n == 0) return fail(e, EVAL, "empty corpus: %s", "oracle");
    idset seen = idset_make(n);
    int rc = OK;
    for (int64_t i = 0; i < n; ++i) {
        if (v[i].length < 1) {
            rc = fail(e, EVAL, "sample %lld has non-positive length %lld", (long long)v[i].id,
                      (long long)v[i].length);
            break;
        }
        if (!idset_insert(&seen, v[i].id)) {
            rc = fail(e, EVAL, "duplicate sample id %lld", (long long)v[i].id);
            break;
        }
    }
    idset_free(&seen);
    return rc;
}

static int validate_groups(const hbp_groups* g, errbuf* e) {
    if (g->count < 1) return fail(e, EVAL, "no packing groups");
    int64_t prev = 0;
    for (int32_t i = 0; i < g->count; ++i) {
        if (g->groups[i].length <= prev)
            return fail(e, EVAL, "group lengths must be strictly increasing");
        if (g->groups[i].sp < 1 || g->groups[i].ckpt < 0)
            return fail(e, EVAL, "invalid group runtime config");
        prev = g->groups[i].length;
    }
    if (g->groups[g->count - 1].length != g->l_max) return fail(e, EVAL, "last group must carry l_max");
    return OK;
}

static sample* make_samples(const int64_t* ids, const int64_t* lengths, int64_t n) {
    sample* v = (sample*)xmalloc(sizeof(sample) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        v[i].id = ids ? ids[i] : i;
        v[i].length = lengths[i];
    }
    return v;
}

/* ------------------------------------------------------------------------ */
/* group_data: balance.cpp:25-44                                              */
/* ------------------------------------------------------------------------ */

static int group_data(const sample* v, int64_t n, const hbp_groups* g, svec* parts, errbuf* e) {
    int rc = validate_groups(g, e);
    if (rc) return rc;
    for (int64_t i = 0; i < n; ++i) {
        if (v[i].length > g->l_max)
            return fail(e, EVAL, "sample %lld exceeds the largest packing length %lld",
                        (long long)v[i].id, (long long)g->l_max);
        int32_t idx = 0;
        while (v[i].length > g->groups[idx].length) ++idx; /* (l_{i-1}, l_i] */
        sv_push(&parts[idx], v[i]);
    }
    return OK;
}

/* ------------------------------------------------------------------------ */
/* packing strategies: packing.cpp                                            */
/* ------------------------------------------------------------------------ */

static int cmp_decreasing(const void* a, const void* b) { /* packing.cpp:55-60 */
    const sample* x = (const sample*)a;
    const sample* y = (const sample*)b;
    if (x->length != y->length) return x->length > y->length ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}
static int cmp_by_id(const void* a, const void* b) {
    const sample* x = (const sample*)a;
    const sample* y = (const sample*)b;
    return (x->id > y->id) - (x->id < y->id);
}

/* next fit, packing.cpp:69-82 */
static void sequential_fill(const sample* order, int64_t n, int64_t capacity, plist* out) {
    pack cur = pack_make(capacity);
    for (int64_t i = 0; i < n; ++i) {
        if (cur.total + order[i].length > capacity) {
            if (cur.samples.n) pl_push(out, cur);
            else sv_free(&cur.samples);
            cur = pack_make(capacity);
        }
        pack_add(&cur, order[i]);
    }
    if (cur.samples.n) pl_push(out, cur);
    else sv_free(&cur.samples);
}

/* first fit, packing.cpp:86-103. The scan "first pack with total + len <=
 * capacity" is answered by a max-residual segment tree over pack slots. */
typedef struct segtree {
    int64_t* t;
    int64_t size; /* leaves, power of two */
} segtree;

static segtree seg_make(int64_t leaves) {
    segtree s;
    s.size = 1;
    while (s.size < leaves) s.size <<= 1;
    s.t = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(2 * s.size));
    for (int64_t i = 0; i < 2 * s.size; ++i) s.t[i] = -1; /* empty slot: never fits */
    return s;
}
static void seg_set(segtree* s, int64_t i, int64_t v) {
    int64_t k = i + s->size;
    s->t[k] = v;
    for (k >>= 1; k >= 1; k >>= 1) s->t[k] = s->t[2 * k] > s->t[2 * k + 1] ? s->t[2 * k] : s->t[2 * k + 1];
}
static int64_t seg_first_ge(const segtree* s, int64_t need) { /* leftmost leaf >= need */
    if (s->t[1] < need) return -1;
    int64_t k = 1;
    while (k < s->size) k = s->t[2 * k] >= need ? 2 * k : 2 * k + 1;
    return k - s->size;
}

static void first_fit(const sample* order, int64_t n, int64_t capacity, plist* out) {
    const int64_t base = out->n;
    segtree st = seg_make(n > 0 ? n : 1);
    int64_t used = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t b = seg_first_ge(&st, order[i].length);
        if (b < 0) {
            pl_push(out, pack_make(capacity));
            b = used++;
        }
        pack* p = &out->v[base + b];
        pack_add(p, order[i]);
        seg_set(&st, b, pack_residual(p));
    }
    free(st.t);
}

/* best fit, packing.cpp:107-127: tightest pack with room, earliest on ties */
static void best_fit(const sample* order, int64_t n, int64_t capacity, plist* out) {
    const int64_t base = out->n;
    for (int64_t i = 0; i < n; ++i) {
        int64_t best = -1;
        int64_t best_res = capacity + 1;
        for (int64_t b = base; b < out->n; ++b) {
            const int64_t r = pack_residual(&out->v[b]);
            if (r >= order[i].length && r < best_res) {
                best = b;
                best_res = r;
            }
        }
        if (best < 0) {
            pl_push(out, pack_make(capacity));
            best = out->n - 1;
        }
        pack_add(&out->v[best], order[i]);
    }
}

/* SPFHP, packing.cpp:132-162: lengths longest first (ids ascending), each
 * sample joins the open pack with the largest residual (lowest index on
 * ties) when that residual fits, else opens a pack. A max-heap keyed by
 * (residual desc, index asc) returns the same pack as the reference's
 * residual -> index-set map. */
typedef struct hentry {
    int64_t residual, index;
} hentry;
static int h_less(hentry a, hentry b) { /* a above b */
    if (a.residual != b.residual) return a.residual > b.residual;
    return a.index < b.index;
}
static void h_push(hentry* h, int64_t* n, hentry x) {
    int64_t i = (*n)++;
    h[i] = x;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!h_less(h[i], h[p])) break;
        hentry t = h[i];
        h[i] = h[p];
        h[p] = t;
        i = p;
    }
}
static hentry h_pop(hentry* h, int64_t* n) {
    hentry top = h[0];
    h[0] = h[--(*n)];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && h_less(h[l], h[m])) m = l;
        if (r < *n && h_less(h[r], h[m])) m = r;
        if (m == i) break;
        hentry t = h[i];
        h[i] = h[m];
        h[m] = t;
        i = m;
    }
    return top;
}
static void spfhp(sample* v, int64_t n, int64_t capacity, plist* out) {
    qsort(v, (size_t)n, sizeof(sample), cmp_decreasing);
    hentry* heap = (hentry*)xmalloc(sizeof(hentry) * (size_t)(n + 1));
    int64_t hn = 0;
    const int64_t base = out->n;
    for (int64_t i = 0; i < n; ++i) {
        if (hn > 0 && heap[0].residual >= v[i].length) {
            hentry top = h_pop(heap, &hn);
            pack* p = &out->v[base + top.index];
            pack_add(p, v[i]);
            hentry e = {pack_residual(p), top.index};
            h_push(heap, &hn, e);
        } else {
            pl_push(out, pack_make(capacity));
            pack* p = &out->v[out->n - 1];
            pack_add(p, v[i]);
            hentry e = {pack_residual(p), out->n - 1 - base};
            h_push(heap, &hn, e);
        }
    }
    free(heap);
}

/* ISF, packing.cpp:164-206 */
static void isf(sample* pool, int64_t n, int64_t capacity, int32_t rounds, double threshold, uint64_t seed,
                plist* out) {
    sample* next = (sample*)xmalloc(sizeof(sample) * (size_t)(n + 1));
    for (int32_t round = 0; round < rounds && n > 0; ++round) {
        rng r = rng_make(derive_seed_i(seed, "isf-round", (uint64_t)round));
        rng_shuffle(&r, pool, n, sizeof(sample));
        plist packs;
        memset(&packs, 0, sizeof packs);
        sequential_fill(pool, n, capacity, &packs);
        const double min_fill = (double)capacity * threshold;
        int64_t m = 0;
        for (int64_t p = 0; p < packs.n; ++p) {
            if ((double)packs.v[p].total >= min_fill) {
                pl_push(out, packs.v[p]);
            } else {
                for (int64_t k = 0; k < packs.v[p].samples.n; ++k) next[m++] = packs.v[p].samples.v[k];
                sv_free(&packs.v[p].samples);
            }
        }
        free(packs.v);
        memcpy(pool, next, sizeof(sample) * (size_t)m);
        n = m;
    }
    free(next);
    qsort(pool, (size_t)n, sizeof(sample), cmp_decreasing);
    first_fit(pool, n, capacity, out);
}

static int strategy_validate(const hbp_strategy* s, errbuf* e) { /* packing.cpp:33-42 */
    if (s->kind == HBP_STRATEGY_ISF) {
        if (s->isf_iterations < 1) return fail(e, EVAL, "isf_iterations must be >= 1");
        if (s->isf_fill_threshold <= 0.0 || s->isf_fill_threshold > 1.0)
            return fail(e, EVAL, "isf fill threshold must lie in (0, 1]");
    }
    return OK;
}

/* pack(), packing.cpp:210-261 */
static int do_pack(const sample* in, int64_t n, int64_t capacity, const hbp_strategy* s, uint64_t seed, plist* out,
                   errbuf* e) {
    int rc = strategy_validate(s, e);
    if (rc) return rc;
    if (capacity < 1) return fail(e, EVAL, "pack capacity must be >= 1");
    for (int64_t i = 0; i < n; ++i) {
        if (in[i].length > capacity)
            return fail(e, EVAL, "sample %lld length %lld exceeds pack capacity %lld", (long long)in[i].id,
                        (long long)in[i].length, (long long)capacity);
        if (in[i].length < 1) return fail(e, EVAL, "sample %lld has non-positive length", (long long)in[i].id);
    }
    sample* order = (sample*)xmalloc(sizeof(sample) * (size_t)(n + 1));
    memcpy(order, in, sizeof(sample) * (size_t)n);
    rng r;
    switch (s->kind) {
        case HBP_STRATEGY_RANDOM:
            r = rng_make(derive_seed(seed, "random-pack"));
            rng_shuffle(&r, order, n, sizeof(sample));
            sequential_fill(order, n, capacity, out);
            break;
        case HBP_STRATEGY_ISF:
            isf(order, n, capacity, s->isf_iterations, s->isf_fill_threshold, seed, out);
            break;
        case HBP_STRATEGY_FFS:
            r = rng_make(derive_seed(seed, "ffs"));
            rng_shuffle(&r, order, n, sizeof(sample));
            first_fit(order, n, capacity, out);
            break;
        case HBP_STRATEGY_FFD:
            qsort(order, (size_t)n, sizeof(sample), cmp_decreasing);
            first_fit(order, n, capacity, out);
            break;
        case HBP_STRATEGY_BFS:
            r = rng_make(derive_seed(seed, "bfs"));
            rng_shuffle(&r, order, n, sizeof(sample));
            best_fit(order, n, capacity, out);
            break;
        case HBP_STRATEGY_SPFHP:
            spfhp(order, n, capacity, out);
            break;
        default:
            free(order);
            return fail(e, EVAL, "unknown packing strategy");
    }
    free(order);
    return OK;
}

/* ------------------------------------------------------------------------ */
/* greedy fill: balance.cpp:46-101                                            */
/* ------------------------------------------------------------------------ */

/* One pool: for each length, its samples sorted by id; ids <= -2 form a
 * prefix (the reference probe {residual, id=-1} skips them at the exact
 * length, balance.cpp:82-83). `avail` is a 64-ary bitmap over lengths. */
typedef struct fpool {
    int64_t maxlen;
    int64_t* start;  /* [maxlen + 2] CSR over lengths 0..maxlen */
    int64_t* neg_head;
    int64_t* neg_end; /* ids <= -2 in [start, neg_end) */
    int64_t* pos_head; /* ids >= -1 in [neg_end, start[L+1]) */
    int64_t* pos_of;  /* entry -> position in the input pool */
    int64_t* ids;
    uint64_t* bits[4];
    int64_t nwords[4];
    int levels;
    int64_t remaining;
} fpool;

static void fp_setbit(fpool* f, int64_t L, int on) {
    for (int lv = 0; lv < f->levels; ++lv) {
        const int64_t w = L >> 6;
        const uint64_t m = 1ULL << (L & 63);
        if (on) {
            const int was = f->bits[lv][w] != 0;
            f->bits[lv][w] |= m;
            if (was) return;
        } else {
            f->bits[lv][w] &= ~m;
            if (f->bits[lv][w]) return;
        }
        L = w;
    }
}

/* largest length <= x with a set bit, or -1 */
static int64_t fp_pred(const fpool* f, int64_t x) {
    if (x < 0) return -1;
    if (x > f->maxlen) x = f->maxlen;
    int lv = 0;
    int64_t pos = x;
    /* climb until a word holds a bit at or below pos */
    for (;;) {
        const int64_t w = pos >> 6;
        const int b = (int)(pos & 63);
        const uint64_t m = b == 63 ? ~0ULL : ((1ULL << (b + 1)) - 1);
        const uint64_t v = f->bits[lv][w] & m;
        if (v) {
            pos = (w << 6) + 63 - __builtin_clzll(v);
            break;
        }
        if (lv + 1 >= f->levels || w == 0) {
            /* scan left at this level (top level is tiny) */
            int64_t ww = w - 1;
            while (ww >= 0 && f->bits[lv][ww] == 0) --ww;
            if (ww < 0) return -1;
            pos = (ww << 6) + 63 - __builtin_clzll(f->bits[lv][ww]);
            break;
        }
        pos = w - 1;
        lv++;
        if (pos < 0) return -1;
    }
    /* descend: take the highest set bit in each child word */
    while (lv > 0) {
        lv--;
        const uint64_t v = f->bits[lv][pos];
        pos = (pos << 6) + 63 - __builtin_clzll(v);
    }
    return pos;
}

static int cmp_len_id(const void* a, const void* b) { /* length asc, id asc */
    const int64_t* x = (const int64_t*)a;
    const int64_t* y = (const int64_t*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}

static void fp_build(fpool* f, const svec* pool) {
    memset(f, 0, sizeof *f);
    int64_t maxlen = 1;
    for (int64_t k = 0; k < pool->n; ++k)
        if (pool->v[k].length > maxlen) maxlen = pool->v[k].length;
    f->maxlen = maxlen;
    const int64_t n = pool->n;
    int64_t* tri = (int64_t*)xmalloc(sizeof(int64_t) * 3 * (size_t)(n + 1));
    for (int64_t k = 0; k < n; ++k) {
        tri[3 * k] = pool->v[k].length;
        tri[3 * k + 1] = pool->v[k].id;
        tri[3 * k + 2] = k;
    }
    qsort(tri, (size_t)n, 3 * sizeof(int64_t), cmp_len_id);
    f->start = (int64_t*)xcalloc((size_t)(maxlen + 2), sizeof(int64_t));
    f->neg_head = (int64_t*)xcalloc((size_t)(maxlen + 1), sizeof(int64_t));
    f->neg_end = (int64_t*)xcalloc((size_t)(maxlen + 1), sizeof(int64_t));
    f->pos_head = (int64_t*)xcalloc((size_t)(maxlen + 1), sizeof(int64_t));
    f->pos_of = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(n + 1));
    f->ids = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t k = 0; k < n; ++k) {
        f->start[tri[3 * k] + 1]++;
        f->ids[k] = tri[3 * k + 1];
        f->pos_of[k] = tri[3 * k + 2];
    }
    for (int64_t L = 0; L <= maxlen; ++L) f->start[L + 1] += f->start[L];
    int64_t words = (maxlen >> 6) + 1;
    f->levels = 0;
    for (;;) {
        f->nwords[f->levels] = words;
        f->bits[f->levels] = (uint64_t*)xcalloc((size_t)words, sizeof(uint64_t));
        f->levels++;
        if (words <= 1 || f->levels == 4) break;
        words = ((words - 1) >> 6) + 1;
    }
    for (int64_t L = 0; L <= maxlen; ++L) {
        int64_t a = f->start[L], b = f->start[L + 1];
        int64_t m = a;
        while (m < b && f->ids[m] <= -2) ++m;
        f->neg_head[L] = a;
        f->neg_end[L] = m;
        f->pos_head[L] = m;
        if (b > a) fp_setbit(f, L, 1);
    }
    f->remaining = n;
    free(tri);
}

static void fp_free(fpool* f) {
    free(f->start);
    free(f->neg_head);
    free(f->neg_end);
    free(f->pos_head);
    free(f->pos_of);
    free(f->ids);
    for (int lv = 0; lv < f->levels; ++lv) free(f->bits[lv]);
}

static int fp_empty_at(const fpool* f, int64_t L) {
    return f->neg_head[L] == f->neg_end[L] && f->pos_head[L] == f->start[L + 1];
}

/* Take the entry the reference's lower_bound({residual, -1}) returns, or -1. */
static int64_t fp_take(fpool* f, int64_t residual) {
    if (residual <= 0) return -1;
    int64_t entry = -1;
    if (residual <= f->maxlen && f->pos_head[residual] < f->start[residual + 1]) {
        entry = f->pos_head[residual]++; /* exact length, lowest id >= -1 */
        if (fp_empty_at(f, residual)) fp_setbit(f, residual, 0);
        f->remaining--;
        return entry;
    }
    const int64_t L = fp_pred(f, residual - 1); /* largest shorter length */
    if (L < 0) return -1;
    if (f->neg_head[L] < f->neg_end[L]) entry = f->neg_head[L]++;
    else entry = f->pos_head[L]++;
    if (fp_empty_at(f, L)) fp_setbit(f, L, 0);
    f->remaining--;
    return entry;
}

static int64_t fp_len_of(const fpool* f, int64_t entry) {
    /* binary search the CSR for the entry's length */
    int64_t lo = 0, hi = f->maxlen;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        if (f->start[mid] <= entry) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

static void greedy_fill(plist* packs, svec* pools, int32_t n_pools) {
    fpool* fp = (fpool*)xcalloc((size_t)(n_pools > 0 ? n_pools : 1), sizeof(fpool));
    unsigned char** consumed = (unsigned char**)xcalloc((size_t)(n_pools > 0 ? n_pools : 1), sizeof(void*));
    for (int32_t j = 0; j < n_pools; ++j) {
        fp_build(&fp[j], &pools[j]);
        consumed[j] = (unsigned char*)xcalloc((size_t)(pools[j].n + 1), 1);
    }
    for (int64_t p = 0; p < packs->n; ++p) {
        pack* pk = &packs->v[p];
        for (int32_t j = n_pools - 1; j >= 0; --j) { /* nearest smaller group first */
            int64_t residual = pack_residual(pk);
            while (residual > 0 && fp[j].remaining > 0) {
                const int64_t entry = fp_take(&fp[j], residual);
                if (entry < 0) break;
                sample s = {fp[j].ids[entry], fp_len_of(&fp[j], entry)};
                pack_add(pk, s);
                residual = pack_residual(pk);
                consumed[j][fp[j].pos_of[entry]] = 1;
            }
        }
    }
    for (int32_t j = 0; j < n_pools; ++j) {
        int64_t m = 0;
        for (int64_t k = 0; k < pools[j].n; ++k)
            if (!consumed[j][k]) pools[j].v[m++] = pools[j].v[k];
        pools[j].n = m;
        fp_free(&fp[j]);
        free(consumed[j]);
    }
    free(fp);
    free(consumed);
}

/* ------------------------------------------------------------------------ */
/* batching: balance.cpp:105-205                                              */
/* ------------------------------------------------------------------------ */

static void chunk_packs(pack* ordered, int64_t np, int32_t device_count, int32_t group_index, int sp_comm,
                        int64_t capacity, ilist* out) {
    const int64_t n = device_count;
    int64_t i = 0;
    for (; i + n <= np; i += n) {
        iteration it;
        it.group_index = group_index;
        it.n_devices = device_count;
        it.devices = (dbatch*)xcalloc((size_t)n, sizeof(dbatch));
        for (int64_t d = 0; d < n; ++d) {
            plist one;
            memset(&one, 0, sizeof one);
            pl_push(&one, ordered[i + d]);
            it.devices[d] = dbatch_build((int32_t)d, one, sp_comm);
        }
        il_push(out, it);
    }
    if (i == np) return;

    /* final partial run: redistribute the samples (balance.cpp:121-151) */
    svec spill;
    memset(&spill, 0, sizeof spill);
    for (int64_t k = i; k < np; ++k)
        for (int64_t m = 0; m < ordered[k].samples.n; ++m) sv_push(&spill, ordered[k].samples.v[m]);
    qsort(spill.v, (size_t)spill.n, sizeof(sample), cmp_decreasing);
    pack* batches = (pack*)xcalloc((size_t)n, sizeof(pack));
    for (int64_t d = 0; d < n; ++d) batches[d] = pack_make(capacity);
    int ok = 1;
    for (int64_t k = 0; k < spill.n; ++k) {
        int64_t target = n;
        int64_t best_attention = 0;
        for (int64_t d = 0; d < n; ++d) {
            if (pack_residual(&batches[d]) < spill.v[k].length) continue;
            if (target == n || batches[d].attention < best_attention) {
                target = d;
                best_attention = batches[d].attention;
            }
        }
        if (target == n) {
            ok = 0;
            break;
        }
        pack_add(&batches[target], spill.v[k]);
    }
    sv_free(&spill);

    iteration it;
    it.group_index = group_index;
    it.n_devices = device_count;
    it.devices = (dbatch*)xcalloc((size_t)n, sizeof(dbatch));
    if (ok) {
        for (int64_t d = 0; d < n; ++d) {
            batches[d].capacity = batches[d].total; /* unpadded */
            plist ps;
            memset(&ps, 0, sizeof ps);
            if (batches[d].samples.n) pl_push(&ps, batches[d]);
            else sv_free(&batches[d].samples);
            it.devices[d] = dbatch_build((int32_t)d, ps, sp_comm);
        }
        for (int64_t k = i; k < np; ++k) sv_free(&ordered[k].samples);
    } else {
        for (int64_t d = 0; d < n; ++d) sv_free(&batches[d].samples);
        for (int64_t d = 0; d < n; ++d) {
            plist ps;
            memset(&ps, 0, sizeof ps);
            if (i + d < np) pl_push(&ps, ordered[i + d]);
            it.devices[d] = dbatch_build((int32_t)d, ps, sp_comm);
        }
    }
    free(batches);
    il_push(out, it);
}

/* stable sort by attention descending (balance.cpp:185-189) */
static void stable_sort_attention(pack* v, int64_t n) {
    if (n < 2) return;
    pack* tmp = (pack*)xmalloc(sizeof(pack) * (size_t)n);
    for (int64_t width = 1; width < n; width *= 2) {
        for (int64_t lo = 0; lo < n; lo += 2 * width) {
            int64_t mid = lo + width < n ? lo + width : n;
            int64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
            int64_t a = lo, b = mid, k = lo;
            while (a < mid && b < hi) {
                if (v[b].attention > v[a].attention) tmp[k++] = v[b++];
                else tmp[k++] = v[a++];
            }
            while (a < mid) tmp[k++] = v[a++];
            while (b < hi) tmp[k++] = v[b++];
        }
        memcpy(v, tmp, sizeof(pack) * (size_t)n);
    }
    free(tmp);
}

/* takes ownership of packs */
static int batch_packs(plist* packs, int64_t capacity, int32_t device_count, int32_t group_index, int sp_comm,
                       int random, uint64_t seed, ilist* out, errbuf* e) {
    if (device_count < 1) return fail(e, EVAL, "device count must be >= 1");
    if (packs->n == 0) return OK;
    if (random) {
        rng r = rng_make(derive_seed_i(seed, "pack-batching", (uint64_t)group_index));
        rng_shuffle(&r, packs->v, packs->n, sizeof(pack));
    } else {
        stable_sort_attention(packs->v, packs->n);
    }
    chunk_packs(packs->v, packs->n, device_count, group_index, sp_comm, capacity, out);
    free(packs->v);
    packs->v = NULL;
    packs->n = packs->cap = 0;
    return OK;
}

/* ------------------------------------------------------------------------ */
/* build_plan: balance.cpp:207-258                                            */
/* ------------------------------------------------------------------------ */

static int build_plan(const sample* v, int64_t n, const hbp_groups* g, const hbp_plan_options* o, ilist* out,
                      errbuf* e) {
    int rc = validate_samples(v, n, e);
    if (rc) return rc;
    rc = validate_groups(g, e);
    if (rc) return rc;
    if (o->device_count < 1) return fail(e, EVAL, "device count must be >= 1");
    svec* pools = (svec*)xcalloc((size_t)g->count, sizeof(svec));
    rc = group_data(v, n, g, pools, e);
    for (int32_t gi = g->count - 1; rc == OK && gi >= 0; --gi) {
        if (pools[gi].n == 0) continue;
        svec mine = pools[gi];
        memset(&pools[gi], 0, sizeof(svec));
        plist packed;
        memset(&packed, 0, sizeof packed);
        rc = do_pack(mine.v, mine.n, g->groups[gi].length, &o->strategy,
                     derive_seed_i(o->seed, "pack", (uint64_t)gi), &packed, e);
        sv_free(&mine);
        if (rc) {
            pl_free(&packed);
            break;
        }
        if (o->greedy_fill && gi > 0) greedy_fill(&packed, pools, gi);
        rc = batch_packs(&packed, g->groups[gi].length, o->device_count, gi, g->groups[gi].sp > 1,
                         !o->balance_batching, o->seed, out, e);
        pl_free(&packed);
    }
    for (int32_t gi = 0; gi < g->count; ++gi) sv_free(&pools[gi]);
    free(pools);
    if (rc) return rc;
    rng r = rng_make(derive_seed(o->seed, "plan-shuffle"));
    rng_shuffle(&r, out->v, out->n, sizeof(iteration));
    return OK;
}

/* ------------------------------------------------------------------------ */
/* metrics: metrics.cpp:22-144                                                */
/* ------------------------------------------------------------------------ */

static int iter_dbr_abr(const hbp_plan_view* p, int64_t i, double* dbr, double* abr, errbuf* e) {
    const int64_t d0 = p->iter_dev_offsets[i], d1 = p->iter_dev_offsets[i + 1];
    if (d1 == d0) return fail(e, EVAL, "dbr: no devices");
    int64_t tmax = 0, amax = 0;
    for (int64_t d = d0; d < d1; ++d) {
        int64_t t = 0, a = 0;
        for (int64_t k = p->dev_pack_offsets[d]; k < p->dev_pack_offsets[d + 1]; ++k) {
            t += p->pack_total[k];
            a += p->pack_attention[k];
        }
        if (t > tmax) tmax = t;
        if (a > amax) amax = a;
    }
    if (tmax == 0) return fail(e, EVAL, "dbr undefined: all devices carry zero tokens");
    double gap = 0.0;
    for (int64_t d = d0; d < d1; ++d) {
        int64_t t = 0;
        for (int64_t k = p->dev_pack_offsets[d]; k < p->dev_pack_offsets[d + 1]; ++k) t += p->pack_total[k];
        gap += (double)(tmax - t);
    }
    *dbr = gap / ((double)tmax * (double)(d1 - d0));
    if (amax == 0) return fail(e, EVAL, "abr undefined: all devices carry zero attention");
    gap = 0.0;
    for (int64_t d = d0; d < d1; ++d) {
        int64_t a = 0;
        for (int64_t k = p->dev_pack_offsets[d]; k < p->dev_pack_offsets[d + 1]; ++k) a += p->pack_attention[k];
        gap += (double)(amax - a);
    }
    *abr = gap / ((double)amax * (double)(d1 - d0));
    return OK;
}

static int report(const hbp_plan_view* p, hbp_metrics* out, double* dbr_out, double* abr_out, errbuf* e) {
    if (p->n_iterations == 0) return fail(e, EVAL, "metrics report: empty plan");
    double comm = 0.0, total = 0.0, pad_gap = 0.0, pad_cap = 0.0;
    double* dbrs = (double*)xmalloc(sizeof(double) * (size_t)p->n_iterations);
    double* abrs = (double*)xmalloc(sizeof(double) * (size_t)p->n_iterations);
    for (int64_t i = 0; i < p->n_iterations; ++i) {
        int rc = iter_dbr_abr(p, i, &dbrs[i], &abrs[i], e);
        if (rc) {
            free(dbrs);
            free(abrs);
            return rc;
        }
        const int sp = p->groups.groups[p->iter_group[i]].sp > 1;
        for (int64_t d = p->iter_dev_offsets[i]; d < p->iter_dev_offsets[i + 1]; ++d) {
            int64_t t = 0;
            for (int64_t k = p->dev_pack_offsets[d]; k < p->dev_pack_offsets[d + 1]; ++k) t += p->pack_total[k];
            comm += (double)(sp ? t : 0);
            total += (double)t;
            for (int64_t k = p->dev_pack_offsets[d]; k < p->dev_pack_offsets[d + 1]; ++k) {
                pad_gap += (double)(p->pack_capacity[k] - p->pack_total[k]);
                pad_cap += (double)p->pack_capacity[k];
            }
        }
    }
    double ds = 0.0, as = 0.0;
    for (int64_t i = 0; i < p->n_iterations; ++i) {
        ds += dbrs[i];
        as += abrs[i];
        if (dbr_out) dbr_out[i] = dbrs[i];
        if (abr_out) abr_out[i] = abrs[i];
    }
    const double ni = (double)p->n_iterations;
    out->dbr = ds / ni;
    out->abr = as / ni;
    out->cr = total > 0.0 ? comm / total : 0.0;
    out->pr = pad_cap > 0.0 ? pad_gap / pad_cap : 0.0;
    out->ave_t = total / (ni * (double)p->device_count);
    free(dbrs);
    free(abrs);
    return OK;
}

/* ------------------------------------------------------------------------ */
/* cost model: costmodel.cpp:14-104                                           */
/* ------------------------------------------------------------------------ */

static int profile_validate(const hbp_hardware_profile* p, errbuf* e) { /* costmodel.cpp:14-35 */
    if (p->per_token_linear_cost < 0 || p->per_token2_attention_cost < 0 || p->sp_comm_cost < 0 ||
        p->gc_recompute_factor < 0 || p->fixed_iteration_cost < 0)
        return fail(e, EVAL, "profile costs must be >= 0");
    if (p->layer_count < 1) return fail(e, EVAL, "layer_count must be >= 1");
    if (p->device_memory <= p->base_memory) return fail(e, EVAL, "device_memory must exceed base_memory");
    if (p->per_token_activation_memory < 0 || p->gc_memory_saving_per_layer < 0)
        return fail(e, EVAL, "memory constants must be >= 0");
    if (p->reference_length < 1) return fail(e, EVAL, "reference_length must be >= 1");
    if (p->gc_memory_saving_per_layer > p->per_token_activation_memory * (double)p->reference_length)
        return fail(e, EVAL, "gc_memory_saving_per_layer exceeds per-layer activation memory");
    return OK;
}

static int memory_used(int64_t l, int32_t sp, int32_t ckpt, const hbp_hardware_profile* p, int64_t* out,
                       errbuf* e) { /* costmodel.cpp:37-53 */
    if (sp < 1) return fail(e, EVAL, "sp must be >= 1");
    if (ckpt < 0 || ckpt > p->layer_count) return fail(e, EVAL, "ckpt must lie in [0, layer_count]");
    const double shard = (double)l / (double)sp;
    const double activations = p->per_token_activation_memory * shard * (double)p->layer_count;
    const double saved = p->gc_memory_saving_per_layer * (double)ckpt * shard / (double)p->reference_length;
    *out = p->base_memory + (int64_t)ceil(activations - saved);
    return OK;
}

typedef struct dwork { /* costmodel.hpp:56-61 */
    int64_t padded, real, attention, max_cap;
} dwork;

static int iter_time_work(const dwork* w, int32_t sp, int32_t ckpt, const hbp_hardware_profile* p, double* out,
                          errbuf* e) { /* costmodel.cpp:69-99 */
    int rc = profile_validate(p, e);
    if (rc) return rc;
    if (w->padded == 0) {
        *out = 0.0;
        return OK;
    }
    int64_t used;
    rc = memory_used(w->max_cap, sp, ckpt, p, &used, e);
    if (rc) return rc;
    if (used > p->device_memory)
        return fail(e, EINF, "configuration sp=%d ckpt=%d at length %lld requires %lld bytes, %lld available", sp,
                    ckpt, (long long)w->max_cap, (long long)used, (long long)p->device_memory);
    const double tokens = (double)w->padded;
    const double compute =
        p->per_token_linear_cost * tokens + p->per_token2_attention_cost * (double)w->attention / (double)sp;
    const double recompute = p->gc_recompute_factor * (double)ckpt / (double)p->layer_count * compute;
    const double comm = sp > 1 ? p->sp_comm_cost * tokens * (double)(sp - 1) : 0.0;
    *out = compute + recompute + comm + p->fixed_iteration_cost;
    return OK;
}

static dwork device_work(const int64_t* cap, const int64_t* tot, const int64_t* att, int64_t a, int64_t b) {
    dwork w = {0, 0, 0, 0}; /* costmodel.cpp:55-67 */
    for (int64_t k = a; k < b; ++k) {
        w.padded += cap[k];
        w.real += tot[k];
        w.attention += att[k];
        const int64_t pad = cap[k] - tot[k];
        w.attention += pad * pad;
        if (cap[k] > w.max_cap) w.max_cap = cap[k];
    }
    return w;
}

static int simulate(const hbp_plan_view* p, const hbp_hardware_profile* prof, hbp_sim_totals* out, double* iter_s,
                    double* dcomp, double* dcomm, double* didle, errbuf* e) { /* sim.cpp:9-60 */
    int rc = profile_validate(prof, e);
    if (rc) return rc;
    if (p->n_iterations == 0) return fail(e, EVAL, "simulate: empty plan");
    rc = report(p, &out->metrics, NULL, NULL, e);
    if (rc) return rc;
    out->device_count = p->device_count;
    int32_t switches = 0; /* schedule.cpp:67-79 */
    for (int64_t i = 1; i < p->n_iterations; ++i) {
        const hbp_group_config* a = &p->groups.groups[p->iter_group[i]];
        const hbp_group_config* b = &p->groups.groups[p->iter_group[i - 1]];
        if (a->sp != b->sp || a->ckpt != b->ckpt) ++switches;
    }
    out->switch_count = switches;
    double total = 0.0;
    for (int64_t i = 0; i < p->n_iterations; ++i) {
        const hbp_group_config* c = &p->groups.groups[p->iter_group[i]];
        double imax = 0.0;
        const int64_t d0 = p->iter_dev_offsets[i], d1 = p->iter_dev_offsets[i + 1];
        for (int64_t d = d0; d < d1; ++d) {
            const dwork w = device_work(p->pack_capacity, p->pack_total, p->pack_attention, p->dev_pack_offsets[d],
                                        p->dev_pack_offsets[d + 1]);
            double busy = 0.0;
            char inner[512];
            errbuf ie = {inner, sizeof inner};
            rc = iter_time_work(&w, c->sp, c->ckpt, prof, &busy, &ie);
            if (rc == EINF) return fail(e, EINF, "iteration %lld: %s", (long long)i, inner);
            if (rc) return fail(e, rc, "%s", inner);
            const double comm = c->sp > 1 ? prof->sp_comm_cost * (double)w.padded * (double)(c->sp - 1) : 0.0;
            if (dcomm) dcomm[d] = comm;
            if (dcomp) dcomp[d] = busy - comm;
            if (busy > imax) imax = busy;
        }
        for (int64_t d = d0; d < d1 && didle; ++d) didle[d] = imax - ((dcomp ? dcomp[d] : 0) + (dcomm ? dcomm[d] : 0));
        if (iter_s) iter_s[i] = imax;
        total += imax;
    }
    out->total_seconds = total;
    out->gpu_days = total * (double)p->device_count / 86400.0;
    return OK;
}

/* ------------------------------------------------------------------------ */
/* profilers: costmodel.cpp:110-325                                           */
/* ------------------------------------------------------------------------ */

static const hbp_profile_row* table_find(const hbp_profiler* pr, int64_t l, int32_t sp) {
    for (int64_t i = 0; i < pr->n_rows; ++i)
        if (pr->rows[i].length == l && pr->rows[i].sp == sp) return &pr->rows[i];
    return NULL;
}

static int profiler_check(const hbp_profiler* pr, int32_t* cmin, int32_t* cmax, errbuf* e) {
    if (pr->kind == HBP_PROFILER_ANALYTIC) { /* costmodel.cpp:110-121 */
        int rc = profile_validate(&pr->profile, e);
        if (rc) return rc;
        *cmin = pr->ckpt_min;
        *cmax = pr->ckpt_max < 0 ? pr->profile.layer_count : pr->ckpt_max;
        if (*cmin < 0 || *cmin >= *cmax || *cmax > pr->profile.layer_count)
            return fail(e, EVAL, "ckpt probe bounds must satisfy 0 <= ckpt_min < ckpt_max <= layer_count");
        return OK;
    }
    for (int64_t i = 0; i < pr->n_rows; ++i) /* costmodel.cpp:144-156 */
        for (int64_t j = 0; j < i; ++j)
            if (pr->rows[i].length == pr->rows[j].length && pr->rows[i].sp == pr->rows[j].sp)
                return fail(e, EVAL, "duplicate profile row for length %lld, sp %d", (long long)pr->rows[i].length,
                            pr->rows[i].sp);
    return OK;
}

static int p_time(const hbp_profiler* pr, int64_t l, int32_t sp, int32_t ckpt, double* out, errbuf* e) {
    if (pr->kind == HBP_PROFILER_ANALYTIC) { /* costmodel.cpp:123-129 */
        dwork w = {l, l, l * l, l};
        return iter_time_work(&w, sp, ckpt, &pr->profile, out, e);
    }
    const hbp_profile_row* r = table_find(pr, l, sp); /* costmodel.cpp:223-240 */
    if (!r) return fail(e, EINF, "no profile row for length %lld, sp %d", (long long)l, sp);
    if (r->oom)
        return fail(e, EINF, "profiled configuration is out of memory at length %lld, sp %d", (long long)l, sp);
    if (r->ckpt != ckpt)
        return fail(e, EINF, "no profile row for length %lld, sp %d, ckpt %d", (long long)l, sp, ckpt);
    *out = r->seconds;
    return OK;
}

static int p_memory(const hbp_profiler* pr, int64_t l, int32_t sp, int32_t ckpt, int64_t* out, errbuf* e) {
    if (pr->kind == HBP_PROFILER_ANALYTIC) { /* costmodel.cpp:131-134 */
        int64_t used;
        int rc = memory_used(l, sp, ckpt, &pr->profile, &used, e);
        if (rc) return rc;
        *out = pr->profile.device_memory - used;
        return OK;
    }
    const hbp_profile_row* r = table_find(pr, l, sp); /* costmodel.cpp:242-251 */
    if (!r) return fail(e, EINF, "no profile row for length %lld, sp %d", (long long)l, sp);
    *out = r->oom ? -1 : pr->device_memory - r->memory_bytes;
    return OK;
}

static int greedy_ckpt(const hbp_profiler* pr, int64_t l, int32_t sp, int32_t cmin, int32_t cmax, int32_t* out,
                       errbuf* e) { /* costmodel.cpp:271-292 */
    if (cmin >= cmax) return fail(e, EVAL, "greedy_profile_ckpt: ckpt_min must be < ckpt_max");
    int64_t a, b;
    int rc = p_memory(pr, l, sp, cmin, &a, e);
    if (rc) return rc;
    rc = p_memory(pr, l, sp, cmax, &b, e);
    if (rc) return rc;
    const double m1r = (double)a, m2r = (double)b;
    const double m_ave = (m2r - m1r) / (double)(cmax - cmin);
    if (m_ave <= 0.0)
        return fail(e, EINF, "GC does not reduce memory under this profile (slope %f bytes/layer)", m_ave);
    const double c_o = (double)cmax - m2r / m_ave;
    int32_t rounded = (int32_t)ceil(c_o);
    if (rounded < 0) rounded = 0;
    if (rounded > cmax) rounded = cmax;
    *out = rounded;
    return OK;
}

static int p_ckpt(const hbp_profiler* pr, int64_t l, int32_t sp, int32_t* out, errbuf* e) {
    if (pr->kind == HBP_PROFILER_ANALYTIC) { /* costmodel.cpp:136-138 */
        int32_t cmin, cmax;
        int rc = profiler_check(pr, &cmin, &cmax, e);
        if (rc) return rc;
        return greedy_ckpt(pr, l, sp, cmin, cmax, out, e);
    }
    const hbp_profile_row* r = table_find(pr, l, sp); /* costmodel.cpp:253-265 */
    if (!r) return fail(e, EINF, "no profile row for length %lld, sp %d", (long long)l, sp);
    if (r->oom)
        return fail(e, EINF, "profiled configuration is out of memory at length %lld, sp %d", (long long)l, sp);
    *out = r->ckpt;
    return OK;
}

/* Appends to a growing failure string like the reference's std::string. */
typedef struct sbuf {
    char* s;
    size_t n, cap;
} sbuf;
static void sb_add(sbuf* b, const char* t) {
    size_t k = strlen(t);
    if (b->n + k + 1 > b->cap) {
        b->cap = (b->n + k + 1) * 2;
        b->s = (char*)xrealloc(b->s, b->cap);
    }
    memcpy(b->s + b->n, t, k + 1);
    b->n += k;
}

static int best_sp_ckpt(const hbp_profiler* pr, int64_t l, const int32_t* sps, int32_t nsp, int32_t* osp,
                        int32_t* ockpt, double* osec, errbuf* e) { /* costmodel.cpp:294-325 */
    if (nsp < 1) return fail(e, EVAL, "find_best_sp_ckpt: no sp candidates");
    int have = 0;
    sbuf failures = {NULL, 0, 0};
    sb_add(&failures, "");
    for (int32_t k = 0; k < nsp; ++k) {
        const int32_t sp = sps[k];
        char msg[1024];
        errbuf ie = {msg, sizeof msg};
        int32_t ckpt = 0;
        int rc = p_ckpt(pr, l, sp, &ckpt, &ie);
        int64_t mem = 0;
        if (!rc) rc = p_memory(pr, l, sp, ckpt, &mem, &ie);
        if (!rc && mem < 0) rc = fail(&ie, EINF, "sp=%d does not fit device memory even at ckpt %d", sp, ckpt);
        double sec = 0.0;
        if (!rc) rc = p_time(pr, l, sp, ckpt, &sec, &ie);
        if (rc) {
            char head[64];
            if (failures.n) sb_add(&failures, "; ");
            snprintf(head, sizeof head, "sp=%d: ", sp);
            sb_add(&failures, head);
            sb_add(&failures, msg);
            continue;
        }
        if (!have || sec < *osec) {
            have = 1;
            *osp = sp;
            *ockpt = ckpt;
            *osec = sec;
        }
    }
    int rc = OK;
    if (!have) rc = fail(e, EINF, "no feasible (sp, ckpt) for length %lld: %s", (long long)l, failures.s);
    free(failures.s);
    return rc;
}

static int is_pow2(int32_t v) { return v > 0 && (v & (v - 1)) == 0; }

static int nearest_sp(double target, int64_t length, const hbp_profiler* pr, const int32_t* sps, int32_t nsp,
                      int32_t* out_sp, int32_t* out_ckpt, errbuf* e) { /* autoselect.cpp:41-72 */
    int32_t best_sp = -1, best_ckpt = 0;
    double best_gap = 0.0;
    for (int32_t k = 0; k < nsp; ++k) {
        const int32_t sp = sps[k];
        if (!is_pow2(sp)) continue;
        char msg[1024];
        errbuf ie = {msg, sizeof msg};
        int32_t ckpt;
        if (p_ckpt(pr, length, sp, &ckpt, &ie)) continue;
        int64_t mem;
        if (p_memory(pr, length, sp, ckpt, &mem, &ie)) continue;
        if (mem < 0) continue;
        const double gap = fabs(log2((double)sp) - log2(target));
        if (best_sp < 0 || gap < best_gap || (gap == best_gap && sp < best_sp)) {
            best_sp = sp;
            best_gap = gap;
            best_ckpt = ckpt;
        }
    }
    if (best_sp < 0) return fail(e, EINF, "no feasible sp for mid-level group of length %lld", (long long)length);
    *out_sp = best_sp;
    *out_ckpt = best_ckpt;
    return OK;
}

static int select_groups(const int64_t* lengths, int32_t nl, const hbp_profiler* pr, const int32_t* sps,
                         int32_t nsp, hbp_group_config* out, int32_t* out_n, int64_t* l_best_out,
                         int64_t* l_max_out, errbuf* e) { /* autoselect.cpp:76-168 */
    if (nl < 1) return fail(e, EVAL, "select_groups: no candidate lengths");
    for (int32_t i = 1; i < nl; ++i)
        if (lengths[i] <= lengths[i - 1]) return fail(e, EVAL, "candidate lengths must be strictly ascending");
    for (int32_t k = 0; k < nsp; ++k)
        if (!is_pow2(sps[k])) return fail(e, EVAL, "sp candidates must be powers of two, got %d", sps[k]);
    int64_t* pl = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)nl);
    int32_t* psp = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)nl);
    int32_t* pck = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)nl);
    double* psec = (double*)xmalloc(sizeof(double) * (size_t)nl);
    int32_t np = 0;
    sbuf failures = {NULL, 0, 0};
    sb_add(&failures, "");
    for (int32_t i = 0; i < nl; ++i) {
        char msg[4096];
        errbuf ie = {msg, sizeof msg};
        if (best_sp_ckpt(pr, lengths[i], sps, nsp, &psp[np], &pck[np], &psec[np], &ie)) {
            if (failures.n) sb_add(&failures, "; ");
            sb_add(&failures, msg);
            continue;
        }
        pl[np++] = lengths[i];
    }
    int rc = OK;
    if (np == 0) {
        rc = fail(e, EINF, "no candidate length is feasible: %s", failures.s);
    } else if (pl[np - 1] != lengths[nl - 1]) {
        rc = fail(e, EINF, "largest candidate length %lld is infeasible: %s", (long long)lengths[nl - 1],
                  failures.s);
    }
    if (rc == OK) {
        int32_t bi = 0;
        for (int32_t i = 1; i < np; ++i)
            if (psec[i] < psec[bi]) bi = i;
        const int64_t l_best = pl[bi], l_max = pl[np - 1];
        const int32_t s_best = psp[bi], c_best = pck[bi], s_max = psp[np - 1], c_max = pck[np - 1];
        const int64_t l1 = l_best / s_best;
        const int64_t l2 = l_max / s_max;
        hbp_group_config raw[4];
        int32_t nraw = 0;
        int32_t c1;
        rc = p_ckpt(pr, l1, 1, &c1, e);
        if (rc == OK) {
            raw[nraw++] = (hbp_group_config){l1, 1, c1};
            raw[nraw++] = (hbp_group_config){l_best, s_best, c_best};
            if (l2 > l_best) {
                int32_t sp2 = 1, c2 = 0;
                rc = nearest_sp((double)l2 / (double)l1, l2, pr, sps, nsp, &sp2, &c2, e);
                if (rc == OK) raw[nraw++] = (hbp_group_config){l2, sp2, c2};
            }
        }
        if (rc == OK) {
            raw[nraw++] = (hbp_group_config){l_max, s_max, c_max};
            /* dedup by length keeping the lower sp; ascending (std::map) */
            hbp_group_config ded[4];
            int32_t nd = 0;
            for (int32_t k = 0; k < nraw; ++k) {
                int32_t f = -1;
                for (int32_t q = 0; q < nd; ++q)
                    if (ded[q].length == raw[k].length) f = q;
                if (f < 0) ded[nd++] = raw[k];
                else if (raw[k].sp < ded[f].sp) ded[f] = raw[k];
            }
            for (int32_t a = 1; a < nd; ++a)
                for (int32_t b = a; b > 0 && ded[b].length < ded[b - 1].length; --b) {
                    hbp_group_config t = ded[b];
                    ded[b] = ded[b - 1];
                    ded[b - 1] = t;
                }
            hbp_groups g = {ded, nd, l_best, l_max};
            rc = validate_groups(&g, e);
            if (rc == OK) {
                memcpy(out, ded, sizeof(hbp_group_config) * (size_t)nd);
                *out_n = nd;
                *l_best_out = l_best;
                *l_max_out = l_max;
            }
        }
    }
    free(failures.s);
    free(pl);
    free(psp);
    free(pck);
    free(psec);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* synthetic corpora: ingest.cpp:188-329                                      */
/* ------------------------------------------------------------------------ */

typedef struct dist {
    int family; /* 0 constant 1 uniform 2 normal 3 lognormal */
    double a, b;
} dist;

static int parse_dist(const char* text, dist* d, errbuf* e) { /* ingest.cpp:207-244 */
    char buf[256];
    snprintf(buf, sizeof buf, "%s", text);
    /* split on ':' like std::getline (empty fields kept, no trailing one) */
    char* parts[8];
    int np = 0;
    if (buf[0]) {
        char* t = buf;
        for (;;) {
            char* c = strchr(t, ':');
            if (np < 8) parts[np++] = t;
            if (!c) break;
            *c = '\0';
            t = c + 1;
            if (!*t) break;
        }
    }
    if (np == 0) return fail(e, EVAL, "empty distribution spec");
    int want;
    if (!strcmp(parts[0], "constant")) d->family = 0, want = 2;
    else if (!strcmp(parts[0], "uniform")) d->family = 1, want = 3;
    else if (!strcmp(parts[0], "normal")) d->family = 2, want = 3;
    else if (!strcmp(parts[0], "lognormal")) d->family = 3, want = 3;
    else return fail(e, EVAL, "unknown distribution family: %s", parts[0]);
    if (np != want) {
        static const char* names[] = {"constant needs 1 parameter", "uniform needs 2 parameters",
                                      "normal needs 2 parameters", "lognormal needs 2 parameters"};
        return fail(e, EVAL, "%s", names[d->family]);
    }
    char* end;
    d->a = strtod(parts[1], &end);
    if (end == parts[1]) return fail(e, EVAL, "bad distribution parameter in '%s'", text);
    d->b = 0.0;
    if (want == 3) {
        d->b = strtod(parts[2], &end);
        if (end == parts[2]) return fail(e, EVAL, "bad distribution parameter in '%s'", text);
    }
    switch (d->family) { /* ingest.cpp:188-205 */
        case 0:
            if (d->a < 1.0) return fail(e, EVAL, "constant length must be >= 1");
            break;
        case 1:
            if (d->a < 1.0 || d->b < d->a) return fail(e, EVAL, "uniform bounds must satisfy 1 <= low <= high");
            break;
        case 2:
            if (d->b < 0.0) return fail(e, EVAL, "normal stddev must be >= 0");
            break;
        default:
            if (d->b < 0.0) return fail(e, EVAL, "lognormal sigma must be >= 0");
    }
    return OK;
}

static int64_t draw_length(const dist* d, rng* r, int64_t max_length) { /* ingest.cpp:279-300 */
    double v = 1.0;
    switch (d->family) {
        case 0:
            v = d->a;
            break;
        case 1:
            v = (double)rng_uniform(r, (int64_t)d->a, (int64_t)d->b);
            break;
        case 2:
            v = d->a + d->b * rng_normal(r);
            break;
        default:
            v = exp(d->a + d->b * rng_normal(r));
    }
    int64_t len = (int64_t)llround(v);
    if (len < 1) len = 1;
    if (len > max_length) len = max_length;
    return len;
}

/* ------------------------------------------------------------------------ */
/* exported ABI                                                               */
/* ------------------------------------------------------------------------ */

void oracle_plan_free(oracle_plan* p) {
    if (!p) return;
    free(p->iter_group);
    free(p->iter_dev_offsets);
    free(p->dev_index);
    free(p->dev_pack_offsets);
    free(p->pack_capacity);
    free(p->pack_total);
    free(p->pack_attention);
    free(p->pack_member_offsets);
    free(p->member_id);
    free(p->member_length);
    free(p);
}

int oracle_kind(void) { return 1; }

int oracle_synth_lengths(int64_t count, const char* short_dist, double long_fraction, const char* long_dist,
                         int64_t max_length, uint64_t seed, int64_t* lengths, char* err, int errlen) {
    errbuf e = {err, errlen};
    dist sd, ld;
    int rc = parse_dist(short_dist, &sd, &e);
    if (rc) return rc;
    if (long_dist && long_dist[0]) {
        rc = parse_dist(long_dist, &ld, &e);
        if (rc) return rc;
    } else {
        ld = sd;
    }
    if (count < 1) return fail(&e, EVAL, "synth count must be >= 1"); /* ingest.cpp:267-275 */
    if (long_fraction < 0.0 || long_fraction > 1.0) return fail(&e, EVAL, "long_fraction must lie in [0, 1]");
    if (max_length < 1) return fail(&e, EVAL, "max_length must be >= 1");
    const int64_t long_count = (int64_t)llround((double)count * long_fraction);
    const int64_t short_count = count - long_count;
    rng rs = rng_make(derive_seed(seed, "synth-short"));
    rng rl = rng_make(derive_seed(seed, "synth-long"));
    for (int64_t i = 0; i < short_count; ++i) lengths[i] = draw_length(&sd, &rs, max_length);
    for (int64_t i = 0; i < long_count; ++i) lengths[short_count + i] = draw_length(&ld, &rl, max_length);
    return OK;
}

int oracle_shuffle_positions(uint64_t seed, int64_t m, uint32_t* out) {
    for (int64_t i = 0; i < m; ++i) out[i] = (uint32_t)i;
    rng r = rng_make(seed);
    rng_shuffle(&r, out, m, sizeof(uint32_t));
    return OK;
}

int oracle_validate(const int64_t* ids, const int64_t* lengths, int64_t n, char* err, int errlen) {
    errbuf e = {err, errlen};
    sample* v = make_samples(ids, lengths, n);
    int rc = validate_samples(v, n, &e);
    free(v);
    return rc;
}

int oracle_fingerprint(const int64_t* ids, const int64_t* lengths, int64_t n, uint64_t* hash, int64_t* count,
                       int64_t* tokens) { /* types.cpp:52-72 */
    sample* v = make_samples(ids, lengths, n);
    qsort(v, (size_t)n, sizeof(sample), cmp_by_id);
    uint64_t h = 0xcbf29ce484222325ULL;
    int64_t t = 0;
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t vals[2] = {(uint64_t)v[i].id, (uint64_t)v[i].length};
        for (int q = 0; q < 2; ++q)
            for (int b = 0; b < 8; ++b) {
                h ^= (vals[q] >> (8 * b)) & 0xffu;
                h *= 0x100000001b3ULL;
            }
        t += v[i].length;
    }
    *hash = h;
    *count = n;
    *tokens = t;
    free(v);
    return OK;
}

int oracle_group_data(const int64_t* ids, const int64_t* lengths, int64_t n, const hbp_groups* groups,
                      oracle_plan** out, char* err, int errlen) {
    errbuf e = {err, errlen};
    sample* v = make_samples(ids, lengths, n);
    int rc = validate_groups(groups, &e);
    svec* parts = NULL;
    if (rc == OK) {
        parts = (svec*)xcalloc((size_t)groups->count, sizeof(svec));
        rc = group_data(v, n, groups, parts, &e);
    }
    if (rc == OK) {
        flat f;
        flat_init(&f);
        for (int32_t g = 0; g < groups->count; ++g) {
            pack p = pack_make(groups->groups[g].length);
            for (int64_t k = 0; k < parts[g].n; ++k) pack_add(&p, parts[g].v[k]);
            flat_pack(&f, &p);
            sv_free(&p.samples);
        }
        *out = flat_finish(&f, 0, 0);
    }
    if (parts)
        for (int32_t g = 0; g < groups->count; ++g) sv_free(&parts[g]);
    free(parts);
    free(v);
    return rc;
}

int oracle_pack(const int64_t* ids, const int64_t* lengths, int64_t n, int64_t capacity, const hbp_strategy* strategy,
                uint64_t seed, oracle_plan** out, char* err, int errlen) {
    errbuf e = {err, errlen};
    sample* v = make_samples(ids, lengths, n);
    plist packs;
    memset(&packs, 0, sizeof packs);
    int rc = do_pack(v, n, capacity, strategy, seed, &packs, &e);
    if (rc == OK) {
        flat f;
        flat_init(&f);
        for (int64_t p = 0; p < packs.n; ++p) flat_pack(&f, &packs.v[p]);
        *out = flat_finish(&f, 0, seed);
    }
    pl_free(&packs);
    free(v);
    return rc;
}

int oracle_greedy_fill(const oracle_plan* packs, const oracle_plan* pools, oracle_plan** out_packs,
                       oracle_plan** out_pools, char* err, int errlen) {
    (void)err;
    (void)errlen;
    plist l = plist_from_flat(packs);
    const int32_t np = (int32_t)pools->n_packs;
    svec* ps = (svec*)xcalloc((size_t)(np > 0 ? np : 1), sizeof(svec));
    for (int32_t j = 0; j < np; ++j)
        for (int64_t k = pools->pack_member_offsets[j]; k < pools->pack_member_offsets[j + 1]; ++k) {
            sample s = {pools->member_id[k], pools->member_length[k]};
            sv_push(&ps[j], s);
        }
    greedy_fill(&l, ps, np);
    flat a;
    flat_init(&a);
    for (int64_t p = 0; p < l.n; ++p) flat_pack(&a, &l.v[p]);
    *out_packs = flat_finish(&a, 0, 0);
    flat b;
    flat_init(&b);
    for (int32_t j = 0; j < np; ++j) {
        pack p = pack_make(pools->pack_capacity[j]);
        for (int64_t k = 0; k < ps[j].n; ++k) pack_add(&p, ps[j].v[k]);
        flat_pack(&b, &p);
        sv_free(&p.samples);
        sv_free(&ps[j]);
    }
    *out_pools = flat_finish(&b, 0, 0);
    free(ps);
    pl_free(&l);
    return OK;
}

int oracle_balance_batching(const oracle_plan* packs, int32_t device_count, int32_t group_index, int32_t sp_comm,
                            int32_t random_batching, uint64_t seed, oracle_plan** out, char* err, int errlen) {
    errbuf e = {err, errlen};
    plist l = plist_from_flat(packs);
    ilist its;
    memset(&its, 0, sizeof its);
    const int64_t capacity = packs->n_packs > 0 ? packs->pack_capacity[0] : 0;
    int rc = batch_packs(&l, capacity, device_count, group_index, sp_comm, random_batching, seed, &its, &e);
    if (rc == OK) {
        flat f;
        flat_init(&f);
        for (int64_t i = 0; i < its.n; ++i) flat_iteration(&f, &its.v[i]);
        *out = flat_finish(&f, device_count, seed);
    }
    pl_free(&l);
    il_free(&its);
    return rc;
}

int oracle_build_plan(const int64_t* ids, const int64_t* lengths, int64_t n, const hbp_groups* groups,
                      const hbp_plan_options* options, oracle_plan** out, char* err, int errlen) {
    errbuf e = {err, errlen};
    sample* v = make_samples(ids, lengths, n);
    ilist its;
    memset(&its, 0, sizeof its);
    int rc = build_plan(v, n, groups, options, &its, &e);
    if (rc == OK) {
        flat f;
        flat_init(&f);
        for (int64_t i = 0; i < its.n; ++i) flat_iteration(&f, &its.v[i]);
        *out = flat_finish(&f, options->device_count, options->seed);
    }
    il_free(&its);
    free(v);
    return rc;
}

int oracle_report(const hbp_plan_view* plan, hbp_metrics* out, double* dbr, double* abr, char* err, int errlen) {
    errbuf e = {err, errlen};
    return report(plan, out, dbr, abr, &e);
}

int oracle_simulate(const hbp_plan_view* plan, const hbp_hardware_profile* profile, hbp_sim_totals* out,
                    double* iteration_seconds, double* device_compute, double* device_comm, double* device_idle,
                    char* err, int errlen) {
    errbuf e = {err, errlen};
    return simulate(plan, profile, out, iteration_seconds, device_compute, device_comm, device_idle, &e);
}

int oracle_memory_used(int64_t length, int32_t sp, int32_t ckpt, const hbp_hardware_profile* profile, int64_t* out,
                       char* err, int errlen) {
    errbuf e = {err, errlen};
    return memory_used(length, sp, ckpt, profile, out, &e);
}

int oracle_iter_time(const int64_t* capacity, const int64_t* total, const int64_t* attention, int64_t n_packs,
                     int32_t sp, int32_t ckpt, const hbp_hardware_profile* profile, double* out, char* err,
                     int errlen) {
    errbuf e = {err, errlen};
    const dwork w = device_work(capacity, total, attention, 0, n_packs);
    return iter_time_work(&w, sp, ckpt, profile, out, &e);
}

int oracle_profile_time(const hbp_profiler* profiler, int64_t length, int32_t sp, int32_t ckpt, double* out,
                        char* err, int errlen) {
    errbuf e = {err, errlen};
    int32_t a, b;
    int rc = profiler_check(profiler, &a, &b, &e);
    return rc ? rc : p_time(profiler, length, sp, ckpt, out, &e);
}

int oracle_profile_memory(const hbp_profiler* profiler, int64_t length, int32_t sp, int32_t ckpt, int64_t* out,
                          char* err, int errlen) {
    errbuf e = {err, errlen};
    int32_t a, b;
    int rc = profiler_check(profiler, &a, &b, &e);
    return rc ? rc : p_memory(profiler, length, sp, ckpt, out, &e);
}

int oracle_derive_ckpt(const hbp_profiler* profiler, int64_t length, int32_t sp, int32_t* out, char* err,
                       int errlen) {
    errbuf e = {err, errlen};
    int32_t a, b;
    int rc = profiler_check(profiler, &a, &b, &e);
    return rc ? rc : p_ckpt(profiler, length, sp, out, &e);
}

int oracle_greedy_profile_ckpt(const hbp_profiler* profiler, int64_t length, int32_t sp, int32_t ckpt_min,
                               int32_t ckpt_max, int32_t* out, char* err, int errlen) {
    errbuf e = {err, errlen};
    int32_t a, b;
    int rc = profiler_check(profiler, &a, &b, &e);
    return rc ? rc : greedy_ckpt(profiler, length, sp, ckpt_min, ckpt_max, out, &e);
}

int oracle_find_best_sp_ckpt(const hbp_profiler* profiler, int64_t length, const int32_t* sp, int32_t n_sp,
                             int32_t* out_sp, int32_t* out_ckpt, double* out_seconds, char* err, int errlen) {
    errbuf e = {err, errlen};
    int32_t a, b;
    int rc = profiler_check(profiler, &a, &b, &e);
    return rc ? rc : best_sp_ckpt(profiler, length, sp, n_sp, out_sp, out_ckpt, out_seconds, &e);
}

int oracle_select_groups(const int64_t* lengths, int32_t n_lengths, const hbp_profiler* profiler, const int32_t* sp,
                         int32_t n_sp, hbp_group_config* out_groups, int32_t* out_count, int64_t* out_l_best,
                         int64_t* out_l_max, char* err, int errlen) {
    errbuf e = {err, errlen};
    int32_t a, b;
    int rc = profiler_check(profiler, &a, &b, &e);
    return rc ? rc
              : select_groups(lengths, n_lengths, profiler, sp, n_sp, out_groups, out_count, out_l_best, out_l_max,
                              &e);
}

int oracle_sweep(const int64_t* ids, const int64_t* lengths, int64_t n, const hbp_group_config* cand_groups,
                 const int64_t* cand_offsets, const int64_t* cand_l_best, int64_t n_candidates,
                 const hbp_plan_options* options, const hbp_hardware_profile* profile, double* out_seconds,
                 int64_t* out_best, char* err, int errlen) {
    errbuf e = {err, errlen};
    sample* v = make_samples(ids, lengths, n);
    int64_t best = -1;
    int rc = OK;
    for (int64_t c = 0; c < n_candidates && rc == OK; ++c) {
        hbp_groups g = {cand_groups + cand_offsets[c], (int32_t)(cand_offsets[c + 1] - cand_offsets[c]),
                        cand_l_best[c], cand_groups[cand_offsets[c + 1] - 1].length};
        ilist its;
        memset(&its, 0, sizeof its);
        char msg[1024];
        errbuf ie = {msg, sizeof msg};
        double t = INFINITY;
        int r = build_plan(v, n, &g, options, &its, &ie);
        if (r == OK) {
            flat f;
            flat_init(&f);
            for (int64_t i = 0; i < its.n; ++i) flat_iteration(&f, &its.v[i]);
            oracle_plan* o = flat_finish(&f, options->device_count, options->seed);
            hbp_plan_view pv;
            memset(&pv, 0, sizeof pv);
            pv.device_count = o->device_count;
            pv.seed = o->seed;
            pv.groups = g;
            pv.n_iterations = o->n_iterations;
            pv.n_devices = o->n_devices;
            pv.n_packs = o->n_packs;
            pv.n_members = o->n_members;
            pv.iter_group = o->iter_group;
            pv.iter_dev_offsets = o->iter_dev_offsets;
            pv.dev_index = o->dev_index;
            pv.dev_pack_offsets = o->dev_pack_offsets;
            pv.pack_capacity = o->pack_capacity;
            pv.pack_total = o->pack_total;
            pv.pack_attention = o->pack_attention;
            pv.pack_member_offsets = o->pack_member_offsets;
            hbp_sim_totals st;
            r = simulate(&pv, profile, &st, NULL, NULL, NULL, NULL, &ie);
            if (r == OK) t = st.total_seconds;
            oracle_plan_free(o);
        }
        il_free(&its);
        if (r != OK && r != EINF) rc = fail(&e, r, "%s", msg);
        out_seconds[c] = t;
        if (t != INFINITY && (best < 0 || t < out_seconds[best])) best = c;
    }
    *out_best = best;
    free(v);
    return rc;
}
