/*
 * HalftimeHash CPU oracle -- scalar C restatement of the reference hash path.
 *
 * TEST INFRASTRUCTURE ONLY.  The product library (paper_2104_08865_b200/)
 * never links, loads or calls this code.  It is used by tests/ as the
 * checker for the CUDA engine at sizes the numpy oracle cannot reach
 * (e.g. the 16 GiB single string of config 5), by __graft_entry__.smoke()
 * as the checker, and by bench.py as the CPU baseline ("port").
 *
 * Restates the reference package halftimehash 0.1.0
 * (/root/reference/pkg/src/halftimehash), following the scalar engine
 * hasher.py:217-269 and the contract it implements:
 *   seed stream          hasher.py:29-67      (splitmix64 counter form)
 *   seed layout          hasher.py:126-158
 *   words                hasher.py:179-183    (LE u64, zero-padded last word)
 *   GF(16) scale         gf16.py:17-32        (bit-sliced, 16 elements/u64)
 *   codes / matrices     params.py:105-130, 185-227
 *   EHC leaf             ehc.py:23-118
 *   NH / tree node       nh.py:48-121
 *   stack construction   tree.py:63-100
 *   finalize             tree.py:103-134
 *   Toeplitz tail        hasher.py:186-206
 * Pinned by tests/test_oracle_golden.py against the reference's golden
 * digests (pkg/tests/test_hasher.py:30-53) and reference-generated fixtures.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXLEV 24

typedef struct {
    int k, e, d, w, b, f, m, ew;
    int parity[4][7];
    int matrix[5][10];
} hto_variant;

static int gf_xt4(int a) { int t = (a >> 3) & 1; return ((a << 1) & 0xF) ^ t ^ (t << 1); }
static int gf_mul4(int a, int b) {
    int acc = 0, t = b;
    for (int i = 0; i < 4; i++) { if ((a >> i) & 1) acc ^= t; t = gf_xt4(t); }
    return acc;
}
static int gf_inv4(int a) { for (int b = 1; b < 16; b++) if (gf_mul4(a, b) == 1) return b; return 0; }

static const int MAT16[2][7] = {{1,0,1,1,2,1,4},{0,1,1,2,1,4,1}};
static const int MAT24[3][9] = {{0,0,1,4,1,1,2,2,1},{1,1,0,0,1,4,1,2,2},{1,4,1,1,0,0,2,1,2}};
static const int MAT32[4][10] = {{0,0,0,1,1,4,2,4,1,1},{0,1,2,0,0,1,1,2,4,1},
                                 {2,0,1,0,4,0,1,1,1,1},{1,1,0,1,0,0,4,1,2,8}};
static const int MAT40[5][9] = {{1,0,0,0,0,1,1,2,4},{0,1,0,0,0,1,2,1,7},{0,0,1,0,0,1,3,8,5},
                                {0,0,0,1,0,1,4,9,8},{0,0,0,0,1,1,5,3,9}};

static int get_variant(int out_bytes, hto_variant* v) {
    memset(v, 0, sizeof *v);
    v->b = 8; v->f = 8;
    int p = 0;
    switch (out_bytes) {  /* params.py:217-227 */
    case 16: v->k=2; v->e=7; v->d=6; v->w=2; break;
    case 24: v->k=3; v->e=9; v->d=7; v->w=3; break;
    case 32: v->k=4; v->e=10; v->d=7; v->w=3; break;
    case 40: v->k=5; v->e=9; v->d=5; v->w=3; break;
    default: return -1;
    }
    v->m = v->d * v->w * v->b;
    v->ew = v->e * v->w;
    p = v->e - v->d;
    for (int j = 0; j < p; j++)
        for (int i = 0; i < v->d; i++)
            v->parity[j][i] = out_bytes == 16 ? 1 : gf_inv4(j ^ (p + i)); /* params.py:105-130 */
    for (int r = 0; r < v->k; r++)
        for (int c = 0; c < v->e; c++)
            v->matrix[r][c] = out_bytes == 16 ? MAT16[r][c] : out_bytes == 24 ? MAT24[r][c]
                            : out_bytes == 32 ? MAT32[r][c] : MAT40[r][c];
    return 0;
}

/* ---------------------------------------------------------------- seeds */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void hto_splitmix(uint64_t fold, uint64_t start, uint64_t count, uint64_t* out, int threads) {
    (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
    for (int64_t i = 0; i < (int64_t)count; i++)
        out[i] = mix64(fold + (start + (uint64_t)i + 1) * 0x9E3779B97F4A7C15ULL);
}

static int level_count(uint64_t n) { int l = 1; while (n >= 8) { n >>= 3; l++; } return l; }

typedef struct { uint64_t n_inst; int L; uint64_t T[5], F[5], R, total; } hto_layout;

static void get_layout(const hto_variant* v, uint64_t n_bytes, hto_layout* lay) {
    uint64_t nw = (n_bytes + 7) / 8;
    lay->n_inst = nw / (uint64_t)v->m;
    lay->L = lay->n_inst ? level_count(lay->n_inst) : 1;
    uint64_t t0 = v->ew, f0 = t0 + 7ull * lay->L * v->k;
    for (int r = 0; r < v->k; r++) { lay->T[r] = t0 + 7ull * lay->L * r; lay->F[r] = f0 + 64ull * lay->L * r; }
    lay->R = f0 + 64ull * lay->L * v->k;
    lay->total = lay->R + v->m + v->k - 1;
}

uint64_t hto_seed_words_needed(int out_bytes, uint64_t n_bytes) {
    hto_variant v; hto_layout lay;
    if (get_variant(out_bytes, &v)) return 0;
    get_layout(&v, n_bytes, &lay);
    return lay.total;
}

/* ------------------------------------------------------------ primitives */
static inline uint64_t nh(uint64_t x, uint64_t s) {
    uint32_t lo = (uint32_t)x + (uint32_t)s, hi = (uint32_t)(x >> 32) + (uint32_t)(s >> 32);
    return (uint64_t)lo * hi;
}
static inline uint64_t xtime(uint64_t v) { uint64_t t = v >> 48; return (v << 16) ^ t ^ (t << 16); }
static inline uint64_t scale(int c, uint64_t v) {
    uint64_t acc = 0;
    for (int i = 0; i < 4; i++) { if ((c >> i) & 1) acc ^= v; v = xtime(v); }
    return acc;
}

/* word t of a string (LE, zero-padded past n) */
static inline uint64_t load_word(const uint8_t* p, uint64_t n, uint64_t t) {
    uint64_t off = t * 8;
    if (off + 8 <= n) { uint64_t x; memcpy(&x, p + off, 8); return x; }
    uint64_t x = 0;
    for (uint64_t i = off; i < n; i++) x |= (uint64_t)p[i] << (8 * (i - off));
    return x;
}

/* leaf for instance t: C[r][j] (ehc.py:102-118 == hasher.py:356-364) */
static void leaf(const hto_variant* v, const uint8_t* p, uint64_t n, uint64_t t,
                 const uint64_t* S, uint64_t C[5][8]) {
    uint64_t X[7][3], E[10][3], H[10];
    for (int j = 0; j < 8; j++) {
        for (int i = 0; i < v->d; i++)
            for (int u = 0; u < v->w; u++)
                X[i][u] = load_word(p, n, t * v->m + (uint64_t)(i * v->w + u) * 8 + j);
        for (int i = 0; i < v->d; i++)
            for (int u = 0; u < v->w; u++) E[i][u] = X[i][u];
        for (int q = 0; q < v->e - v->d; q++)
            for (int u = 0; u < v->w; u++) {
                uint64_t a = 0;
                for (int i = 0; i < v->d; i++) if (v->parity[q][i]) a ^= scale(v->parity[q][i], X[i][u]);
                E[v->d + q][u] = a;
            }
        for (int i = 0; i < v->e; i++) {
            uint64_t h = 0;
            for (int u = 0; u < v->w; u++) h += nh(E[i][u], S[i * v->w + u]);
            H[i] = h;
        }
        for (int r = 0; r < v->k; r++) {
            uint64_t a = 0;
            for (int i = 0; i < v->e; i++) a += (uint64_t)v->matrix[r][i] * H[i];
            C[r][j] = a;
        }
    }
}

/* --------------------------------------------------- stack construction */
typedef struct {
    int cnt[MAXLEV];
    int top;  /* number of levels touched */
    uint64_t blk[MAXLEV][8][5][8];
} stack_t_;

static void push(const hto_variant* v, stack_t_* st, int lvl, uint64_t B[5][8],
                 const hto_layout* lay, const uint64_t* S) {
    for (;;) {
        if (lvl >= st->top) st->top = lvl + 1;
        memcpy(st->blk[lvl][st->cnt[lvl]], B, sizeof(uint64_t) * 5 * 8);
        if (++st->cnt[lvl] < 8) return;
        /* nh_blockwise over the 8 blocks with level seeds (tree.py:63-100, nh.py:70-121) */
        uint64_t N[5][8];
        for (int r = 0; r < v->k; r++) {
            const uint64_t* s = S + lay->T[r] + 7ull * lvl;
            for (int j = 0; j < 8; j++) {
                uint64_t a = st->blk[lvl][7][r][j];
                for (int q = 0; q < 7; q++) a += nh(st->blk[lvl][q][r][j], s[q]);
                N[r][j] = a;
            }
        }
        st->cnt[lvl] = 0;
        memcpy(B, N, sizeof N);
        lvl++;
    }
}

/* finalize + tail for a completed stack (tree.py:103-134, hasher.py:258-269) */
static void finish(const hto_variant* v, const stack_t_* st, const uint8_t* p, uint64_t n,
                   const hto_layout* lay, const uint64_t* S, uint64_t* out) {
    for (int r = 0; r < v->k; r++) {
        uint64_t acc = 0;
        if (lay->n_inst) {
            const uint64_t* s = S + lay->F[r];
            for (int l = 0; l < lay->L; l++)
                for (int q = 0; q < 7; q++)
                    for (int j = 0; j < 8; j++) {
                        uint64_t z = q < st->cnt[l] ? st->blk[l][q][r][j] : 0;
                        acc += nh(z, s[l * 56 + q * 8 + j]);
                    }
            acc += nh(n, s[lay->L * 56]);
        } else {
            acc += nh(n, S[lay->F[r]]);
        }
        uint64_t nw = (n + 7) / 8, t0 = lay->n_inst * v->m;
        for (uint64_t t = t0; t < nw; t++) acc += nh(load_word(p, n, t), S[lay->R + r + (t - t0)]);
        out[r] = acc;
    }
}

static int check(int out_bytes, uint64_t n, uint64_t cap, hto_variant* v, hto_layout* lay) {
    if (get_variant(out_bytes, v)) return -1;
    get_layout(v, n, lay);
    if (cap < lay->total) return -2;
    if (lay->L >= MAXLEV) return -1;
    return 0;
}

int hto_hash_one(int out_bytes, const uint8_t* p, uint64_t n, const uint64_t* S, uint64_t cap,
                 uint64_t* out) {
    hto_variant v; hto_layout lay;
    int rc = check(out_bytes, n, cap, &v, &lay);
    if (rc) return rc;
    stack_t_* st = (stack_t_*)calloc(1, sizeof *st);
    uint64_t C[5][8];
    for (uint64_t t = 0; t < lay.n_inst; t++) {
        leaf(&v, p, n, t, S, C);
        push(&v, st, 0, C, &lay, S);
    }
    finish(&v, st, p, n, &lay, S, out);
    free(st);
    return 0;
}

int hto_hash_fixed(int out_bytes, const uint8_t* data, uint64_t n_strings, uint64_t stride,
                   uint64_t n, const uint64_t* S, uint64_t cap, uint64_t* out, int threads) {
    hto_variant v; hto_layout lay;
    int rc = check(out_bytes, n, cap, &v, &lay);
    if (rc) return rc;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1)
    for (int64_t s = 0; s < (int64_t)n_strings; s++)
        hto_hash_one(out_bytes, data + (uint64_t)s * stride, n, S, cap, out + (uint64_t)s * v.k);
    return 0;
}

int hto_hash_varlen(int out_bytes, const uint8_t* data, const uint64_t* off, uint64_t n_strings,
                    const uint64_t* S, uint64_t cap, uint64_t* out, int threads) {
    hto_variant v;
    if (get_variant(out_bytes, &v)) return -1;
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads > 0 ? threads : 1) reduction(|:bad)
    for (int64_t s = 0; s < (int64_t)n_strings; s++)
        bad |= hto_hash_one(out_bytes, data + off[s], off[s + 1] - off[s], S, cap, out + (uint64_t)s * v.k) != 0;
    return bad ? -2 : 0;
}

/*
 * One long string, parallel over f^c-aligned subtrees.  Each full chunk of
 * 8^c instances reduces to exactly one level-c block; the chunk roots then
 * continue the stack construction from level c.  Bit-identical to
 * hto_hash_one because the stack groups are front-aligned (tree.py:63-100).
 */
int hto_hash_huge(int out_bytes, const uint8_t* p, uint64_t n, const uint64_t* S, uint64_t cap,
                  uint64_t* out, int threads) {
    hto_variant v; hto_layout lay;
    int rc = check(out_bytes, n, cap, &v, &lay);
    if (rc) return rc;
    int c = 3;
    while (c < 12 && (lay.n_inst >> (3 * (c + 1))) >= (uint64_t)(threads > 0 ? threads : 1) * 8) c++;
    uint64_t chunk = 1ull << (3 * c), nfull = lay.n_inst / chunk;
    uint64_t (*roots)[5][8] = (uint64_t(*)[5][8])malloc(sizeof(uint64_t) * 40 * (nfull + 1));
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
    {
        stack_t_* st = (stack_t_*)calloc(1, sizeof *st);
        uint64_t C[5][8];
#pragma omp for schedule(dynamic, 1)
        for (int64_t g = 0; g < (int64_t)nfull; g++) {
            memset(st, 0, sizeof *st);
            for (uint64_t t = g * chunk; t < (g + 1) * chunk; t++) {
                leaf(&v, p, n, t, S, C);
                push(&v, st, 0, C, &lay, S);
            }
            memcpy(roots[g], st->blk[c][0], sizeof(uint64_t) * 40);
        }
        free(st);
    }
    stack_t_* st = (stack_t_*)calloc(1, sizeof *st);
    for (uint64_t g = 0; g < nfull; g++) push(&v, st, c, roots[g], &lay, S);
    uint64_t C[5][8];
    for (uint64_t t = nfull * chunk; t < lay.n_inst; t++) {
        leaf(&v, p, n, t, S, C);
        push(&v, st, 0, C, &lay, S);
    }
    /* levels below c that the roots skipped are empty but still "touched" */
    finish(&v, st, p, n, &lay, S, out);
    free(st); free(roots);
    return 0;
}

/*
 * Slice / merge restatement of the same hash, for checking the multi-device
 * decomposition (test infrastructure).  A string cut at multiples of 8^c
 * instances splits into independent level-c subtrees because the stack
 * construction groups blocks front-aligned (tree.py:63-100).  The finalize
 * NH (tree.py:103-134) and the tail (hasher.py:186-206) are sums of terms,
 * so each slice contributes a partial sum; level-c roots that are not
 * leftovers ("frontier") are finished by the merge.
 */
static uint64_t fin_term(const hto_variant* v, const hto_layout* lay, const uint64_t* S, int r, int lvl,
                         uint64_t slot, const uint64_t blk[8]) {
    uint64_t acc = 0;
    for (int j = 0; j < 8; j++) acc += nh(blk[j], S[lay->F[r] + 56ull * lvl + slot * 8 + j]);
    (void)v;
    return acc;
}

int hto_slice(int out_bytes, const uint8_t* p, uint64_t n, uint64_t a, uint64_t b, int c, const uint64_t* S,
              uint64_t cap, uint64_t* frontier, uint64_t* partial) {
    hto_variant v; hto_layout lay;
    int rc = check(out_bytes, n, cap, &v, &lay);
    if (rc) return rc;
    for (int r = 0; r < v.k; r++) partial[r] = 0;
    const uint64_t keep = (lay.n_inst >> (3 * c)) & ~7ull, fbase = a >> (3 * c);
    stack_t_* st = (stack_t_*)calloc(1, sizeof *st);
    uint64_t C[5][8];
    for (uint64_t t = a; t < b; t++) {
        leaf(&v, p, n, t, S, C);
        push(&v, st, 0, C, &lay, S);
        if (st->cnt[c] == 1) {  /* a level-c root just completed */
            uint64_t idx = t >> (3 * c);
            if (idx < keep) {
                for (int r = 0; r < v.k; r++) memcpy(frontier + (idx - fbase) * 8 * v.k + r * 8, st->blk[c][0][r], 64);
            } else {
                for (int r = 0; r < v.k; r++) partial[r] += fin_term(&v, &lay, S, r, c, idx & 7, st->blk[c][0][r]);
            }
            st->cnt[c] = 0;
        }
    }
    if (b == lay.n_inst) {  /* last slice: leftovers below c, every zero slot, tag, tail */
        for (int r = 0; r < v.k; r++) {
            uint64_t acc = 0;
            if (lay.n_inst) {
                const uint64_t* s = S + lay.F[r];
                for (int l = 0; l < lay.L; l++) {
                    const int digit = (int)((lay.n_inst >> (3 * l)) & 7);
                    for (int q = 0; q < 7; q++)
                        for (int j = 0; j < 8; j++) {
                            if (q >= digit) acc += nh(0, s[l * 56 + q * 8 + j]);             /* zero slot */
                            else if (l < c) acc += nh(st->blk[l][q][r][j], s[l * 56 + q * 8 + j]);
                        }
                }
                acc += nh(n, s[lay.L * 56]);
            } else {
                acc += nh(n, S[lay.F[r]]);
            }
            uint64_t nw = (n + 7) / 8, t0 = lay.n_inst * v.m;
            for (uint64_t t = t0; t < nw; t++) acc += nh(load_word(p, n, t), S[lay.R + r + (t - t0)]);
            partial[r] += acc;
        }
    }
    free(st);
    return 0;
}

int hto_merge(int out_bytes, uint64_t n, int c, const uint64_t* frontier, uint64_t nf, const uint64_t* partials,
              uint64_t np, const uint64_t* S, uint64_t cap, uint64_t* out) {
    hto_variant v; hto_layout lay;
    int rc = check(out_bytes, n, cap, &v, &lay);
    if (rc) return rc;
    for (int r = 0; r < v.k; r++) {
        uint64_t acc = 0;
        for (uint64_t q = 0; q < np; q++) acc += partials[q * v.k + r];
        out[r] = acc;
    }
    uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * 40 * (nf + 8));
    uint64_t* nxt = (uint64_t*)malloc(sizeof(uint64_t) * 40 * (nf / 8 + 8));
    memcpy(cur, frontier, sizeof(uint64_t) * 8 * v.k * nf);
    int lvl = c;
    while (nf >= 8) {
        uint64_t nn = nf / 8, keep = nn & ~7ull;
        for (uint64_t g = 0; g < nn; g++)
            for (int r = 0; r < v.k; r++) {
                uint64_t blk[8];
                for (int j = 0; j < 8; j++) {
                    uint64_t a = cur[(8 * g + 7) * 8 * v.k + r * 8 + j];
                    for (int q = 0; q < 7; q++) a += nh(cur[(8 * g + q) * 8 * v.k + r * 8 + j], S[lay.T[r] + 7ull * lvl + q]);
                    blk[j] = a;
                }
                if (g >= keep) out[r] += fin_term(&v, &lay, S, r, lvl + 1, g & 7, blk);
                else memcpy(nxt + g * 8 * v.k + r * 8, blk, 64);
            }
        uint64_t* t = cur; cur = nxt; nxt = t;
        nf = keep;
        lvl++;
    }
    free(cur); free(nxt);
    return 0;
}
