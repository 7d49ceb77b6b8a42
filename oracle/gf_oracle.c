/*
 * oracle/gf_oracle.c -- PLAIN, SLOW, OBVIOUSLY-CORRECT CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
 * this library.  The product path (paper_2306_11686_b200/, include/gf_xs.h) never links, imports or
 * calls it, and this file includes none of the product's headers: the two share no code, tables or
 * constant generators.  Every constant below is typed here independently of the CUDA path.
 *
 * What it computes: the XSBench v20 / RSBench v13 macroscopic cross-section lookup that GPU First
 * runs on the GPU (Sec. 5.3.1 "XSBench and RSBench"; Fig. 8).
 * PAPER.md itself states only "perform the cross-section lookup ... event-based lookup and
 * history-based lookup" on "two different input sizes".  The
 * step-by-step semantics follow the reading recorded in SURVEY.md Sec. 8(c) c.2 (and the readings
 * R-* of its ambiguity register c.3), which DESIGN.md Sec. 3 lists.  Function-level comments cite
 * the SURVEY line that each step follows.
 *
 * Arithmetic: IEEE fp64, round-to-nearest, every operation in the order written.  Build with
 * -O2 -ffp-contract=off (no FMA contraction, no -ffast-math): R-FP, SURVEY.md:655.
 *
 * Parity status per function:
 *   o_lcg_*, o_fast_forward, o_thresholds, o_pick_mat, xs grid build, grid_search, ig/hg entries,
 *   xs lookups, RS Faddeeva constants: pinned (tests/test_oracle_*.py).
 *   xso_history_batch / rso_history_batch (NEXT-1): pinned by the L = 1 reduction to event lookups,
 *   an independent Python transcription of the particle chain (exact-integer LCG, per-step macro
 *   from the pinned xso_macro / rso_macro) and hash bounds / additivity (tests/test_oracle_history.py).
 *   Results vs the real XSBench/RSBench binaries: parity unpinned (no implementation exists to
 *   compare against; SURVEY.md:691).  RS generator layout: pinned only to the survey's reading
 *   (golden values SURVEY.md:996-997).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- LCG (SURVEY.md:540-547) */
#define O_LCG_A 2806196910506780709ULL
#define O_LCG_MASK 0x7FFFFFFFFFFFFFFFULL /* mod 2^63 */

uint64_t o_lcg_step(uint64_t s) { return (O_LCG_A * s + 1ULL) & O_LCG_MASK; }

double o_lcg_double(uint64_t *s) {
    *s = o_lcg_step(*s);
    return (double)(*s) / 9223372036854775808.0; /* (double)s / 2^63 */
}

uint64_t o_lcg_int(uint64_t *s) {
    *s = o_lcg_step(*s);
    return *s;
}

/* fast_forward(s, n): n LCG steps in O(log n) (SURVEY.md:544-547). */
uint64_t o_fast_forward(uint64_t seed, uint64_t n) {
    uint64_t a = O_LCG_A, c = 1ULL, a_new = 1ULL, c_new = 0ULL;
    n = n & O_LCG_MASK;
    while (n > 0) {
        if (n & 1ULL) {
            a_new = a_new * a;
            c_new = c_new * a + c;
        }
        c = c * (a + 1ULL);
        a = a * a;
        n >>= 1;
    }
    return (a_new * seed + c_new) & O_LCG_MASK;
}

/* ---------------------------------------------------------------- materials (SURVEY.md:549-558) */
static const double O_DIST[12] = {0.140, 0.052, 0.275, 0.134, 0.154, 0.064,
                                  0.066, 0.055, 0.008, 0.015, 0.025, 0.013};

/* T[m] = dist[m] + dist[m-1] + ... + dist[1], summed in that (descending) order; T[0] = 0 (R-PICK). */
void o_thresholds(double T[12]) {
    for (int m = 0; m < 12; m++) {
        double running = 0.0;
        for (int j = m; j > 0; j--) running += O_DIST[j];
        T[m] = running;
    }
}

/* pick_mat: first m in 1..11 with roll < T[m], else 0 (fuel) (SURVEY.md:551). */
int o_pick_mat(double roll) {
    double T[12];
    o_thresholds(T);
    for (int m = 0; m < 12; m++)
        if (roll < T[m]) return m;
    return 0;
}

static const int O_FUEL_SMALL[34] = {58, 59, 60, 61, 40, 42, 43, 44, 45, 46, 1,  2,  3,  7,  8,  9,  10,
                                     29, 57, 47, 48, 0,  62, 15, 33, 34, 52, 53, 54, 55, 56, 18, 23, 41};
static const int O_M1[5] = {63, 64, 65, 66, 67};
static const int O_M2[4] = {24, 41, 4, 5};
static const int O_M4[27] = {19, 20, 21, 22, 35, 36, 37, 38, 39, 25, 27, 28, 29, 30,
                             31, 32, 26, 49, 50, 51, 11, 12, 13, 14, 6,  16, 17};
static const int O_M5[21] = {24, 41, 4, 5, 19, 20, 21, 22, 35, 36, 37, 38, 39, 25, 27, 28, 29, 30, 31, 32, 26};
static const int O_M10[9] = {24, 41, 4, 5, 63, 64, 65, 66, 67};

/* Built-in Hoogenboom-Martin tables for n_iso = 68 (small) or 355 (large).  Row-major
 * mats[12][max_num_nucs].  Returns max_num_nucs, or -1 if n_iso is neither 68 nor 355. */
int o_builtin_tables(int n_iso, int num_nucs[12], int *mats /* may be NULL: sizes only */) {
    if (n_iso != 68 && n_iso != 355) return -1;
    static const int rest[11] = {5, 4, 4, 27, 21, 21, 21, 21, 21, 9, 9};
    num_nucs[0] = (n_iso == 68) ? 34 : 321;
    for (int m = 1; m < 12; m++) num_nucs[m] = rest[m - 1];
    int mx = num_nucs[0];
    if (mats) {
        for (int j = 0; j < 34; j++) mats[0 * mx + j] = O_FUEL_SMALL[j];
        if (n_iso == 355)
            for (int j = 0; j < 321 - 34; j++) mats[0 * mx + 34 + j] = 68 + j;
        for (int j = 0; j < 5; j++) mats[1 * mx + j] = O_M1[j];
        for (int j = 0; j < 4; j++) mats[2 * mx + j] = O_M2[j];
        for (int j = 0; j < 4; j++) mats[3 * mx + j] = O_M2[j];
        for (int j = 0; j < 27; j++) mats[4 * mx + j] = O_M4[j];
        for (int m = 5; m <= 9; m++)
            for (int j = 0; j < 21; j++) mats[m * mx + j] = O_M5[j];
        for (int m = 10; m <= 11; m++)
            for (int j = 0; j < 9; j++) mats[m * mx + j] = O_M10[j];
    }
    return mx;
}

/* ================================================================ XSBench */
enum { O_NUCLIDE = 0, O_UNIONIZED = 1, O_HASH = 2 };

typedef struct {
    int n_iso;
    long n_gp;
    int grid_type;
    int bins;
    int num_nucs[12];
    int max_num_nucs;
    int *mats;      /* [12][max_num_nucs] */
    double *concs;  /* [12][max_num_nucs] */
    double *G;      /* nuclide grid [n_iso][n_gp][6]: E, total, elastic, absorption, fission, nu-fission */
    double *U;      /* unionized energies [n_iso*n_gp] (unionized only) */
    int32_t *HG;    /* hash grid [bins][n_iso] (hash only) */
} xs_oracle;

typedef struct {
    double v[6];
    long gen; /* generation index inside the nuclide: the stable-sort tie-break (R-TIE-SORT) */
} o_rec;

static int cmp_rec(const void *a, const void *b) {
    const o_rec *x = (const o_rec *)a, *y = (const o_rec *)b;
    if (x->v[0] < y->v[0]) return -1;
    if (x->v[0] > y->v[0]) return 1;
    return (x->gen < y->gen) ? -1 : (x->gen > y->gen);
}

static int cmp_double(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x < y) ? -1 : (x > y);
}

/* XSBench grid_search / grid_search_nuclide: lower-bound bisection on [lo, hi] that returns lo
 * (SURVEY.md:569-570).  `A` is read with stride `stride` doubles (6 for the nuclide grid). */
long o_grid_search(const double *A, long stride, double q, long lo, long hi) {
    long length = hi - lo;
    while (length > 1) {
        long mid = lo + length / 2;
        if (A[mid * stride] > q)
            hi = mid;
        else
            lo = mid;
        length = hi - lo;
    }
    return lo;
}

/* #{k in [0,n) : A[k*stride] <= q}, by bisection on the sorted array. */
static long o_count_le(const double *A, long stride, long n, double q) {
    long lo = 0, hi = n; /* answer in [lo, hi] */
    while (lo < hi) {
        long mid = lo + (hi - lo) / 2;
        if (A[mid * stride] <= q)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

/* Build the grids (A0; SURVEY.md:560-567).  custom_num_nucs/custom_mats NULL = built-in tables. */
xs_oracle *xso_create(int n_iso, long n_gp, int grid_type, int bins, uint64_t seed,
                      const int *custom_num_nucs, const int *custom_mats, int custom_max) {
    if (n_iso < 1 || n_gp < 2 || grid_type < 0 || grid_type > 2) return NULL;
    if (grid_type == O_HASH && bins < 1) return NULL;
    xs_oracle *o = (xs_oracle *)calloc(1, sizeof(xs_oracle));
    o->n_iso = n_iso;
    o->n_gp = n_gp;
    o->grid_type = grid_type;
    o->bins = bins;
    if (custom_num_nucs) {
        for (int m = 0; m < 12; m++) o->num_nucs[m] = custom_num_nucs[m];
        o->max_num_nucs = custom_max;
        o->mats = (int *)malloc(sizeof(int) * 12 * (size_t)custom_max);
        memcpy(o->mats, custom_mats, sizeof(int) * 12 * (size_t)custom_max);
    } else {
        int mx = o_builtin_tables(n_iso, o->num_nucs, NULL);
        if (mx < 0) {
            free(o);
            return NULL;
        }
        o->max_num_nucs = mx;
        o->mats = (int *)calloc(12 * (size_t)mx, sizeof(int));
        o_builtin_tables(n_iso, o->num_nucs, o->mats);
    }
    for (int m = 0; m < 12; m++)
        for (int j = 0; j < o->num_nucs[m]; j++) {
            int nuc = o->mats[m * o->max_num_nucs + j];
            if (nuc < 0 || nuc >= n_iso) { /* table references a nuclide that does not exist */
                free(o->mats);
                free(o);
                return NULL;
            }
        }

    /* A0.1: one LCG stream from `seed`, 6 draws per gridpoint in field order, nuclide-major. */
    size_t npts = (size_t)n_iso * (size_t)n_gp;
    o->G = (double *)malloc(sizeof(double) * 6 * npts);
    uint64_t s = seed;
    for (size_t p = 0; p < npts; p++)
        for (int f = 0; f < 6; f++) o->G[p * 6 + f] = o_lcg_double(&s);

    /* A0.6 (R-CONC): concentrations continue the same stream, m ascending then j ascending. */
    o->concs = (double *)calloc(12 * (size_t)o->max_num_nucs, sizeof(double));
    for (int m = 0; m < 12; m++)
        for (int j = 0; j < o->num_nucs[m]; j++) o->concs[m * o->max_num_nucs + j] = o_lcg_double(&s);

    /* A0.2: sort each nuclide's points by E, stable by generation index. */
    o_rec *tmp = (o_rec *)malloc(sizeof(o_rec) * (size_t)n_gp);
    for (int i = 0; i < n_iso; i++) {
        double *base = o->G + (size_t)i * n_gp * 6;
        for (long k = 0; k < n_gp; k++) {
            memcpy(tmp[k].v, base + k * 6, sizeof(double) * 6);
            tmp[k].gen = k;
        }
        qsort(tmp, (size_t)n_gp, sizeof(o_rec), cmp_rec);
        for (long k = 0; k < n_gp; k++) memcpy(base + k * 6, tmp[k].v, sizeof(double) * 6);
    }
    free(tmp);

    /* A0.3: U = sorted multiset of all energies. */
    if (grid_type == O_UNIONIZED) {
        o->U = (double *)malloc(sizeof(double) * npts);
        for (size_t p = 0; p < npts; p++) o->U[p] = o->G[p * 6];
        qsort(o->U, npts, sizeof(double), cmp_double);
    }
    /* A0.5: HG[b][i] = grid_search(A_i.E, b*du, 0, n_gp-1), du = 1.0/bins (R-HASHQ). */
    if (grid_type == O_HASH) {
        o->HG = (int32_t *)malloc(sizeof(int32_t) * (size_t)bins * n_iso);
        double du = 1.0 / bins;
        for (long b = 0; b < bins; b++) {
            double energy = b * du;
            for (int i = 0; i < n_iso; i++)
                o->HG[b * n_iso + i] =
                    (int32_t)o_grid_search(o->G + (size_t)i * n_gp * 6, 6, energy, 0, n_gp - 1);
        }
    }
    return o;
}

void xso_free(xs_oracle *o) {
    if (!o) return;
    free(o->mats);
    free(o->concs);
    free(o->G);
    free(o->U);
    free(o->HG);
    free(o);
}

/* Accessors (the caller copies out what it needs). */
const double *xso_nuclide_grid(const xs_oracle *o) { return o->G; }
const double *xso_unionized(const xs_oracle *o) { return o->U; }
const int32_t *xso_hash_grid(const xs_oracle *o) { return o->HG; }
int xso_max_num_nucs(const xs_oracle *o) { return o->max_num_nucs; }
void xso_tables(const xs_oracle *o, int num_nucs[12], int *mats, double *concs) {
    memcpy(num_nucs, o->num_nucs, sizeof(int) * 12);
    memcpy(mats, o->mats, sizeof(int) * 12 * (size_t)o->max_num_nucs);
    memcpy(concs, o->concs, sizeof(double) * 12 * (size_t)o->max_num_nucs);
}

/* A0.4 (R-IG, closed form): IG[e][i] = clamp(#{k : A_i[k].E <= U[e]} - 1, 0, n_gp - 2).
 * Computed on demand, element by element (no 5.7 GB table is needed to check one entry). */
int32_t xso_ig_entry(const xs_oracle *o, long e, int i) {
    const double *A = o->G + (size_t)i * o->n_gp * 6;
    long c = o_count_le(A, 6, o->n_gp, o->U[e]) - 1;
    if (c < 0) c = 0;
    if (c > o->n_gp - 2) c = o->n_gp - 2;
    return (int32_t)c;
}

/* Fill IG rows [e0, e1) energy-major: out[(e-e0)*n_iso + i]. */
void xso_ig_rows(const xs_oracle *o, long e0, long e1, int32_t *out) {
#pragma omp parallel for schedule(static)
    for (long e = e0; e < e1; e++)
        for (int i = 0; i < o->n_iso; i++) out[(e - e0) * o->n_iso + i] = xso_ig_entry(o, e, i);
}

/* A3-A5 for one (E, mat): macro[0..4] (SURVEY.md:574-590). */
void xso_macro(const xs_oracle *o, double E, int mat, double macro[5]) {
    const long n_gp = o->n_gp;
    long u = 0, b = 0;
    if (o->grid_type == O_UNIONIZED) {
        long n_u = (long)o->n_iso * n_gp;
        u = o_grid_search(o->U, 1, E, 0, n_u - 1);
    } else if (o->grid_type == O_HASH) {
        double du = 1.0 / o->bins;
        b = (long)(E / du);
        if (b > o->bins - 1) b = o->bins - 1; /* R-E1 */
        if (b < 0) b = 0;                     /* energies below 0 (energies API only) */
    }
    for (int c = 0; c < 5; c++) macro[c] = 0.0;
    for (int j = 0; j < o->num_nucs[mat]; j++) {
        int nuc = o->mats[mat * o->max_num_nucs + j];
        double conc = o->concs[mat * o->max_num_nucs + j];
        const double *A = o->G + (size_t)nuc * n_gp * 6;
        long k;
        if (o->grid_type == O_NUCLIDE) {
            k = o_grid_search(A, 6, E, 0, n_gp - 1);
        } else if (o->grid_type == O_UNIONIZED) {
            k = xso_ig_entry(o, u, nuc);
        } else {
            long lo_ = o->HG[b * o->n_iso + nuc];
            long hi_ = (b == o->bins - 1) ? n_gp - 1 : (long)o->HG[(b + 1) * o->n_iso + nuc] + 1;
            if (E <= A[lo_ * 6])
                k = 0;
            else if (E >= A[hi_ * 6])
                k = n_gp - 1;
            else
                k = o_grid_search(A, 6, E, lo_, hi_);
        }
        if (k == n_gp - 1) k = k - 1;
        const double *lo = A + k * 6;
        const double *hi = lo + 6;
        double f = (hi[0] - E) / (hi[0] - lo[0]);
        for (int c = 0; c < 5; c++) {
            double x = hi[c + 1] - f * (hi[c + 1] - lo[c + 1]);
            macro[c] = macro[c] + x * conc;
        }
    }
}

/* A6: v = 1 + first index of the strict maximum, starting from max = -1.0 (R-ARGMAX, R-PLUS1). */
int o_argmax5_plus1(const double macro[5]) {
    double mx = -1.0;
    int idx = 0;
    for (int c = 0; c < 5; c++)
        if (macro[c] > mx) {
            mx = macro[c];
            idx = c;
        }
    return idx + 1;
}

/* A1: lookup i samples from the stream fast_forward(seed, 2i): E first, then the material roll. */
void o_sample(uint64_t i, uint64_t seed, double *E, int *mat) {
    uint64_t s = o_fast_forward(seed, 2ULL * i);
    *E = o_lcg_double(&s);
    *mat = o_pick_mat(o_lcg_double(&s));
}

/* Event-based batch over GLOBAL indices [first, first+n).  Returns the exact raw sum of v.
 * macro_out: NULL or [n][5].  nthreads <= 0: OpenMP default. */
uint64_t xso_lookup_batch(const xs_oracle *o, uint64_t first, uint64_t n, uint64_t seed, double *macro_out,
                          int nthreads) {
    uint64_t raw = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : raw)
    for (long long t = 0; t < (long long)n; t++) {
        double E, macro[5];
        int mat;
        o_sample(first + (uint64_t)t, seed, &E, &mat);
        xso_macro(o, E, mat, macro);
        raw += (uint64_t)o_argmax5_plus1(macro);
        if (macro_out)
            for (int c = 0; c < 5; c++) macro_out[(size_t)t * 5 + c] = macro[c];
    }
    return raw;
}

/* Same, for an explicit list of global indices (sampled parity at full size). */
uint64_t xso_lookup_indices(const xs_oracle *o, const uint64_t *idx, uint64_t n, uint64_t seed,
                            double *macro_out) {
    uint64_t raw = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : raw)
    for (long long t = 0; t < (long long)n; t++) {
        double E, macro[5];
        int mat;
        o_sample(idx[t], seed, &E, &mat);
        xso_macro(o, E, mat, macro);
        raw += (uint64_t)o_argmax5_plus1(macro);
        if (macro_out)
            for (int c = 0; c < 5; c++) macro_out[(size_t)t * 5 + c] = macro[c];
    }
    return raw;
}

/* Caller-supplied (E, mat) pairs (the energies entry point).  Input domain (DESIGN.md Sec. 3,
 * "caller energies"): a material id in 0..11 (the 12 Hoogenboom-Martin materials, SURVEY.md:552) and a
 * finite energy; anything else is rejected as a whole with UINT64_MAX (errors as values),
 * before any lookup runs. */
uint64_t xso_lookup_energies(const xs_oracle *o, const double *E, const int *mat, uint64_t n, double *macro_out) {
    for (uint64_t t = 0; t < n; t++)
        if (mat[t] < 0 || mat[t] >= 12 || !isfinite(E[t])) return UINT64_MAX;
    uint64_t raw = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : raw)
    for (long long t = 0; t < (long long)n; t++) {
        double macro[5];
        xso_macro(o, E[t], mat[t], macro);
        raw += (uint64_t)o_argmax5_plus1(macro);
        if (macro_out)
            for (int c = 0; c < 5; c++) macro_out[(size_t)t * 5 + c] = macro[c];
    }
    return raw;
}

/* History-based mode (NEXT-1; "event-based lookup and
 * history-based lookup"; reading R-HIST, SURVEY.md:679 and DESIGN.md Sec. 3).  Particle p (GLOBAL
 * index) runs L dependent lookups:
 *     s = fast_forward(seed, p * L * 2 * 4);  E = lcg_double(&s);  mat = pick_mat(lcg_double(&s))
 *     for i in 0 .. L-1:
 *         macro = lookup(E, mat);  raw += 1 + argmax(macro)
 *         n_forward = #{c : macro[c] > 1.0};  if n_forward > 0: s = fast_forward(s, n_forward)
 *         E = lcg_double(&s);  mat = pick_mat(lcg_double(&s))
 * Particles [first_p, first_p + n_p).  macro_out: NULL or [n_p][L][5].  Returns the exact raw sum. */
uint64_t xso_history_batch(const xs_oracle *o, uint64_t first_p, uint64_t n_p, int L, uint64_t seed,
                           double *macro_out, int nthreads) {
    uint64_t raw = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : raw)
    for (long long t = 0; t < (long long)n_p; t++) {
        uint64_t p = first_p + (uint64_t)t;
        uint64_t s = o_fast_forward(seed, p * (uint64_t)L * 2ULL * 4ULL);
        double E = o_lcg_double(&s);
        int mat = o_pick_mat(o_lcg_double(&s));
        for (int i = 0; i < L; i++) {
            double macro[5];
            xso_macro(o, E, mat, macro);
            raw += (uint64_t)o_argmax5_plus1(macro);
            if (macro_out)
                for (int c = 0; c < 5; c++) macro_out[((size_t)t * L + i) * 5 + c] = macro[c];
            uint64_t n_forward = 0;
            for (int c = 0; c < 5; c++)
                if (macro[c] > 1.0) n_forward++;
            if (n_forward > 0) s = o_fast_forward(s, n_forward);
            E = o_lcg_double(&s);
            mat = o_pick_mat(o_lcg_double(&s));
        }
    }
    return raw;
}

/* ================================================================ RSBench (SURVEY.md:594-633) */
typedef struct {
    double r, i;
} o_cplx;

static o_cplx c_add(o_cplx a, o_cplx b) { o_cplx z = {a.r + b.r, a.i + b.i}; return z; }
static o_cplx c_sub(o_cplx a, o_cplx b) { o_cplx z = {a.r - b.r, a.i - b.i}; return z; }
/* (a+bi)(c+di) = (ac - bd) + (ad + bc)i */
static o_cplx c_mul(o_cplx A, o_cplx B) {
    double a = A.r, b = A.i, c = B.r, d = B.i;
    o_cplx z = {a * c - b * d, a * d + b * c};
    return z;
}
/* textbook division, no scaling: ((ac + bd) + (bc - ad)i) / (c^2 + d^2) */
static o_cplx c_div(o_cplx A, o_cplx B) {
    double a = A.r, b = A.i, c = B.r, d = B.i;
    double den = c * c + d * d;
    o_cplx z = {(a * c + b * d) / den, (b * c - a * d) / den};
    return z;
}
static double c_abs(o_cplx A) { return sqrt(A.r * A.r + A.i * A.i); }

/* fast_exp(x) = (1 + x/4096)^4096 by twelve squarings (SURVEY.md:629). */
double o_fast_exp(double x) {
    x = 1.0 + x * 0.000244140625;
    for (int k = 0; k < 12; k++) x = x * x;
    return x;
}
static o_cplx fast_cexp(o_cplx z) {
    o_cplx t5 = {o_fast_exp(z.r), 0.0};
    o_cplx t4 = {cos(z.i), sin(z.i)};
    return c_mul(t5, t4);
}

static const double O_AN[10] = {2.758402e-01, 2.245740e-01, 1.594149e-01, 9.866577e-02, 5.324414e-02,
                                2.505215e-02, 1.027747e-02, 3.676164e-03, 1.146494e-03, 3.117570e-04};
static const double O_DENL[10] = {9.869604e+00, 3.947842e+01, 8.882644e+01, 1.579137e+02, 2.467401e+02,
                                  3.553058e+02, 4.836106e+02, 6.316547e+02, 7.994380e+02, 9.869604e+02};
static const double O_NEG1N[10] = {-1.0, 1.0, -1.0, 1.0, -1.0, 1.0, -1.0, 1.0, -1.0, 1.0};
static const double O_QA = 0.512424224754768462984202823134979415014943561548661637413182;
static const double O_QB = 0.275255128608410950901357962647054304017026259671664935783653;
static const double O_QC = 0.051765358792987823963876628425793170829107067780337219430904;
static const double O_QD = 2.724744871391589049098642037352945695982973740328335064216346;

/* Faddeeva proxy: Abrarov-Quine (tau_m = 12, N = 10) if |Z| < 6, else the 4-point Gauss-Hermite
 * asymptotic form (SURVEY.md:620-632). */
void rso_fast_nuclear_W(double zr, double zi, double *wr, double *wi) {
    o_cplx Z = {zr, zi}, W;
    if (c_abs(Z) < 6.0) {
        o_cplx prefactor = {0.0, 8.124330e+01};
        o_cplx t1 = {0.0, 12.0}, t2 = {12.0, 0.0}, I = {0.0, 1.0}, one = {1.0, 0.0};
        W = c_div(c_mul(I, c_sub(one, fast_cexp(c_mul(t1, Z)))), c_mul(t2, Z));
        o_cplx sum = {0.0, 0.0};
        for (int n = 0; n < 10; n++) {
            o_cplx t3 = {O_NEG1N[n], 0.0};
            o_cplx top = c_sub(c_mul(t3, fast_cexp(c_mul(t1, Z))), one);
            o_cplx t4 = {O_DENL[n], 0.0}, t5 = {144.0, 0.0};
            o_cplx bot = c_sub(t4, c_mul(t5, c_mul(Z, Z)));
            o_cplx t6 = {O_AN[n], 0.0};
            sum = c_add(sum, c_mul(t6, c_div(top, bot)));
        }
        W = c_add(W, c_mul(prefactor, c_mul(Z, sum)));
    } else {
        o_cplx a = {O_QA, 0.0}, b = {O_QB, 0.0}, c = {O_QC, 0.0}, d = {O_QD, 0.0}, I = {0.0, 1.0};
        o_cplx Z2 = c_mul(Z, Z);
        W = c_mul(c_mul(Z, I), c_add(c_div(a, c_sub(Z2, b)), c_div(c, c_sub(Z2, d))));
    }
    *wr = W.r;
    *wi = W.i;
}

typedef struct {
    int n_nuc, numL, avg_poles, avg_windows;
    int num_nucs[12];
    int max_num_nucs;
    int *mats;
    double *concs;
    int *n_poles, *n_windows;
    long *pole_off, *win_off;  /* per-nuclide offsets into the flat arrays */
    double *pole;              /* [total_poles][8]: EA.r EA.i RT.r RT.i RA.r RA.i RF.r RF.i */
    int *pole_l;               /* [total_poles] */
    double *win;               /* [total_windows][3]: T A F */
    int *win_start, *win_end;  /* [total_windows]; end is inclusive as generated (R-RSEND) */
    double *K0RS;              /* [n_nuc][numL] */
    int doppler;               /* 1 (default): Doppler-broadened poles via W(z); 0: the 0 K kernel (R-RS0) */
} rs_oracle;

/* NEXT-3: select the 0 K (doppler = 0) or Doppler-broadened (doppler = 1) pole kernel. */
void rso_set_doppler(rs_oracle *o, int doppler) { o->doppler = doppler ? 1 : 0; }

/* RS data, one stream from `seed`, consumed in this order (SURVEY.md:594-603, R-RSGEN). */
rs_oracle *rso_create(int n_nuc, int avg_poles, int avg_windows, int numL, uint64_t seed) {
    if (numL != 4 || avg_poles < 1 || avg_windows < 1) return NULL;
    rs_oracle *o = (rs_oracle *)calloc(1, sizeof(rs_oracle));
    o->n_nuc = n_nuc;
    o->numL = numL;
    o->avg_poles = avg_poles;
    o->avg_windows = avg_windows;
    int mx = o_builtin_tables(n_nuc, o->num_nucs, NULL);
    if (mx < 0) {
        free(o);
        return NULL;
    }
    o->max_num_nucs = mx;
    o->mats = (int *)calloc(12 * (size_t)mx, sizeof(int));
    o_builtin_tables(n_nuc, o->num_nucs, o->mats);
    uint64_t s = seed;
    o->concs = (double *)calloc(12 * (size_t)mx, sizeof(double));
    for (int m = 0; m < 12; m++)
        for (int j = 0; j < o->num_nucs[m]; j++) o->concs[m * mx + j] = o_lcg_double(&s);
    o->n_poles = (int *)malloc(sizeof(int) * n_nuc);
    o->n_windows = (int *)malloc(sizeof(int) * n_nuc);
    for (int i = 0; i < n_nuc; i++) o->n_poles[i] = 1;
    for (long r = 0; r < (long)avg_poles * n_nuc - n_nuc; r++) o->n_poles[o_lcg_int(&s) % (uint64_t)n_nuc]++;
    for (int i = 0; i < n_nuc; i++) o->n_windows[i] = 1;
    for (long r = 0; r < (long)avg_windows * n_nuc - n_nuc; r++) o->n_windows[o_lcg_int(&s) % (uint64_t)n_nuc]++;
    o->pole_off = (long *)malloc(sizeof(long) * (n_nuc + 1));
    o->win_off = (long *)malloc(sizeof(long) * (n_nuc + 1));
    o->pole_off[0] = o->win_off[0] = 0;
    for (int i = 0; i < n_nuc; i++) {
        o->pole_off[i + 1] = o->pole_off[i] + o->n_poles[i];
        o->win_off[i + 1] = o->win_off[i] + o->n_windows[i];
    }
    long tp = o->pole_off[n_nuc], tw = o->win_off[n_nuc];
    o->pole = (double *)malloc(sizeof(double) * 8 * tp);
    o->pole_l = (int *)malloc(sizeof(int) * tp);
    for (int i = 0; i < n_nuc; i++)
        for (int j = 0; j < o->n_poles[i]; j++) {
            long p = o->pole_off[i] + j;
            for (int f = 0; f < 4; f++) { /* EA, RT, RA, RF */
                double r = o_lcg_double(&s);
                double im = o_lcg_double(&s);
                o->pole[p * 8 + 2 * f] = 152.5 * r;
                o->pole[p * 8 + 2 * f + 1] = 152.5 * im;
            }
            o->pole_l[p] = (int)(o_lcg_int(&s) % (uint64_t)numL);
        }
    o->win = (double *)malloc(sizeof(double) * 3 * tw);
    o->win_start = (int *)malloc(sizeof(int) * tw);
    o->win_end = (int *)malloc(sizeof(int) * tw);
    for (int i = 0; i < n_nuc; i++) {
        int space = o->n_poles[i] / o->n_windows[i];
        int rem = o->n_poles[i] - space * o->n_windows[i];
        int ctr = 0;
        for (int w = 0; w < o->n_windows[i]; w++) {
            long q = o->win_off[i] + w;
            o->win[q * 3 + 0] = o_lcg_double(&s);
            o->win[q * 3 + 1] = o_lcg_double(&s);
            o->win[q * 3 + 2] = o_lcg_double(&s);
            o->win_start[q] = ctr;
            o->win_end[q] = ctr + space - 1;
            ctr += space;
            if (w < rem) {
                ctr += 1;
                o->win_end[q] += 1;
            }
        }
    }
    o->K0RS = (double *)malloc(sizeof(double) * n_nuc * numL);
    for (int i = 0; i < n_nuc; i++)
        for (int l = 0; l < numL; l++) o->K0RS[i * numL + l] = o_lcg_double(&s);
    o->doppler = 1;
    return o;
}

void rso_free(rs_oracle *o) {
    if (!o) return;
    free(o->mats); free(o->concs); free(o->n_poles); free(o->n_windows); free(o->pole_off); free(o->win_off);
    free(o->pole); free(o->pole_l); free(o->win); free(o->win_start); free(o->win_end); free(o->K0RS);
    free(o);
}

/* Accessors for data-parity tests. */
long rso_total_poles(const rs_oracle *o) { return o->pole_off[o->n_nuc]; }
long rso_total_windows(const rs_oracle *o) { return o->win_off[o->n_nuc]; }
void rso_counts(const rs_oracle *o, int *n_poles, int *n_windows) {
    memcpy(n_poles, o->n_poles, sizeof(int) * o->n_nuc);
    memcpy(n_windows, o->n_windows, sizeof(int) * o->n_nuc);
}
void rso_data(const rs_oracle *o, double *pole, int *pole_l, double *win, int *win_start, int *win_end,
              double *K0RS, double *concs) {
    long tp = o->pole_off[o->n_nuc], tw = o->win_off[o->n_nuc];
    memcpy(pole, o->pole, sizeof(double) * 8 * tp);
    memcpy(pole_l, o->pole_l, sizeof(int) * tp);
    memcpy(win, o->win, sizeof(double) * 3 * tw);
    memcpy(win_start, o->win_start, sizeof(int) * tw);
    memcpy(win_end, o->win_end, sizeof(int) * tw);
    memcpy(K0RS, o->K0RS, sizeof(double) * o->n_nuc * o->numL);
    memcpy(concs, o->concs, sizeof(double) * 12 * o->max_num_nucs);
}

/* B2-B3: micro xs (sigT, sigA, sigF, sigE) of nuclide `nuc` at E, Doppler-broadened
 * (SURVEY.md:609-617), or at 0 K when o->doppler == 0 (NEXT-3, reading R-RS0).  *scale receives sum of |terms| (the R-UNIQ cancellation scale). */
static void rso_micro(const rs_oracle *o, int nuc, double E, double micro[4], double *scale) {
    double spacing = 1.0 / o->n_windows[nuc];
    int w = (int)(E / spacing);
    if (w == o->n_windows[nuc]) w--;
    if (w < 0) w = 0;
    if (w > o->n_windows[nuc] - 1) w = o->n_windows[nuc] - 1;
    o_cplx fac[4];
    for (int l = 0; l < 4; l++) {
        double phi = o->K0RS[nuc * o->numL + l] * sqrt(E);
        if (l == 1)
            phi -= -atan(phi);
        else if (l == 2)
            phi -= atan(3.0 * phi / (3.0 - phi * phi));
        else if (l == 3)
            phi -= atan(phi * (15.0 - phi * phi) / (15.0 - 6.0 * phi * phi));
        phi *= 2.0;
        fac[l].r = cos(phi);
        fac[l].i = -sin(phi);
    }
    long q = o->win_off[nuc] + w;
    double sigT = E * o->win[q * 3 + 0];
    double sigA = E * o->win[q * 3 + 1];
    double sigF = E * o->win[q * 3 + 2];
    double S = fabs(sigT) + fabs(sigA) + fabs(sigF);
    for (int p = o->win_start[q]; p < o->win_end[q]; p++) { /* [start, end): R-RSEND */
        const double *P = o->pole + (o->pole_off[nuc] + p) * 8;
        o_cplx EA = {P[0], P[1]}, RT = {P[2], P[3]}, RA = {P[4], P[5]}, RF = {P[6], P[7]};
        o_cplx W;
        if (o->doppler) {
            o_cplx Ec = {E, 0.0}, dopp = {0.5, 0.0};
            o_cplx Z = c_mul(c_sub(Ec, EA), dopp);
            rso_fast_nuclear_W(Z.r, Z.i, &W.r, &W.i);
        } else { /* 0 K (R-RS0): PSIIKI = i / (EA - sqrt(E)); CDUM = PSIIKI / E; W := CDUM */
            o_cplx t1 = {0.0, 1.0}, t2 = {sqrt(E), 0.0}, Ec = {E, 0.0};
            o_cplx psiiki = c_div(t1, c_sub(EA, t2));
            W = c_div(psiiki, Ec);
        }
        double t = c_mul(RT, c_mul(W, fac[o->pole_l[o->pole_off[nuc] + p]])).r;
        double a = c_mul(RA, W).r;
        double f = c_mul(RF, W).r;
        sigT += t;
        sigA += a;
        sigF += f;
        S += fabs(t) + fabs(a) + fabs(f);
    }
    micro[0] = sigT;
    micro[1] = sigA;
    micro[2] = sigF;
    micro[3] = sigT - sigA;
    *scale = S;
}

void rso_macro(const rs_oracle *o, double E, int mat, double macro[4], double *scale) {
    double S = 0.0;
    for (int c = 0; c < 4; c++) macro[c] = 0.0;
    for (int j = 0; j < o->num_nucs[mat]; j++) {
        int nuc = o->mats[mat * o->max_num_nucs + j];
        double conc = o->concs[mat * o->max_num_nucs + j];
        double micro[4], s;
        rso_micro(o, nuc, E, micro, &s);
        for (int c = 0; c < 4; c++) macro[c] += micro[c] * conc;
        S += s * fabs(conc);
    }
    if (scale) *scale = S;
}

/* B4: v = 1 + first strict maximum, starting from -DBL_MAX (R-ARGMAX). */
int o_argmax4_plus1(const double macro[4]) {
    double mx = -DBL_MAX;
    int idx = 0;
    for (int c = 0; c < 4; c++)
        if (macro[c] > mx) {
            mx = macro[c];
            idx = c;
        }
    return idx + 1;
}

uint64_t rso_lookup_batch(const rs_oracle *o, uint64_t first, uint64_t n, uint64_t seed, double *macro_out,
                          double *scale_out, int nthreads) {
    uint64_t raw = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : raw)
    for (long long t = 0; t < (long long)n; t++) {
        double E, macro[4], S;
        int mat;
        o_sample(first + (uint64_t)t, seed, &E, &mat);
        rso_macro(o, E, mat, macro, &S);
        raw += (uint64_t)o_argmax4_plus1(macro);
        if (macro_out)
            for (int c = 0; c < 4; c++) macro_out[(size_t)t * 4 + c] = macro[c];
        if (scale_out) scale_out[t] = S;
    }
    return raw;
}

uint64_t rso_lookup_indices(const rs_oracle *o, const uint64_t *idx, uint64_t n, uint64_t seed,
                            double *macro_out, double *scale_out) {
    uint64_t raw = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : raw)
    for (long long t = 0; t < (long long)n; t++) {
        double E, macro[4], S;
        int mat;
        o_sample(idx[t], seed, &E, &mat);
        rso_macro(o, E, mat, macro, &S);
        raw += (uint64_t)o_argmax4_plus1(macro);
        if (macro_out)
            for (int c = 0; c < 4; c++) macro_out[(size_t)t * 4 + c] = macro[c];
        if (scale_out) scale_out[t] = S;
    }
    return raw;
}

/* RSBench history-based mode (NEXT-1; reading R-HIST-RS).  Particle p (GLOBAL
 * index) runs L dependent lookups:
 *     s = fast_forward(seed, p * L * 2);  E = lcg_double(&s);  mat = pick_mat(lcg_double(&s))
 *     for i in 0 .. L-1:
 *         macro = lookup(E, mat);  raw += 1 + argmax4(macro)
 *         for x in 0..3: s += (macro[x] > 0) ? 1337 * p : 42          (u64 wraparound)
 *         E = lcg_double(&s);  mat = pick_mat(lcg_double(&s))
 * macro_out: NULL or [n_p][L][4]; scale_out: NULL or [n_p][L] (the R-UNIQ scale S). */
uint64_t rso_history_batch(const rs_oracle *o, uint64_t first_p, uint64_t n_p, int L, uint64_t seed,
                           double *macro_out, double *scale_out, int nthreads) {
    uint64_t raw = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : raw)
    for (long long t = 0; t < (long long)n_p; t++) {
        uint64_t p = first_p + (uint64_t)t;
        uint64_t s = o_fast_forward(seed, p * (uint64_t)L * 2ULL);
        double E = o_lcg_double(&s);
        int mat = o_pick_mat(o_lcg_double(&s));
        for (int i = 0; i < L; i++) {
            double macro[4], S;
            rso_macro(o, E, mat, macro, &S);
            raw += (uint64_t)o_argmax4_plus1(macro);
            if (macro_out)
                for (int c = 0; c < 4; c++) macro_out[((size_t)t * L + i) * 4 + c] = macro[c];
            if (scale_out) scale_out[(size_t)t * L + i] = S;
            for (int x = 0; x < 4; x++) s += (macro[x] > 0.0) ? 1337ULL * p : 42ULL;
            E = o_lcg_double(&s);
            mat = o_pick_mat(o_lcg_double(&s));
        }
    }
    return raw;
}

int o_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ================================================================ NEXT-4: page-rank propagation
 * HeCBench page-rank, "the propagation step is measured" (Fig. 9c; SURVEY.md
 * Sec. 8(f) NEXT-4).  The paper gives no generator or formula; readings R-PR-GRAPH / R-PR-STEP
 * (DESIGN.md Sec. 3):
 *   graph: N nodes; node u draws from s = fast_forward(seed, 2 D u): out-degree
 *          d_u = 1 + floor(lcg_double(&s) * (2 D - 1)), then d_u targets v = floor(lcg_double(&s) * N)
 *          (clamped to N - 1); in-edges of v are ordered by (u, j) -- j the draw order.
 *   step:  contrib[u] = r[u] / d_u;  r'[v] = (1 - 0.85) / N + 0.85 * (sum over in-edges in order of
 *          contrib[u]), every operation fp64 round-to-nearest, sums left to right. */
typedef struct {
    long n, nnz;
    int D;
    long *rowptr;   /* [n + 1] in-edge CSR by destination */
    int32_t *col;   /* [nnz] source of each in-edge */
    int32_t *outdeg;/* [n] */
} pr_oracle;

pr_oracle *pro_create(long n, int D, uint64_t seed) {
    if (n < 1 || D < 1) return NULL;
    pr_oracle *o = (pr_oracle *)calloc(1, sizeof(pr_oracle));
    o->n = n;
    o->D = D;
    o->outdeg = (int32_t *)malloc(sizeof(int32_t) * n);
    o->rowptr = (long *)calloc((size_t)n + 1, sizeof(long));
    /* pass 1: degrees and in-degree counts */
    for (long u = 0; u < n; u++) {
        uint64_t s = o_fast_forward(seed, 2ULL * (uint64_t)D * (uint64_t)u);
        int d = 1 + (int)(o_lcg_double(&s) * (double)(2 * D - 1));
        if (d > 2 * D - 1) d = 2 * D - 1;
        o->outdeg[u] = d;
        for (int j = 0; j < d; j++) {
            long v = (long)(o_lcg_double(&s) * (double)n);
            if (v > n - 1) v = n - 1;
            o->rowptr[v + 1]++;
        }
    }
    for (long v = 0; v < n; v++) o->rowptr[v + 1] += o->rowptr[v];
    o->nnz = o->rowptr[n];
    o->col = (int32_t *)malloc(sizeof(int32_t) * (size_t)(o->nnz > 0 ? o->nnz : 1));
    long *fill = (long *)malloc(sizeof(long) * n);
    memcpy(fill, o->rowptr, sizeof(long) * n);
    /* pass 2: sources in (u, j) order -- appending in generation order keeps rows sorted */
    for (long u = 0; u < n; u++) {
        uint64_t s = o_fast_forward(seed, 2ULL * (uint64_t)D * (uint64_t)u);
        (void)o_lcg_double(&s);
        for (int j = 0; j < o->outdeg[u]; j++) {
            long v = (long)(o_lcg_double(&s) * (double)n);
            if (v > n - 1) v = n - 1;
            o->col[fill[v]++] = (int32_t)u;
        }
    }
    free(fill);
    return o;
}

void pro_free(pr_oracle *o) {
    if (!o) return;
    free(o->rowptr);
    free(o->col);
    free(o->outdeg);
    free(o);
}

long pro_nnz(const pr_oracle *o) { return o->nnz; }
void pro_arrays(const pr_oracle *o, long *rowptr, int32_t *col, int32_t *outdeg) {
    memcpy(rowptr, o->rowptr, sizeof(long) * (o->n + 1));
    memcpy(col, o->col, sizeof(int32_t) * o->nnz);
    memcpy(outdeg, o->outdeg, sizeof(int32_t) * o->n);
}

/* R-PR-STEP on any in-edge CSR (also used by the pins with hand-made graphs). */
void pro_propagate_csr(long n, const long *rowptr, const int32_t *col, const int32_t *outdeg, const double *r,
                       double *out, int nthreads) {
    double *contrib = (double *)malloc(sizeof(double) * n);
    const double base = (1.0 - 0.85) / (double)n;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(static)
    for (long u = 0; u < n; u++) contrib[u] = r[u] / (double)outdeg[u];
#pragma omp parallel for schedule(dynamic, 1024)
    for (long v = 0; v < n; v++) {
        double s = 0.0;
        for (long e = rowptr[v]; e < rowptr[v + 1]; e++) s = s + contrib[col[e]];
        out[v] = base + 0.85 * s;
    }
    free(contrib);
}

void pro_propagate(const pr_oracle *o, const double *r, double *out, int nthreads) {
    pro_propagate_csr(o->n, o->rowptr, o->col, o->outdeg, r, out, nthreads);
}

/* ================================================================ NEXT-4: AMGmk relax
 * "The first measures only the relax kernel of the original AMGmk proxy application".
 * Readings R-AMG-MAT / R-AMG-RELAX: the 27-point Laplacian on an nx x ny x nz grid
 * (row i = x + nx (y + ny z)), CSR with the diagonal (26) first and then the existing neighbours (-1)
 * in increasing column order; one Jacobi relaxation sweep
 *     u'[i] = (f[i] - sum_{jj > first} a[jj] u[col[jj]]) / a[first],
 * fp64 round-to-nearest, the row sum from the right-hand side down, left to right. */
long amo_nnz(int nx, int ny, int nz) {
    long c = 0;
    for (int z = 0; z < nz; z++)
        for (int y = 0; y < ny; y++)
            for (int x = 0; x < nx; x++) {
                int cnt = 0;
                for (int dz = -1; dz <= 1; dz++)
                    for (int dy = -1; dy <= 1; dy++)
                        for (int dx = -1; dx <= 1; dx++) {
                            int X = x + dx, Y = y + dy, Z = z + dz;
                            if (X >= 0 && X < nx && Y >= 0 && Y < ny && Z >= 0 && Z < nz) cnt++;
                        }
                c += cnt;
            }
    return c;
}

void amo_matrix(int nx, int ny, int nz, long *rowptr, int32_t *col, double *val) {
    long e = 0, i = 0;
    rowptr[0] = 0;
    for (int z = 0; z < nz; z++)
        for (int y = 0; y < ny; y++)
            for (int x = 0; x < nx; x++, i++) {
                col[e] = (int32_t)i;
                val[e++] = 26.0;
                for (int dz = -1; dz <= 1; dz++)
                    for (int dy = -1; dy <= 1; dy++)
                        for (int dx = -1; dx <= 1; dx++) {
                            if (!dx && !dy && !dz) continue;
                            int X = x + dx, Y = y + dy, Z = z + dz;
                            if (X >= 0 && X < nx && Y >= 0 && Y < ny && Z >= 0 && Z < nz) {
                                col[e] = (int32_t)(X + (long)nx * (Y + (long)ny * Z));
                                val[e++] = -1.0;
                            }
                        }
                rowptr[i + 1] = e;
            }
}

void amo_relax(long n, const long *rowptr, const int32_t *col, const double *val, const double *f, const double *u,
               double *out, int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; i++) {
        double res = f[i];
        for (long jj = rowptr[i] + 1; jj < rowptr[i + 1]; jj++) res = res - val[jj] * u[col[jj]];
        out[i] = res / val[rowptr[i]];
    }
}
