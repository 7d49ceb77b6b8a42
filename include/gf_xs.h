/*
 * gf_xs.h -- C ABI of the B200-native XSBench / RSBench macroscopic cross-section lookup.
 *
 * The operation is the data-parallel loop that GPU First (arXiv 2306.11686) runs on the GPU:
 * "two alternative methods are available to perform the cross-section lookup as part of the
 * neutron transport simulation: event-based lookup and history-based lookup" (PAPER.md:1408,
 * Sec. 5.3.1 "XSBench and RSBench"; Fig. 8), on XSBench
 * v20 / RSBench v13 inputs of "two different input sizes".  The paper states no
 * more than that; the step-by-step semantics this library implements are the readings recorded
 * in DESIGN.md Sec. 3 (taken from SURVEY.md Sec. 8(c)).  The entry-point names follow
 * BASELINE.json's north_star: gf_xs_grid_init, gf_xs_lookup_batch, gf_xs_verify.
 *
 * Conventions (all functions):
 *   - extern "C", noexcept: nothing throws across the boundary or aborts the process.  Faults are
 *     returned as gf_status values; gf_xs_last_error() gives a thread-local message for the last
 *     non-OK status.
 *   - Ownership: the CALLER owns every byte of device memory (e.g. torch.empty(..., device='cuda')).
 *     The library never allocates device memory.  A gf_xs_grid handle holds non-owning views into
 *     caller memory; the caller keeps that memory alive until gf_xs_grid_free().
 *   - Asynchrony: argument validation is synchronous (GF_E_INVAL is returned before anything is
 *     enqueued).  Device work is enqueued on `stream` (0 = legacy default stream) and the call
 *     returns after enqueue, except where GF_HOST_IO is set (see below).  Device faults surface as
 *     GF_E_CUDA at the next call or at the caller's synchronisation.
 *   - Device: every call runs on the CUDA device that was current when the grid was initialised;
 *     the library sets it for the duration of a call and restores the caller's current device.
 *   - Threading: a grid is immutable after init.  Concurrent lookup calls on different streams are
 *     legal if their scratch buffers and outputs do not alias.
 *   - There is no CPU fallback: without a usable sm_100a device every compute call returns
 *     GF_E_CUDA (or GF_E_UNSUPPORTED).
 */
#ifndef GF_XS_H
#define GF_XS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GF_XS_ABI_VERSION 1u
#define GF_HASH_MODULUS 999983ull /* BASELINE.json north_star: "argmax-of-5 index summed mod 999983" */

typedef struct CUstream_st *gf_stream_t; /* == cudaStream_t */

typedef enum {
    GF_OK = 0,
    GF_E_INVAL = 1,       /* bad argument; nothing was enqueued */
    GF_E_NOMEM = 2,       /* a caller buffer is smaller than the matching *_bytes() query */
    GF_E_CUDA = 3,        /* CUDA runtime / launch / device fault (message has cudaGetErrorString) */
    GF_E_UNSUPPORTED = 4, /* a valid request this build does not implement (e.g. history mode) */
    GF_E_MISMATCH = 5     /* gf_xs_verify: hash differs from the expected value */
} gf_status;

typedef enum { GF_XSBENCH = 0, GF_RSBENCH = 1 } gf_bench;

/* XSBench energy-grid acceleration: plain per-nuclide bisection, the
 * unionized grid with its index grid, or the hash grid with `hash_bins` bins. */
typedef enum { GF_GRID_NUCLIDE = 0, GF_GRID_UNIONIZED = 1, GF_GRID_HASH = 2 } gf_grid_type;

typedef struct {
    uint32_t abi_version;   /* must equal GF_XS_ABI_VERSION */
    int32_t bench;          /* gf_bench */
    int32_t n_isotopes;     /* 68 = small, 355 = large (built-in tables); any >= 1 with custom tables */
    int64_t n_gridpoints;   /* XS: gridpoints per nuclide, 11303 in both sizes (XL 238,847); 2 <= n <= 2^20;
                               the unionized grid needs <= 65,536 points per nuclide per band */
    int32_t grid_type;      /* XS: gf_grid_type */
    int32_t hash_bins;      /* XS hash grid: bins (10000); >= 1 */
    int32_t avg_n_poles;    /* RS: average poles per nuclide (1000); >= 1 */
    int32_t avg_n_windows;  /* RS: average windows per nuclide (100); >= 1 */
    int32_t numL;           /* RS: must be 4 */
    int32_t doppler;        /* RS: 1 = Doppler-broadened poles through the Faddeeva function (default);
                               0 = the 0 K kernel, sigma += Re(R i / ((EA - sqrt E) E) [fac_l])
                               (NEXT-3, reading R-RS0); other values GF_E_INVAL */
    uint64_t init_seed;     /* grid / data generation LCG seed (42) */
    const int32_t *num_nucs;/* NULL = built-in Hoogenboom-Martin tables; else HOST int32[12] ...   */
    const int32_t *mats;    /* ... and HOST int32[12 * max_num_nucs] row-major nuclide ids        */
    int32_t max_num_nucs;   /* row length of `mats` when custom tables are given                  */
    int32_t n_bands;        /* NEXT-2 energy-band sharding of the UNIONIZED grid: 1 = whole grid     */
    int32_t band;           /* (default).  With W = n_bands > 1 this grid replica holds the unionized */
                            /* energies and index grid of band r = `band` only: E in [r/W, (r+1)/W),   */
                            /* band 0 open below, band W-1 open above; the nuclide grid stays whole.   */
                            /* Its lookup calls process only the lookups whose E falls in the band, so */
                            /* W replicas (one per GPU) sum to the whole batch.  Needed when the whole */
                            /* index grid does not fit (XL: 355 x 84.8 M entries).  Sorted event       */
                            /* lookups only (GF_SORT_LOCALITY); other calls GF_E_UNSUPPORTED.          */
} gf_xs_params;

/* Fills *p with the defaults of BASELINE.json configs[2] (XSBench large, unionized) for
 * bench = GF_XSBENCH, or configs[4] (RSBench large) for GF_RSBENCH.  Host-only. */
gf_status gf_xs_default_params(int32_t bench, gf_xs_params *p);

typedef struct gf_xs_grid gf_xs_grid; /* opaque; immutable after init */

/* Sizes (bytes) of the caller-owned grid buffer and of the init-only scratch buffer.
 * Host-only; no CUDA calls.  Both buffers must be device memory, 256-byte aligned. */
gf_status gf_xs_grid_bytes(const gf_xs_params *p, size_t *grid_bytes, size_t *init_scratch_bytes);

/* A0 ("data initialization is also performed on the GPU"):
 * builds every grid array on `device` into grid_mem, asynchronously on `stream`.  The scratch
 * buffer may be reused by the caller once the stream has passed the init work.  *out receives a
 * host handle (free with gf_xs_grid_free). */
gf_status gf_xs_grid_init(const gf_xs_params *p, int device, void *grid_mem, size_t grid_bytes, void *scratch,
                          size_t scratch_bytes, gf_stream_t stream, gf_xs_grid **out);

/* Frees the handle only; the buffers belong to the caller.  NULL is a no-op. */
gf_status gf_xs_grid_free(gf_xs_grid *g);

/* Read-only device views of the grid arrays, for tests and tools.  Layouts (all row-major):
 *   GF_ARR_NUCLIDE_GRID  double [n_iso][n_gp][6]  (E, total, elastic, absorption, fission, nu-fission)
 *   GF_ARR_ENERGY        double [n_iso][n_gp]     (E column, SoA copy used by the searches)
 *   GF_ARR_UNIONIZED     double [n_iso*n_gp]      (unionized grid only)
 *   GF_ARR_INDEX_GRID    uint16 [n_iso][pitch]    nuclide-major IG, pitch = *pitch_out >= n_iso*n_gp
 *   GF_ARR_HASH_GRID     uint16 [n_iso][pitch]    nuclide-major HG, pitch >= hash_bins
 *   GF_ARR_UNION_BINS    uint32 [2^20 + 1]        #{U < b / 2^20}: top level of the unionized search
 *   GF_ARR_RECIP_WIDTH   double [n_iso][n_gp]     RN(1 / (E[k+1] - E[k])) per interval (exact division)
 *   GF_ARR_NUCLIDE_BINS  uint16 [n_iso][pitch]    unionized whole grids with n_gp < 65536: #{E_nuc <= b / 2^14},
 *                                                 b = 0..2^14 -- the sparse-batch search (history waves)
 *   GF_ARR_INTERVALS     double [n_iso][n_gp][16] unionized / hash grids: per interval k < n_gp-1 the
 *                        sorted kernel's 128-B record E[k+1], E[k+1]-E[k], (xs_c[k+1], xs_c[k+1]-xs_c[k])
 *                        for c = 0..4, RN(1/(E[k+1]-E[k])), E[k], 0, 0 (all RN); record n_gp-1 is zero
 *   GF_ARR_CONCS         double [total]           concentrations in (material, j) order
 *   GF_ARR_MAT_NUCS      int32  [total]           nuclide ids in (material, j) order
 *   GF_ARR_MAT_OFFSETS   int32  [13]              CSR offsets of the two arrays above
 *   GF_ARR_THRESHOLDS    double [12]              pick_mat thresholds T[m]
 *   GF_ARR_RS_POLES      double [total_poles][8]  EA, RT, RA, RF (re, im)         (RSBench)
 *   GF_ARR_RS_POLE_L     int32  [total_poles]                                      (RSBench)
 *   GF_ARR_RS_WINDOWS    double [total_windows][4] T, A, F, (int start, int end) packed  (RSBench)
 *   GF_ARR_RS_K0RS       double [n_iso][4]                                         (RSBench)
 *   GF_ARR_RS_POLE_OFF   int32  [n_iso+1], GF_ARR_RS_WIN_OFF int32 [n_iso+1]       (RSBench)
 * Returns GF_E_INVAL for an array this grid does not have. */
typedef enum {
    GF_ARR_NUCLIDE_GRID = 0, GF_ARR_ENERGY = 1, GF_ARR_UNIONIZED = 2, GF_ARR_INDEX_GRID = 3, GF_ARR_HASH_GRID = 4,
    GF_ARR_CONCS = 5, GF_ARR_MAT_NUCS = 6, GF_ARR_MAT_OFFSETS = 7, GF_ARR_THRESHOLDS = 8,
    GF_ARR_RS_POLES = 9, GF_ARR_RS_POLE_L = 10, GF_ARR_RS_WINDOWS = 11, GF_ARR_RS_K0RS = 12,
    GF_ARR_RS_POLE_OFF = 13, GF_ARR_RS_WIN_OFF = 14, GF_ARR_UNION_BINS = 15,
    GF_ARR_RECIP_WIDTH = 16, GF_ARR_INTERVALS = 17, GF_ARR_NUCLIDE_BINS = 18
} gf_array;
gf_status gf_xs_grid_array(const gf_xs_grid *g, int32_t which, const void **ptr, size_t *bytes, int64_t *pitch_out);

/* Lookup flags. */
enum {
    GF_SORT_LOCALITY = 1u << 0, /* A2: bin lookups by (material, energy) before the lookup kernel
                                   (default in bench).  Results are identical either way. */
    GF_HISTORY = 1u << 1,       /* history-based mode is a separate call (gf_xs_history_batch): in
                                   the event-lookup calls this flag returns GF_E_UNSUPPORTED */
    GF_HOST_IO = 1u << 2,       /* outputs (and, for gf_xs_lookup_energies, inputs) are HOST
                                   pointers; the call stages them through `scratch`, copies inside
                                   the call and synchronises `stream` before returning */
    GF_HIST_WAVES = 1u << 3     /* gf_xs_history_batch: run step i of all particles as one event-style
                                   batch (implied by GF_SORT_LOCALITY); without it, one thread per
                                   particle runs its L lookups back to back */
};

/* Scratch bytes a lookup call of n lookups with `flags` needs (caller allocates on the device).  With
 * GF_HOST_IO this is the chunked pipeline's bound (two 2^22-lookup chunk slots): device memory does not
 * grow with n. */
gf_status gf_xs_batch_bytes(const gf_xs_grid *g, uint64_t n_lookups, uint32_t flags, size_t *scratch_bytes);
/* The larger scratch of the whole-batch host-I/O mode (gf_xs_lookup_energies, GF_HOST_IO |
 * GF_SORT_LOCALITY, no per-lookup outputs): the chunk copies overlap the sort's counting pass, then one
 * sort and one lookup pass run over the whole batch (O(n) device scratch, ~25 B per lookup).  A call
 * given at least this much scratch runs that mode; with less, the chunked pipeline (same results). */
gf_status gf_xs_batch_bytes_whole(const gf_xs_grid *g, uint64_t n_lookups, uint32_t flags, size_t *scratch_bytes);

/* A1-A6 / B1-B4: event-based lookups with GLOBAL indices [first, first+n).
 * Lookup i samples (E, material) from the LCG stream fast_forward(starting_seed, 2i) (1070 in the
 * benchmarks), finds each nuclide's energy interval with the grid's search, interpolates the 5
 * (XS) micro cross sections or evaluates the windowed multipole poles (RS), accumulates them by
 * concentration and takes v_i = 1 + argmax over the channels.
 *   d_macro_out: NULL, or fp64 [n][5] (XS) / [n][4] (RS), row i - first, original order.
 *   d_vsum:      uint64; the call ADDS sum(v_i) to it (caller zeroes it), so batches and shards
 *                compose by integer addition; the hash is computed once at the end (gf_xs_verify).
 * n must be < 2^32 per call (split larger jobs into batches).  n == 0 enqueues nothing. */
gf_status gf_xs_lookup_batch(const gf_xs_grid *g, uint64_t first, uint64_t n, uint64_t starting_seed, uint32_t flags,
                             double *d_macro_out, uint64_t *d_vsum, void *scratch, size_t scratch_bytes,
                             gf_stream_t stream);

/* Stage timing (bench / profiling): cudaEvent_t handles (as void*; any may be NULL) recorded on
 * `stream` before the sort stage (A1-A2), between it and the lookup kernel (A3-A6), and after the
 * lookup kernel.  Without GF_SORT_LOCALITY the first two coincide. */
typedef struct {
    void *before_sort;
    void *before_lookup;
    void *after_lookup;
} gf_stage_events;

/* gf_xs_lookup_batch with stage events; identical launches and results. */
gf_status gf_xs_lookup_batch_ev(const gf_xs_grid *g, uint64_t first, uint64_t n, uint64_t starting_seed,
                                uint32_t flags, double *d_macro_out, uint64_t *d_vsum, void *scratch,
                                size_t scratch_bytes, gf_stream_t stream, const gf_stage_events *ev);

/* Same lookup for CALLER-SUPPLIED particle states (a transport code's energies and materials):
 * E[n] finite (the method samples [0, 1); other finite energies follow the literal algorithm, e.g.
 * hash bin / RS window clamped at 0), mat[n] in 0..11.  Device pointers, or host pointers with
 * GF_HOST_IO.  macro_out [n][5|4] (may be NULL) and vsum as in gf_xs_lookup_batch.
 * Inputs outside that domain (mat > 11, NaN or +-inf energies) are errors.  They cannot be checked
 * before enqueue without reading device memory, so the kernels that read the inputs flag them: bit 63
 * of *vsum is set (a valid raw sum is < 2^63) and gf_xs_verify returns GF_E_INVAL for such a sum; the
 * other lookups' results are still computed and the flagged ones' outputs are unspecified.  With
 * GF_HOST_IO the call completes before returning and returns GF_E_INVAL itself (*vsum untouched). */
gf_status gf_xs_lookup_energies(const gf_xs_grid *g, const double *E, const uint8_t *mat, uint64_t n, uint32_t flags,
                                double *macro_out, uint64_t *vsum, void *scratch, size_t scratch_bytes,
                                gf_stream_t stream);

/* Streaming form of the host-I/O call, for back-to-back batches: caller energies and materials from
 * (pinned) HOST memory, everything ENQUEUED on `stream` with no host wait -- the copies of E[n] (8 B) and
 * mat[n] (1 B) into the scratch, the sorted lookup (flags must be GF_SORT_LOCALITY: the whole-batch sort,
 * PAPER.md:1408 event lookups), and the raw sum ADDED to the DEVICE accumulator *d_vsum.  A caller
 * alternating two scratch buffers on two streams overlaps batch k+1's copies with batch k's lookups.
 * The host arrays must stay unchanged and the scratch unused until the stream has passed this call.
 * Scratch: gf_xs_batch_bytes_whole(g, n, GF_SORT_LOCALITY | GF_HOST_IO).  No per-lookup outputs.
 * Invalid inputs (mat > 11, non-finite E) set bit 63 of *d_vsum (gf_xs_verify: GF_E_INVAL).  Not for
 * band grids (their batches are sampled).  n < 2^32. */
gf_status gf_xs_lookup_energies_async(const gf_xs_grid *g, const double *E_host, const uint8_t *mat_host, uint64_t n,
                                      uint32_t flags, uint64_t *d_vsum, void *scratch, size_t scratch_bytes,
                                      gf_stream_t stream);

/* NEXT-1: HISTORY-BASED lookups, PAPER.md:1408 ("event-based lookup and
 * history-based lookup").  Particles with GLOBAL indices [first_particle, first_particle + n_particles)
 * each run `lookups_per_particle` (L, 34 in XSBench / RSBench) DEPENDENT lookups; the readings
 * are
 *   XSBench (R-HIST):    s = fast_forward(seed, 8 L p); E, mat drawn; after each lookup
 *                        s = fast_forward(s, #{c : macro_c > 1.0}), then E, mat drawn again.
 *   RSBench (R-HIST-RS): s = fast_forward(seed, 2 L p); E, mat drawn; after each lookup
 *                        s += (macro_c > 0 ? 1337 p : 42) for c = 0..3 (u64), then E, mat drawn.
 * flags: 0 = one thread per particle (GPU First's mapping of the particle loop); GF_HIST_WAVES =
 * step-synchronous waves of n_particles event lookups; GF_SORT_LOCALITY (implies waves) = waves with
 * the A2 locality sort.  Results are identical in every mode.
 *   d_macro_out: NULL, or fp64 [n_particles][L][5] (XS) / [n_particles][L][4] (RS), row
 *                (p - first_particle) * L + i.
 *   d_vsum:      uint64; the call ADDS sum(1 + argmax) over all n_particles * L lookups.
 * n_particles < 2^32, 1 <= L <= 2^20.  Enqueued on `stream`; scratch from gf_xs_history_bytes.
 * (RSBench: the sign test macro_c > 0 decides the stream.  The RS macro xs agree with the oracle to
 * 1e-10 S (R-UNIQ), so a channel within that distance of 0 could branch differently; the parity
 * tests report the smallest |macro_c| / S seen.) */
gf_status gf_xs_history_bytes(const gf_xs_grid *g, uint64_t n_particles, uint32_t flags, size_t *scratch_bytes);
gf_status gf_xs_history_batch(const gf_xs_grid *g, uint64_t first_particle, uint64_t n_particles,
                              int32_t lookups_per_particle, uint64_t starting_seed, uint32_t flags,
                              double *d_macro_out, uint64_t *d_vsum, void *scratch, size_t scratch_bytes,
                              gf_stream_t stream);

/* Grid facts: *fastdiv = 1 when the lookup kernels use the exact reciprocal division (every
 * interval of the nuclide grid has a normal, non-zero width), 0 when they use __ddiv_rn. */
gf_status gf_xs_grid_info(const gf_xs_grid *g, int32_t *fastdiv);

/* A/B and test hook: forces the kernel of the sorted lookup path of an XSBench grid (default: chosen
 * at grid init -- the warp-tile kernel for batches of at least tile_min lookups, one lookup per thread
 * below).  kern: GF_KERN_AUTO, or one kernel for every batch size; tile_min: the auto crossover
 * (0 = keep); nb_on: sparse batches and nuclide grids search the per-nuclide bin brackets (1) or the
 * index grid / warp search (0).  Every choice gives bit-identical results.  Not synchronised with
 * lookups in flight on the same grid: call it between batches.  GF_E_INVAL for an unknown kernel or
 * an RSBench grid. */
enum { GF_KERN_AUTO = 0, GF_KERN_GROUP = 1, GF_KERN_THREAD = 2, /* 3 retired */ GF_KERN_TILE = 4,
       GF_KERN_TILE_NB = 5, GF_KERN_WARP_SEARCH = 6 };
gf_status gf_xs_debug_set_kernel(gf_xs_grid *g, int32_t kern, uint64_t tile_min, int32_t nb_on);
/* Test hook: ieee = 1 makes the lookup kernels of this grid divide with IEEE __ddiv_rn (the path grids
 * with a zero-width interval take) instead of the exact reciprocal scheme; ieee = 0 restores the
 * grid's own choice.  Results are bit-identical either way (both give the RN quotient). */
gf_status gf_xs_debug_set_division(gf_xs_grid *g, int32_t ieee);
/* Test hook: unionized warp-tile batches of at least n lookups (default 2^23) find each tile's union
 * indices per tile (one pass before the lookup kernel) and search the rare leftover lookups by bisection;
 * smaller ones use per-lookup union indices.  Identical results either way. */
gf_status gf_xs_debug_set_prep_min(gf_xs_grid *g, uint64_t n);
/* The sorted-path kernel (GF_KERN_*) a batch of n lookups with `flags` runs on this grid (the nuclide
 * grid reports GF_KERN_THREAD for its NB-bracket kernel); -1 for RSBench grids and unsorted batches,
 * which have one kernel each.  For reports (bench) and tests. */
gf_status gf_xs_kernel_for(const gf_xs_grid *g, uint64_t n, uint32_t flags, int32_t *kern);

/* Diagnostics: d_out[i] = the lookup kernels' reciprocal division of d_a[i] by d_b[i] (device
 * arrays of n doubles), d_ref[i] = IEEE a / b (__ddiv_rn).  The two must agree bit for bit for
 * |a| <= 4 and normal non-zero b.  Enqueued on `stream`. */
gf_status gf_xs_selftest_div(const double *d_a, const double *d_b, double *d_out, double *d_ref, uint64_t n,
                             gf_stream_t stream);

/* Host-only finalisation: *hash = raw_sum % 999983 (R-MOD: once, after all batches and shards).
 * If expected != UINT64_MAX and *hash != expected, returns GF_E_MISMATCH (hash still written).
 * A raw sum with bit 63 set carries the invalid-input flag of gf_xs_lookup_energies: GF_E_INVAL,
 * *hash not written. */
gf_status gf_xs_verify(uint64_t raw_sum, uint64_t expected, uint64_t *hash);

/* Thread-local text for the last non-OK status returned on this thread ("" if none). */
const char *gf_xs_last_error(void);

/* Build identification: "gf_xs <abi> sm_100a <nvcc version>". */
const char *gf_xs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GF_XS_H */
