// xs_lookup.cu -- A1-A6: the XSBench event-based lookup on sm_100a.
//
//   A1  sampling        lookup i draws (E, material) from fast_forward(seed, 2i).  A thread handles
//                       a run of consecutive lookups: one skip-ahead, then 2 LCG steps per lookup.
//   A2  locality sort   counting sort by (material, energy bin): count -> two-kernel scan -> scatter
//                       of E (and the original position when per-lookup outputs are requested).
//                       Results are order-independent (integer hash; outputs go back by position).
//   A3  energy search   unionized: two-level search of U (the 2^20-bin table ubin narrows the
//                       bisection to one energy bin; same result as XSBench's grid_search, which is
//                       clamp(#{U <= E} - 1, 0, n-2)); hash: (int64)(E / (1.0/bins)); nuclide: per
//                       nuclide bisection of the SoA energy column.
//   A4  micro xs        per nuclide of the material, in table order: interval k (u16 index grid),
//                       the 96-B record pair as 6 x 16-B vector loads, f and the 5 interpolations.
//                       f's IEEE quotient comes from the per-interval reciprocal (div_rn, exact;
//                       5 FP64 instructions instead of ~13).  Software-pipelined with two pair
//                       buffers: the pair of nuclide j+1 and the interval of j+2 are in flight while
//                       j is accumulated; the sorted unionized kernel also prefetches the index-grid
//                       line kPrefetch nuclides ahead into L2.
//   A5  macro xs        macro_c += micro_c * conc_c, RN multiply then RN add, j ascending.
//   A6  hash            v = 1 + argmax (first strict max above -1.0); warp redux -> SMEM -> one u64
//                       atomic per CTA.
// Material tables (CSR: offsets / nuclide ids / concentrations) and pick_mat thresholds are staged
// in shared memory per CTA.
#include "gf_internal.cuh"

namespace gf {

constexpr int kLookupTpb = 128;  // lookup CTA size
constexpr int kPrefetch = 8;     // nuclides of index-grid L2 prefetch lookahead

// A1/A2 (sampling, locality sort): sort.cu.
static inline unsigned nblk(long long n, int b) { return (unsigned)((n + b - 1) / b); }

// ------------------------------------------------------------------------------------------ A3
// Per-lookup energy-grid index: u (unionized) or b (hash); unused for the nuclide grid.
template <int GT>
__device__ __forceinline__ long long energy_index(const XsDev &X, double E) {
  if (GT == GF_GRID_UNIONIZED) {
    return union_search(X.ubin, X.U, X.n_union, E);
  } else if (GT == kGridNB) {
    // bin b = floor(E 2^kNbLog2) of the per-nuclide tables for E in [0, 1); otherwise -1 (the interval
    // then comes from the index grid)
    if (E >= 0.0 && E < 1.0) return (long long)__dmul_rn(E, (double)(1 << kNbLog2));
    return -1;
  } else if (GT == GF_GRID_HASH) {
    const double du = __ddiv_rn(1.0, (double)X.bins);
    long long b = (long long)__ddiv_rn(E, du);  // truncation toward zero, as the C cast
    b = b > X.bins - 1 ? X.bins - 1 : b;          // R-E1
    return b < 0 ? 0 : b;
  }
  return 0;
}

// ------------------------------------------------------------------------------------------ A4/A5
// SMEM tables, XSBench flavour: per CSR entry j the nuclide's record base (nuc * n_gp) and its row
// base in the index / hash grid (nuc * pitch), so the inner loop does 32-bit index math only.
struct XsTables {
  const int32_t *off;
  const double *conc;
  const uint2 *ent;  // {nuc * n_gp, nuc * pitch}
  const double *thr;
  const uint4 *pk;   // {nuc * n_gp, nuc * pitch, conc (2 words)}: ent + conc in one 16-B LDS
};

// PK: the group kernel's packed layout, one 16-B entry {nuc * n_gp, nuc * pitch, conc} (ent and conc
// stay unset); otherwise the separate ent / conc arrays.
// NBP: the row base of entry j is nuc * nb_pitch (kGridNB kernels) instead of the index / hash grid's.
template <bool PK = false, bool NBP = false>
__device__ __forceinline__ XsTables stage_xs_tables(const XsDev &X, unsigned char *smem) {
  int32_t *s_off = reinterpret_cast<int32_t *>(smem);          // 16 ints
  double *s_thr = reinterpret_cast<double *>(smem + 64);       // 12 doubles -> 160
  double *s_conc = reinterpret_cast<double *>(smem + 160);     // total doubles
  uint2 *s_ent = reinterpret_cast<uint2 *>(smem + 160 + 8 * (size_t)X.total);
  uint4 *s_pk = reinterpret_cast<uint4 *>(smem + 160);         // PK: 16-B aligned (160 % 16 == 0)
  const uint32_t pitch =
      NBP ? (uint32_t)X.nb_pitch : (uint32_t)(X.grid_type == GF_GRID_UNIONIZED ? X.ig_pitch : X.hg_pitch);
  for (int t = threadIdx.x; t < X.total; t += blockDim.x) {
    const uint32_t nuc = (uint32_t)X.mnuc[t];
    const double c = X.mconc[t];
    // record base of the nuclide; a band grid's index grid holds intervals relative to k0[nuc]
    const uint32_t rb = nuc * (uint32_t)X.n_gp + (X.k0 ? X.k0[nuc] : 0u);
    if (PK) {
      const unsigned long long cb = (unsigned long long)__double_as_longlong(c);
      s_pk[t] = make_uint4(rb, nuc * pitch, (uint32_t)cb, (uint32_t)(cb >> 32));
    } else {
      s_conc[t] = c;
      s_ent[t] = make_uint2(rb, nuc * pitch);
    }
  }
  if (threadIdx.x < kMats + 1) s_off[threadIdx.x] = X.moff[threadIdx.x];
  if (threadIdx.x < kMats) s_thr[threadIdx.x] = X.thr[threadIdx.x];
  __syncthreads();
  if (PK) return XsTables{s_off, nullptr, nullptr, s_thr, s_pk};
  return XsTables{s_off, s_conc, s_ent, s_thr, nullptr};
}

__device__ __forceinline__ uint2 tab_ent(const XsTables &T, int j, bool pk) {
  if (pk) {
    const uint4 v = T.pk[j];
    return make_uint2(v.x, v.y);
  }
  return T.ent[j];
}
__device__ __forceinline__ double tab_conc(const XsTables &T, int j, bool pk) {
  if (pk) {
    const uint4 v = T.pk[j];
    return __longlong_as_double((long long)(((unsigned long long)v.w << 32) | v.z));
  }
  return T.conc[j];
}

__host__ __device__ inline size_t xs_table_smem(int total) { return 160 + 16 * (size_t)total; }

// Interval index k (clamped so that k + 1 is a gridpoint) of the nuclide of entry e.
template <int GT>
__device__ __forceinline__ uint32_t interval(const XsDev &X, uint2 e, double E, long long idx) {
  const int n_gp = X.n_gp;
  int k;
  if (GT == GF_GRID_NUCLIDE) {
    k = bisect<int>(X.Ed + e.x, E, 0, n_gp - 1);
  } else if (GT == GF_GRID_UNIONIZED) {
    k = __ldg(X.IG + e.y + (uint32_t)idx);
  } else if (GT == kGridNB) {
    // sparse batches: #{E_nuc <= E} lies in [NB[b], NB[b+1]] (a 2^14-bin table per nuclide, L2-resident,
    // ~0.7 points per bin), finished by a bisection over that bracket -- the same interval as the
    // index grid's, without a DRAM sector of the index grid per (lookup, nuclide)
    if ((unsigned long long)idx < (1ull << kNbLog2)) {  // (a u32 0xFFFFFFFF from idx_prep also fails it)
      const uint16_t *nb = X.NB + e.y + (uint32_t)idx;
      int lo = __ldg(nb), hi = __ldg(nb + 1);
      const double *A = X.Ed + e.x;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(A + mid) <= E) lo = mid + 1; else hi = mid;
      }
      k = lo > 0 ? lo - 1 : 0;
    } else if (X.IG) {
      const uint32_t nuc = e.y / (uint32_t)X.nb_pitch;
      k = __ldg(X.IG + (size_t)nuc * X.ig_pitch + (uint32_t)energy_index<GF_GRID_UNIONIZED>(X, E));
    } else {  // nuclide grid: the literal search
      k = bisect<int>(X.Ed + e.x, E, 0, n_gp - 1);
    }
  } else {
    const double *Ed = X.Ed + e.x;
    int lo_, hi_;
    if (X.hg32) {  // XL / XXL point counts (NEXT-2): u32 entries
      const uint32_t *hg = reinterpret_cast<const uint32_t *>(X.HG) + e.y + (uint32_t)idx;
      lo_ = (int)__ldg(hg);
      hi_ = (idx == X.bins - 1) ? n_gp - 1 : (int)__ldg(hg + 1) + 1;
    } else {
      const uint16_t *hg = X.HG + e.y + (uint32_t)idx;
      lo_ = __ldg(hg);
      hi_ = (idx == X.bins - 1) ? n_gp - 1 : (int)__ldg(hg + 1) + 1;
    }
    if (E <= __ldg(Ed + lo_))
      k = 0;
    else if (E >= __ldg(Ed + hi_))
      k = n_gp - 1;
    else
      k = bisect<int>(Ed, E, lo_, hi_);
  }
  return (uint32_t)(k == n_gp - 1 ? k - 1 : k);
}

struct Pair {  // records k (lo) and k+1 (hi): E, total, elastic, absorption, fission, nu-fission; y
  double2 l0, l1, l2, h0, h1, h2;
  double y;    // RN(1 / (hi.E - lo.E)) (fast division path only)
};

template <bool FAST>
__device__ __forceinline__ void load_pair(const XsDev &X, uint32_t rec, Pair &P) {
  const double2 *p = reinterpret_cast<const double2 *>(X.G) + (size_t)rec * 3;
  P.l0 = __ldg(p + 0);
  P.l1 = __ldg(p + 1);
  P.l2 = __ldg(p + 2);
  P.h0 = __ldg(p + 3);
  P.h1 = __ldg(p + 4);
  P.h2 = __ldg(p + 5);
  if (FAST) P.y = __ldg(X.Rd + rec);
}

// f = (hi.E - E) / (hi.E - lo.E); x_c = hi_c - f (hi_c - lo_c); m_c += x_c * conc, every operation
// rounded to nearest and none contracted; the quotient is IEEE RN either way (div_rn is exact).
template <bool FAST>
__device__ __forceinline__ void accumulate(const Pair &P, double E, double conc, double m[5]) {
  const double a = __dsub_rn(P.h0.x, E), b = __dsub_rn(P.h0.x, P.l0.x);
  const double f = FAST ? div_rn(a, b, P.y) : __ddiv_rn(a, b);
  const double lo[5] = {P.l0.y, P.l1.x, P.l1.y, P.l2.x, P.l2.y};
  const double hi[5] = {P.h0.y, P.h1.x, P.h1.y, P.h2.x, P.h2.y};
#pragma unroll
  for (int c = 0; c < 5; c++) {
    const double x = __dsub_rn(hi[c], __dmul_rn(f, __dsub_rn(hi[c], lo[c])));
    m[c] = __dadd_rn(m[c], __dmul_rn(x, conc));
  }
}

// Nuclides j0..j1-1 in table order, software-pipelined with two record-pair buffers (A, B): the
// pair of j+1 and the interval of j+2 are loaded while j is accumulated.  With PF, each thread also
// prefetches into L2 the index-grid line of nuclide j + kPrefetch.
template <int GT, bool FAST, bool PF>
__device__ __forceinline__ void nuclide_loop(const XsDev &X, const XsTables &T, double E, long long idx, int j0,
                                             int j1, double m[5]) {
  Pair A, B;
  uint32_t kA = interval<GT>(X, T.ent[j0], E, idx);
  load_pair<FAST>(X, T.ent[j0].x + kA, A);
  uint32_t kB = (j0 + 1 < j1) ? interval<GT>(X, T.ent[j0 + 1], E, idx) : 0u;
  for (int j = j0; j < j1; j += 2) {
    if (PF && j + kPrefetch < j1)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(X.IG + T.ent[j + kPrefetch].y + (uint32_t)idx));
    if (j + 1 < j1) load_pair<FAST>(X, T.ent[j + 1].x + kB, B);
    if (j + 2 < j1) kA = interval<GT>(X, T.ent[j + 2], E, idx);
    accumulate<FAST>(A, E, T.conc[j], m);
    if (j + 1 >= j1) break;
    if (PF && j + 1 + kPrefetch < j1)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(X.IG + T.ent[j + 1 + kPrefetch].y + (uint32_t)idx));
    if (j + 2 < j1) load_pair<FAST>(X, T.ent[j + 2].x + kA, A);
    if (j + 3 < j1) kB = interval<GT>(X, T.ent[j + 3], E, idx);
    accumulate<FAST>(B, E, T.conc[j + 1], m);
  }
}

// kGridNB with E in [0, 1) (bin b): a three-stage ring so that no step waits on a load issued in the
// same step -- step j issues the NB bracket loads of nuclide j+3, the one probe Ed[lo] of nuclide j+2
// (when its bracket holds one point: c = lo + (Ed[lo] <= E)), resolves the interval of j+1 and issues
// its record pair, then accumulates j.  Brackets of two or more points (~15%) bisect at resolve time.
// Same intervals as interval<kGridNB>; the accumulation order is unchanged.
#ifndef GF_NB_RING
#define GF_NB_RING 1
#endif
#ifndef GF_NB_RING_MIN
#define GF_NB_RING_MIN 64  // materials with at least this many nuclides take the ring (the large fuel, 321)
#endif
__device__ __forceinline__ void nb_bracket(const XsDev &X, uint2 e, uint32_t b, int &lo, int &hi) {
  const uint16_t *q = X.NB + e.y + b;
  lo = __ldg(q);
  hi = __ldg(q + 1);
}
__device__ __forceinline__ double nb_probe(const XsDev &X, uint2 e, int lo, int hi) {
  return hi - lo == 1 ? __ldg(X.Ed + e.x + lo) : 0.0;
}
__device__ __forceinline__ uint32_t nb_resolve(const XsDev &X, uint2 e, double E, int lo, int hi, double pr) {
  int c;
  if (hi - lo <= 0) {
    c = lo;
  } else if (hi - lo == 1) {
    c = lo + (pr <= E ? 1 : 0);
  } else {
    const double *A = X.Ed + e.x;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(A + mid) <= E) lo = mid + 1; else hi = mid;
    }
    c = lo;
  }
  const int k = c > 0 ? c - 1 : 0;
  return (uint32_t)(k > X.n_gp - 2 ? X.n_gp - 2 : k);
}

template <bool FAST>
__device__ __forceinline__ void nuclide_loop_nb(const XsDev &X, const XsTables &T, double E, uint32_t b, int j0,
                                                int j1, double m[5]) {
  int lo1 = 0, hi1 = 0, lo2 = 0, hi2 = 0, lo3 = 0, hi3 = 0;
  double pr1 = 0.0, pr2 = 0.0;
  Pair P, Q;
  {
    int lo0, hi0;
    nb_bracket(X, T.ent[j0], b, lo0, hi0);
    const double pr0 = nb_probe(X, T.ent[j0], lo0, hi0);
    if (j0 + 1 < j1) nb_bracket(X, T.ent[j0 + 1], b, lo1, hi1);
    if (j0 + 2 < j1) nb_bracket(X, T.ent[j0 + 2], b, lo2, hi2);
    if (j0 + 1 < j1) pr1 = nb_probe(X, T.ent[j0 + 1], lo1, hi1);
    load_pair<FAST>(X, T.ent[j0].x + nb_resolve(X, T.ent[j0], E, lo0, hi0, pr0), P);
  }
#pragma unroll 2
  for (int j = j0; j < j1; j++) {
    if (j + 3 < j1) nb_bracket(X, T.ent[j + 3], b, lo3, hi3);
    if (j + 2 < j1) pr2 = nb_probe(X, T.ent[j + 2], lo2, hi2);
    if (j + 1 < j1) load_pair<FAST>(X, T.ent[j + 1].x + nb_resolve(X, T.ent[j + 1], E, lo1, hi1, pr1), Q);
    accumulate<FAST>(P, E, T.conc[j], m);
    P = Q;
    lo1 = lo2; hi1 = hi2; pr1 = pr2;
    lo2 = lo3; hi2 = hi3;
  }
}

template <int GT, bool PF>
__device__ __forceinline__ void macro_xs(const XsDev &X, const XsTables &T, double E, long long idx, int mat,
                                         double m[5]) {
#pragma unroll
  for (int c = 0; c < 5; c++) m[c] = 0.0;
  const int j0 = T.off[mat], j1 = T.off[mat + 1];
  if (j0 >= j1) return;
  if (GT == kGridNB && GF_NB_RING && j1 - j0 >= GF_NB_RING_MIN && (unsigned long long)idx < (1ull << kNbLog2)) {
    if (X.fastdiv)
      nuclide_loop_nb<true>(X, T, E, (uint32_t)idx, j0, j1, m);
    else
      nuclide_loop_nb<false>(X, T, E, (uint32_t)idx, j0, j1, m);
    return;
  }
  // the reciprocal division needs |hi.E - E| <= 4 (all sampled energies are in [0, 1])
  if (X.fastdiv && fabs(E) <= 2.0)
    nuclide_loop<GT, true, PF>(X, T, E, idx, j0, j1, m);
  else
    nuclide_loop<GT, false, PF>(X, T, E, idx, j0, j1, m);
}

__device__ __forceinline__ uint32_t argmax5_plus1(const double m[5]) {
  double mx = -1.0;
  uint32_t idx = 0;
#pragma unroll
  for (int c = 0; c < 5; c++)
    if (m[c] > mx) {
      mx = m[c];
      idx = c;
    }
  return idx + 1;
}

// ------------------------------------------------------------------------------------------ kernels
// Lookups in global-index order (no sort): thread t handles lookup first + t.
template <int GT>
__global__ void __launch_bounds__(kLookupTpb) xs_lookup_direct(XsDev X, uint64_t first, uint32_t n, uint64_t seed,
                                                               const double *__restrict__ src_E,
                                                               const uint8_t *__restrict__ src_mat,
                                                               OutSpec out,
                                                               unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(128) unsigned char smem[];
  const XsTables T = stage_xs_tables(X, smem);
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t v = 0;
  if (t < n) {
    double E;
    int mat;
    if (src_E) {
      E = src_E[t];
      mat = src_mat[t];
      if (mat >= kMats || !isfinite(E)) invalid_input(vsum);
      mat = mat < kMats ? mat : kMats - 1;
    } else {
      uint64_t s = lcg_skip(seed, 2ull * (first + t));
      E = lcg_draw(s);
      mat = pick_material(lcg_draw(s), T.thr);
    }
    double m[5];
    macro_xs<GT, false>(X, T, E, energy_index<GT>(X, E), mat, m);
    v = argmax5_plus1(m);
    if (out.any()) write_out<5>(out, t, m);
  }
  hash_epilogue(v, vsum);
}

// Lookups over the locality-sorted order: position p holds energy Es[p]; its material is the
// segment of mstart that contains p; its original position is idx[p] (outputs only).
#ifndef GF_SORTED_MINB
#define GF_SORTED_MINB 5  // 5 CTAs per SM (with the NB ring: H3 14.2 -> 13.3 ms; 6 CTAs spill 176 B)
#endif
template <int GT>
__global__ void __launch_bounds__(kLookupTpb, GF_SORTED_MINB) xs_lookup_sorted(XsDev X, uint32_t n, const double *__restrict__ Es,
                                                               const uint32_t *__restrict__ idx,
                                                               const uint32_t *__restrict__ mstart,
                                                               OutSpec out,
                                                               unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(128) unsigned char smem[];
  const XsTables T = stage_xs_tables<false, GT == kGridNB>(X, smem);
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  n = min(n, __ldg(mstart + kMats));  // lookups kept by the sort (band grids keep their band's)
  uint32_t v = 0;
  if (p < n) {
    int mat = 0;
#pragma unroll
    for (int mm = 1; mm < kMats; mm++)
      if (p >= __ldg(mstart + mm)) mat = mm;
    const double E = Es[p];
    double m[5];
    macro_xs<GT, GT == GF_GRID_UNIONIZED>(X, T, E, energy_index<GT>(X, E), mat, m);
    v = argmax5_plus1(m);
    if (out.any()) write_out<5>(out, idx[p], m);
  }
  hash_epilogue(v, vsum);
}

// ------------------------------------------------------------------------------------------ production
#include "xs_sorted_u.cuh"
#include "xs_warp_nuclide.cuh"

#include "xs_tile.cuh"

#ifndef GF_TILE_PREP
#define GF_TILE_PREP 0  // A/B: 1 = every unionized tile batch takes tile_prep (exact extremes), no scatter tix
#endif

// Kernel for the sorted path (XsDev::kern, chosen once at grid init).  Default: the warp-tile kernel
// for dense batches (n >= tile_min; unionized and hash grids), the group kernel (4 lookups per
// thread, per-lookup searches) for medium ones and the one-lookup-per-thread kernel below group_min:
// a sparse batch (a history wave, a host-IO chunk) spreads a tile over many intervals, beyond its
// staged records (measured).  The nuclide grid searches the
// per-nuclide bin brackets (NB).  The alternatives stay selectable for A/B measurements
// (GF_XS_KERNEL at grid init): group (4 lookups per thread, per-lookup index-grid loads), thread,
// tilenb (tile runs from the NB brackets), warp (warp-cooperative nuclide-grid search).
static int sorted_kernel(const XsDev &X, uint32_t n) {
  if (X.kern != kKernAuto) return X.kern;
  return n >= X.tile_min ? kKernTile : n >= X.group_min ? kKernGroup : kKernThread;
}

template <int GT>
static cudaError_t launch_gt(const XsDev &X, uint64_t first, uint32_t n, uint64_t seed, const double *src_E,
                             const uint8_t *src_mat, bool sort, const SortScratch &S, const OutSpec &out,
                             unsigned long long *vsum, cudaStream_t st, cudaEvent_t ev_mid) {
  const size_t smem = xs_table_smem(X.total);
  cudaError_t e;
  if (sort) {
    const int kern = sorted_kernel(X, n);
    // sampled unionized warp-tile batches with per-tile union indices: the scatter writes them (TixSpec);
    // caller energies (possibly clamped into a material's last bin) take tile_prep's exact tile extremes
    const bool tix = GT == GF_GRID_UNIONIZED && kern == kKernTile && n >= X.prep_min && !src_E && !GF_TILE_PREP;
    const TixSpec T{reinterpret_cast<uint2 *>(S.us), X.ubin, X.U, X.n_union};
    if ((e = launch_locality_sort(first, n, seed, src_E, src_mat, X.thr, S, out.any(), vsum, st, X.band_lo, X.band_hi,
                                  tix ? &T : nullptr)) != cudaSuccess)
      return e;
    if (ev_mid && (e = cudaEventRecord(ev_mid, st)) != cudaSuccess) return e;
    if (GT != GF_GRID_NUCLIDE && kern == kKernGroup)
      return X.fastdiv ? launch_group<GT, true>(X, n, S, out, vsum, st)
                       : launch_group<GT, false>(X, n, S, out, vsum, st);
    if constexpr (GT != GF_GRID_NUCLIDE) {
      if (kern == kKernTile)
        return X.fastdiv ? launch_tile<GT, true>(X, n, S, out, vsum, st, !tix)
                         : launch_tile<GT, false>(X, n, S, out, vsum, st, !tix);
    }
    if constexpr (GT == GF_GRID_UNIONIZED) {
      if (kern == kKernTileNB && X.NB)
        return X.fastdiv ? launch_tile<kGridNB, true>(X, n, S, out, vsum, st, false)
                         : launch_tile<kGridNB, false>(X, n, S, out, vsum, st, false);
    }
    if constexpr (GT == GF_GRID_NUCLIDE) {  // the warp-tile kernel with runs from the NB brackets
      if ((kern == kKernTile || kern == kKernTileNB) && X.XR && X.NB)
        return X.fastdiv ? launch_tile<kGridNB, true>(X, n, S, out, vsum, st, false)
                         : launch_tile<kGridNB, false>(X, n, S, out, vsum, st, false);
    }
    if (GT == GF_GRID_NUCLIDE && X.NB && X.nb_on && kern != kKernWarpSearch) {
      if ((e = allow_smem(xs_lookup_sorted<kGridNB>, smem)) != cudaSuccess) return e;
      xs_lookup_sorted<kGridNB><<<nblk(n, kLookupTpb), kLookupTpb, smem, st>>>(X, n, S.Es, S.idx, S.mstart, out,
                                                                               vsum);
      return cudaGetLastError();
    }
    if (GT == GF_GRID_NUCLIDE && kern != kKernThread) {
      if ((e = allow_smem(xs_lookup_warp_nuclide, smem)) != cudaSuccess) return e;
      xs_lookup_warp_nuclide<<<nblk(n, kLookupTpb), kLookupTpb, smem, st>>>(X, n, S.Es, S.idx, S.mstart, out,
                                                                           vsum);
      return cudaGetLastError();
    }
    if (GT == GF_GRID_UNIONIZED && X.NB && X.nb_on) {
      if ((e = allow_smem(xs_lookup_sorted<kGridNB>, smem)) != cudaSuccess) return e;
      xs_lookup_sorted<kGridNB><<<nblk(n, kLookupTpb), kLookupTpb, smem, st>>>(X, n, S.Es, S.idx, S.mstart, out,
                                                                               vsum);
      return cudaGetLastError();
    }
    if ((e = allow_smem(xs_lookup_sorted<GT>, smem)) != cudaSuccess) return e;
    xs_lookup_sorted<GT><<<nblk(n, kLookupTpb), kLookupTpb, smem, st>>>(X, n, S.Es, S.idx, S.mstart, out, vsum);
  } else {
    if (ev_mid && (e = cudaEventRecord(ev_mid, st)) != cudaSuccess) return e;
    if ((e = allow_smem(xs_lookup_direct<GT>, smem)) != cudaSuccess) return e;
    xs_lookup_direct<GT><<<nblk(n, kLookupTpb), kLookupTpb, smem, st>>>(X, first, n, seed, src_E, src_mat, out,
                                                                        vsum);
  }
  return cudaGetLastError();
}

cudaError_t launch_xs_lookup(const XsDev &X, uint64_t first, uint32_t n, uint64_t seed, const double *src_E,
                             const uint8_t *src_mat, bool sort, const SortScratch &S, const OutSpec &out,
                             unsigned long long *vsum, cudaStream_t st, cudaEvent_t ev_mid) {
  switch (X.grid_type) {
    case GF_GRID_NUCLIDE:
      return launch_gt<GF_GRID_NUCLIDE>(X, first, n, seed, src_E, src_mat, sort, S, out, vsum, st, ev_mid);
    case GF_GRID_UNIONIZED:
      return launch_gt<GF_GRID_UNIONIZED>(X, first, n, seed, src_E, src_mat, sort, S, out, vsum, st, ev_mid);
    default:
      return launch_gt<GF_GRID_HASH>(X, first, n, seed, src_E, src_mat, sort, S, out, vsum, st, ev_mid);
  }
}

// ------------------------------------------------------------------------------------------ NEXT-1
// History-based mode, direct mapping (history.cu): one thread per particle runs its L dependent
// lookups (R-HIST): start at fast_forward(seed, 8 L p); after each lookup skip #{c : macro_c > 1.0}
// draws, then draw E and the material.  macro: NULL or [np][L][5].
template <int GT>
__global__ void __launch_bounds__(kLookupTpb) xs_history_direct(XsDev X, uint64_t first_p, uint32_t np, int L,
                                                                uint64_t seed, double *__restrict__ macro,
                                                                unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(128) unsigned char smem[];
  const XsTables T = stage_xs_tables(X, smem);
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t v = 0;
  if (t < np) {
    const uint64_t p = first_p + t;
    uint64_t s = lcg_skip(seed, p * (uint64_t)L * 8ull);
    double E = lcg_draw(s);
    int mat = pick_material(lcg_draw(s), T.thr);
    for (int i = 0; i < L; i++) {
      double m[5];
      macro_xs<GT, false>(X, T, E, energy_index<GT>(X, E), mat, m);
      v += argmax5_plus1(m);
      if (macro) {
#pragma unroll
        for (int c = 0; c < 5; c++) macro[((size_t)t * L + i) * 5 + c] = m[c];
      }
      uint32_t nf = 0;
#pragma unroll
      for (int c = 0; c < 5; c++) nf += m[c] > 1.0 ? 1u : 0u;
      for (uint32_t k = 0; k < nf; k++) s = lcg_next(s);
      E = lcg_draw(s);
      mat = pick_material(lcg_draw(s), T.thr);
    }
  }
  hash_epilogue(v, vsum);
}

cudaError_t launch_xs_history_direct(const XsDev &X, uint64_t first_p, uint32_t np, int L, uint64_t seed,
                                     double *macro, unsigned long long *vsum, cudaStream_t st) {
  const size_t smem = xs_table_smem(X.total);
  const unsigned g = nblk(np, kLookupTpb);
  cudaError_t e;
  switch (X.grid_type) {
    case GF_GRID_NUCLIDE:
      if ((e = allow_smem(xs_history_direct<GF_GRID_NUCLIDE>, smem)) != cudaSuccess) return e;
      xs_history_direct<GF_GRID_NUCLIDE><<<g, kLookupTpb, smem, st>>>(X, first_p, np, L, seed, macro, vsum);
      break;
    case GF_GRID_UNIONIZED:
      if ((e = allow_smem(xs_history_direct<GF_GRID_UNIONIZED>, smem)) != cudaSuccess) return e;
      xs_history_direct<GF_GRID_UNIONIZED><<<g, kLookupTpb, smem, st>>>(X, first_p, np, L, seed, macro, vsum);
      break;
    default:
      if ((e = allow_smem(xs_history_direct<GF_GRID_HASH>, smem)) != cudaSuccess) return e;
      xs_history_direct<GF_GRID_HASH><<<g, kLookupTpb, smem, st>>>(X, first_p, np, L, seed, macro, vsum);
  }
  return cudaGetLastError();
}

// Self-test hook for the exact reciprocal division (tests): out[i] = div_rn(a[i], b[i], RN(1/b[i]))
// and ref[i] = __ddiv_rn(a[i], b[i]).
__global__ void div_selftest(const double *a, const double *b, double *out, double *ref, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = div_rn(a[i], b[i], __drcp_rn(b[i]));
  ref[i] = __ddiv_rn(a[i], b[i]);
}

cudaError_t launch_div_selftest(const double *a, const double *b, double *out, double *ref, int n, cudaStream_t st) {
  div_selftest<<<nblk(n, 256), 256, 0, st>>>(a, b, out, ref, n);
  return cudaGetLastError();
}

}  // namespace gf
