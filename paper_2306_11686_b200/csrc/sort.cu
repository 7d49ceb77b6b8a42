// sort.cu -- A1/A2: sampling and the locality sort on sm_100a.
//
// Lookups are ordered by the key (material, floor(E 2^b)) -- b = 17 at 17 M: 12 x 2^17 bins, ~18-36
// lookups per bin (smaller batches: fewer bins, sort_bits) -- so that neighbouring lookups share
// intervals in the lookup kernels; order inside a bin is arbitrary (results are order-independent:
// integer hash, outputs scattered back through idx).
// Counting sort: sort_count (sample, one global atomic per lookup on its bin), a two-kernel scan (which
// also writes the material starts and, for unionized tile batches, the per-tile union indices),
// sort_scatter (sample again, atomic cursor, store E and the lookup position; sampled batches in two
// energy slices so that each slice's destinations stay in L2).  Sampling is index-addressed (lookup i
// draws from fast_forward(seed, 2i)): warp 0 composes the CTA's skip (lcg_skip_warp), each thread starts
// from it through an offset map and steps through 16 consecutive lookups as two interleaved LCG chains;
// the material roll is decided on the integer LCG state (pick_material_tab, exact).
// A band grid (NEXT-2) keeps only lookups with band_lo <= E < band_hi: its count pass (sort_count_band)
// samples the whole batch once, keeps the ~n/W in-band LCG states in a compact list (per-warp segments)
// with each one's rank inside its bin (the count atomic's return value), and the scatter
// (sort_scatter_band) places that list without re-sampling or atomics.
// Measured alternatives: a two-level sort (coarse buckets per CTA run, then a
// per-bucket fine sort), and a two-pass MSD radix sort without global atomics (per-CTA bucket histograms,
// shared-memory ranks, one CTA per bucket): both moved fewer atomics but were not faster at 17 M.
#include "gf_internal.cuh"

#include <cstdlib>
#include <algorithm>
#include <cmath>

namespace gf {

constexpr int kRun = 16;  // lookups per sampling thread (registers hold them between phases)
constexpr int kSampTpb = 256;
static_assert(kRun == 16 && kSampTpb == 256, "the offset maps (kOffMapOff) are for 256 x 16 lookups");

// A sampling CTA (kSampTpb threads x 16 consecutive lookups): the integer thresholds and the material
// bucket table go to shared memory; warp 0 skips to the CTA's first lookup once (gen: sampled, not
// caller, energies; lcg_skip_warp) and every thread starts from it through the offset map of its 32 t
// steps -- one affine map instead of a ~25-step skip per thread.
struct SampleSmem {
  unsigned long long sT[kMats];
  unsigned long long base;
  alignas(16) uint8_t tab[1 << kMatTabLog2];
};
__device__ __forceinline__ void stage_sampler(SampleSmem &Q, const double *thr, uint64_t first, uint64_t seed,
                                              bool gen) {
  const unsigned char *tb = reinterpret_cast<const unsigned char *>(thr);
  if (threadIdx.x < kMats) Q.sT[threadIdx.x] = reinterpret_cast<const unsigned long long *>(thr)[kMats + threadIdx.x];
  reinterpret_cast<uint4 *>(Q.tab)[threadIdx.x] = __ldg(reinterpret_cast<const uint4 *>(tb + kMatTabOff) + threadIdx.x);
  if (gen && threadIdx.x < 32) {  // (warp 0: the skip as one warp-wide composition, not one thread's chain)
    const uint64_t b = lcg_skip_warp(seed, 2ull * (first + (uint64_t)blockIdx.x * kSampTpb * kRun));
    if (threadIdx.x == 0) Q.base = b;
  }
  __syncthreads();
}
__device__ __forceinline__ uint64_t thread_start(const double *thr, const SampleSmem &Q) {
  const ulonglong2 m =
      __ldg(reinterpret_cast<const ulonglong2 *>(reinterpret_cast<const unsigned char *>(thr) + kOffMapOff) + threadIdx.x);
  return (m.x * Q.base + m.y) & kLcgMask;
}

// Sort bins within a material: 2^nbl bins, bin = floor((E - b0) 2^sl) clamped (a whole grid: b0 = 0,
// sl = nbl, exact scaling).  A band grid's batch covers only its band [b0, b0 + 1/W): its bins span the
// band at the whole grid's density (sl = nbl + floor(log2 W)), so the zeroing and the scans shrink W-fold.
// Sampled lookups are filtered on the LCG state instead: E = RN(s) 2^-63 is non-decreasing in s, so
// band_lo <= E < band_hi exactly when slo <= s < shi (state_threshold), and a lookup outside the band
// costs its LCG step and one compare.
struct SortBins {
  double b0;
  int sl, nbl;
  unsigned long long slo, shi;          // the band on the LCG state (whole grid: 0, 2^63)
  unsigned long long a2, c2, a16, c16;  // affine maps of 2 and 16 LCG steps (one / eight lookups)
};
__device__ __forceinline__ int sort_bin(double E, const SortBins &B) {
  int b = (int)__dmul_rn(__dsub_rn(E, B.b0), (double)(1 << B.sl));
  b = b < 0 ? 0 : b;
  return b > (1 << B.nbl) - 1 ? (1 << B.nbl) - 1 : b;
}
__device__ __forceinline__ uint32_t bin_of(double E, int mat, const SortBins &B) {
  return (uint32_t)((mat << B.nbl) + sort_bin(E, B));
}

// The thread's 16 lookups t0 + r as two interleaved chains of energy states (r and r + 8; the second
// started through the 16-step map, both stepped by the 2-step map): f(r, s1) with the energy state s1 of
// lookup t0 + r (its material state is lcg_next(s1)).
template <typename F>
__device__ __forceinline__ void sample_run(uint64_t s, const SortBins &B, F &&f) {
  uint64_t sa = lcg_next(s);
  uint64_t sb = (B.a16 * sa + B.c16) & kLcgMask;
#pragma unroll
  for (int r = 0; r < 8; r++) {
    f(r, sa);
    f(r + 8, sb);
    sa = (B.a2 * sa + B.c2) & kLcgMask;
    sb = (B.a2 * sb + B.c2) & kLcgMask;
  }
}

__global__ void __launch_bounds__(kSampTpb) sort_count(uint64_t first, uint32_t n, uint64_t seed,
                                                  const double *__restrict__ src_E,
                                                  const uint8_t *__restrict__ src_mat,
                                                  const double *__restrict__ thr, uint32_t *__restrict__ counts,
                                                  SortBins B, unsigned long long *__restrict__ flag) {
  __shared__ SampleSmem Q;
  stage_sampler(Q, thr, first, seed, !src_E);
  const uint64_t t0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRun;
  if (t0 >= n) return;
  if (!src_E) {
    const int rem = (int)min((uint64_t)kRun, n - t0);
    sample_run(thread_start(thr, Q), B, [&](int r, uint64_t s1) {
      if (r < rem) atomicAdd(counts + bin_of(lcg_unit(s1), pick_material_tab(lcg_next(s1), Q.tab, Q.sT), B), 1u);
    });
    return;
  }
  for (int r = 0; r < kRun; r++) {
    const uint64_t t = t0 + r;
    if (t >= n) break;
    const double E = src_E[t];
    int mat = src_mat[t];
    if (mat >= kMats || !isfinite(E)) invalid_input(flag);  // outside the input domain: flagged
    mat = mat < kMats ? mat : kMats - 1;
    atomicAdd(counts + bin_of(E, mat, B), 1u);
  }
}

// Block-exclusive scan of kScanBlk counts per CTA (coalesced); writes local offsets and the CTA total.
__global__ void __launch_bounds__(kScanBlk) scan_local(const uint32_t *__restrict__ counts,
                                                       uint32_t *__restrict__ cursor, uint32_t *__restrict__ btot) {
  __shared__ uint32_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int b = blockIdx.x * kScanBlk + tid;
  const uint32_t c = counts[b];
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  cursor[b] = x - c + (wid > 0 ? wsum[wid - 1] : 0u);
  if (tid == kScanBlk - 1) btot[blockIdx.x] = wsum[31];
}

// Per-tile union indices (TixSpec, gf_internal.cuh) for sampled batches: bin k of a material holds
// sorted positions [start, start + count); a full tile t (positions 128 t .. 128 t + 127) takes the lower
// edge of the bin holding 128 t and the upper edge of the bin holding 128 t + 127.  Bin edges are
// b0 + k 2^-sl: the lookups of bin k satisfy edge(k) <= E < edge(k + 1) (E - b0 is exact: b0 = 0, or
// Sterbenz for a band's E in [b0, 2 b0]), and RN is monotone, so RN(edge) bounds E on the same side (bin 0
// of a material: u = 0).  The batch's last, partial tile is left to the lookup kernel.
// u(e) at a bin edge e: a multiple of 2^-20 (whole grids, power-of-two bands) is a top-level bin edge of
// the two-level search, so #{U <= e} = ubin[e 2^20] + #{U == e} (two dependent loads); else the search.
__device__ __forceinline__ uint32_t edge_union(const TixSpec &T, double e) {
  const double t = __dmul_rn(e, (double)kUBins);  // (exact scaling)
  if (t >= 0.0 && t <= (double)kUBins && t == floor(t)) {
    long long k = __ldg(T.ubin + (int)t);
    while (k < T.n_union && __ldg(T.U + k) == e) k++;
    long long u = k - 1;
    u = u < 0 ? 0 : u;
    return (uint32_t)(u > T.n_union - 2 ? T.n_union - 2 : u);
  }
  return (uint32_t)union_search(T.ubin, T.U, T.n_union, e);
}
__device__ __forceinline__ void tile_bounds(const TixSpec &T, const SortBins &B, uint32_t lb, uint32_t start,
                                            uint32_t count) {
  const uint32_t end = start + count;
  const double w = exp2(-(double)B.sl);
  for (uint32_t p = (start + 127u) & ~127u; p < end; p += 128u)
    T.tix[p >> 7].x = lb == 0u ? 0u : edge_union(T, __dadd_rn(B.b0, __dmul_rn((double)lb, w)));
  for (uint32_t p = start | 127u; p < end; p += 128u)
    T.tix[p >> 7].y = edge_union(T, __dadd_rn(B.b0, __dmul_rn((double)(lb + 1u), w)));
}

// Adds the exclusive prefix of the CTA totals; records material starts mstart[m] (mstart[12] = n) and,
// for sampled unionized tile batches, the per-tile union indices (T.tix).
__global__ void __launch_bounds__(kScanBlk) scan_add(uint32_t *__restrict__ cursor, const uint32_t *__restrict__ btot,
                                                     uint32_t *__restrict__ mstart, const uint32_t *__restrict__ counts,
                                                     SortBins B, TixSpec T) {
  __shared__ uint32_t s_off;
  const int nb_log2 = B.nbl;
  const int nblocks = (kMats << nb_log2) / kScanBlk;
  if (threadIdx.x < 32) {
    uint32_t acc = 0;
    for (int i = threadIdx.x; i < (int)blockIdx.x; i += 32) acc += btot[i];
    acc = __reduce_add_sync(0xffffffffu, acc);
    if (threadIdx.x == 0) s_off = acc;
    if (blockIdx.x == nblocks - 1) {
      uint32_t all = 0;
      for (int i = threadIdx.x; i < nblocks; i += 32) all += btot[i];
      all = __reduce_add_sync(0xffffffffu, all);
      if (threadIdx.x == 0) mstart[kMats] = all;
    }
  }
  __syncthreads();
  const int b = blockIdx.x * kScanBlk + threadIdx.x;
  const uint32_t v = cursor[b] + s_off;
  cursor[b] = v;
  if ((b & ((1 << nb_log2) - 1)) == 0) mstart[b >> nb_log2] = v;
  if (T.tix) {
    const uint32_t c = counts[b];
    if (c) tile_bounds(T, B, (uint32_t)b & ((1u << nb_log2) - 1u), v, c);
  }
}

__global__ void __launch_bounds__(kSampTpb) sort_scatter(uint64_t first, uint32_t n, uint64_t seed,
                                                    const double *__restrict__ src_E,
                                                    const uint8_t *__restrict__ src_mat,
                                                    const double *__restrict__ thr, uint32_t *__restrict__ cursor,
                                                    double *__restrict__ Es, uint32_t *__restrict__ idx, SortBins B,
                                                    unsigned long long slo, unsigned long long sspan) {
  __shared__ SampleSmem Q;
  stage_sampler(Q, thr, first, seed, !src_E);
  const uint64_t t0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRun;
  if (t0 >= n) return;
  const int cnt = (int)min((uint64_t)kRun, n - t0);
  // three phases so that the kRun cursor atomics (each an L2 round trip) are in flight together
  double E[kRun];
  uint32_t pos[kRun];
  if (src_E) {
#pragma unroll
    for (int r = 0; r < kRun; r++) {
      pos[r] = 0xFFFFFFFFu;  // (beyond the batch: none)
      if (r < cnt) {
        E[r] = src_E[t0 + r];
        const int mat = src_mat[t0 + r];
        pos[r] = bin_of(E[r], mat < kMats ? mat : kMats - 1, B);
      }
    }
  } else {
    sample_run(thread_start(thr, Q), B, [&](int r, uint64_t s1) {
      E[r] = lcg_unit(s1);
      pos[r] = (r < cnt && s1 - slo < sspan) ? bin_of(E[r], pick_material_tab(lcg_next(s1), Q.tab, Q.sT), B)
                                              : 0xFFFFFFFFu;
    });
  }
#pragma unroll
  for (int r = 0; r < kRun; r++)
    if (pos[r] != 0xFFFFFFFFu) pos[r] = atomicAdd(cursor + pos[r], 1u);
#pragma unroll
  for (int r = 0; r < kRun; r++) {
    if (pos[r] != 0xFFFFFFFFu) {
      Es[pos[r]] = E[r];
      if (idx) idx[pos[r]] = (uint32_t)(t0 + r);
    }
  }
}

// Band grids, count pass, one warp per 512 consecutive lookups (a segment) and no CTA barrier: the warp
// skips to its segment (lcg_skip_warp), every lane samples its 16 lookups and queues the in-band energy
// states in its own shared-memory row (no divergent work per step); then the warp processes its queue 32
// entries at a time with every lane active: one returning atomic per kept lookup (its bin count, and its
// rank inside the bin for the scatter), the state and rank stored at the segment's slots of the compact
// list (capacity 512 per segment) and the segment's length in segcnt.
constexpr int kSeg = 32 * kRun;     // lookups per warp segment
constexpr int kQStride = kRun + 1;  // (row stride in u64: lanes' rows in different banks)
__global__ void __launch_bounds__(kSampTpb) sort_count_band(uint64_t first, uint32_t n, uint64_t seed,
                                                       const double *__restrict__ thr, uint32_t *__restrict__ counts,
                                                       SortBins B, uint64_t *__restrict__ cs,
                                                       uint32_t *__restrict__ rk, uint32_t *__restrict__ cidx,
                                                       uint32_t *__restrict__ segcnt, unsigned long long a_stride,
                                                       unsigned long long c_stride) {
  __shared__ unsigned long long q[kSampTpb * kQStride];
  __shared__ uint8_t qp[kSampTpb * kRun];
  __shared__ uint32_t wpre[kSampTpb / 32][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t nwarps = gridDim.x * (kSampTpb / 32);
  const uint32_t nseg = (uint32_t)(((uint64_t)n + kSeg - 1) / kSeg);
  uint32_t g = blockIdx.x * (kSampTpb / 32) + w;  // this warp's first segment; then every nwarps-th
  if (g >= nseg) return;  // (warp-uniform)
  const unsigned char *tb = reinterpret_cast<const unsigned char *>(thr);
  const uint8_t *tab = tb + kMatTabOff;
  const unsigned long long *sT = reinterpret_cast<const unsigned long long *>(thr) + kMats;
  const ulonglong2 m = __ldg(reinterpret_cast<const ulonglong2 *>(tb + kOffMapOff) + lane);  // 32 lane steps
  // the lane's start state for its 16 lookups of segment g; the next segment's is one affine map away
  uint64_t s0 = (m.x * lcg_skip_warp(seed, 2ull * (first + (uint64_t)g * kSeg)) + m.y) & kLcgMask;
  const unsigned long long span = B.shi - B.slo;
  unsigned long long *row = q + threadIdx.x * kQStride;
  uint8_t *prow = qp + threadIdx.x * kRun;
  for (; g < nseg; g += nwarps) {
    const uint64_t w0 = (uint64_t)g * kSeg, t0 = w0 + (uint64_t)lane * kRun;
    const int rem = t0 < n ? (int)min((uint64_t)kRun, n - t0) : 0;  // (32-bit compares in the unrolled loop)
    uint32_t cnt = 0;
    sample_run(s0, B, [&](int r, uint64_t s1) {
      if (r < rem && s1 - B.slo < span) {
        row[cnt] = s1;
        prow[cnt] = (uint8_t)r;
        cnt++;
      }
    });
    s0 = (a_stride * s0 + c_stride) & kLcgMask;
    uint32_t x = cnt;  // warp prefix of the queue lengths
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    wpre[w][lane] = x - cnt;
    const uint32_t wn = __shfl_sync(0xffffffffu, x, 31);
    if (lane == 0) segcnt[g] = wn;
    __syncwarp();
    for (uint32_t j = lane; j < wn; j += 32) {
      int o = 0;  // the lane whose queue holds entry j: max{o : wpre[o] <= j}
#pragma unroll
      for (int step = 16; step > 0; step >>= 1)
        if (wpre[w][o + step] <= j) o += step;
      const uint32_t k = j - wpre[w][o];
      const int src = w * 32 + o;
      const uint64_t s1 = q[src * kQStride + k];
      const size_t slot = (size_t)w0 + j;
      rk[slot] = atomicAdd(counts + bin_of(lcg_unit(s1), pick_material_tab(lcg_next(s1), tab, sT), B), 1u);
      cs[slot] = s1;
      if (cidx) cidx[slot] = (uint32_t)(w0 + (uint64_t)o * kRun + qp[src * kRun + k]);
    }
    __syncwarp();  // (the queue rows are refilled by the next segment)
  }
}

// Band grids, scatter: one warp per segment places its kept lookups at bin start + rank (no atomics).
__global__ void __launch_bounds__(256) sort_scatter_band(const uint64_t *__restrict__ cs, const uint32_t *__restrict__ rk,
                                                         const uint32_t *__restrict__ cidx,
                                                         const uint32_t *__restrict__ segcnt, uint32_t nseg,
                                                         const double *__restrict__ thr,
                                                         const uint32_t *__restrict__ cursor, double *__restrict__ Es,
                                                         uint32_t *__restrict__ idx, SortBins B) {
  const int lane = threadIdx.x & 31;
  const uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (g >= nseg) return;
  const unsigned char *tb = reinterpret_cast<const unsigned char *>(thr);
  const uint8_t *tab = tb + kMatTabOff;
  const unsigned long long *sT = reinterpret_cast<const unsigned long long *>(thr) + kMats;
  const uint32_t c = __ldg(segcnt + g);
  for (uint32_t j = lane; j < c; j += 32) {
    const size_t slot = (size_t)g * kSeg + j;
    const uint64_t s1 = __ldg(cs + slot);
    const double E = lcg_unit(s1);
    const uint32_t p = __ldg(cursor + bin_of(E, pick_material_tab(lcg_next(s1), tab, sT), B)) + __ldg(rk + slot);
    Es[p] = E;
    if (idx) idx[p] = __ldg(cidx + slot);
  }
}

static inline unsigned nblk(long long n, int b) { return (unsigned)((n + b - 1) / b); }

// Bins per material: 2^17 from 1 M lookups (17 M: ~18-36 lookups per fuel / water bin; the tile kernel's
// lanes want energy-adjacent lookups, so a 2.1 M shard keeps 2^17 too), fewer for small batches so that
// the zeroing and the two scans over 12 x 2^b counters stay small next to the batch (a 500 k-lookup
// history wave: 2^13), i.e. ~4 lookups per bin of the average material, b in [10, 17].
static int sort_bits_override() {  // A/B override GF_SORT_BITS in [10, 17], read once per process
  static const int v = [] {
    const char *f = getenv("GF_SORT_BITS");
    const int b = f ? atoi(f) : 0;
    return (b >= 10 && b <= 17) ? b : 0;
  }();
  return v;
}

// Energy slices of the whole-grid scatter: 2 (gpurun_out/r02al, C3 17 M step: 1 slice 2.680 ms (DRAM
// 162 MB read + 371 MB written by the scatter: partial sectors evicted), 2 slices 2.612, 3 2.616, 4 2.626:
// each slice re-samples the batch).  GF_SCATTER_SLICES overrides (A/B), read once per process.
static int scatter_slices() {
  static const int v = [] {
    const char *f = getenv("GF_SCATTER_SLICES");
    const int k = f ? atoi(f) : 2;
    return (k >= 1 && k <= 16) ? k : 2;
  }();
  return v;
}

static int sort_bits(uint32_t n) {
  if (const int v = sort_bits_override()) return v;
  if (n >= (1u << 20)) return 17;  // tile-kernel batches: the finest bins (C3 8-way shard 0.708 -> 0.681 ms)
  int b = 10;
  while (b < 17 && ((uint64_t)kMats << (b + 2)) < n) b++;
  return b;
}

// min{s in [0, 2^63] : RN(s) 2^-63 >= T} (2^63: none), by bisection with the samplers' conversion (the
// host's int64 -> double conversion rounds to nearest like __ull2double_rn; the scaling is exact).
static unsigned long long state_threshold(double T) {
  unsigned long long lo = 0ull, hi = 1ull << 63;
  while (lo < hi) {
    const unsigned long long mid = lo + ((hi - lo) >> 1);
    if ((double)(long long)mid * 0x1p-63 >= T) hi = mid; else lo = mid + 1;
  }
  return lo;
}

static SortBins with_maps(SortBins B) {
  uint64_t A, C;
  lcg_skip_map(2, A, C);
  B.a2 = A;
  B.c2 = C;
  lcg_skip_map(16, A, C);
  B.a16 = A;
  B.c16 = C;
  return B;
}
static SortBins whole_bins(int nb) { return with_maps(SortBins{0.0, nb, nb, 0ull, 1ull << 63}); }

// The bins of an n-lookup batch on a grid with band [lo, hi) ((-inf, inf): whole grid; band 0 is open
// below, the last band above, their lookups still lie in [0, 1/W) / [(W-1)/W, 1)).
static SortBins sort_bins(uint32_t n, double lo, double hi) {
  const int nb = sort_bits(n);
  const bool flo = std::isfinite(lo), fhi = std::isfinite(hi);
  if (!flo && !fhi) return whole_bins(nb);
  const double width = (flo && fhi) ? hi - lo : (fhi ? hi : 1.0 - lo);
  const long W = width > 0.0 ? std::lround(1.0 / width) : 1;
  int wl = 0;  // floor(log2 W)
  while (wl < 20 && (2l << wl) <= W) wl++;
  // a band's bins one level finer than the whole grid's (2^18 per unit energy from 1 M lookups: the band's
  // tiles narrower; gpurun_out/r02bp, C3 W = 8: 0.390 vs 0.393 ms), within the 12 x 2^17 counters
  const int nbb = std::min(nb + 1 - wl, 17);
  const int nbl = nbb < 10 ? 10 : nbb;
  return with_maps(SortBins{flo ? lo : 0.0, nbl + wl, nbl, flo ? state_threshold(lo) : 0ull,
                            fhi ? state_threshold(hi) : 1ull << 63});
}

// Words of the count / cursor arrays (12 x 2^17 bins).
size_t sort_hist_words(uint64_t) { return ((size_t)kMats << 17) + 1; }

cudaError_t launch_sort_zero(uint32_t n, const SortScratch &S, cudaStream_t st) {
  return cudaMemsetAsync(S.counts, 0, sizeof(uint32_t) * ((size_t)kMats << sort_bits(n)), st);
}

// Counts caller lookups [0, cn) of a chunk (src_E / src_mat point at the chunk) into the bins of an
// n_total-lookup batch (no band grids: the host-IO path rejects them).
cudaError_t launch_sort_count(uint32_t n_total, uint32_t cn, const double *src_E, const uint8_t *src_mat,
                              const double *thr, const SortScratch &S, unsigned long long *flag, cudaStream_t st) {
  const unsigned gc = nblk(((long long)cn + kRun - 1) / kRun, kSampTpb);
  sort_count<<<gc, kSampTpb, 0, st>>>(0, cn, 0, src_E, src_mat, thr, S.counts, whole_bins(sort_bits(n_total)), flag);
  return cudaGetLastError();
}

cudaError_t launch_locality_sort(uint64_t first, uint32_t n, uint64_t seed, const double *src_E,
                                 const uint8_t *src_mat, const double *thr, const SortScratch &S, bool want_idx,
                                 unsigned long long *flag, cudaStream_t st, double band_lo, double band_hi,
                                 const TixSpec *tix) {
  cudaError_t e;
  const SortBins B = S.counted ? whole_bins(sort_bits(n)) : sort_bins(n, band_lo, band_hi);
  const int bins = kMats << B.nbl;  // a multiple of kScanBlk for nbl >= 10
  const TixSpec T = (tix && !src_E) ? *tix : TixSpec{};  // (bin edges bound sampled energies only)
  // band grids take sampled lookups only (abi.cu): the compact-list path
  const bool band = B.slo != 0ull || B.shi != (1ull << 63);
  if (band && (src_E || S.counted)) return cudaErrorInvalidValue;
  if (!S.counted) {
    if ((e = cudaMemsetAsync(S.counts, 0, sizeof(uint32_t) * bins, st)) != cudaSuccess) return e;
    const unsigned gc = nblk(((long long)n + kRun - 1) / kRun, kSampTpb);
    if (band) {  // persistent: the resident warps walk the segments, stepping their states by one map
      int dev = 0, sms = 0, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sort_count_band, kSampTpb, 0);
      const unsigned gb = std::min(gc, (unsigned)(sms * std::max(per_sm, 1)));
      uint64_t A, C;
      lcg_skip_map(2ull * kSeg * gb * (kSampTpb / 32), A, C);
      sort_count_band<<<gb, kSampTpb, 0, st>>>(first, n, seed, thr, S.counts, B, reinterpret_cast<uint64_t *>(S.Et),
                                                S.rk, want_idx ? S.idxt : nullptr, S.segcnt, A, C);
    } else {
      sort_count<<<gc, kSampTpb, 0, st>>>(first, n, seed, src_E, src_mat, thr, S.counts, B, flag);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  scan_local<<<bins / kScanBlk, kScanBlk, 0, st>>>(S.counts, S.cursor, S.btot);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  scan_add<<<bins / kScanBlk, kScanBlk, 0, st>>>(S.cursor, S.btot, S.mstart, S.counts, B, T);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (band) {
    const uint32_t nseg = (uint32_t)(((uint64_t)n + kSeg - 1) / kSeg);
    sort_scatter_band<<<nblk((long long)nseg * 32, 256), 256, 0, st>>>(
        reinterpret_cast<const uint64_t *>(S.Et), S.rk, S.idxt, S.segcnt, nseg, thr, S.cursor, S.Es,
        want_idx ? S.idx : nullptr, B);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  } else {
    // sampled batches scatter in energy slices (one launch each, the others' lookups skipped on the LCG
    // state): a slice's destinations (1/K of the sorted array) stay in L2 until its sectors are complete,
    // instead of partial sectors going to DRAM read-modify-write
    const int K = src_E ? 1 : scatter_slices();
    for (int k = 0; k < K; k++) {
      const unsigned long long lo = k ? state_threshold((double)k / K) : 0ull;
      const unsigned long long hi = k + 1 < K ? state_threshold((double)(k + 1) / K) : 1ull << 63;
      sort_scatter<<<nblk(((long long)n + kRun - 1) / kRun, kSampTpb), kSampTpb, 0, st>>>(
          first, n, seed, src_E, src_mat, thr, S.cursor, S.Es, want_idx ? S.idx : nullptr, B, lo, hi - lo);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  }
  return cudaGetLastError();
}

}  // namespace gf
