// sort.cu -- A1/A2: sampling and the locality sort on sm_100a.
//
// Lookups are ordered by the key (material, floor(E 2^b)) -- b = 17 at 17 M: 12 x 2^17 bins, ~18-36
// lookups per bin (smaller batches: fewer bins, sort_bits) -- so that neighbouring lookups share intervals in the lookup kernels; order inside a
// bin is arbitrary (results are order-independent: integer hash, outputs scattered back through idx).
// Counting sort: sort_count (sample, one global atomic per lookup on its bin), a two-kernel scan,
// sort_scatter (sample again, atomic cursor, store E and the lookup position).  Sampling is
// index-addressed (lookup i draws from fast_forward(seed, 2i)): a thread skips once and steps
// through kRun consecutive lookups; the material roll is decided on the integer LCG state
// (pick_material_state, exact).  A band grid (NEXT-2) keeps only lookups with band_lo <= E < band_hi
// (the defaults keep all).  Measured alternative: a two-level sort (coarse
// buckets per CTA run, then a per-bucket fine sort) moved fewer DRAM bytes but was not faster.
#include "gf_internal.cuh"

#include <cstdlib>
#include <algorithm>
#include <cmath>

namespace gf {

constexpr int kRun = 16;   // sort_scatter: lookups per thread (registers hold them between phases)
constexpr int kRunC = 16;  // sort_count: lookups per thread (64 measured: no faster at 17 M, slower for small batches)
constexpr int kSampTpb = 256;
static_assert(kRun == 16 && kRunC == 16 && kSampTpb == 256, "the offset maps (kOffMapOff) are for 256 x 16 lookups");

// A sampling CTA (kSampTpb threads x 16 consecutive lookups): the integer thresholds and the material
// bucket table go to shared memory; thread 0 skips to the CTA's first lookup once (gen: sampled, not
// caller, energies) and every thread starts from it through the offset map of its 32 t steps -- one
// affine map instead of a ~25-step skip per thread.
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
  if (gen && threadIdx.x == 0) Q.base = lcg_skip(seed, 2ull * (first + (uint64_t)blockIdx.x * kSampTpb * kRun));
  __syncthreads();
}
__device__ __forceinline__ uint64_t thread_start(const double *thr, const SampleSmem &Q) {
  const ulonglong2 m =
      __ldg(reinterpret_cast<const ulonglong2 *>(reinterpret_cast<const unsigned char *>(thr) + kOffMapOff) + threadIdx.x);
  return (m.x * Q.base + m.y) & kLcgMask;
}

// Band filter of a NEXT-2 band grid: [lo, hi).  The defaults (-inf, +inf) mean "no band" and keep
// every lookup, +-inf and NaN energies included.
// Sort bins within a material: 2^nbl bins, bin = floor((E - b0) 2^sl) clamped (a whole grid: b0 = 0,
// sl = nbl, exact scaling).  A band grid's batch covers only its band [b0, b0 + 1/W): its bins span the
// band at the whole grid's density (sl = nbl + floor(log2 W)), so the zeroing and the scans shrink W-fold.
// Sampled lookups are filtered on the LCG state instead: E = RN(s) 2^-63 is non-decreasing in s, so
// band_lo <= E < band_hi exactly when slo <= s < shi (state_threshold), and a lookup outside the band
// costs its two LCG steps and two compares only.
struct SortBins {
  double b0;
  int sl, nbl;
  unsigned long long slo, shi;  // the band on the LCG state (whole grid: 0, 2^63)
};
__device__ __forceinline__ int sort_bin(double E, const SortBins &B) {
  int b = (int)__dmul_rn(__dsub_rn(E, B.b0), (double)(1 << B.sl));
  b = b < 0 ? 0 : b;
  return b > (1 << B.nbl) - 1 ? (1 << B.nbl) - 1 : b;
}

__device__ __forceinline__ bool in_band(double E, double lo, double hi) {
  const bool whole = lo == -__longlong_as_double(0x7ff0000000000000ll) && hi == __longlong_as_double(0x7ff0000000000000ll);
  return whole || (E >= lo && E < hi);
}  // consecutive lookups per thread in the sampling kernels
__global__ void __launch_bounds__(kSampTpb) sort_count(uint64_t first, uint32_t n, uint64_t seed,
                                                  const double *__restrict__ src_E,
                                                  const uint8_t *__restrict__ src_mat,
                                                  const double *__restrict__ thr, uint32_t *__restrict__ counts,
                                                  double band_lo, double band_hi, SortBins B,
                                                  unsigned long long *__restrict__ flag) {
  __shared__ SampleSmem Q;
  stage_sampler(Q, thr, first, seed, !src_E);
  uint64_t t0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRunC;
  if (t0 >= n) return;
  uint64_t s = 0;
  if (!src_E) s = thread_start(thr, Q);
  for (int r = 0; r < kRunC; r++) {
    uint64_t t = t0 + r;
    if (t >= n) break;
    double E;
    int mat;
    if (src_E) {
      E = src_E[t];
      mat = src_mat[t];
      if (mat >= kMats || !isfinite(E)) invalid_input(flag);  // outside the input domain: flagged
      mat = mat < kMats ? mat : kMats - 1;
      if (!in_band(E, band_lo, band_hi)) continue;
    } else {
      const uint64_t s1 = lcg_next(s);
      s = lcg_next(s1);
      if (s1 < B.slo || s1 >= B.shi) continue;  // outside the band
      E = lcg_unit(s1);
      mat = pick_material_tab(s, Q.tab, Q.sT);  // == pick_material(RN(s) 2^-63, T), exact
    }
    atomicAdd(counts + (mat << B.nbl) + sort_bin(E, B), 1u);
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

// Adds the exclusive prefix of the CTA totals; records material starts mstart[m] (mstart[12] = n).
__global__ void __launch_bounds__(kScanBlk) scan_add(uint32_t *__restrict__ cursor, const uint32_t *__restrict__ btot,
                                                     uint32_t *__restrict__ mstart, int nb_log2) {
  __shared__ uint32_t s_off;
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
}

__global__ void __launch_bounds__(kSampTpb) sort_scatter(uint64_t first, uint32_t n, uint64_t seed,
                                                    const double *__restrict__ src_E,
                                                    const uint8_t *__restrict__ src_mat,
                                                    const double *__restrict__ thr, uint32_t *__restrict__ cursor,
                                                    double *__restrict__ Es, uint32_t *__restrict__ idx,
                                                    double band_lo, double band_hi, SortBins B) {
  __shared__ SampleSmem Q;
  stage_sampler(Q, thr, first, seed, !src_E);
  uint64_t t0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRun;
  if (t0 >= n) return;
  const int cnt = (int)min((uint64_t)kRun, n - t0);
  uint64_t s = 0;
  if (!src_E) s = thread_start(thr, Q);
  // three phases so that the kRun cursor atomics (each an L2 round trip) are in flight together
  double E[kRun];
  uint32_t pos[kRun];
#pragma unroll
  for (int r = 0; r < kRun; r++) {
    if (r < cnt) {
      const uint64_t t = t0 + r;
      pos[r] = 0xFFFFFFFFu;  // (outside the band: dropped)
      if (src_E) {
        E[r] = src_E[t];
        int mat = src_mat[t];
        mat = mat < kMats ? mat : kMats - 1;
        if (in_band(E[r], band_lo, band_hi)) pos[r] = (uint32_t)((mat << B.nbl) + sort_bin(E[r], B));
      } else {
        const uint64_t s1 = lcg_next(s);
        s = lcg_next(s1);
        if (s1 >= B.slo && s1 < B.shi) {
          E[r] = lcg_unit(s1);
          const int mat = pick_material_tab(s, Q.tab, Q.sT);  // == pick_material(RN(s) 2^-63, T), exact
          pos[r] = (uint32_t)((mat << B.nbl) + sort_bin(E[r], B));
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kRun; r++)
    if (r < cnt && pos[r] != 0xFFFFFFFFu) pos[r] = atomicAdd(cursor + pos[r], 1u);
#pragma unroll
  for (int r = 0; r < kRun; r++) {
    if (r < cnt && pos[r] != 0xFFFFFFFFu) {
      Es[pos[r]] = E[r];
      if (idx) idx[pos[r]] = (uint32_t)(t0 + r);
    }
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

static int sort_bits(uint32_t n) {
  if (const int v = sort_bits_override()) return v;
  if (n >= (1u << 20)) return 17;  // tile-kernel batches: the finest bins (C3 8-way shard 0.708 -> 0.681 ms)
  int b = 10;
  while (b < 17 && ((uint64_t)kMats << (b + 2)) < n) b++;
  return b;
}

// The bins of an n-lookup batch on a grid with band [lo, hi) ((-inf, inf): whole grid; band 0 is open
// below, the last band above, their lookups still lie in [0, 1/W) / [(W-1)/W, 1)).
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

static SortBins whole_bins(int nb) { return SortBins{0.0, nb, nb, 0ull, 1ull << 63}; }

static SortBins sort_bins(uint32_t n, double lo, double hi) {
  const int nb = sort_bits(n);
  const bool flo = std::isfinite(lo), fhi = std::isfinite(hi);
  if (!flo && !fhi) return whole_bins(nb);
  const double width = (flo && fhi) ? hi - lo : (fhi ? hi : 1.0 - lo);
  const long W = width > 0.0 ? std::lround(1.0 / width) : 1;
  int wl = 0;  // floor(log2 W)
  while (wl < 20 && (2l << wl) <= W) wl++;
  const int nbl = nb - wl < 10 ? 10 : nb - wl;
  return SortBins{flo ? lo : 0.0, nbl + wl, nbl, flo ? state_threshold(lo) : 0ull,
                  fhi ? state_threshold(hi) : 1ull << 63};
}

cudaError_t launch_sort_zero(uint32_t n, const SortScratch &S, cudaStream_t st) {
  return cudaMemsetAsync(S.counts, 0, sizeof(uint32_t) * (kMats << sort_bits(n)), st);
}

// Counts caller lookups [0, cn) of a chunk (src_E / src_mat point at the chunk) into the bins of an
// n_total-lookup batch (no band grids: the host-IO path rejects them).
cudaError_t launch_sort_count(uint32_t n_total, uint32_t cn, const double *src_E, const uint8_t *src_mat,
                              const double *thr, const SortScratch &S, unsigned long long *flag, cudaStream_t st) {
  const double inf = HUGE_VAL;
  const unsigned gc = nblk(((long long)cn + kRunC - 1) / kRunC, kSampTpb);
  const int nb = sort_bits(n_total);
  sort_count<<<gc, kSampTpb, 0, st>>>(0, cn, 0, src_E, src_mat, thr, S.counts, -inf, inf, whole_bins(nb), flag);
  return cudaGetLastError();
}

cudaError_t launch_locality_sort(uint64_t first, uint32_t n, uint64_t seed, const double *src_E,
                                 const uint8_t *src_mat, const double *thr, const SortScratch &S, bool want_idx,
                                 unsigned long long *flag, cudaStream_t st, double band_lo, double band_hi) {
  cudaError_t e;
  const SortBins B = S.counted ? whole_bins(sort_bits(n)) : sort_bins(n, band_lo, band_hi);
  const int nbl = B.nbl;
  const int bins = kMats << nbl;  // a multiple of kScanBlk for nbl >= 10
  const unsigned g = nblk(((long long)n + kRun - 1) / kRun, kSampTpb);
  if (!S.counted) {
    if ((e = cudaMemsetAsync(S.counts, 0, sizeof(uint32_t) * bins, st)) != cudaSuccess) return e;
    const unsigned gc = nblk(((long long)n + kRunC - 1) / kRunC, kSampTpb);
    sort_count<<<gc, kSampTpb, 0, st>>>(first, n, seed, src_E, src_mat, thr, S.counts, band_lo, band_hi, B, flag);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  scan_local<<<bins / kScanBlk, kScanBlk, 0, st>>>(S.counts, S.cursor, S.btot);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  scan_add<<<bins / kScanBlk, kScanBlk, 0, st>>>(S.cursor, S.btot, S.mstart, nbl);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  sort_scatter<<<g, kSampTpb, 0, st>>>(first, n, seed, src_E, src_mat, thr, S.cursor, S.Es, want_idx ? S.idx : nullptr,
                                band_lo, band_hi, B);
  return cudaGetLastError();
}

}  // namespace gf
