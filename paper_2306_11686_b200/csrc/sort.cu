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
#include <cmath>

namespace gf {

constexpr int kRun = 16;   // sort_scatter: lookups per thread (registers hold them between phases)
constexpr int kRunC = 16;  // sort_count: lookups per thread (64 measured: no faster at 17 M, slower for small batches)

// Band filter of a NEXT-2 band grid: [lo, hi).  The defaults (-inf, +inf) mean "no band" and keep
// every lookup, +-inf and NaN energies included.
// Sort bin of E within its material with 2^nb_log2 bins: floor(E 2^nb_log2) clamped (exact scaling).
__device__ __forceinline__ int sort_bin_bits(double E, int nb_log2) {
  int b = (int)__dmul_rn(E, (double)(1 << nb_log2));
  b = b < 0 ? 0 : b;
  return b > (1 << nb_log2) - 1 ? (1 << nb_log2) - 1 : b;
}

__device__ __forceinline__ bool in_band(double E, double lo, double hi) {
  const bool whole = lo == -__longlong_as_double(0x7ff0000000000000ll) && hi == __longlong_as_double(0x7ff0000000000000ll);
  return whole || (E >= lo && E < hi);
}  // consecutive lookups per thread in the sampling kernels
__global__ void __launch_bounds__(256) sort_count(uint64_t first, uint32_t n, uint64_t seed,
                                                  const double *__restrict__ src_E,
                                                  const uint8_t *__restrict__ src_mat,
                                                  const double *__restrict__ thr, uint32_t *__restrict__ counts,
                                                  double band_lo, double band_hi, int nb_log2,
                                                  unsigned long long *__restrict__ flag) {
  __shared__ unsigned long long sT[kMats];  // integer thresholds S[m] (thresholds_kernel)
  if (threadIdx.x < kMats) sT[threadIdx.x] = reinterpret_cast<const unsigned long long *>(thr)[kMats + threadIdx.x];
  __syncthreads();
  uint64_t t0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRunC;
  if (t0 >= n) return;
  uint64_t s = 0;
  if (!src_E) s = lcg_skip(seed, 2ull * (first + t0));
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
    } else {
      E = lcg_draw(s);
      s = lcg_next(s);
      mat = pick_material_state(s, sT);  // == pick_material(RN(s) 2^-63, T), exact
    }
    if (in_band(E, band_lo, band_hi)) atomicAdd(counts + (mat << nb_log2) + sort_bin_bits(E, nb_log2), 1u);
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

__global__ void __launch_bounds__(256) sort_scatter(uint64_t first, uint32_t n, uint64_t seed,
                                                    const double *__restrict__ src_E,
                                                    const uint8_t *__restrict__ src_mat,
                                                    const double *__restrict__ thr, uint32_t *__restrict__ cursor,
                                                    double *__restrict__ Es, uint32_t *__restrict__ idx,
                                                    double band_lo, double band_hi, int nb_log2) {
  __shared__ unsigned long long sT[kMats];  // integer thresholds S[m] (thresholds_kernel)
  if (threadIdx.x < kMats) sT[threadIdx.x] = reinterpret_cast<const unsigned long long *>(thr)[kMats + threadIdx.x];
  __syncthreads();
  uint64_t t0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRun;
  if (t0 >= n) return;
  const int cnt = (int)min((uint64_t)kRun, n - t0);
  uint64_t s = 0;
  if (!src_E) s = lcg_skip(seed, 2ull * (first + t0));
  // three phases so that the kRun cursor atomics (each an L2 round trip) are in flight together
  double E[kRun];
  uint32_t pos[kRun];
#pragma unroll
  for (int r = 0; r < kRun; r++) {
    if (r < cnt) {
      const uint64_t t = t0 + r;
      int mat;
      if (src_E) {
        E[r] = src_E[t];
        mat = src_mat[t];
        mat = mat < kMats ? mat : kMats - 1;
      } else {
        E[r] = lcg_draw(s);
        s = lcg_next(s);
        mat = pick_material_state(s, sT);  // == pick_material(RN(s) 2^-63, T), exact
      }
      pos[r] = in_band(E[r], band_lo, band_hi) ? (uint32_t)((mat << nb_log2) + sort_bin_bits(E[r], nb_log2))
                                               : 0xFFFFFFFFu;
    }
  }
#pragma unroll
  for (int r = 0; r < kRun; r++)
    if (r < cnt && pos[r] != 0xFFFFFFFFu) pos[r] = atomicAdd(cursor + pos[r], 1u);
#pragma unroll
  for (int r = 0; r < kRun; r++) {
    if (r < cnt && pos[r] != 0xFFFFFFFFu) {  // (outside the band: dropped)
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

cudaError_t launch_sort_zero(uint32_t n, const SortScratch &S, cudaStream_t st) {
  return cudaMemsetAsync(S.counts, 0, sizeof(uint32_t) * (kMats << sort_bits(n)), st);
}

// Counts caller lookups [0, cn) of a chunk (src_E / src_mat point at the chunk) into the bins of an
// n_total-lookup batch (no band grids: the host-IO path rejects them).
cudaError_t launch_sort_count(uint32_t n_total, uint32_t cn, const double *src_E, const uint8_t *src_mat,
                              const double *thr, const SortScratch &S, unsigned long long *flag, cudaStream_t st) {
  const double inf = HUGE_VAL;
  const unsigned gc = nblk(((long long)cn + kRunC - 1) / kRunC, 256);
  sort_count<<<gc, 256, 0, st>>>(0, cn, 0, src_E, src_mat, thr, S.counts, -inf, inf, sort_bits(n_total), flag);
  return cudaGetLastError();
}

cudaError_t launch_locality_sort(uint64_t first, uint32_t n, uint64_t seed, const double *src_E,
                                 const uint8_t *src_mat, const double *thr, const SortScratch &S, bool want_idx,
                                 unsigned long long *flag, cudaStream_t st, double band_lo, double band_hi) {
  cudaError_t e;
  const int nbl = sort_bits(n);
  const int bins = kMats << nbl;  // a multiple of kScanBlk for nbl >= 10
  const unsigned g = nblk(((long long)n + kRun - 1) / kRun, 256);
  if (!S.counted) {
    if ((e = cudaMemsetAsync(S.counts, 0, sizeof(uint32_t) * bins, st)) != cudaSuccess) return e;
    const unsigned gc = nblk(((long long)n + kRunC - 1) / kRunC, 256);
    sort_count<<<gc, 256, 0, st>>>(first, n, seed, src_E, src_mat, thr, S.counts, band_lo, band_hi, nbl, flag);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  scan_local<<<bins / kScanBlk, kScanBlk, 0, st>>>(S.counts, S.cursor, S.btot);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  scan_add<<<bins / kScanBlk, kScanBlk, 0, st>>>(S.cursor, S.btot, S.mstart, nbl);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  sort_scatter<<<g, 256, 0, st>>>(first, n, seed, src_E, src_mat, thr, S.cursor, S.Es, want_idx ? S.idx : nullptr,
                                band_lo, band_hi, nbl);
  return cudaGetLastError();
}

}  // namespace gf
