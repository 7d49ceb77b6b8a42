// xs_lookup.cu -- A1-A6: the XSBench event-based lookup on sm_100a.
//
//   A1  sampling        lookup i draws (E, material) from fast_forward(seed, 2i).  A thread handles
//                       a run of consecutive lookups: one skip-ahead, then 2 LCG steps per lookup.
//   A2  locality sort   counting sort by (material, energy bin): count -> scan -> scatter of E (and
//                       the original position when per-lookup outputs are requested).  The result
//                       is order-independent (integer hash; outputs scattered back by position).
//   A3  energy search   unionized: bisection of U; hash: (int64)(E / (1.0/bins)); nuclide: per
//                       nuclide bisection of the SoA energy column.
//   A4  micro xs        per nuclide of the material, in table order: interval k, the 96-B record
//                       pair read as 6 x 16-B vector loads, f and the 5 interpolations.
//   A5  macro xs        macro_c += micro_c * conc_c, RN multiply then RN add, j ascending.
//   A6  hash            v = 1 + argmax (first strict max above -1.0); warp redux -> SMEM -> one u64
//                       atomic per CTA.
// Material tables (CSR: offsets / nuclide ids / concentrations) and pick_mat thresholds are staged
// in shared memory per CTA.
#include "gf_internal.cuh"

namespace gf {

constexpr int kRun = 8;       // consecutive lookups per thread in the sampling kernels
constexpr int kLookupTpb = 256;

// ------------------------------------------------------------------------------------------ A1/A2
__device__ __forceinline__ int energy_bin(double E) {
  int b = (int)(E * (double)kNB);
  b = b < 0 ? 0 : b;
  return b > kNB - 1 ? kNB - 1 : b;
}

__global__ void __launch_bounds__(256) sort_count(uint64_t first, uint32_t n, uint64_t seed,
                                                  const double *__restrict__ src_E,
                                                  const uint8_t *__restrict__ src_mat,
                                                  const double *__restrict__ thr, uint32_t *__restrict__ counts) {
  __shared__ double sT[kMats];
  if (threadIdx.x < kMats) sT[threadIdx.x] = thr[threadIdx.x];
  __syncthreads();
  uint64_t t0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRun;
  if (t0 >= n) return;
  uint64_t s = 0;
  if (!src_E) s = lcg_skip(seed, 2ull * (first + t0));
  for (int r = 0; r < kRun; r++) {
    uint64_t t = t0 + r;
    if (t >= n) break;
    double E;
    int mat;
    if (src_E) {
      E = src_E[t];
      mat = src_mat[t];
      mat = mat < kMats ? mat : kMats - 1;
    } else {
      E = lcg_draw(s);
      mat = pick_material(lcg_draw(s), sT);
    }
    atomicAdd(counts + mat * kNB + energy_bin(E), 1u);
  }
}

// Exclusive scan of kBins counts by one CTA of 1024 threads; cursor = offsets; mstart[m] = start
// of material m (mstart[12] = n).
__global__ void __launch_bounds__(1024) sort_scan(const uint32_t *__restrict__ counts, uint32_t *__restrict__ cursor,
                                                  uint32_t *__restrict__ mstart) {
  constexpr int kPer = kBins / 1024;
  __shared__ uint32_t warp_tot[32];
  const int tid = threadIdx.x;
  uint32_t sum = 0;
  for (int k = 0; k < kPer; k++) sum += counts[tid * kPer + k];
  // block exclusive scan of `sum`
  uint32_t x = sum;
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_tot[lane] = w;  // inclusive
  }
  __syncthreads();
  uint32_t run = x - sum + (wid > 0 ? warp_tot[wid - 1] : 0u);
  for (int k = 0; k < kPer; k++) {
    int b = tid * kPer + k;
    if (b % kNB == 0) mstart[b / kNB] = run;
    cursor[b] = run;
    run += counts[b];
  }
  if (tid == 1023) mstart[kMats] = run;
}

__global__ void __launch_bounds__(256) sort_scatter(uint64_t first, uint32_t n, uint64_t seed,
                                                    const double *__restrict__ src_E,
                                                    const uint8_t *__restrict__ src_mat,
                                                    const double *__restrict__ thr, uint32_t *__restrict__ cursor,
                                                    double *__restrict__ Es, uint32_t *__restrict__ idx) {
  __shared__ double sT[kMats];
  if (threadIdx.x < kMats) sT[threadIdx.x] = thr[threadIdx.x];
  __syncthreads();
  uint64_t t0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kRun;
  if (t0 >= n) return;
  uint64_t s = 0;
  if (!src_E) s = lcg_skip(seed, 2ull * (first + t0));
  for (int r = 0; r < kRun; r++) {
    uint64_t t = t0 + r;
    if (t >= n) break;
    double E;
    int mat;
    if (src_E) {
      E = src_E[t];
      mat = src_mat[t];
      mat = mat < kMats ? mat : kMats - 1;
    } else {
      E = lcg_draw(s);
      mat = pick_material(lcg_draw(s), sT);
    }
    uint32_t pos = atomicAdd(cursor + mat * kNB + energy_bin(E), 1u);
    Es[pos] = E;
    if (idx) idx[pos] = (uint32_t)t;
  }
}

static inline unsigned nblk(long long n, int b) { return (unsigned)((n + b - 1) / b); }

cudaError_t launch_locality_sort(uint64_t first, uint32_t n, uint64_t seed, const double *src_E,
                                 const uint8_t *src_mat, const double *thr, const SortScratch &S, bool want_idx,
                                 cudaStream_t st) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(S.counts, 0, sizeof(uint32_t) * kBins, st)) != cudaSuccess) return e;
  unsigned g = nblk(((long long)n + kRun - 1) / kRun, 256);
  sort_count<<<g, 256, 0, st>>>(first, n, seed, src_E, src_mat, thr, S.counts);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  sort_scan<<<1, 1024, 0, st>>>(S.counts, S.cursor, S.mstart);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  sort_scatter<<<g, 256, 0, st>>>(first, n, seed, src_E, src_mat, thr, S.cursor, S.Es, want_idx ? S.idx : nullptr);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------ A3-A5
template <int GT>
__device__ __forceinline__ void macro_xs(const XsDev &X, const Tables &T, double E, int mat, double m[5]) {
  long long u = 0;
  int b = 0;
  if (GT == GF_GRID_UNIONIZED) {
    u = bisect<long long>(X.U, E, 0ll, X.n_union - 1);
  } else if (GT == GF_GRID_HASH) {
    double du = __ddiv_rn(1.0, (double)X.bins);
    double q = __ddiv_rn(E, du);
    long long bb = (long long)q;  // truncation toward zero, as the C cast
    bb = bb > X.bins - 1 ? X.bins - 1 : bb;  // R-E1
    bb = bb < 0 ? 0 : bb;
    b = (int)bb;
  }
#pragma unroll
  for (int c = 0; c < 5; c++) m[c] = 0.0;
  const int j1 = T.off[mat + 1];
  const int n_gp = X.n_gp;
  for (int j = T.off[mat]; j < j1; j++) {
    const int nuc = T.nuc[j];
    const double conc = T.conc[j];
    const double *Ed = X.Ed + (size_t)nuc * n_gp;
    int k;
    if (GT == GF_GRID_NUCLIDE) {
      k = bisect<int>(Ed, E, 0, n_gp - 1);
    } else if (GT == GF_GRID_UNIONIZED) {
      k = __ldg(X.IG + (size_t)nuc * X.ig_pitch + u);
    } else {
      const int32_t *hg = X.HG + (size_t)nuc * X.hg_pitch + b;
      int lo_ = __ldg(hg);
      int hi_ = (b == X.bins - 1) ? n_gp - 1 : __ldg(hg + 1) + 1;
      if (E <= __ldg(Ed + lo_))
        k = 0;
      else if (E >= __ldg(Ed + hi_))
        k = n_gp - 1;
      else
        k = bisect<int>(Ed, E, lo_, hi_);
    }
    if (k == n_gp - 1) k = k - 1;
    const double2 *p = reinterpret_cast<const double2 *>(X.G + ((size_t)nuc * n_gp + k) * 6);
    const double2 l0 = __ldg(p + 0), l1 = __ldg(p + 1), l2 = __ldg(p + 2);
    const double2 h0 = __ldg(p + 3), h1 = __ldg(p + 4), h2 = __ldg(p + 5);
    const double f = __ddiv_rn(__dsub_rn(h0.x, E), __dsub_rn(h0.x, l0.x));
    const double lo[5] = {l0.y, l1.x, l1.y, l2.x, l2.y};
    const double hi[5] = {h0.y, h1.x, h1.y, h2.x, h2.y};
#pragma unroll
    for (int c = 0; c < 5; c++) {
      const double x = __dsub_rn(hi[c], __dmul_rn(f, __dsub_rn(hi[c], lo[c])));
      m[c] = __dadd_rn(m[c], __dmul_rn(x, conc));
    }
  }
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


// Lookups in global-index order (no sort): thread t handles lookup first + t.
template <int GT>
__global__ void __launch_bounds__(kLookupTpb) xs_lookup_direct(XsDev X, uint64_t first, uint32_t n, uint64_t seed,
                                                               const double *__restrict__ src_E,
                                                               const uint8_t *__restrict__ src_mat,
                                                               double *__restrict__ macro_out,
                                                               unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Tables T = stage_tables(X.total, X.moff, X.mnuc, X.mconc, X.thr, smem);
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t v = 0;
  if (t < n) {
    double E;
    int mat;
    if (src_E) {
      E = src_E[t];
      mat = src_mat[t];
      mat = mat < kMats ? mat : kMats - 1;
    } else {
      uint64_t s = lcg_skip(seed, 2ull * (first + t));
      E = lcg_draw(s);
      mat = pick_material(lcg_draw(s), T.thr);
    }
    double m[5];
    macro_xs<GT>(X, T, E, mat, m);
    v = argmax5_plus1(m);
    if (macro_out) {
#pragma unroll
      for (int c = 0; c < 5; c++) macro_out[(size_t)t * 5 + c] = m[c];
    }
  }
  hash_epilogue(v, vsum);
}

// Lookups over the locality-sorted order: position p holds energy Es[p]; its material is the
// segment of mstart that contains p; its original position is idx[p] (outputs only).
template <int GT>
__global__ void __launch_bounds__(kLookupTpb) xs_lookup_sorted(XsDev X, uint32_t n, const double *__restrict__ Es,
                                                               const uint32_t *__restrict__ idx,
                                                               const uint32_t *__restrict__ mstart,
                                                               double *__restrict__ macro_out,
                                                               unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Tables T = stage_tables(X.total, X.moff, X.mnuc, X.mconc, X.thr, smem);
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t v = 0;
  if (p < n) {
    int mat = 0;
#pragma unroll
    for (int m = 1; m < kMats; m++)
      if (p >= __ldg(mstart + m)) mat = m;
    const double E = Es[p];
    double m[5];
    macro_xs<GT>(X, T, E, mat, m);
    v = argmax5_plus1(m);
    if (macro_out) {
      const size_t o = (size_t)idx[p] * 5;
#pragma unroll
      for (int c = 0; c < 5; c++) macro_out[o + c] = m[c];
    }
  }
  hash_epilogue(v, vsum);
}

template <int GT>
static cudaError_t launch_gt(const XsDev &X, uint64_t first, uint32_t n, uint64_t seed, const double *src_E,
                             const uint8_t *src_mat, bool sort, const SortScratch &S, double *macro_out,
                             unsigned long long *vsum, cudaStream_t st, cudaEvent_t ev_mid) {
  const size_t smem = table_smem(X.total);
  cudaError_t e;
  if (sort) {
    if ((e = launch_locality_sort(first, n, seed, src_E, src_mat, X.thr, S, macro_out != nullptr, st)) != cudaSuccess)
      return e;
    if (ev_mid && (e = cudaEventRecord(ev_mid, st)) != cudaSuccess) return e;
    xs_lookup_sorted<GT><<<nblk(n, kLookupTpb), kLookupTpb, smem, st>>>(X, n, S.Es, S.idx, S.mstart, macro_out, vsum);
  } else {
    if (ev_mid && (e = cudaEventRecord(ev_mid, st)) != cudaSuccess) return e;
    xs_lookup_direct<GT><<<nblk(n, kLookupTpb), kLookupTpb, smem, st>>>(X, first, n, seed, src_E, src_mat, macro_out,
                                                                        vsum);
  }
  return cudaGetLastError();
}

cudaError_t launch_xs_lookup(const XsDev &X, uint64_t first, uint32_t n, uint64_t seed, const double *src_E,
                             const uint8_t *src_mat, bool sort, const SortScratch &S, double *macro_out,
                             unsigned long long *vsum, cudaStream_t st, cudaEvent_t ev_mid) {
  switch (X.grid_type) {
    case GF_GRID_NUCLIDE: return launch_gt<GF_GRID_NUCLIDE>(X, first, n, seed, src_E, src_mat, sort, S, macro_out, vsum, st, ev_mid);
    case GF_GRID_UNIONIZED: return launch_gt<GF_GRID_UNIONIZED>(X, first, n, seed, src_E, src_mat, sort, S, macro_out, vsum, st, ev_mid);
    default: return launch_gt<GF_GRID_HASH>(X, first, n, seed, src_E, src_mat, sort, S, macro_out, vsum, st, ev_mid);
  }
}

}  // namespace gf
