// xs_grid.cu -- A0: device-side XSBench grid build (PAPER.md:1415
// "data initialization is also performed on the GPU").
//
//   K0a+b  xs_sort_fill      one CTA per nuclide: regenerate the nuclide's energies from the LCG by
//                            skip-ahead, bitonic-sort (E, generation index) pairs in SMEM (stable by
//                            generation index, R-TIE-SORT), then write the 48-B records in sorted
//                            order, regenerating each record's 6 draws from its stream position.
//   K0c    merge_round       unionized energies U = ceil(log2 n_iso) rounds of pairwise merges of the
//                            sorted per-nuclide runs (rank of each element in its partner run).
//   K0d    ig_build          nuclide-major index grid IG[i][e] = clamp(#{A_i <= U[e]} - 1, 0, n_gp-2)
//                            (R-IG closed form, u16): one bisection per 32 entries, then a linear walk.
//          ubin_build        top-level table of the two-level unionized search.
//   K0e    hg_build          nuclide-major u16 hash grid HG[i][b] = grid_search(A_i, b * (1.0/bins)).
//   K0f    concs_fill        concentrations continue the grid stream (R-CONC).
//   thresholds               pick_mat thresholds, summed in the stated order (R-PICK).
#include "gf_internal.cuh"

namespace gf {

// Volume fractions of the 12 materials (SURVEY.md:549), typed for the product independently.
__constant__ double c_dist[kMats] = {0.140, 0.052, 0.275, 0.134, 0.154, 0.064,
                                     0.066, 0.055, 0.008, 0.015, 0.025, 0.013};

// T[m] = dist[m] + dist[m-1] + ... + dist[1] in that order; T[0] = 0 (R-PICK: the order fixes bits).
__global__ void thresholds_kernel(double *thr) {
  if (threadIdx.x == 0) {
    for (int m = 0; m < kMats; m++) {
      double run = 0.0;
      for (int j = m; j > 0; j--) run = __dadd_rn(run, c_dist[j]);
      thr[m] = run;
    }
  }
  __syncthreads();
  // Integer form for the samplers: roll = RN(s) 2^-63 is non-decreasing in the LCG state s, so
  // roll < T[m]  <=>  s < S[m] = min{s : RN(s) 2^-63 >= T[m]} -- found by bisection over s with the
  // same conversion, stored as u64 in thr[kMats + m].
  const int m = threadIdx.x;
  if (m < kMats) {
    unsigned long long lo = 0ull, hi = 1ull << 63;  // predicate false at lo? search min s with P(s)
    const double T = thr[m];
    while (lo < hi) {
      const unsigned long long mid = lo + ((hi - lo) >> 1);
      if (__dmul_rn(__ull2double_rn(mid), 0x1p-63) >= T) hi = mid; else lo = mid + 1;
    }
    reinterpret_cast<unsigned long long *>(thr)[kMats + m] = lo;
  }
}

// The sampling tables after the thresholds (gf_internal.cuh, kMatTabOff / kOffMapOff): one thread per
// material-table bucket, the first 256 threads also write the offset maps.
__global__ void __launch_bounds__(256) sample_tables_kernel(double *thr) {
  const unsigned long long *S = reinterpret_cast<const unsigned long long *>(thr) + kMats;
  unsigned char *base = reinterpret_cast<unsigned char *>(thr);
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < (1u << kMatTabLog2)) {
    const unsigned long long lo = (unsigned long long)k << (63 - kMatTabLog2);
    const unsigned long long hi = lo + (1ull << (63 - kMatTabLog2));
    bool inside = false;
    for (int m = 1; m < kMats; m++) inside = inside || (S[m] > lo && S[m] < hi);
    base[kMatTabOff + k] = inside ? 0xFF : (unsigned char)pick_material_state(lo, S);
  }
  if (k < 256) {
    uint64_t A, C;
    lcg_skip_map(32ull * k, A, C);
    reinterpret_cast<unsigned long long *>(base + kOffMapOff)[2 * k] = A;
    reinterpret_cast<unsigned long long *>(base + kOffMapOff)[2 * k + 1] = C;
  }
}

cudaError_t launch_tables(const double *, double *thr, cudaStream_t st) {
  thresholds_kernel<<<1, 32, 0, st>>>(thr);
  sample_tables_kernel<<<(1u << kMatTabLog2) / 256, 256, 0, st>>>(thr);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------ K0a+b
__global__ void __launch_bounds__(1024) xs_sort_fill(double *__restrict__ G, double *__restrict__ Ed,
                                                     double *__restrict__ Rd, int *__restrict__ zero_width,
                                                     int n_gp, int npow, uint64_t seed) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long *key = reinterpret_cast<unsigned long long *>(smem);
  uint32_t *gen = reinterpret_cast<uint32_t *>(key + npow);
  const int nuc = blockIdx.x;
  const uint64_t base = 6ull * (uint64_t)nuc * (uint64_t)n_gp;  // draws before this nuclide

  for (int k = threadIdx.x; k < npow; k += blockDim.x) {
    if (k < n_gp) {
      uint64_t s = lcg_skip(seed, base + 6ull * k);
      double E = lcg_draw(s);
      key[k] = (unsigned long long)__double_as_longlong(E);  // E in [0, 1]: bit order == value order
      gen[k] = (uint32_t)k;
    } else {
      key[k] = ~0ull;  // padding sorts last
      gen[k] = 0xFFFFFFFFu;
    }
  }
  __syncthreads();

  // Bitonic sort of (key, gen) pairs, ascending, lexicographic: equal energies keep generation order.
  for (int size = 2; size <= npow; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (npow >> 1); t += blockDim.x) {
        int lo = 2 * stride * (t / stride) + (t % stride);
        int hi = lo + stride;
        bool asc = (lo & size) == 0;
        unsigned long long ka = key[lo], kb = key[hi];
        uint32_t ga = gen[lo], gb = gen[hi];
        bool a_gt_b = (ka > kb) || (ka == kb && ga > gb);
        if (a_gt_b == asc) {
          key[lo] = kb;
          key[hi] = ka;
          gen[lo] = gb;
          gen[hi] = ga;
        }
      }
      __syncthreads();
    }
  }

  // Write the records in sorted order; each record's 6 draws are regenerated from its position.
  for (int k = threadIdx.x; k < n_gp; k += blockDim.x) {
    uint32_t g = gen[k];
    uint64_t s = lcg_skip(seed, base + 6ull * g);
    double v[6];
#pragma unroll
    for (int f = 0; f < 6; f++) v[f] = lcg_draw(s);
    double2 *rec = reinterpret_cast<double2 *>(G + ((size_t)nuc * n_gp + k) * 6);
    rec[0] = make_double2(v[0], v[1]);
    rec[1] = make_double2(v[2], v[3]);
    rec[2] = make_double2(v[4], v[5]);
    Ed[(size_t)nuc * n_gp + k] = v[0];
    // per-interval reciprocal width for the exact reciprocal division (gf_internal.cuh div_rn)
    double r = 0.0;
    if (k + 1 < n_gp) {
      const double w = __dsub_rn(__longlong_as_double((long long)key[k + 1]), v[0]);
      if (!(w >= 0x1p-960)) atomicOr(zero_width, 1);  // zero / near-underflow width: exact path off
      r = __drcp_rn(w);
    }
    Rd[(size_t)nuc * n_gp + k] = r;
  }
}

// ------------------------------------------------------------------------------------------ K0a/b, large n_gp
// NEXT-2 (XL / XXL point counts): a nuclide's points do not fit one CTA's SMEM
// sort above kMaxSortGp.  Same result (per-nuclide sort by (E, generation index)) in global passes:
// keys -> SMEM bitonic sort of kMaxSortGp-point chunks -> stable pairwise merges of runs inside each
// nuclide's segment -> records regenerated from the sorted generation indices.
__global__ void __launch_bounds__(256) big_keys(unsigned long long *__restrict__ K, uint32_t *__restrict__ Gn,
                                                long long npts, int n_gp, uint64_t seed) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= npts) return;
  uint64_t s = lcg_skip(seed, 6ull * (uint64_t)g);  // point k of nuclide i is draw block i n_gp + k
  K[g] = (unsigned long long)__double_as_longlong(lcg_draw(s));  // E in [0, 1]: bit order == value order
  Gn[g] = (uint32_t)(g % n_gp);
}

// One CTA per (chunk, nuclide): bitonic sort of up to kMaxSortGp (key, gen) pairs in SMEM.
__global__ void __launch_bounds__(1024) big_chunk_sort(unsigned long long *__restrict__ K, uint32_t *__restrict__ Gn,
                                                       int n_gp) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long *key = reinterpret_cast<unsigned long long *>(smem);
  uint32_t *gen = reinterpret_cast<uint32_t *>(key + kMaxSortGp);
  const int nuc = blockIdx.y;
  const int c0 = blockIdx.x * kMaxSortGp, len = min(kMaxSortGp, n_gp - c0);
  const size_t base = (size_t)nuc * n_gp + c0;
  for (int k = threadIdx.x; k < kMaxSortGp; k += blockDim.x) {
    key[k] = k < len ? K[base + k] : ~0ull;
    gen[k] = k < len ? Gn[base + k] : 0xFFFFFFFFu;
  }
  __syncthreads();
  for (int size = 2; size <= kMaxSortGp; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (kMaxSortGp >> 1); t += blockDim.x) {
        const int lo = 2 * stride * (t / stride) + (t % stride), hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const unsigned long long ka = key[lo], kb = key[hi];
        const uint32_t ga = gen[lo], gb = gen[hi];
        if (((ka > kb) || (ka == kb && ga > gb)) == asc) {
          key[lo] = kb;
          key[hi] = ka;
          gen[lo] = gb;
          gen[hi] = ga;
        }
      }
      __syncthreads();
    }
  }
  for (int k = threadIdx.x; k < len; k += blockDim.x) {
    K[base + k] = key[k];
    Gn[base + k] = gen[k];
  }
}

// Merge sorted runs of length L pairwise inside each nuclide's segment.  Generation indices of a
// left run all precede the right run's, so "left before equal right" (lower bound for left
// elements, upper bound for right ones) keeps the (E, gen) order.
__global__ void __launch_bounds__(256) big_merge_round(const unsigned long long *__restrict__ Ki,
                                                       const uint32_t *__restrict__ Gi,
                                                       unsigned long long *__restrict__ Ko, uint32_t *__restrict__ Go,
                                                       long long npts, int n_gp, int L) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= npts) return;
  const long long seg = (g / n_gp) * (long long)n_gp;
  const int loc = (int)(g - seg), run = loc / L, start = run * L;
  const int pstart = (run ^ 1) * L;
  const unsigned long long v = Ki[g];
  int rank = 0, base = start;
  if (pstart < n_gp) {
    const int plen = min(L, n_gp - pstart);
    const unsigned long long *P = Ki + seg + pstart;
    int lo = 0, hi = plen;
    if (run & 1) {  // right run: #{left <= v}
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (P[mid] <= v) lo = mid + 1; else hi = mid;
      }
    } else {  // left run: #{right < v}
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (P[mid] < v) lo = mid + 1; else hi = mid;
      }
    }
    rank = lo;
    base = min(start, pstart);
  }
  const long long o = seg + base + (loc - start) + rank;
  Ko[o] = v;
  Go[o] = Gi[g];
}

// Records in sorted order, regenerated from the generation index; Ed, Rd and the zero-width flag.
__global__ void __launch_bounds__(256) big_write(const unsigned long long *__restrict__ K,
                                                 const uint32_t *__restrict__ Gn, double *__restrict__ Gr,
                                                 double *__restrict__ Ed, double *__restrict__ Rd,
                                                 int *__restrict__ zero_width, long long npts, int n_gp,
                                                 uint64_t seed) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= npts) return;
  const long long seg = (g / n_gp) * (long long)n_gp;
  const int k = (int)(g - seg);
  uint64_t s = lcg_skip(seed, 6ull * (uint64_t)(seg + Gn[g]));
  double v[6];
#pragma unroll
  for (int f = 0; f < 6; f++) v[f] = lcg_draw(s);
  double2 *rec = reinterpret_cast<double2 *>(Gr + g * 6);
  rec[0] = make_double2(v[0], v[1]);
  rec[1] = make_double2(v[2], v[3]);
  rec[2] = make_double2(v[4], v[5]);
  Ed[g] = v[0];
  double r = 0.0;
  if (k + 1 < n_gp) {
    const double w = __dsub_rn(__longlong_as_double((long long)K[g + 1]), v[0]);
    if (!(w >= 0x1p-960)) atomicOr(zero_width, 1);
    r = __drcp_rn(w);
  }
  Rd[g] = r;
}

// ------------------------------------------------------------------------------------------ K0b'
// Interval records for the sorted lookup kernel, one 128-B line per interval k < n_gp - 1 of each
// nuclide (layout in gf_internal.cuh XsDev::XR).  Every stored difference / reciprocal is the RN
// operation the lookup would otherwise do per micro evaluation (R-FP), so results are unchanged.
__global__ void __launch_bounds__(256) xr_build(const double *__restrict__ G, const double *__restrict__ Rd,
                                                double *__restrict__ XR, long long npts, int n_gp) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= npts) return;
  double2 *o = reinterpret_cast<double2 *>(XR + r * 16);
  if ((int)(r % n_gp) == n_gp - 1) {  // no interval starts at the last gridpoint
#pragma unroll
    for (int q = 0; q < 8; q++) o[q] = make_double2(0.0, 0.0);
    return;
  }
  const double *lo = G + r * 6, *hi = lo + 6;
  o[0] = make_double2(hi[0], __dsub_rn(hi[0], lo[0]));
#pragma unroll
  for (int c = 0; c < 5; c++) o[1 + c] = make_double2(hi[1 + c], __dsub_rn(hi[1 + c], lo[1 + c]));
  o[6] = make_double2(Rd[r], lo[0]);
  o[7] = make_double2(0.0, 0.0);
}

// ------------------------------------------------------------------------------------------ K0c
// One merge round: runs of length L (last may be shorter) are merged pairwise.  An element of a
// left run goes before partner elements equal to it (lower bound), an element of a right run after
// them (upper bound); the result is a permutation and U is the sorted multiset.
__global__ void merge_round(const double *__restrict__ in, double *__restrict__ out, long long N, long long L) {
  long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= N) return;
  long long run = g / L, start = run * L;
  long long pr = run ^ 1ll, pstart = pr * L;
  double v = in[g];
  long long rank = 0, base = start;
  if (pstart < N) {
    long long plen = min(L, N - pstart);
    const double *P = in + pstart;
    long long lo = 0, hi = plen;
    if (run & 1ll) {  // right run: #{P <= v}
      while (lo < hi) {
        long long mid = (lo + hi) >> 1;
        if (__ldg(P + mid) <= v) lo = mid + 1; else hi = mid;
      }
    } else {  // left run: #{P < v}
      while (lo < hi) {
        long long mid = (lo + hi) >> 1;
        if (__ldg(P + mid) < v) lo = mid + 1; else hi = mid;
      }
    }
    rank = lo;
    base = min(start, pstart);
  }
  out[base + (g - start) + rank] = v;
}

// ------------------------------------------------------------------------------------------ K0d
// 32 consecutive entries per thread: a bisection for the first, then a monotone walk (U is sorted,
// so #{A <= U[e]} is non-decreasing in e).  u16 entries (n_gp <= 16384); rows are 128-B aligned
// (pitch % 64 == 0): 4 x 16-B stores per thread.
__global__ void __launch_bounds__(256) ig_build(const double *__restrict__ Ed, const double *__restrict__ U,
                                                uint16_t *__restrict__ IG, int n_gp, long long n_union,
                                                long long pitch, const uint32_t *__restrict__ k0) {
  const int nuc = blockIdx.y;
  long long e0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 32;
  if (e0 >= pitch) return;
  const double *A = Ed + (size_t)nuc * n_gp;
  long long eq = min(e0, n_union - 1);
  double q = __ldg(U + eq);
  int lo = 0, hi = n_gp;  // c = #{A <= q}
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldg(A + mid) <= q) lo = mid + 1; else hi = mid;
  }
  int c = lo;
  uint32_t w[16];
#pragma unroll
  for (int k = 0; k < 32; k++) {
    long long e = e0 + k;
    if (e < n_union) {
      q = __ldg(U + e);
      while (c < n_gp && __ldg(A + c) <= q) c++;
    }
    int v = c - 1;
    v = v < 0 ? 0 : v;
    v = v > n_gp - 2 ? n_gp - 2 : v;
    if (k0) v -= (int)k0[nuc];  // band grid: relative to the nuclide's interval at the band's low edge
    if (k & 1) w[k >> 1] |= (uint32_t)v << 16; else w[k >> 1] = (uint32_t)v;
  }
  uint4 *dst = reinterpret_cast<uint4 *>(IG + (size_t)nuc * pitch + e0);
#pragma unroll
  for (int k = 0; k < 4; k++) dst[k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
}

// Per-nuclide bin counts of the sparse-batch search: NB[nuc][b] = #{E_nuc[j] <= b 2^-kNbLog2}
// (exact edges; a bisection over the sorted energies).  For E in [b, b+1) 2^-kNbLog2 the count
// #{E_nuc <= E} lies in [NB[b], NB[b+1]].
__global__ void nb_build(const double *__restrict__ Ed, uint16_t *__restrict__ NB, int n_gp, int pitch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x, nuc = blockIdx.y;
  if (b > (1 << kNbLog2)) return;
  const double e = ldexp((double)b, -kNbLog2);
  const double *A = Ed + (size_t)nuc * n_gp;
  int lo = 0, hi = n_gp;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A[mid] <= e) lo = mid + 1; else hi = mid;
  }
  NB[(size_t)nuc * pitch + b] = (uint16_t)lo;
}

cudaError_t launch_nb_build(const XsDev &X, uint16_t *NB, cudaStream_t st) {
  dim3 grid(((1 << kNbLog2) + 1 + 255) / 256, X.n_iso);
  nb_build<<<grid, 256, 0, st>>>(X.Ed, NB, X.n_gp, X.nb_pitch);
  return cudaGetLastError();
}

// Top-level table of the two-level unionized search: ubin[b] = #{U < b / 2^20}, ubin[2^20] = n.
__global__ void ubin_build(const double *__restrict__ U, uint32_t *__restrict__ ubin, long long n_union) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > kUBins) return;
  if (b == kUBins) {
    ubin[b] = (uint32_t)n_union;
    return;
  }
  const double edge = __dmul_rn((double)b, 1.0 / kUBins);  // exact
  long long lo = 0, hi = n_union;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (__ldg(U + mid) < edge) lo = mid + 1; else hi = mid;
  }
  ubin[b] = (uint32_t)lo;
}

// ------------------------------------------------------------------------------------------ K0e
__global__ void hg_build(const double *__restrict__ Ed, uint16_t *__restrict__ HG, uint32_t *__restrict__ HG32,
                         int n_iso, int n_gp, int bins, int pitch) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)n_iso * pitch) return;
  int nuc = (int)(t / pitch), b = (int)(t % pitch);
  int v = 0;
  if (b < bins) {
    double du = __ddiv_rn(1.0, (double)bins);
    double energy = __dmul_rn((double)b, du);
    v = bisect<int>(Ed + (size_t)nuc * n_gp, energy, 0, n_gp - 1);
  }
  if (HG32)
    HG32[(size_t)nuc * pitch + b] = (uint32_t)v;  // n_gp > 65536 (XL / XXL)
  else
    HG[(size_t)nuc * pitch + b] = (uint16_t)v;
}

// ------------------------------------------------------------------------------------------ K0f
__global__ void concs_fill(double *__restrict__ conc, int total, uint64_t seed, uint64_t draws_before) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= total) return;
  uint64_t s = lcg_skip(seed, draws_before + (uint64_t)c);
  conc[c] = lcg_draw(s);
}

static inline unsigned nblk(long long n, int b) { return (unsigned)((n + b - 1) / b); }

cudaError_t launch_xs_grid(const XsDev &X, double *G, double *Ed, double *Rd, double *XR, int *zero_width,
                           double *U, uint16_t *IG, uint16_t *HG, uint32_t *ubin, double *mconc, uint64_t seed,
                           double *scratch, cudaStream_t st) {
  cudaError_t e;
  const long long npts = (long long)X.n_iso * X.n_gp;
  if ((e = cudaMemsetAsync(zero_width, 0, sizeof(int), st)) != cudaSuccess) return e;
  if (X.n_gp <= kMaxSortGp) {
    int npow = 2;
    while (npow < X.n_gp) npow <<= 1;
    size_t smem = (size_t)npow * (sizeof(unsigned long long) + sizeof(uint32_t));
    if ((e = cudaFuncSetAttribute(xs_sort_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
      return e;
    int threads = npow >= 1024 ? 1024 : (npow < 64 ? 64 : npow);
    xs_sort_fill<<<X.n_iso, threads, smem, st>>>(G, Ed, Rd, zero_width, X.n_gp, npow, seed);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  } else {  // NEXT-2 point counts: chunked sort + segment merges in the init scratch (24 B per point)
    unsigned long long *K0 = reinterpret_cast<unsigned long long *>(scratch);
    unsigned long long *K1 = K0 + npts;
    uint32_t *G0 = reinterpret_cast<uint32_t *>(K1 + npts), *G1 = G0 + npts;
    big_keys<<<nblk(npts, 256), 256, 0, st>>>(K0, G0, npts, X.n_gp, seed);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const size_t smem = (size_t)kMaxSortGp * (sizeof(unsigned long long) + sizeof(uint32_t));
    if ((e = cudaFuncSetAttribute(big_chunk_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
        cudaSuccess)
      return e;
    big_chunk_sort<<<dim3((X.n_gp + kMaxSortGp - 1) / kMaxSortGp, X.n_iso), 1024, smem, st>>>(K0, G0, X.n_gp);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    for (int L = kMaxSortGp; L < X.n_gp; L <<= 1) {
      big_merge_round<<<nblk(npts, 256), 256, 0, st>>>(K0, G0, K1, G1, npts, X.n_gp, L);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      unsigned long long *kt = K0; K0 = K1; K1 = kt;
      uint32_t *gt = G0; G0 = G1; G1 = gt;
    }
    big_write<<<nblk(npts, 256), 256, 0, st>>>(K0, G0, G, Ed, Rd, zero_width, npts, X.n_gp, seed);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (XR) {
    xr_build<<<nblk(npts, 256), 256, 0, st>>>(G, Rd, XR, npts, X.n_gp);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }

  concs_fill<<<nblk(X.total, 256), 256, 0, st>>>(mconc, X.total, seed, 6ull * (uint64_t)npts);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;

  if (X.grid_type == GF_GRID_UNIONIZED && !X.k0) {  // (band grids: launch_band_union / _index)
    int rounds = 0;
    for (long long L = X.n_gp; L < npts; L <<= 1) rounds++;
    if (rounds == 0) {
      if ((e = cudaMemcpyAsync(U, Ed, sizeof(double) * npts, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
    } else {
      // ping-pong so that the last round writes U
      const double *in = Ed;
      long long L = X.n_gp;
      for (int r = 0; r < rounds; r++, L <<= 1) {
        double *out = ((rounds - r) % 2 == 1) ? U : scratch;
        merge_round<<<nblk(npts, 256), 256, 0, st>>>(in, out, npts, L);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        in = out;
      }
    }
    dim3 grid(nblk(X.ig_pitch, 256 * 32), X.n_iso);
    ig_build<<<grid, 256, 0, st>>>(Ed, U, IG, X.n_gp, X.n_union, X.ig_pitch, nullptr);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ubin_build<<<nblk(kUBins + 1, 256), 256, 0, st>>>(U, ubin, X.n_union);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  } else if (X.grid_type == GF_GRID_HASH) {
    hg_build<<<nblk((long long)X.n_iso * X.hg_pitch, 256), 256, 0, st>>>(
        Ed, X.hg32 ? nullptr : HG, X.hg32 ? reinterpret_cast<uint32_t *>(HG) : nullptr, X.n_iso, X.n_gp, X.bins,
        X.hg_pitch);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------------------------------ NEXT-2 bands
// Energy-band sharding of the unionized grid (SURVEY.md Sec. 8(e) alternative, 8(f) NEXT-2): the band
// [lo, hi) keeps U_band = {lo} + sorted {A : lo <= A < hi} + {hi} and the index grid over it.  For a
// lookup E in the band, #{U_band <= E} - 1 indexes the last U_band entry <= E, and every grid point
// <= E is either < lo or in U_band, so IG_band[u] = clamp(#{A <= E} - 1, 0, n_gp - 2) - k0 with k0 the
// interval at lo (the sentinels keep u inside [0, n_band - 2] for every E in the band).  The record
// base of each table entry adds k0, so the lookup kernels are unchanged; results are identical.
__global__ void band_counts(const double *__restrict__ Ed, int n_iso, int n_gp, double lo, double hi, int cap,
                            uint32_t *__restrict__ k0, uint32_t *__restrict__ first, uint32_t *__restrict__ cnt,
                            uint32_t *__restrict__ info) {
  const int nuc = blockIdx.x * blockDim.x + threadIdx.x;
  if (nuc >= n_iso) return;
  const double *A = Ed + (size_t)nuc * n_gp;
  auto count_lt = [&](double q) {  // #{A < q}
    int l = 0, h = n_gp;
    while (l < h) {
      const int m = (l + h) >> 1;
      if (A[m] < q) l = m + 1; else h = m;
    }
    return l;
  };
  int l = 0, h = n_gp;  // #{A <= lo}
  while (l < h) {
    const int m = (l + h) >> 1;
    if (A[m] <= lo) l = m + 1; else h = m;
  }
  int k = l - 1;
  k = k < 0 ? 0 : (k > n_gp - 2 ? n_gp - 2 : k);
  k0[nuc] = (uint32_t)k;
  const int a = count_lt(lo), b = count_lt(hi);
  first[nuc] = (uint32_t)a;
  cnt[nuc] = (uint32_t)(b - a);
  atomicAdd(info, (uint32_t)(b - a));
  if (b - a > cap) atomicOr(info + 1, 1u);  // more points than the layout bound
}

// Padded runs: run[nuc][j] = A[first + j] for j < cnt, +inf after (sorts last).
__global__ void band_runs(const double *__restrict__ Ed, int n_iso, int n_gp, int cap,
                          const uint32_t *__restrict__ first, const uint32_t *__restrict__ cnt,
                          double *__restrict__ run) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)n_iso * cap) return;
  const int nuc = (int)(t / cap), j = (int)(t % cap);
  const uint32_t c = min(cnt[nuc], (uint32_t)cap);
  run[t] = (uint32_t)j < c ? Ed[(size_t)nuc * n_gp + first[nuc] + j] : __longlong_as_double(0x7ff0000000000000ll);
}

__global__ void band_finish(const double *__restrict__ S, double *__restrict__ U, const uint32_t *__restrict__ info,
                            double lo, double hi) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long tot = info[0];
  if (t == 0) U[0] = lo;
  if (t < tot) U[t + 1] = S[t];
  if (t == tot) U[tot + 1] = hi;
}

cudaError_t launch_band_union(const XsDev &X, int cap, uint32_t *k0, uint32_t *cnt, double *U, uint32_t *info,
                              double *scratch, cudaStream_t st) {
  cudaError_t e;
  const long long N = (long long)X.n_iso * cap;
  uint32_t *first = cnt + X.n_iso;
  if ((e = cudaMemsetAsync(info, 0, 16, st)) != cudaSuccess) return e;
  band_counts<<<nblk(X.n_iso, 128), 128, 0, st>>>(X.Ed, X.n_iso, X.n_gp, X.band_lo, X.band_hi, cap, k0, first, cnt,
                                                  info);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  double *a = scratch, *b = scratch + N;
  band_runs<<<nblk(N, 256), 256, 0, st>>>(X.Ed, X.n_iso, X.n_gp, cap, first, cnt, a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  for (long long L = cap; L < N; L <<= 1) {
    merge_round<<<nblk(N, 256), 256, 0, st>>>(a, b, N, L);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    double *t = a; a = b; b = t;
  }
  band_finish<<<nblk(N + 2, 256), 256, 0, st>>>(a, U, info, X.band_lo, X.band_hi);
  return cudaGetLastError();
}

cudaError_t launch_band_index(const XsDev &X, const double *U, uint16_t *IG, uint32_t *ubin, cudaStream_t st) {
  cudaError_t e;
  dim3 grid(nblk(X.ig_pitch, 256 * 32), X.n_iso);
  ig_build<<<grid, 256, 0, st>>>(X.Ed, U, IG, X.n_gp, X.n_union, X.ig_pitch, X.k0);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ubin_build<<<nblk(kUBins + 1, 256), 256, 0, st>>>(U, ubin, X.n_union);
  return cudaGetLastError();
}

}  // namespace gf
