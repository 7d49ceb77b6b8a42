// xs_warp_nuclide.cuh -- the sorted nuclide-grid lookup (C1) with a warp-cooperative binary search
// (BASELINE.json north_star: "a warp-cooperative binary search"; included by xs_lookup.cu).
//
// On the nuclide grid every micro evaluation needs the interval k = clamp(#{A <= E} - 1, 0, n - 2)
// of its own nuclide (XSBench grid_search, SURVEY.md:569-570): a per-thread bisection is 14
// dependent loads for n = 11,303.  After the locality sort a warp's 32 lookups share one material
// and lie in a narrow energy range [Emin, Emax], so the warp searches once per nuclide for that
// range, 32-ary:
//   round:  the 32 lanes load A[s_0..s_31] at evenly spaced positions of the current window and two
//           ballots count the samples <= Emin and <= Emax; both count ranges shrink ~33-fold
//           (11,303 -> ~343 -> ~10: two rounds), each round one dependent load per lane;
//   final:  once the window holds <= 32 positions, lane l loads A[lo + l] (one coalesced load) and
//           every lane finds its own count with a 5-step binary search over the window through
//           __shfl_sync -- no further memory access.
// Every lane's count c(E) lies in the window because c is monotone and Emin <= E <= Emax; positions
// left of the window are <= Emin and right of it > Emax.  The result is the exact count, i.e.
// grid_search's k (bit-identical; NaN energies, for which grid_search is not the count, and warps
// that straddle a material boundary take the per-lane bisection; a warp whose energies span most of
// the window, as without the sort, finishes with a per-lane bisection inside the narrowed window).
#pragma once

constexpr unsigned kFull = 0xffffffffu;

// k = clamp(#{A[0..n) <= E} - 1, 0, n - 2) for this lane's E; Emin / Emax are warp-uniform bounds
// of the participating lanes' energies.  All 32 lanes must call it.
__device__ __forceinline__ int warp_interval(const double *__restrict__ A, int n, double E, double Emin,
                                             double Emax) {
  const int lane = threadIdx.x & 31;
  int lo_a = 0, hi_a = n;  // c(Emin) in [lo_a, hi_a]
  int lo_b = 0, hi_b = n;  // c(Emax) in [lo_b, hi_b]
  while (hi_b - lo_a > 32) {
    const int L = lo_a, R = hi_b, W = R - L;  // sample positions s_t = L + (t + 1) W / 33 in [L, R)
    const double a = __ldg(A + L + (int)(((long long)(lane + 1) * W) / 33));
    const int ta = __popc(__ballot_sync(kFull, a <= Emin));  // prefix masks: A is sorted
    const int tb = __popc(__ballot_sync(kFull, a <= Emax));
    // A[s_t] <= q  <=>  c(q) >= s_t + 1
    if (ta > 0) lo_a = max(lo_a, L + (int)(((long long)ta * W) / 33) + 1);
    if (ta < 32) hi_a = min(hi_a, L + (int)(((long long)(ta + 1) * W) / 33));
    if (tb > 0) lo_b = max(lo_b, L + (int)(((long long)tb * W) / 33) + 1);
    if (tb < 32) hi_b = min(hi_b, L + (int)(((long long)(tb + 1) * W) / 33));
    if (lo_a == L && hi_b == R) break;  // the warp's counts span ~the whole window: no joint progress
  }
  int c;
  const int W = hi_b - lo_a;
  if (W <= 32) {  // window [lo_a, hi_b): lane l holds A[lo_a + l], lanes beyond it NaN (never <= E,
                  // so "v <= E" stays a prefix predicate even for E = +inf)
    const double a = lane < W ? __ldg(A + lo_a + lane) : __longlong_as_double(0x7ff8000000000000ll);
    c = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const double v = __shfl_sync(kFull, a, c + step - 1);
      if (v <= E) c += step;
    }
    const double last = __shfl_sync(kFull, a, 31);  // c == 31: is the 32nd element <= E too?
    c += (c == 31 && last <= E) ? 1 : 0;
    c += lo_a;
  } else {  // wide warp (not locality-sorted): per-lane upper bound within the narrowed window
    int lo = lo_a, hi = hi_b;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(A + mid) <= E) lo = mid + 1; else hi = mid;
    }
    c = lo;
  }
  const int k = c - 1;
  return k < 0 ? 0 : (k > n - 2 ? n - 2 : k);
}

template <bool FAST>
__device__ __forceinline__ void warp_nuclide_loop(const XsDev &X, const XsTables &T, double E, double Emin,
                                                  double Emax, int j0, int j1, double m[5]) {
  const int n_gp = X.n_gp;
  Pair A, B;
  uint32_t kA = warp_interval(X.Ed + T.ent[j0].x, n_gp, E, Emin, Emax);
  load_pair<FAST>(X, T.ent[j0].x + kA, A);
  uint32_t kB = (j0 + 1 < j1) ? warp_interval(X.Ed + T.ent[j0 + 1].x, n_gp, E, Emin, Emax) : 0u;
  for (int j = j0; j < j1; j += 2) {
    if (j + 1 < j1) load_pair<FAST>(X, T.ent[j + 1].x + kB, B);
    if (j + 2 < j1) kA = warp_interval(X.Ed + T.ent[j + 2].x, n_gp, E, Emin, Emax);
    accumulate<FAST>(A, E, T.conc[j], m);
    if (j + 1 >= j1) break;
    if (j + 2 < j1) load_pair<FAST>(X, T.ent[j + 2].x + kA, A);
    if (j + 3 < j1) kB = warp_interval(X.Ed + T.ent[j + 3].x, n_gp, E, Emin, Emax);
    accumulate<FAST>(B, E, T.conc[j + 1], m);
  }
}

// Sorted nuclide-grid lookups, one per lane; the warp's 32 consecutive sorted lookups search together.
__global__ void __launch_bounds__(kLookupTpb) xs_lookup_warp_nuclide(XsDev X, uint32_t n,
                                                                     const double *__restrict__ Es,
                                                                     const uint32_t *__restrict__ idx,
                                                                     const uint32_t *__restrict__ mstart,
                                                                     OutSpec out,
                                                                     unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(128) unsigned char smem[];
  const XsTables T = stage_xs_tables(X, smem);
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  n = min(n, __ldg(mstart + kMats));  // lookups kept by the sort
  const bool act = p < n;
  uint32_t v = 0;
  if (__any_sync(kFull, act)) {  // warp-uniform: every lane of a live warp takes part
    const uint32_t q = act ? p : n - 1;  // idle tail lanes clone the last lookup (results dropped)
    int mat = 0;
#pragma unroll
    for (int mm = 1; mm < kMats; mm++)
      if (q >= __ldg(mstart + mm)) mat = mm;
    const double E = Es[q];
    double m[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    const int mat0 = __shfl_sync(kFull, mat, 0);
    const bool coop = __all_sync(kFull, mat == mat0 && E == E);
    if (coop) {
      double lo = E, hi = E;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(kFull, lo, o));
        hi = fmax(hi, __shfl_xor_sync(kFull, hi, o));
      }
      const int j0 = T.off[mat], j1 = T.off[mat + 1];
      if (j1 > j0) {
        // reciprocal division needs |hi.E - E| <= 4 (sampled energies are in [0, 1])
        if (X.fastdiv && __all_sync(kFull, fabs(E) <= 2.0))
          warp_nuclide_loop<true>(X, T, E, lo, hi, j0, j1, m);
        else
          warp_nuclide_loop<false>(X, T, E, lo, hi, j0, j1, m);
      }
    } else {  // material boundary inside the warp (at most 11 per batch) or NaN energies
      macro_xs<GF_GRID_NUCLIDE, false>(X, T, E, 0, mat, m);
    }
    if (act) {
      v = argmax5_plus1(m);
      if (out.any()) write_out<5>(out, idx[p], m);
    }
  }
  hash_epilogue(v, vsum);
}
