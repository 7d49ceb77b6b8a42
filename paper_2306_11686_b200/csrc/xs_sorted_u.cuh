// xs_sorted_u.cuh -- the production sorted lookup kernel for the unionized and hash grids (included
// by xs_lookup.cu).
//
// Each thread owns kL = 4 consecutive locality-sorted lookups.  Sorted neighbours nearly always fall
// into the same interval of a nuclide, so one record-pair load (6 x 16 B + the 8-B reciprocal width)
// feeds kL interpolations.  This is what the L1 data path needs: with one lookup per thread a warp
// pulls 32 x 104 B per nuclide through the 128-B/clk L1 -> register path, more cycles than the warp's
// FP64 work, while here that traffic drops kL-fold and each thread carries kL independent FP64
// chains.  A lookup whose interval differs from the staged pair reloads it (rare).
//
// The nuclide loop is software-pipelined at three distances: the interval indices of the kL lookups
// 3 nuclides ahead (register ring, unrolled by 4 so it is statically indexed), the index- / hash-grid
// line kIgPf nuclides ahead (prefetch.global.L2, no register cost), the interval record 2 ahead
// (prefetch.global.L1) and the record of the next nuclide (two register buffers).  CTAs are
// persistent (grid = SMs x resident CTAs) and stage the material tables in SMEM once.  A3 runs in a separate massively parallel pass (idx_prep) so its dependent
// search latency is not on this kernel's critical path.
// Measured alternatives: one lookup per thread; a TMA/mbarrier producer-consumer
// ring (removed in round 2: 2x slower); deeper register rings (instruction-cache or register-file
// overflow).
#pragma once

#ifndef GF_GROUP_L
#define GF_GROUP_L 4
#endif
#ifndef GF_GROUP_MINB
#define GF_GROUP_MINB 4
#endif
constexpr int kL = GF_GROUP_L;  // lookups per thread (A/B: -DGF_GROUP_L=2 -DGF_GROUP_MINB=5)
constexpr int kTpbL = 128;
constexpr int kIgPf = 10;  // index-/hash-grid L2 prefetch distance (nuclides)

// A3 for every sorted lookup in a separate, massively parallel pass: ix[p] = u (unionized) or b
// (hash) of lookup p.
// Four consecutive sorted lookups per thread: one 32-B energy load, one 16-B index store, and their
// searches are independent (their probes overlap in flight; neighbours hit the same U lines).
template <int GT>
__global__ void __launch_bounds__(256) idx_prep(XsDev X, uint32_t n, const double *__restrict__ Es,
                                                const uint32_t *__restrict__ mstart, uint32_t *__restrict__ ix) {
  n = min(n, __ldg(mstart + kMats));
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (p + 4 <= n) {
    double e0, e1, e2, e3;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(e0), "=d"(e1), "=d"(e2), "=d"(e3) : "l"(Es + p));
    uint4 r;
    r.x = (uint32_t)energy_index<GT>(X, e0);
    r.y = (uint32_t)energy_index<GT>(X, e1);
    r.z = (uint32_t)energy_index<GT>(X, e2);
    r.w = (uint32_t)energy_index<GT>(X, e3);
    *reinterpret_cast<uint4 *>(ix + p) = r;
  } else {
    for (uint32_t q = p; q < n; q++) ix[q] = (uint32_t)energy_index<GT>(X, Es[q]);
  }
}

// One interval record of XsDev::XR: v0 = (E[k+1], E[k+1] - E[k]), v(1+c) = (xs_c[k+1],
// xs_c[k+1] - xs_c[k]), y = RN(1 / (E[k+1] - E[k])).  Six 16-B loads and one 8-B load from one
// 128-B line (4 sectors), the same instruction count as the 96-B record pair of G plus Rd.
struct Rec {
  double2 v0, v1, v2, v3, v4, v5;
  double y;  // fast division path only
};

#ifndef GF_PACKTAB
#define GF_PACKTAB 1  // group loop: record base + concentration from one 16-B shared load
#endif

#ifndef GF_LD256
#define GF_LD256 1
#endif

// 32-B vector load through the read-only path (sm_100: LDG.E.ENL2.256): one LSU request instead of two.
__device__ __forceinline__ void ldg256(const double *p, double2 &a, double2 &b) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y) : "l"(p));
}

template <bool FAST>
__device__ __forceinline__ void load_rec(const XsDev &X, uint32_t r, Rec &R) {
#if GF_LD256  // records are 128-B aligned: three 32-B loads + the 8-B reciprocal (4 requests, not 7)
  const double *q = X.XR + (size_t)r * 16;
  ldg256(q, R.v0, R.v1);
  ldg256(q + 4, R.v2, R.v3);
  ldg256(q + 8, R.v4, R.v5);
  if (FAST) R.y = __ldg(q + 12);
#else
  const double2 *p = reinterpret_cast<const double2 *>(X.XR) + (size_t)r * 8;
  R.v0 = __ldg(p + 0);
  R.v1 = __ldg(p + 1);
  R.v2 = __ldg(p + 2);
  R.v3 = __ldg(p + 3);
  R.v4 = __ldg(p + 4);
  R.v5 = __ldg(p + 5);
  if (FAST) R.y = __ldg(X.XR + (size_t)r * 16 + 12);
#endif
}

// f = (hi.E - E) / (hi.E - lo.E); x_c = hi_c - f (hi_c - lo_c); m_c += x_c * conc -- the same RN
// operations as accumulate() with the two grid-only differences read from the record.
template <bool FAST>
__device__ __forceinline__ void accumulate_rec(const Rec &R, double E, double conc, double m[5]) {
  const double a = __dsub_rn(R.v0.x, E), b = R.v0.y;
  const double f = FAST ? div_rn(a, b, R.y) : __ddiv_rn(a, b);
  const double2 hd[5] = {R.v1, R.v2, R.v3, R.v4, R.v5};
#pragma unroll
  for (int c = 0; c < 5; c++) {
    const double x = __dsub_rn(hd[c].x, __dmul_rn(f, hd[c].y));
    m[c] = __dadd_rn(m[c], __dmul_rn(x, conc));
  }
}

template <bool FAST>
__device__ __forceinline__ void accumulate_group(const XsDev &X, uint32_t rec_base, const uint32_t (&k)[kL], Rec &P,
                                                 uint32_t &kP, const double (&E)[kL], double conc, double (&m)[kL][5]) {
#pragma unroll
  for (int i = 0; i < kL; i++) {
    if (k[i] != kP) {  // another interval than the staged pair (rare): reload
      load_rec<FAST>(X, rec_base + k[i], P);
      kP = k[i];
    }
    accumulate_rec<FAST>(P, E[i], conc, m[i]);
  }
}

// Prefetches (measured): on the unionized grid both pay (C3 lookup 2.90 ms vs 3.46
// without); on the hash grid they cost more than they hide (C4 46.7 vs 44.5 ms without), and
// issuing them from the first lane of each run of equal lines only (shuffle + compare) is slower.
#ifndef GF_PF_L1
#define GF_PF_L1 1
#endif
#ifndef GF_PF_L2
#define GF_PF_L2 1
#endif

#ifndef GF_ONEBUF
#define GF_ONEBUF 1  // one record register buffer: 128 registers, 16 warps/SM (measured: C3 lookup 3.61 -> 2.98 ms)
#endif

#ifndef GF_SHORTCUT
#define GF_SHORTCUT 1
#endif

// Interval indices of the kL lookups for the nuclide of table entry e.
// Unionized grid: one u16 index-grid load per lookup.
// Hash grid: interval shortcut (DESIGN.md R-SHORT).  Lookup 0's interval k0 is searched literally;
// a lookup i in the same hash bin with A[k0] < E_i < A[k0+1] has interval k0 as well -- the bin's
// edge rules cannot fire for it and the bisection returns the unique k with A[k] <= E_i < A[k+1] --
// so only the rare others are searched.  Grid energies are LCG doubles in [+0, 1): the test compares
// bit patterns as signed 64-bit integers, which order exactly like the doubles for every E_i (NaN,
// -0 and negatives fail it and take the literal search).  (Measured: splitting
// the hash search into two pipeline stages, with or without L1 prefetch of the energies, is slower.)
template <int GT>
__device__ __forceinline__ void load_k(const XsDev &X, uint2 e, const double (&E)[kL], const uint32_t (&ix)[kL],
                                       uint32_t (&k)[kL]) {
  if (GT == GF_GRID_HASH && GF_SHORTCUT) {
    const uint32_t k0 = interval<GT>(X, e, E[0], ix[0]);
    const long long lo = __double_as_longlong(__ldg(X.Ed + e.x + k0));
    const long long hi = __double_as_longlong(__ldg(X.Ed + e.x + k0 + 1));
    k[0] = k0;
#pragma unroll
    for (int i = 1; i < kL; i++) {
      const long long v = __double_as_longlong(E[i]);
      k[i] = (ix[i] == ix[0] && lo < v && v < hi) ? k0 : interval<GT>(X, e, E[i], ix[i]);
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < kL; i++) {
    if (GT == GF_GRID_UNIONIZED)
      k[i] = __ldg(X.IG + e.y + ix[i]);  // never n_gp - 1 (IG is clamped to n_gp - 2)
    else
      k[i] = interval<GT>(X, e, E[i], ix[i]);
  }
}

template <int GT>
__device__ __forceinline__ const void *grid_line(const XsDev &X, uint2 e, uint32_t ix) {
  if (GT == GF_GRID_UNIONIZED) return X.IG + e.y + ix;
  return X.hg32 ? (const void *)(reinterpret_cast<const uint32_t *>(X.HG) + e.y + ix) : (const void *)(X.HG + e.y + ix);
}

#ifndef GF_LOCAL_SORT
#define GF_LOCAL_SORT 1
#endif

// The group's kL lookups in ascending energy (odd-even transposition network, unrolled).  The
// counting sort leaves lookups unordered inside a sort bin; in energy order the intervals k of
// every nuclide are non-decreasing across the slots (k is monotone in E), so a thread reloads its
// record only where a run of equal k ends, and a warp executes the reload of slot i only if some
// lane has a run boundary there (ncu: global load requests 147 M -> 97 M per C3 launch).  Results
// are order-independent; perm maps slots to lookups for the per-lookup outputs.
__device__ __forceinline__ void local_sort(double (&E)[kL], uint32_t (&ix)[kL], uint32_t &perm) {
#pragma unroll
  for (int r = 0; r < kL; r++) {
#pragma unroll
    for (int a = r & 1; a + 1 < kL; a += 2) {
      const int b = a + 1;
      const bool sw = __double_as_longlong(E[b]) < __double_as_longlong(E[a]);  // E >= 0 on this path
      const double e0 = E[a], e1 = E[b];
      E[a] = sw ? e1 : e0;
      E[b] = sw ? e0 : e1;
      const uint32_t i0 = ix[a], i1 = ix[b];
      ix[a] = sw ? i1 : i0;
      ix[b] = sw ? i0 : i1;
      const uint32_t x = ((perm >> (4 * a)) ^ (perm >> (4 * b))) & 15u;
      perm ^= sw ? ((x << (4 * a)) | (x << (4 * b))) : 0u;
    }
  }
}

// Nuclides j0..j1-1 for the kL lookups.
template <int GT, bool FAST>
__device__ __forceinline__ void group_loop(const XsDev &X, const XsTables &T, const double (&E)[kL],
                                           const uint32_t (&ix)[kL], int j0, int j1, double (&m)[kL][5]) {
  uint32_t kq[4][kL];
#pragma unroll
  for (int i = 0; i < 3; i++)
    if (j0 + i < j1) load_k<GT>(X, tab_ent(T, j0 + i, GF_PACKTAB), E, ix, kq[i]);
  Rec A;
  uint32_t kA = kq[0][0];
#if !GF_ONEBUF
  Rec B;
  uint32_t kB = 0xFFFFFFFFu;
  load_rec<FAST>(X, tab_ent(T, j0, GF_PACKTAB).x + kA, A);
#endif
  for (int j = j0; j < j1; j += 4) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int jj = j + i;
      if (jj >= j1) break;
#if GF_ONEBUF  // one record buffer, loaded at the top of the iteration (an L1 hit: prefetched 2 ahead)
      Rec &cur = A;
      uint32_t &kcur = kA;
      kcur = kq[i][0];
      const uint32_t rec_base = tab_ent(T, jj, GF_PACKTAB).x;  // (packed: one 16-B shared load for both)
      const double conc = tab_conc(T, jj, GF_PACKTAB);
      load_rec<FAST>(X, rec_base + kcur, cur);
#else
      Rec &cur = (i & 1) ? B : A;
      Rec &nxt = (i & 1) ? A : B;
      uint32_t &kcur = (i & 1) ? kB : kA;
      uint32_t &knxt = (i & 1) ? kA : kB;
      if (jj + 1 < j1) {
        knxt = kq[(i + 1) & 3][0];
        load_rec<FAST>(X, tab_ent(T, jj + 1, GF_PACKTAB).x + knxt, nxt);
      }
#endif
      constexpr bool kPf = GT != GF_GRID_HASH;
      if (kPf && GF_PF_L2 && jj + kIgPf < j1)  // index-grid line of nuclide jj + kIgPf into L2
        asm volatile("prefetch.global.L2 [%0];" ::"l"(grid_line<GT>(X, tab_ent(T, jj + kIgPf, GF_PACKTAB), ix[0])));
      if (kPf && GF_PF_L1 && jj + 2 < j1)  // the record of nuclide jj + 2 (its interval is in the ring) into L1
        asm volatile("prefetch.global.L1 [%0];" ::"l"(X.XR + (size_t)(tab_ent(T, jj + 2, GF_PACKTAB).x + kq[(i + 2) & 3][0]) * 16));
      if (jj + 3 < j1) load_k<GT>(X, tab_ent(T, jj + 3, GF_PACKTAB), E, ix, kq[(i + 3) & 3]);
#if GF_ONEBUF
      accumulate_group<FAST>(X, rec_base, kq[i], cur, kcur, E, conc, m);
#else
      accumulate_group<FAST>(X, tab_ent(T, jj, GF_PACKTAB).x, kq[i], cur, kcur, E, tab_conc(T, jj, GF_PACKTAB), m);
#endif
    }
  }
}

// Dynamic work distribution (group and tile kernels): lane 0 of a warp takes the next unit of 32
// groups (128 lookups) from a per-launch counter.  Work units come in sorted order, i.e. the
// 321-nuclide fuel first, so the heavy units are handed out first and warps finish together
// (a static grid-stride split left SMs idle for ~25% of the kernel, ncu active vs elapsed cycles).
__device__ __forceinline__ uint32_t next_tile(uint32_t *work) {
  uint32_t t = 0;
  if ((threadIdx.x & 31) == 0) t = atomicAdd(work, 1u);
  return __shfl_sync(0xffffffffu, t, 0);
}

template <int GT, bool FAST>
__global__ void __launch_bounds__(kTpbL, GF_GROUP_MINB)
    xs_lookup_group(XsDev X, uint32_t n, const double *__restrict__ Es, const uint32_t *__restrict__ ixs,
                    const uint32_t *__restrict__ idx, const uint32_t *__restrict__ mstart,
                    OutSpec out, unsigned long long *__restrict__ vsum, uint32_t *__restrict__ work) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t ms[kMats + 1];  // material segment starts (SMEM: registers go to the loop)
  if (threadIdx.x <= kMats) ms[threadIdx.x] = __ldg(mstart + threadIdx.x);
  const XsTables T = stage_xs_tables<GF_PACKTAB>(X, smem);  // (its __syncthreads also publishes ms)
  n = min(n, ms[kMats]);  // lookups kept by the sort (band grids keep their band's)
  uint32_t vacc = 0;
  const uint32_t ngroups = (n + kL - 1) / kL;
  for (uint32_t wg = next_tile(work); wg * 32 < ngroups; wg = next_tile(work)) {
    const uint32_t g = wg * 32 + (threadIdx.x & 31);
    if (g >= ngroups) continue;
    const uint32_t p0 = g * kL;
    const uint32_t nl = min((uint32_t)kL, n - p0);
    int mat0 = 0, mat1 = 0;
#pragma unroll
    for (int mm = 1; mm < kMats; mm++) {
      if (p0 >= ms[mm]) mat0 = mm;
      if (p0 + nl - 1 >= ms[mm]) mat1 = mm;
    }
    double E[kL];
    uint32_t ix[kL];
    double m[kL][5];
#pragma unroll
    for (int i = 0; i < kL; i++) {
      const uint32_t p = p0 + min((uint32_t)i, nl - 1);
      E[i] = Es[p];
      ix[i] = ixs[p];
#pragma unroll
      for (int c = 0; c < 5; c++) m[i][c] = 0.0;
    }
    bool fast = FAST;
#pragma unroll
    for (int i = 0; i < kL; i++) fast = fast && fabs(E[i]) <= 2.0;
    uint32_t perm = 0x76543210u;  // slot i holds the group's lookup (perm >> 4 i) & 15
    if (nl == kL && mat0 == mat1 && fast) {
#if GF_LOCAL_SORT
      local_sort(E, ix, perm);
#endif
      const int j0 = T.off[mat0], j1 = T.off[mat0 + 1];
      if (j1 > j0) group_loop<GT, FAST>(X, T, E, ix, j0, j1, m);
    } else {  // group straddles a material boundary or the batch end, or odd energies: one by one
      for (uint32_t i = 0; i < nl; i++) {
        int mat = 0;
#pragma unroll
        for (int mm = 1; mm < kMats; mm++)
          if (p0 + i >= ms[mm]) mat = mm;
        const int j0 = T.off[mat], j1 = T.off[mat + 1];
        double mi[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        const bool fi = FAST && fabs(E[i]) <= 2.0;
        for (int j = j0; j < j1; j++) {  // plain loop: these lookups are a handful per batch
          Rec P;
          const uint2 ej = tab_ent(T, j, GF_PACKTAB);
          const uint32_t rec = ej.x + interval<GT>(X, ej, E[i], ix[i]);
          const double cj = tab_conc(T, j, GF_PACKTAB);
          if (fi) {
            load_rec<FAST>(X, rec, P);
            accumulate_rec<FAST>(P, E[i], cj, mi);
          } else {
            load_rec<false>(X, rec, P);
            accumulate_rec<false>(P, E[i], cj, mi);
          }
        }
#pragma unroll
        for (int c = 0; c < 5; c++) m[i][c] = mi[c];
      }
    }
    for (uint32_t i = 0; i < nl; i++) {
      vacc += argmax5_plus1(m[i]);
      if (out.any()) write_out<5>(out, idx[p0 + ((perm >> (4 * i)) & 15u)], m[i]);
    }
  }
  hash_epilogue(vacc, vsum);
}

template <int GT, bool FAST>
static cudaError_t launch_group(const XsDev &X, uint32_t n, const SortScratch &S, const OutSpec &out,
                                unsigned long long *vsum, cudaStream_t st) {
  const size_t smem = xs_table_smem(X.total);
  // set per call (the attribute is per device; no cached state shared between host threads)
  int blocks_per_sm = 0;
  cudaError_t e;
  if ((e = allow_smem(xs_lookup_group<GT, FAST>, smem)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, xs_lookup_group<GT, FAST>, kTpbL, smem)) !=
      cudaSuccess)
    return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t ngroups = (n + kL - 1) / kL;
  const uint32_t grid = min((ngroups + kTpbL - 1) / kTpbL, (uint32_t)(sms * max(blocks_per_sm, 1)));
  idx_prep<GT><<<nblk(((long long)n + 3) / 4, 256), 256, 0, st>>>(X, n, S.Es, S.mstart, S.us);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(S.work, 0, sizeof(uint32_t), st)) != cudaSuccess) return e;
  xs_lookup_group<GT, FAST><<<grid, kTpbL, smem, st>>>(X, n, S.Es, S.us, S.idx, S.mstart, out, vsum, S.work);
  return cudaGetLastError();
}
