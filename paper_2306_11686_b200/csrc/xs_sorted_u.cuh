// xs_sorted_u.cuh -- the production sorted unionized lookup (included by xs_lookup.cu).
//
// Persistent CTAs (grid = SMs x resident CTAs) stage the material tables in SMEM once and walk tiles
// of kLookupTpb consecutive sorted lookups, one thread per lookup.  Per lookup the nuclide loop is
// software-pipelined at two depths:
//   * index grid: IG[nuc][u] for the next kDepth nuclides is in flight in registers (u16 values;
//     lanes of a warp hold neighbouring u, so each warp load touches 1-3 sectors of the row) -- the
//     index grid is the one structure this path streams from HBM, kDepth hides its latency;
//   * record pairs: the 96-B pair (and reciprocal width) of nuclide j+1 is loaded while j is
//     accumulated; sorted neighbours share pairs, so these hit L1 (SMEM is kept small for that).
// The loop body is unrolled by kDepth so the register ring is statically indexed.
#pragma once

constexpr int kDepth = 16;  // index-grid lookahead (nuclides)
constexpr int kPairPf = 6;  // record-pair L1 prefetch lookahead (nuclides), < kDepth

// A3 for every sorted lookup in a separate, massively parallel pass: us[p] = u of lookup p.
__global__ void __launch_bounds__(256) us_prep(XsDev X, uint32_t n, const double *__restrict__ Es,
                                               uint32_t *__restrict__ us) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) us[p] = (uint32_t)energy_index<GF_GRID_UNIONIZED>(X, Es[p]);
}

template <bool FAST>
__device__ __forceinline__ void unionized_loop(const XsDev &X, const XsTables &T, double E, uint32_t u, int j0, int j1,
                                               double m[5]) {
  uint32_t kq[kDepth];
#pragma unroll
  for (int i = 0; i < kDepth; i++) kq[i] = (j0 + i < j1) ? (uint32_t)__ldg(X.IG + T.ent[j0 + i].y + u) : 0u;
  Pair A, B;
  load_pair<FAST>(X, T.ent[j0].x + kq[0], A);
  for (int j = j0; j < j1; j += kDepth) {
#pragma unroll
    for (int i = 0; i < kDepth; i++) {
      const int jj = j + i;
      if (jj >= j1) break;
      Pair &cur = (i & 1) ? B : A;
      Pair &nxt = (i & 1) ? A : B;
      if (jj + kPairPf < j1) {  // L1 prefetch of the pair (and reciprocal) kPairPf nuclides ahead
        const uint32_t rec = T.ent[jj + kPairPf].x + kq[(i + kPairPf) % kDepth];
        const char *a = reinterpret_cast<const char *>(X.G + (size_t)rec * 6);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a + 88));
        if (FAST) asm volatile("prefetch.global.L1 [%0];" ::"l"(X.Rd + rec));
      }
      if (jj + 1 < j1) load_pair<FAST>(X, T.ent[jj + 1].x + kq[(i + 1) % kDepth], nxt);
      if (jj + kDepth < j1) kq[i] = (uint32_t)__ldg(X.IG + T.ent[jj + kDepth].y + u);
      accumulate<FAST>(cur, E, T.conc[jj], m);
    }
  }
}

template <bool FAST>
__global__ void __launch_bounds__(kLookupTpb, 4)
    xs_lookup_sorted_u(XsDev X, uint32_t n, const double *__restrict__ Es, const uint32_t *__restrict__ us,
                       const uint32_t *__restrict__ idx, const uint32_t *__restrict__ mstart, double *__restrict__ macro_out,
                       unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(128) unsigned char smem[];
  const XsTables T = stage_xs_tables(X, smem);
  uint32_t ms[kMats + 1];
#pragma unroll
  for (int mm = 0; mm <= kMats; mm++) ms[mm] = __ldg(mstart + mm);
  uint32_t vacc = 0;
  const uint32_t ntiles = (n + kLookupTpb - 1) / kLookupTpb;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t p = tile * kLookupTpb + threadIdx.x;
    if (p >= n) continue;
    int mat = 0;
#pragma unroll
    for (int mm = 1; mm < kMats; mm++)
      if (p >= ms[mm]) mat = mm;
    const double E = Es[p];
    const uint32_t u = us[p];
    double m[5];
#pragma unroll
    for (int c = 0; c < 5; c++) m[c] = 0.0;
    const int j0 = T.off[mat], j1 = T.off[mat + 1];
    if (j1 > j0) {
      if (FAST && fabs(E) <= 2.0)
        unionized_loop<FAST>(X, T, E, u, j0, j1, m);
      else
        unionized_loop<false>(X, T, E, u, j0, j1, m);
    }
    vacc += argmax5_plus1(m);
    if (macro_out) {
      const size_t o = (size_t)idx[p] * 5;
#pragma unroll
      for (int c = 0; c < 5; c++) macro_out[o + c] = m[c];
    }
  }
  hash_epilogue(vacc, vsum);
}

// ------------------------------------------------------------------------------------------ 4 per thread
// Each thread owns kL consecutive sorted lookups.  Sorted neighbours nearly always fall into the
// same interval of a nuclide, so one record-pair load (6 x 16 B) feeds kL interpolations: the L1 ->
// register traffic per micro evaluation drops kL-fold (with one lookup per thread a warp pulls 32 x
// 104 B per nuclide through the 128-B/clk L1 data path, more cycles than its FP64 work) and each
// thread carries kL independent FP64 chains.  A lookup whose interval differs reloads the pair.
constexpr int kL = 4;
constexpr int kTpbL = 128;
constexpr int kIgPf = 10;  // index-grid L2 prefetch distance (nuclides)

template <bool FAST>
__device__ __forceinline__ void accumulate_group(const XsDev &X, uint32_t rec_base, const uint32_t (&k)[kL], Pair &P,
                                                 uint32_t &kP, const double (&E)[kL], double conc, double (&m)[kL][5]) {
#pragma unroll
  for (int i = 0; i < kL; i++) {
    if (k[i] != kP) {  // another interval than the staged pair (rare): reload
      load_pair<FAST>(X, rec_base + k[i], P);
      kP = k[i];
    }
    accumulate<FAST>(P, E[i], conc, m[i]);
  }
}

__device__ __forceinline__ void load_k(const XsDev &X, uint32_t row, const uint32_t (&u)[kL], uint32_t (&k)[kL]) {
#pragma unroll
  for (int i = 0; i < kL; i++) k[i] = __ldg(X.IG + row + u[i]);
}

// Nuclides j0..j1-1 for kL lookups: index-grid values 3 nuclides ahead (register ring) and kIgPf
// ahead in L2 (prefetch), the pair of lookup 0's interval 1 nuclide ahead (two buffers); unrolled
// by 4 so the rings are statically indexed.  (A deeper ring overflows the instruction cache or the
// register file: measured.)
template <bool FAST>
__device__ __forceinline__ void unionized_loop4(const XsDev &X, const XsTables &T, const double (&E)[kL],
                                                const uint32_t (&u)[kL], int j0, int j1, double (&m)[kL][5]) {
  uint32_t kq[4][kL];
#pragma unroll
  for (int i = 0; i < 3; i++)
    if (j0 + i < j1) load_k(X, T.ent[j0 + i].y, u, kq[i]);
  Pair A, B;
  uint32_t kA = kq[0][0], kB = 0xFFFFFFFFu;
  load_pair<FAST>(X, T.ent[j0].x + kA, A);
  for (int j = j0; j < j1; j += 4) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int jj = j + i;
      if (jj >= j1) break;
      Pair &cur = (i & 1) ? B : A;
      Pair &nxt = (i & 1) ? A : B;
      uint32_t &kcur = (i & 1) ? kB : kA;
      uint32_t &knxt = (i & 1) ? kA : kB;
      if (jj + 1 < j1) {
        knxt = kq[(i + 1) & 3][0];
        load_pair<FAST>(X, T.ent[jj + 1].x + knxt, nxt);
      }
      if (jj + kIgPf < j1)  // index-grid line of nuclide jj + kIgPf into L2 (no register cost)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(X.IG + T.ent[jj + kIgPf].y + u[0]));
      if (jj + 3 < j1) load_k(X, T.ent[jj + 3].y, u, kq[(i + 3) & 3]);
      accumulate_group<FAST>(X, T.ent[jj].x, kq[i], cur, kcur, E, T.conc[jj], m);
    }
  }
}

template <bool FAST>
__global__ void __launch_bounds__(kTpbL, 3)
    xs_lookup_sorted_u4(XsDev X, uint32_t n, const double *__restrict__ Es, const uint32_t *__restrict__ us,
                        const uint32_t *__restrict__ idx, const uint32_t *__restrict__ mstart,
                        double *__restrict__ macro_out, unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t ms[kMats + 1];  // material segment starts (SMEM: registers go to the loop)
  if (threadIdx.x <= kMats) ms[threadIdx.x] = __ldg(mstart + threadIdx.x);
  const XsTables T = stage_xs_tables(X, smem);  // (its __syncthreads also publishes ms)
  uint32_t vacc = 0;
  const uint32_t ngroups = (n + kL - 1) / kL;
  for (uint32_t g = blockIdx.x * kTpbL + threadIdx.x; g < ngroups; g += gridDim.x * kTpbL) {
    const uint32_t p0 = g * kL;
    const uint32_t nl = min((uint32_t)kL, n - p0);
    int mat0 = 0, mat1 = 0;
#pragma unroll
    for (int mm = 1; mm < kMats; mm++) {
      if (p0 >= ms[mm]) mat0 = mm;
      if (p0 + nl - 1 >= ms[mm]) mat1 = mm;
    }
    double E[kL];
    uint32_t u[kL];
    double m[kL][5];
#pragma unroll
    for (int i = 0; i < kL; i++) {
      const uint32_t p = p0 + min((uint32_t)i, nl - 1);
      E[i] = Es[p];
      u[i] = us[p];
#pragma unroll
      for (int c = 0; c < 5; c++) m[i][c] = 0.0;
    }
    bool fast = FAST;
#pragma unroll
    for (int i = 0; i < kL; i++) fast = fast && fabs(E[i]) <= 2.0;
    if (nl == kL && mat0 == mat1 && fast) {
      const int j0 = T.off[mat0], j1 = T.off[mat0 + 1];
      if (j1 > j0) unionized_loop4<FAST>(X, T, E, u, j0, j1, m);
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
          Pair P;
          const uint32_t rec = T.ent[j].x + (uint32_t)__ldg(X.IG + T.ent[j].y + u[i]);
          if (fi) {
            load_pair<FAST>(X, rec, P);
            accumulate<FAST>(P, E[i], T.conc[j], mi);
          } else {
            load_pair<false>(X, rec, P);
            accumulate<false>(P, E[i], T.conc[j], mi);
          }
        }
#pragma unroll
        for (int c = 0; c < 5; c++) m[i][c] = mi[c];
      }
    }
    for (uint32_t i = 0; i < nl; i++) {
      vacc += argmax5_plus1(m[i]);
      if (macro_out) {
        const size_t o = (size_t)idx[p0 + i] * 5;
#pragma unroll
        for (int c = 0; c < 5; c++) macro_out[o + c] = m[i][c];
      }
    }
  }
  hash_epilogue(vacc, vsum);
}

template <bool FAST>
static cudaError_t launch_sorted_u4(const XsDev &X, uint32_t n, const SortScratch &S, double *macro_out,
                                    unsigned long long *vsum, cudaStream_t st) {
  const size_t smem = xs_table_smem(X.total);
  static int blocks_per_sm[2] = {0, 0};
  static size_t smem_cfg[2] = {0, 0};
  cudaError_t e;
  if (smem_cfg[FAST] != smem) {
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm[FAST], xs_lookup_sorted_u4<FAST>, kTpbL,
                                                           smem)) != cudaSuccess)
      return e;
    smem_cfg[FAST] = smem;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t ngroups = (n + kL - 1) / kL;
  const uint32_t grid = min((ngroups + kTpbL - 1) / kTpbL, (uint32_t)(sms * max(blocks_per_sm[FAST], 1)));
  us_prep<<<nblk(n, 256), 256, 0, st>>>(X, n, S.Es, S.us);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  xs_lookup_sorted_u4<FAST><<<grid, kTpbL, smem, st>>>(X, n, S.Es, S.us, S.idx, S.mstart, macro_out, vsum);
  return cudaGetLastError();
}

template <bool FAST>
static cudaError_t launch_sorted_u(const XsDev &X, uint32_t n, const SortScratch &S, double *macro_out,
                                   unsigned long long *vsum, cudaStream_t st) {
  const size_t smem = xs_table_smem(X.total);
  static int blocks_per_sm[2] = {0, 0};
  static size_t smem_cfg[2] = {0, 0};
  cudaError_t e;
  if (smem_cfg[FAST] != smem) {
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm[FAST], xs_lookup_sorted_u<FAST>,
                                                           kLookupTpb, smem)) != cudaSuccess)
      return e;
    smem_cfg[FAST] = smem;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t ntiles = (n + kLookupTpb - 1) / kLookupTpb;
  const uint32_t grid = min(ntiles, (uint32_t)(sms * max(blocks_per_sm[FAST], 1)));
  us_prep<<<nblk(n, 256), 256, 0, st>>>(X, n, S.Es, S.us);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  xs_lookup_sorted_u<FAST><<<grid, kLookupTpb, smem, st>>>(X, n, S.Es, S.us, S.idx, S.mstart, macro_out, vsum);
  return cudaGetLastError();
}
