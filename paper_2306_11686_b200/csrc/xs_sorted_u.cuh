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

constexpr int kDepth = 8;   // index-grid lookahead (nuclides)
constexpr int kPairPf = 3;  // record-pair L1 prefetch lookahead (nuclides), < kDepth

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
