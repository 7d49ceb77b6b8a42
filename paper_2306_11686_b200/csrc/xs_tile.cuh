// xs_tile.cuh -- the warp-tile sorted lookup kernel (A3-A6 over a locality-sorted batch; included by
// xs_lookup.cu after xs_sorted_u.cuh).
//
// A warp owns a tile of 128 consecutive sorted lookups (lane l: positions 4l .. 4l+3, sorted by energy
// in registers).  After the locality sort a tile lies in one material and a narrow energy range
// starting at Emin, so for every nuclide of the material the tile's intervals start at
// klo = K(Emin), where K(E) = clamp(#{A <= E} - 1, 0, n_gp - 2) is the plain interval
// (SURVEY.md:520-521).  K is monotone, so for every lookup of the tile (R-TILE)
//     c(E) = #{m in {1, 2} : A[klo + m] <= E},   K(E) = klo + min(c(E), n_gp - 2 - klo)   if c(E) < 2,
// and K(E) >= klo + 2 otherwise (then the literal per-lookup search runs; rare for dense batches).
// The grid-type search therefore runs once per (tile, nuclide) instead of once per (lookup, nuclide),
// and the two interval records klo, klo + 1 -- one contiguous 256-B piece of the interval-record
// array XR, whose first doubles are the boundary energies A[klo + 1], A[klo + 2] -- are staged into
// shared memory by one cp.async.bulk per (tile, nuclide), issued by the lane that found klo.
//
// Pipeline per warp (no producer warp, no CTA barrier): the nuclides of the material are walked in
// chunks of 16; chunk c's records are copied into one of two SMEM buffers while chunk c-1 is
// computed, and the grid-type search of chunk c+2 is issued before chunk c is computed, so neither
// the index-grid load nor the bulk copy is on the critical path after a tile's first two chunks.
// The nuclide loop reads only shared memory: the slot's {record index, clamp}, the two boundaries and
// one record (LDS broadcasts: the lanes of a warp nearly always share the slot's record).
//
// Grid types: unionized (klo from the index grid at the tile's smallest union index), hash (the
// literal hash search at Emin; the tile takes this path only if every lookup lies strictly inside
// its hash bin, RN(b du) < E < RN((b+1) du), where the literal edge rules cannot fire and the
// literal search returns K(E) -- DESIGN.md R-TILE), and kGridNB (per-nuclide bin brackets, no index
// grid).  Tiles that straddle a material boundary or the batch end, or hold energies outside
// [+0, 2] (caller energies), take the one-by-one path with the literal per-lookup search.
#pragma once

constexpr int kTileTpb = 128;  // 4 warps per CTA
constexpr int kTileWarps = kTileTpb / 32;
constexpr int kChunk = 10;     // nuclides per staged chunk (lanes 0..9 stage one each; 4 CTAs fit an SM)
constexpr int kRecs = 4;       // interval records staged per (tile, nuclide): klo .. klo + 3
constexpr int kSlotBytes = 128 * kRecs;

// mbarrier / bulk-copy (TMA 1-D) helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

struct TileSmem {  // per warp
  unsigned char rec[2][kChunk][kSlotBytes];  // [buffer][slot]: records klo .. klo + kRecs - 1
  uint2 meta[2][kChunk];                     // {record index of klo, n_gp - 2 - klo}
  uint64_t bar[2];                           // one mbarrier per buffer (transaction count = staged bytes)
};

__host__ __device__ inline size_t tile_table_bytes(int total) { return (xs_table_smem(total) + 127) & ~size_t(127); }
__host__ __device__ inline size_t tile_smem(int total) {
  return tile_table_bytes(total) + sizeof(TileSmem) * kTileWarps;
}

// klo of the nuclide of entry e for the tile (one lane): the grid type's literal search at Emin.
template <int GT>
__device__ __forceinline__ uint32_t tile_klo(const XsDev &X, uint2 e, double Emin, uint32_t imin) {
  if (GT == GF_GRID_UNIONIZED) return __ldg(X.IG + e.y + imin);  // (the index grid is clamped to n_gp - 2)
  long long ia = imin;
  if (GT == kGridNB) ia = energy_index<kGridNB>(X, Emin);
  return interval<GT>(X, e, Emin, ia);
}

// Stages chunk [c0, c0 + 16) of the material's entries into buffer b: lane l < 16 copies records
// klo, klo + 1 of entry c0 + l.  klo: this lane's tile_klo for that entry.
__device__ __forceinline__ void tile_stage(const XsDev &X, const XsTables &T, TileSmem &S, int b, int c0, int j1,
                                           uint32_t klo) {
  const int lane = threadIdx.x & 31;
  const int cnt = min(kChunk, j1 - c0);
  if (lane == 0) mbar_arrive_tx(&S.bar[b], (uint32_t)(cnt * kSlotBytes));
  __syncwarp();
  if (lane < cnt) {
    const uint2 e = tab_ent(T, c0 + lane, true);
    const uint32_t kb = e.x + klo;
    const uint32_t nucbase = (e.x / (uint32_t)X.n_gp) * (uint32_t)X.n_gp;  // e.x = nuc n_gp (+ k0 < n_gp)
    S.meta[b][lane] = make_uint2(kb, (uint32_t)(X.n_gp - 2) - (kb - nucbase));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the buffer's previous generic reads
    bulk_g2s(S.rec[b][lane], X.XR + (size_t)kb * 16, kSlotBytes, &S.bar[b]);
  }
}

// One interval record from shared memory (its v0.x = E[k+1], ..., y at double 12).  Plain loads through
// a pointer into the extern __shared__ array: they compile to LDS and stay after the mbarrier wait.
template <bool FAST>
__device__ __forceinline__ void load_rec_smem(const unsigned char *a, Rec &R) {
  const double2 *q = reinterpret_cast<const double2 *>(a);
  R.v0 = q[0];
  R.v1 = q[1];
  R.v2 = q[2];
  R.v3 = q[3];
  R.v4 = q[4];
  R.v5 = q[5];
  if (FAST) R.y = reinterpret_cast<const double *>(a)[12];
}

// (unused) The same with volatile LDS: for conditional reloads, which the compiler must not hoist (hoisted
// speculative copies of the record would need another 26 registers per reload).
template <bool FAST>
__device__ __forceinline__ void load_rec_smem_v(const unsigned char *a, Rec &R) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(a);
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(R.v0.x), "=d"(R.v0.y) : "r"(s) : "memory");
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2 + 16];" : "=d"(R.v1.x), "=d"(R.v1.y) : "r"(s) : "memory");
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2 + 32];" : "=d"(R.v2.x), "=d"(R.v2.y) : "r"(s) : "memory");
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2 + 48];" : "=d"(R.v3.x), "=d"(R.v3.y) : "r"(s) : "memory");
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2 + 64];" : "=d"(R.v4.x), "=d"(R.v4.y) : "r"(s) : "memory");
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2 + 80];" : "=d"(R.v5.x), "=d"(R.v5.y) : "r"(s) : "memory");
  if (FAST) asm volatile("ld.shared.f64 %0, [%1 + 96];" : "=d"(R.y) : "r"(s) : "memory");
}

// Predicated reload (one asm statement, no branch): lanes with p reload R from shared address a, the
// others keep it.  A branch around plain loads makes ptxas keep speculative record copies (spills).
__device__ __forceinline__ void reload_rec_smem_if(uint32_t a, bool p, Rec &R) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %14, 0;\n"
      " @q ld.shared.v2.f64 {%0, %1}, [%13];\n @q ld.shared.v2.f64 {%2, %3}, [%13 + 16];\n"
      " @q ld.shared.v2.f64 {%4, %5}, [%13 + 32];\n @q ld.shared.v2.f64 {%6, %7}, [%13 + 48];\n"
      " @q ld.shared.v2.f64 {%8, %9}, [%13 + 64];\n @q ld.shared.v2.f64 {%10, %11}, [%13 + 80];\n"
      " @q ld.shared.f64 %12, [%13 + 96];\n}\n"
      : "+d"(R.v0.x), "+d"(R.v0.y), "+d"(R.v1.x), "+d"(R.v1.y), "+d"(R.v2.x), "+d"(R.v2.y), "+d"(R.v3.x),
        "+d"(R.v3.y), "+d"(R.v4.x), "+d"(R.v4.y), "+d"(R.v5.x), "+d"(R.v5.y), "+d"(R.y)
      : "r"(a), "r"((uint32_t)p)
      : "memory");
}

// c(E) = #{m < min(kRecs, lim) : A[klo + 1 + m] <= E}: the interval of E relative to klo when
// c < kRecs (R-TILE; m < lim masks the slot's records beyond the nuclide's last interval).  Bit
// patterns of non-negative doubles order as signed 64-bit integers.
__device__ __forceinline__ uint32_t slot_count(long long eb, const long long (&bb)[kRecs], const bool (&pm)[kRecs]) {
  uint32_t c = 0;
#pragma unroll
  for (int m = 0; m < kRecs; m++) c += (pm[m] && eb >= bb[m]) ? 1u : 0u;
  return c;
}

__device__ __forceinline__ long long smem_bits(const unsigned char *a) { return *reinterpret_cast<const long long *>(a); }

template <int GT, bool FAST>
__device__ __forceinline__ void tile_loop(const XsDev &X, const XsTables &T, TileSmem &S, uint32_t (&phase),
                                          const double (&E)[kL], const uint32_t (&ix)[kL], int j0, int j1,
                                          double Emin, uint32_t imin, double (&m)[kL][5]) {
  const int lane = threadIdx.x & 31;
  long long eb[kL];
#pragma unroll
  for (int i = 0; i < kL; i++) eb[i] = __double_as_longlong(E[i]);
  __syncwarp();  // the previous tile's readers of S are done
  // prologue: stage chunks 0 and 1
  {
    const bool a = lane < kChunk && j0 + lane < j1, b = lane < kChunk && j0 + kChunk + lane < j1;
    const uint2 ea = tab_ent(T, a ? j0 + lane : j0, true), ebn = tab_ent(T, b ? j0 + kChunk + lane : j0, true);
    const uint32_t ka = a ? tile_klo<GT>(X, ea, Emin, imin) : 0u;
    const uint32_t kbn = b ? tile_klo<GT>(X, ebn, Emin, imin) : 0u;
    tile_stage(X, T, S, 0, j0, j1, ka);
    if (j0 + kChunk < j1) tile_stage(X, T, S, 1, j0 + kChunk, j1, kbn);
  }
  int b = 0;
  for (int c0 = j0; c0 < j1; c0 += kChunk, b ^= 1) {
    // grid-type search of chunk c + 2 (consumed when this chunk is done)
    const int c2 = c0 + 2 * kChunk;
    const bool s2 = lane < kChunk && c2 + lane < j1;
    const uint32_t k2 = s2 ? tile_klo<GT>(X, tab_ent(T, c2 + lane, true), Emin, imin) : 0u;
    mbar_wait(&S.bar[b], (phase >> b) & 1u);
    phase ^= 1u << b;
    __syncwarp();
    const int ce = min(c0 + kChunk, j1);
#pragma unroll 1
    for (int jj = c0; jj < ce; jj++) {
      const int s = jj - c0;
      const uint2 mt = S.meta[b][s];
      const uint32_t kb = mt.x, lim = mt.y;
      const unsigned char *ra = S.rec[b][s];
      // boundaries A[klo + 1 + m] = the staged records' first doubles
      long long bb[kRecs];
      bool pm[kRecs];
#pragma unroll
      for (int q = 0; q < kRecs; q++) {
        bb[q] = smem_bits(ra + 128 * q);
        pm[q] = (uint32_t)q < lim;
      }
      const uint32_t ca = slot_count(eb[0], bb, pm), cd = slot_count(eb[kL - 1], bb, pm);
      const double conc = tab_conc(T, jj, true);
      Rec P;
      // common case: every lookup of the warp lies in a staged record and no thread's lookups span two
      // boundaries; then lookup i > 0 is in record ca + [E_i >= A[klo + 1 + ca]]
      if (!__any_sync(0xffffffffu, cd >= (uint32_t)kRecs || cd > ca + 1u)) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(ra);
        long long bx = bb[0];
#pragma unroll
        for (int q = 1; q < kRecs; q++) bx = ca == (uint32_t)q ? bb[q] : bx;
        uint32_t cP = ca;
        load_rec_smem<FAST>(ra + 128 * ca, P);
        if (!__any_sync(0xffffffffu, ca != cd)) {  // no thread straddles: the 4 chains interleave
#pragma unroll
          for (int i = 0; i < kL; i++) accumulate_rec<FAST>(P, E[i], conc, m[i]);
        } else {
        accumulate_rec<FAST>(P, E[0], conc, m[0]);
#pragma unroll
        for (int i = 1; i < kL; i++) {
          // lanes whose lookup i is past their boundary reload (predicated LDS; ptxas spills if this is
          // a branch around plain loads)
          const uint32_t c = (i == kL - 1) ? cd : ca + (eb[i] >= bx && ca != cd ? 1u : 0u);
          reload_rec_smem_if(sa + 128 * c, c != cP, P);
          cP = c;
          accumulate_rec<FAST>(P, E[i], conc, m[i]);
        }
        }
      } else {  // some thread spans two boundaries or has K(E) >= klo + kRecs: per lookup (rare)
#pragma unroll
        for (int i = 0; i < kL; i++) {
          const uint32_t c = slot_count(eb[i], bb, pm);
          if (c < (uint32_t)kRecs) {
            load_rec_smem<FAST>(ra + 128 * c, P);
          } else {  // the literal search
            const uint2 e = tab_ent(T, jj, true);
            long long id = ix[i];
            if (GT == kGridNB) id = energy_index<kGridNB>(X, E[i]);
            load_rec<FAST>(X, e.x + interval<GT>(X, e, E[i], id), P);
          }
          accumulate_rec<FAST>(P, E[i], conc, m[i]);
        }
      }
    }
    __syncwarp();  // every lane is done with buffer b
    if (c2 < j1) tile_stage(X, T, S, b, c2, j1, k2);
  }
}

// One-by-one path: lookups of a tile that straddles a material boundary or the batch end, or with
// energies outside the tile path's domain.  The literal per-lookup search (interval<GT>).
template <int GT, bool FAST>
__device__ __forceinline__ void lookups_one_by_one(const XsDev &X, const XsTables &T, const uint32_t *ms,
                                                   uint32_t p0, uint32_t nl, const double (&E)[kL],
                                                   const uint32_t (&ix)[kL], double (&m)[kL][5]) {
#pragma unroll
  for (uint32_t i = 0; i < (uint32_t)kL; i++) {  // (unrolled: m stays in registers)
    if (i >= nl) break;
    int mat = 0;
#pragma unroll
    for (int mm = 1; mm < kMats; mm++)
      if (p0 + i >= ms[mm]) mat = mm;
    const int j0 = T.off[mat], j1 = T.off[mat + 1];
    double mi[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    const bool fi = FAST && fabs(E[i]) <= 2.0;
    long long id = ix[i];
    if (GT == kGridNB) id = energy_index<kGridNB>(X, E[i]);
    for (int j = j0; j < j1; j++) {
      Rec P;
      const uint2 ej = tab_ent(T, j, true);
      const uint32_t rec = ej.x + interval<GT>(X, ej, E[i], id);
      const double cj = tab_conc(T, j, true);
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

__device__ __forceinline__ long long warp_min64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

#ifndef GF_TILE_MINB
#define GF_TILE_MINB 4
#endif

// ix: the per-lookup grid index from idx_prep (union index / hash bin); unused for kGridNB.
template <int GT, bool FAST>
__global__ void __launch_bounds__(kTileTpb, GF_TILE_MINB)
    xs_lookup_tile(XsDev X, uint32_t n, const double *__restrict__ Es, const uint32_t *__restrict__ ixs,
                   const uint32_t *__restrict__ idx, const uint32_t *__restrict__ mstart, OutSpec out,
                   unsigned long long *__restrict__ vsum, uint32_t *__restrict__ work) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t ms[kMats + 1];
  if (threadIdx.x <= kMats) ms[threadIdx.x] = __ldg(mstart + threadIdx.x);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  TileSmem &S = reinterpret_cast<TileSmem *>(smem + tile_table_bytes(X.total))[warp];
  if (lane == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const XsTables T = stage_xs_tables<true, GT == kGridNB>(X, smem);  // (its __syncthreads publishes ms, bars)
  uint32_t phase = 0;
  n = min(n, ms[kMats]);  // lookups kept by the sort (band grids keep their band's)
  uint32_t vacc = 0;
  const uint32_t ntiles = (n + 32 * kL - 1) / (32 * kL);
  double du = 0.0;
  if (GT == GF_GRID_HASH) du = __ddiv_rn(1.0, (double)X.bins);
  // dynamic tile scheduling: a warp takes the next tile when it finishes one (tiles of the 321-nuclide
  // fuel come first in the sorted order, so the heavy tiles are handed out first)
  for (uint32_t t = next_tile(work); t < ntiles; t = next_tile(work)) {
    const uint32_t P = t * 32 * kL;
    const uint32_t p0 = P + lane * kL;
    const uint32_t nl = p0 < n ? min((uint32_t)kL, n - p0) : 0u;
    double E[kL];
    uint32_t ix[kL];
    double m[kL][5];
    if (nl == kL) {
      asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(E[0]), "=d"(E[1]), "=d"(E[2]), "=d"(E[3]) : "l"(Es + p0));
      if (GT != kGridNB) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(ixs + p0));
        ix[0] = v.x; ix[1] = v.y; ix[2] = v.z; ix[3] = v.w;
      } else {
#pragma unroll
        for (int i = 0; i < kL; i++) ix[i] = 0;
      }
    } else {
#pragma unroll
      for (int i = 0; i < kL; i++) {
        const uint32_t p = nl ? p0 + min((uint32_t)i, nl - 1) : 0u;
        E[i] = nl ? Es[p] : 0.0;
        ix[i] = (nl && GT != kGridNB) ? ixs[p] : 0u;
      }
    }
#pragma unroll
    for (int i = 0; i < kL; i++)
#pragma unroll
      for (int c = 0; c < 5; c++) m[i][c] = 0.0;
    // tile path: whole tile in one material, energies in [+0, 2] (hash grid: strictly inside the bin)
    bool ok = FAST && nl == kL;
#pragma unroll
    for (int i = 0; i < kL; i++) {
      const long long bits = __double_as_longlong(E[i]);
      ok = ok && bits >= 0 && E[i] <= 2.0;
      if (GT == GF_GRID_HASH) {
        const double lo = __dmul_rn((double)ix[i], du);
        const double hi = (int)ix[i] >= X.bins - 1 ? 1.0 / 0.0 : __dmul_rn((double)(ix[i] + 1), du);
        ok = ok && lo < E[i] && E[i] < hi;
      }
    }
    const uint32_t plast = min(P + 32 * kL, n) - 1;
    int mat0 = 0, mat1 = 0;
#pragma unroll
    for (int mm = 1; mm < kMats; mm++) {
      if (P >= ms[mm]) mat0 = mm;
      if (plast >= ms[mm]) mat1 = mm;
    }
    const bool tile = __all_sync(0xffffffffu, ok) && mat0 == mat1;
    uint32_t perm = 0x76543210u;
    if (tile) {
      local_sort(E, ix, perm);
      const double Emin = __longlong_as_double(warp_min64(__double_as_longlong(E[0])));
      const uint32_t imin = __reduce_min_sync(0xffffffffu, ix[0]);
      const int j0 = T.off[mat0], j1 = T.off[mat0 + 1];
      if (j1 > j0) tile_loop<GT, FAST>(X, T, S, phase, E, ix, j0, j1, Emin, imin, m);
    } else if (nl) {
      lookups_one_by_one<GT, FAST>(X, T, ms, p0, nl, E, ix, m);
    }
#pragma unroll
    for (uint32_t i = 0; i < (uint32_t)kL; i++) {
      if (i < nl) {
        vacc += argmax5_plus1(m[i]);
        if (out.any()) write_out<5>(out, idx[p0 + ((perm >> (4 * i)) & 15u)], m[i]);
      }
    }
  }
  hash_epilogue(vacc, vsum);
}

template <int GT, bool FAST>
static cudaError_t launch_tile(const XsDev &X, uint32_t n, const SortScratch &S, const OutSpec &out,
                               unsigned long long *vsum, cudaStream_t st) {
  const size_t smem = tile_smem(X.total);
  int blocks_per_sm = 0;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(xs_lookup_tile<GT, FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, xs_lookup_tile<GT, FAST>, kTileTpb, smem)) !=
      cudaSuccess)
    return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t ntiles = (n + 32 * kL - 1) / (32 * kL);
  const uint32_t grid =
      max(1u, min((ntiles + kTileWarps - 1) / kTileWarps, (uint32_t)(sms * max(blocks_per_sm, 1))));
  if (GT != kGridNB) {
    idx_prep<GT><<<nblk(((long long)n + 3) / 4, 256), 256, 0, st>>>(X, n, S.Es, S.mstart, S.us);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if ((e = cudaMemsetAsync(S.work, 0, sizeof(uint32_t), st)) != cudaSuccess) return e;
  xs_lookup_tile<GT, FAST><<<grid, kTileTpb, smem, st>>>(X, n, S.Es, S.us, S.idx, S.mstart, out, vsum, S.work);
  return cudaGetLastError();
}
