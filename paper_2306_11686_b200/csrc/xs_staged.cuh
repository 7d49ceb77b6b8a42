// xs_staged.cuh -- the sorted unionized lookup with the index-grid stream on the TMA engine.
// Included by xs_lookup.cu (uses its XsTables / Pair / accumulate / nuclide_loop / energy_index).
//
// Persistent CTAs of 4 consumer warps + 1 producer warp walk tiles of kTile consecutive sorted
// lookups.  staged_prep (a separate, massively parallel pass) computes each sorted lookup's
// unionized index u and each tile's facts: material of its first / last lookup and [min u, max u].
// A tile whose lookups share one material and whose u range spans <= kIgCap entries is "staged":
// for each nuclide j of the material the producer lane issues one cp.async.bulk of the tile's
// index-grid row segment IG[nuc][u_lo..u_hi] into SMEM stage s of a kStages ring (mbarrier full[s]
// completes on the transaction count; empty[s] takes one arrival per consumer warp).  The producer
// has no dependent work, so the ring runs kStages items ahead of the consumers and the DRAM
// latency of the index grid (the one structure this path streams from HBM) is hidden.  Consumers
// read their interval index k from SMEM, release the stage at once, and load the 96-B record pair
// (and reciprocal width) with one item of lookahead -- sorted neighbours share records, so these
// hit L1/L2.  Other tiles (mixed material, sparse materials whose u range is wide) run the
// per-thread pipelined loop.  Results are bit-identical to every other kernel: same index, same
// arithmetic, same order.
#pragma once

constexpr int kTile = 128;                   // lookups per tile = consumer threads
constexpr int kStagedThreads = kTile + 32;   // + producer warp
constexpr int kStages = 24;                  // ring depth (items of lookahead)
constexpr int kIgCap = 1024;                 // index-grid entries per stage (2 KB)
constexpr int kStageBytes = 2 * kIgCap;

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

inline size_t staged_smem(int total) {
  size_t t = (xs_table_smem(total) + 15) & ~size_t(15);
  t += 2 * kStages * 8;
  t = (t + 127) & ~size_t(127);
  return t + (size_t)kStages * kStageBytes;
}

// Tile facts, written by staged_prep, read by the producer and the consumers.
struct TileInfo {
  int staged, j0, cnt, mat;
  uint32_t ubase, ulo, uhi, pad;
};

__device__ __forceinline__ int material_of(const uint32_t *mstart, uint32_t p) {
  int mat = 0;
#pragma unroll
  for (int mm = 1; mm < kMats; mm++)
    if (p >= __ldg(mstart + mm)) mat = mm;
  return mat;
}

// One CTA of kTile threads per tile: us[p] = the unionized index of sorted lookup p (A3, the same
// two-level search as every other kernel), and the tile's facts.
__global__ void __launch_bounds__(kTile) staged_prep(XsDev X, uint32_t n, const double *__restrict__ Es,
                                                     const uint32_t *__restrict__ mstart, uint32_t *__restrict__ us,
                                                     TileInfo *__restrict__ tinfo) {
  __shared__ uint32_t s_lo[kTile / 32], s_hi[kTile / 32];
  const uint32_t tile = blockIdx.x, p0 = tile * kTile, plast = min(n, p0 + kTile) - 1;
  const uint32_t p = p0 + threadIdx.x, pc = min(p, plast);
  const double E = Es[pc];
  const uint32_t u = (uint32_t)energy_index<GF_GRID_UNIONIZED>(X, E);
  if (p < n) us[p] = u;
  const uint32_t lo = __reduce_min_sync(0xffffffffu, u), hi = __reduce_max_sync(0xffffffffu, u);
  // energies outside [-2, 2] (caller-supplied only) need the IEEE division path: not staged
  const int odd = __syncthreads_or(!(fabs(E) <= 2.0));
  if ((threadIdx.x & 31) == 0) {
    s_lo[threadIdx.x >> 5] = lo;
    s_hi[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t ulo = s_lo[0], uhi = s_hi[0];
    for (int w = 1; w < kTile / 32; w++) {
      ulo = min(ulo, s_lo[w]);
      uhi = max(uhi, s_hi[w]);
    }
    const int mlo = material_of(mstart, p0), mhi = material_of(mstart, plast);
    TileInfo t;
    t.mat = mlo;
    t.ubase = ulo & ~7u;
    t.ulo = ulo;
    t.uhi = uhi;
    t.pad = 0;
    const uint32_t uend = (uhi + 8) & ~7u;  // exclusive, 16-B multiple of u16 entries
    t.j0 = __ldg(X.moff + mlo);
    const int j1 = __ldg(X.moff + mlo + 1);
    t.staged = (mlo == mhi) && (uend - t.ubase <= (uint32_t)kIgCap) && (j1 > t.j0) && !odd;
    t.cnt = t.staged ? j1 - t.j0 : 0;
    tinfo[tile] = t;
  }
}

__device__ __forceinline__ TileInfo load_tinfo(const TileInfo *t) {
  const int4 a = __ldg(reinterpret_cast<const int4 *>(t)), b = __ldg(reinterpret_cast<const int4 *>(t) + 1);
  TileInfo r;
  r.staged = a.x;
  r.j0 = a.y;
  r.cnt = a.z;
  r.mat = a.w;
  r.ubase = (uint32_t)b.x;
  r.ulo = (uint32_t)b.y;
  r.uhi = (uint32_t)b.z;
  r.pad = 0;
  return r;
}

// Consumer side of one staged item: wait for stage g, read k, release the stage (one arrival per
// warp), issue the record-pair loads.
template <bool FAST>
__device__ __forceinline__ void staged_fetch(const XsDev &X, unsigned char *stages, uint64_t *full, uint64_t *empty,
                                             uint32_t g, uint32_t urel, uint32_t rec_base, int lane, Pair &P) {
  const uint32_t s = g % kStages, ph = (g / kStages) & 1u;
  mbar_wait(&full[s], ph);
  const uint32_t k = reinterpret_cast<const uint16_t *>(stages + (size_t)s * kStageBytes)[urel];
  __syncwarp();
  if (lane == 0) mbar_arrive(&empty[s]);
  load_pair<FAST>(X, rec_base + k, P);
}

// Look kPeek items ahead in the ring: read that item's interval index from its (landed) stage and
// prefetch its record pair and reciprocal width into L1, so the loads of staged_fetch hit.
constexpr int kPeek = 4;
static_assert(kPeek + 2 < kStages, "the peeked stage must still be held by the consumers");

template <bool FAST>
__device__ __forceinline__ void staged_peek(const XsDev &X, unsigned char *stages, uint64_t *full, uint32_t g,
                                            uint32_t urel, uint32_t rec_base) {
  const uint32_t s = g % kStages, ph = (g / kStages) & 1u;
  mbar_wait(&full[s], ph);
  const uint32_t k = reinterpret_cast<const uint16_t *>(stages + (size_t)s * kStageBytes)[urel];
  const char *a = reinterpret_cast<const char *>(X.G + (size_t)(rec_base + k) * 6);
  asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(a + 88));
  if (FAST) asm volatile("prefetch.global.L1 [%0];" ::"l"(X.Rd + rec_base + k));
}

// Staged tiles only hold energies in [-2, 2] (staged_prep), so FAST needs no per-lookup check.
template <bool FAST>
__device__ __forceinline__ void staged_loop(const XsDev &X, const XsTables &T, unsigned char *stages, uint64_t *full,
                                            uint64_t *empty, uint32_t it, const TileInfo &ti, uint32_t urel,
                                            double E, int lane, double m[5]) {
  Pair A, B;
  const int j0 = ti.j0, cnt = ti.cnt;
  for (int q = 0; q < kPeek && q < cnt; q++) staged_peek<FAST>(X, stages, full, it + q, urel, T.ent[j0 + q].x);
  staged_fetch<FAST>(X, stages, full, empty, it, urel, T.ent[j0].x, lane, A);
  for (int q = 0; q < cnt; q += 2) {
    if (q + kPeek < cnt) staged_peek<FAST>(X, stages, full, it + q + kPeek, urel, T.ent[j0 + q + kPeek].x);
    if (q + 1 + kPeek < cnt)
      staged_peek<FAST>(X, stages, full, it + q + 1 + kPeek, urel, T.ent[j0 + q + 1 + kPeek].x);
    if (q + 1 < cnt) staged_fetch<FAST>(X, stages, full, empty, it + q + 1, urel, T.ent[j0 + q + 1].x, lane, B);
    accumulate<FAST>(A, E, T.conc[j0 + q], m);
    if (q + 1 >= cnt) break;
    if (q + 2 < cnt) staged_fetch<FAST>(X, stages, full, empty, it + q + 2, urel, T.ent[j0 + q + 2].x, lane, A);
    accumulate<FAST>(B, E, T.conc[j0 + q + 1], m);
  }
}

template <bool FAST>
__global__ void __launch_bounds__(kStagedThreads, 3)
    xs_lookup_staged(XsDev X, uint32_t n, const double *__restrict__ Es, const uint32_t *__restrict__ us,
                     const TileInfo *__restrict__ tinfo, const uint32_t *__restrict__ idx,
                     const uint32_t *__restrict__ mstart, OutSpec out,
                     unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(128) unsigned char smem[];
  const XsTables T = stage_xs_tables(X, smem);
  size_t off = (xs_table_smem(X.total) + 15) & ~size_t(15);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + off);
  uint64_t *empty = full + kStages;
  off = (off + 2 * kStages * 8 + 127) & ~size_t(127);
  unsigned char *stages = smem + off;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTile / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t ntiles = (n + kTile - 1) / kTile;

  if (warp == kTile / 32) {
    // ================================================================ producer warp (lane 0 issues)
    uint32_t g = 0;
    TileInfo nxt = load_tinfo(tinfo + min((uint32_t)blockIdx.x, ntiles - 1));
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const TileInfo ti = nxt;
      if (tile + gridDim.x < ntiles) nxt = load_tinfo(tinfo + tile + gridDim.x);  // one tile ahead
      if (!ti.staged) continue;
      const uint32_t bytes = (((ti.uhi + 8) & ~7u) - ti.ubase) * 2;
      for (int q = 0; q < ti.cnt; q++, g++) {
        const uint32_t s = g % kStages, ph = (g / kStages) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        if (lane == 0) {
          mbar_arrive_tx(&full[s], bytes);
          bulk_g2s(stages + (size_t)s * kStageBytes, X.IG + T.ent[ti.j0 + q].y + ti.ubase, bytes, &full[s]);
        }
        __syncwarp();
      }
    }
    hash_epilogue(0u, vsum);
    return;
  }

  // ================================================================== consumer warps
  uint32_t it = 0;  // staged items consumed so far (ring position)
  uint32_t vacc = 0;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t p0 = tile * kTile;
    const uint32_t plast = min(n, p0 + kTile) - 1;
    const uint32_t p = p0 + tid, pc = min(p, plast);
    const TileInfo ti = load_tinfo(tinfo + tile);
    const double E = Es[pc];
    const uint32_t u = us[pc];
    double m[5];
#pragma unroll
    for (int c = 0; c < 5; c++) m[c] = 0.0;
    const bool fast = FAST && fabs(E) <= 2.0;
    if (ti.staged) {
      staged_loop<FAST>(X, T, stages, full, empty, it, ti, u - ti.ubase, E, lane, m);
      it += (uint32_t)ti.cnt;
    } else {
      const int mat = material_of(mstart, pc);
      const int a0 = T.off[mat], a1 = T.off[mat + 1];
      if (a1 > a0) {
        if (fast)
          nuclide_loop<GF_GRID_UNIONIZED, true, false>(X, T, E, u, a0, a1, m);
        else
          nuclide_loop<GF_GRID_UNIONIZED, false, false>(X, T, E, u, a0, a1, m);
      }
    }
    if (p < n) {
      vacc += argmax5_plus1(m);
      if (out.any()) write_out<5>(out, idx[p], m);
    }
  }
  hash_epilogue(vacc, vsum);
}

template <bool FAST>
static cudaError_t launch_staged(const XsDev &X, uint32_t n, const SortScratch &S, const OutSpec &out,
                                 unsigned long long *vsum, cudaStream_t st) {
  const size_t smem = staged_smem(X.total);
  // set per call (the attribute is per device; no cached state shared between host threads)
  int blocks_per_sm = 0;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(xs_lookup_staged<FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, xs_lookup_staged<FAST>, kStagedThreads,
                                                         smem)) != cudaSuccess)
    return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t ntiles = (n + kTile - 1) / kTile;
  TileInfo *tinfo = reinterpret_cast<TileInfo *>(S.tinfo);
  staged_prep<<<ntiles, kTile, 0, st>>>(X, n, S.Es, S.mstart, S.us, tinfo);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const uint32_t grid = min(ntiles, (uint32_t)(sms * max(blocks_per_sm, 1)));
  xs_lookup_staged<FAST><<<grid, kStagedThreads, smem, st>>>(X, n, S.Es, S.us, tinfo, S.idx, S.mstart, out,
                                                             vsum);
  return cudaGetLastError();
}
