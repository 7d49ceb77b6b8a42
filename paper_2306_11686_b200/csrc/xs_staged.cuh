// xs_staged.cuh -- the sorted unionized lookup with its memory side on the TMA engine.
// Included by xs_lookup.cu (uses its XsTables / Pair / accumulate / nuclide_loop / energy_index).
//
// Persistent CTAs of 4 consumer warps + 1 producer warp walk tiles of kTile consecutive sorted
// lookups.  staged_prep (a separate, massively parallel pass) computes each sorted lookup's
// unionized index u and each tile's facts: material of its first / last lookup and [min u, max u].
// A tile whose lookups share one material and whose u range spans <= kIgCap entries is "staged":
// for each nuclide j of the material the producer warp
//   cursor A: issues cp.async.bulk of the tile's index-grid row segment IG[nuc][u_lo..u_hi] into
//             SMEM stage s (mbarrier full_ig[s]), up to kLook items ahead of cursor B;
//   cursor B: once that segment has landed, reads k_lo = IG[u_lo], k_hi = IG[u_hi] (the index grid
//             is monotone in u) and issues cp.async.bulk of the record range [k_lo, k_hi + 1] of the
//             nuclide grid and of the matching reciprocal widths (mbarrier full[s]).
// Stages form a ring of kStages guarded by empty[s] (one arrival per consumer warp).  Consumers
// read their interval index, record pair and reciprocal width from SMEM -- no global access in the
// inner loop; records past kRecCap (rare) fall back to global loads.  Other tiles (mixed
// material, sparse materials whose u range is wide, caller energies outside [-2, 2]) run the
// per-thread pipelined loop.  Results are bit-identical to every other kernel: same index, same
// arithmetic, same order.
#pragma once

constexpr int kTile = 128;                   // lookups per tile = consumer threads
constexpr int kStagedThreads = kTile + 32;   // + producer warp
constexpr int kStages = 24;                  // ring depth
constexpr int kLook = kStages - 2;           // cursor A runs at most kLook items ahead of cursor B
constexpr int kIgCap = 1024;                 // index-grid entries per stage (2 KB)
constexpr int kRecCap = 8;                   // records per stage (k_hi - k_lo + 2 <= 8: >99.9%)
constexpr int kRdCap = kRecCap + 2;          // reciprocal widths per stage (range rounded to 16 B)
// stage layout: ig[kIgCap] u16 | rec[kRecCap] 48-B records | rd[kRdCap] f64 | StageMeta (16 B)
constexpr int kRecOff = 2 * kIgCap;
constexpr int kRdOff = kRecOff + 48 * kRecCap;
constexpr int kMetaOff = kRdOff + 8 * kRdCap;
constexpr int kStageBytes = (kMetaOff + 16 + 127) & ~127;
static_assert(kRecOff % 16 == 0 && kRdOff % 16 == 0 && kMetaOff % 16 == 0, "bulk-copy targets are 16-B aligned");

struct StageMeta {
  int k_lo;        // record index (within the nuclide) of rec[0]
  int n_rec;       // records staged
  uint32_t rd_lo;  // absolute index (into Rd) of rd[0]
  int pad;
};

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
  t += 3 * kStages * 8;
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
  // caller-supplied energies outside [-2, 2] need the IEEE division path: such tiles are not staged
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

// Consumer side of one staged item: wait for stage g, read k and the record pair (SMEM, or global
// past kRecCap), release the stage (one arrival per warp).
template <bool FAST>
__device__ __forceinline__ void staged_fetch(const XsDev &X, unsigned char *stages, uint64_t *full, uint64_t *empty,
                                             uint32_t g, uint32_t urel, uint32_t rec_base, int lane, Pair &P) {
  const uint32_t s = g % kStages, ph = (g / kStages) & 1u;
  const unsigned char *st = stages + (size_t)s * kStageBytes;
  mbar_wait(&full[s], ph);
  const StageMeta meta = *reinterpret_cast<const StageMeta *>(st + kMetaOff);
  const uint32_t k = reinterpret_cast<const uint16_t *>(st)[urel];
  const int rel = (int)k - meta.k_lo;
  if (rel + 1 < meta.n_rec) {
    const double2 *r = reinterpret_cast<const double2 *>(st + kRecOff) + rel * 3;
    P.l0 = r[0];
    P.l1 = r[1];
    P.l2 = r[2];
    P.h0 = r[3];
    P.h1 = r[4];
    P.h2 = r[5];
    if (FAST) P.y = reinterpret_cast<const double *>(st + kRdOff)[rec_base + k - meta.rd_lo];
  } else {
    load_pair<FAST>(X, rec_base + k, P);
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&empty[s]);
}

// Staged tiles only hold energies in [-2, 2] (staged_prep), so FAST needs no per-lookup check.
template <bool FAST>
__device__ __forceinline__ void staged_loop(const XsDev &X, const XsTables &T, unsigned char *stages, uint64_t *full,
                                            uint64_t *empty, uint32_t it, const TileInfo &ti, uint32_t urel,
                                            double E, int lane, double m[5]) {
  const int j0 = ti.j0, cnt = ti.cnt;
  for (int q = 0; q < cnt; q++) {
    Pair P;
    staged_fetch<FAST>(X, stages, full, empty, it + q, urel, T.ent[j0 + q].x, lane, P);
    accumulate<FAST>(P, E, T.conc[j0 + q], m);
  }
}

template <bool FAST>
__global__ void __launch_bounds__(kStagedThreads, 3)
    xs_lookup_staged(XsDev X, uint32_t n, const double *__restrict__ Es, const uint32_t *__restrict__ us,
                     const TileInfo *__restrict__ tinfo, const uint32_t *__restrict__ idx,
                     const uint32_t *__restrict__ mstart, double *__restrict__ macro_out,
                     unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(128) unsigned char smem[];
  const XsTables T = stage_xs_tables(X, smem);
  size_t off = (xs_table_smem(X.total) + 15) & ~size_t(15);
  uint64_t *full_ig = reinterpret_cast<uint64_t *>(smem + off);
  uint64_t *full = full_ig + kStages;
  uint64_t *empty = full + kStages;
  off = (off + 3 * kStages * 8 + 127) & ~size_t(127);
  unsigned char *stages = smem + off;
  __shared__ TileInfo s_ring[kStages];  // producer-private: facts of the staged tiles in flight

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full_ig[s], 1);
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTile / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t ntiles = (n + kTile - 1) / kTile;

  if (warp == kTile / 32) {
    // ================================================================ producer warp
    // All lanes run the control flow; lane 0 issues.
    uint32_t tA = blockIdx.x;  // tile of cursor A
    int qA = 0, qB = 0;        // item within the tile
    uint32_t gA = 0, gB = 0;   // global item counters (ring positions)
    TileInfo iA{}, iB{};
    TileInfo preA = load_tinfo(tinfo + min(tA, ntiles - 1));  // tile facts one tile ahead
    bool haveA = false, haveB = false;
    uint32_t ringA = 0, ringB = 0;
    // Advance a cursor to its next staged item; false at the end of the CTA's tiles.  Only staged
    // tiles enter the ring, so it holds at most kLook + 1 <= kStages tiles between B and A.
    auto advanceA = [&]() -> bool {
      while (true) {
        if (haveA && qA < iA.cnt) return true;
        if (haveA) tA += gridDim.x;
        if (tA >= ntiles) return false;
        iA = preA;
        if (tA + gridDim.x < ntiles) preA = load_tinfo(tinfo + tA + gridDim.x);
        haveA = true;
        qA = 0;
        if (iA.cnt > 0) {
          if (lane == 0) s_ring[ringA % kStages] = iA;
          ringA++;
        }
      }
    };
    auto advanceB = [&]() -> bool {
      if (haveB && qB < iB.cnt) return true;
      if (ringB == ringA) return false;
      __syncwarp();
      iB = s_ring[ringB % kStages];
      ringB++;
      haveB = true;
      qB = 0;
      return true;
    };
    bool moreA = advanceA();
    while (true) {
      // cursor A: index-grid segments, at most kLook items ahead of B
      while (moreA && gA < gB + kLook) {
        const uint32_t s = gA % kStages, ph = (gA / kStages) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        if (lane == 0) {
          const uint32_t bytes = (((iA.uhi + 8) & ~7u) - iA.ubase) * 2;
          mbar_arrive_tx(&full_ig[s], bytes);
          bulk_g2s(stages + (size_t)s * kStageBytes, X.IG + T.ent[iA.j0 + qA].y + iA.ubase, bytes, &full_ig[s]);
        }
        __syncwarp();
        gA++;
        qA++;
        moreA = advanceA();
      }
      if (gB == gA) break;  // A exhausted and B caught up
      if (!advanceB()) break;
      // cursor B: record range of item gB once its index-grid segment has landed
      const uint32_t s = gB % kStages, ph = (gB / kStages) & 1u;
      mbar_wait(&full_ig[s], ph);
      if (lane == 0) {
        unsigned char *st = stages + (size_t)s * kStageBytes;
        const uint16_t *ig = reinterpret_cast<const uint16_t *>(st);
        const int klo = ig[iB.ulo - iB.ubase], khi = ig[iB.uhi - iB.ubase];
        const int nrec = min(khi + 2 - klo, kRecCap);
        const uint32_t rec0 = T.ent[iB.j0 + qB].x + (uint32_t)klo;
        const uint32_t rdlo = rec0 & ~1u;
        const uint32_t rdn = (rec0 + (uint32_t)nrec - rdlo + 1u) & ~1u;
        StageMeta *meta = reinterpret_cast<StageMeta *>(st + kMetaOff);
        meta->k_lo = klo;
        meta->n_rec = nrec;
        meta->rd_lo = rdlo;
        mbar_arrive_tx(&full[s], (uint32_t)nrec * 48u + (FAST ? rdn * 8u : 0u));
        bulk_g2s(st + kRecOff, X.G + (size_t)rec0 * 6, (uint32_t)nrec * 48u, &full[s]);
        if (FAST) bulk_g2s(st + kRdOff, X.Rd + rdlo, rdn * 8u, &full[s]);
      }
      __syncwarp();
      gB++;
      qB++;
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
    if (ti.staged) {
      staged_loop<FAST>(X, T, stages, full, empty, it, ti, u - ti.ubase, E, lane, m);
      it += (uint32_t)ti.cnt;
    } else {
      const int mat = material_of(mstart, pc);
      const int a0 = T.off[mat], a1 = T.off[mat + 1];
      if (a1 > a0) {
        if (FAST && fabs(E) <= 2.0)
          nuclide_loop<GF_GRID_UNIONIZED, FAST, false>(X, T, E, u, a0, a1, m);
        else
          nuclide_loop<GF_GRID_UNIONIZED, false, false>(X, T, E, u, a0, a1, m);
      }
    }
    if (p < n) {
      vacc += argmax5_plus1(m);
      if (macro_out) {
        const size_t o = (size_t)idx[p] * 5;
#pragma unroll
        for (int c = 0; c < 5; c++) macro_out[o + c] = m[c];
      }
    }
  }
  hash_epilogue(vacc, vsum);
}

template <bool FAST>
static cudaError_t launch_staged(const XsDev &X, uint32_t n, const SortScratch &S, double *macro_out,
                                 unsigned long long *vsum, cudaStream_t st) {
  const size_t smem = staged_smem(X.total);
  static int blocks_per_sm[2] = {0, 0};
  static size_t smem_cfg[2] = {0, 0};
  cudaError_t e;
  if (smem_cfg[FAST] != smem) {
    if ((e = cudaFuncSetAttribute(xs_lookup_staged<FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
        cudaSuccess)
      return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm[FAST], xs_lookup_staged<FAST>,
                                                           kStagedThreads, smem)) != cudaSuccess)
      return e;
    smem_cfg[FAST] = smem;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t ntiles = (n + kTile - 1) / kTile;
  TileInfo *tinfo = reinterpret_cast<TileInfo *>(S.tinfo);
  staged_prep<<<ntiles, kTile, 0, st>>>(X, n, S.Es, S.mstart, S.us, tinfo);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const uint32_t grid = min(ntiles, (uint32_t)(sms * max(blocks_per_sm[FAST], 1)));
  xs_lookup_staged<FAST><<<grid, kStagedThreads, smem, st>>>(X, n, S.Es, S.us, tinfo, S.idx, S.mstart, macro_out,
                                                             vsum);
  return cudaGetLastError();
}
