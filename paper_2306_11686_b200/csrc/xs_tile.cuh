// xs_tile.cuh -- the warp-tile sorted lookup kernel (A3-A6 over a locality-sorted batch; included by
// xs_lookup.cu after xs_sorted_u.cuh).
//
// A warp owns a tile of 128 consecutive sorted lookups (lane l: positions 4l .. 4l+3, sorted by energy
// in registers).  After the locality sort a tile lies in one material and a narrow energy range
// [Emin, Emax], so for every nuclide of the material the tile's intervals form a short run
// klo .. khi, klo = K(Emin), khi = K(Emax), where K(E) = clamp(#{A <= E} - 1, 0, n_gp - 2) is the
// plain interval (SURVEY.md:520-521).  K is monotone, so for every lookup of the tile (R-TILE,
// DESIGN.md Sec. 3)
//     K(E) = klo + #{m in 0 .. khi - klo - 1 : A[klo + 1 + m] <= E},
// and the boundaries A[klo + 1 + m] are the first doubles of the interval records klo + m of XR.  The
// grid-type search therefore runs twice per (tile, nuclide) instead of once per (lookup, nuclide), and
// the run's records klo .. khi -- one contiguous piece of XR -- are staged into shared memory by the
// warp (16-B cp.async pieces, the chunk's records spread over the lanes).
//
// Runs are variable-length and packed: a chunk takes as many of the material's nuclides (<= 32, one
// per lane) as fit kCap records (a warp scan of the run lengths), so dense batches (17 M lookups: runs
// of ~1.6 records) stage ~25 nuclides per chunk and sparse ones (2 M lookups, one GPU's share of an
// 8-way split: ~6 records) fewer -- the kernel has no density threshold.  Pipeline per warp (no
// producer warp, no CTA barrier; cp.async groups): two SMEM buffers; chunk c+1 is in flight while chunk c is computed,
// and the searches of the chunk after that are issued before chunk c is computed.  The nuclide loop
// reads only shared memory: the slot's {record index, offset, length}, the boundaries (a count over
// <= 1 boundary in the common case, a binary search in general) and one record (LDS broadcasts).
//
// Grid types: unionized (klo / khi from the index grid at the tile's extreme union indices), hash (the
// literal hash search; the tile takes this path only if every lookup lies strictly inside its hash
// bin, RN(b du) < E < RN((b+1) du), where the literal edge rules cannot fire and the literal search
// returns K(E) -- DESIGN.md R-TILE), and kGridNB (per-nuclide bin brackets, no index grid).  Tiles
// that straddle a material boundary or the batch end, or hold energies outside [+0, 2] (caller
// energies), take the one-by-one path with the literal per-lookup search.
#pragma once

#ifndef GF_TILE_UNROLL
#define GF_TILE_UNROLL 1  // nuclide-loop unroll (measured: 2 is slower, C3 2.89 -> 3.04 ms)
#endif
constexpr int kTileUnroll = GF_TILE_UNROLL;
// Unionized batches from kPrepMin lookups: per-tile union indices (tile_prep) instead of per-lookup ones
// (idx_prep), and the rare per-lookup searches by bisection (PREP).  Measured: C3 17 M 2.885 -> 2.812 ms;
// at 2 M lookups the per-lookup searches are frequent and the per-lookup index wins (0.68 vs 0.76 ms).
constexpr uint32_t kPrepMin = 8u << 20;  // (XsDev::prep_min: default; a test hook lowers it)
#ifndef GF_ODD_FIRST
#define GF_ODD_FIRST 1  // hand out the tiles across material boundaries first
#endif
constexpr int kTileTpb = 128;  // 4 warps per CTA
constexpr int kTileWarps = kTileTpb / 32;
#ifndef GF_TILE_CAP
#define GF_TILE_CAP 40
#endif
constexpr int kCap = GF_TILE_CAP;  // records per staging buffer (5.6 KB; two per warp, 4 CTAs of 4 warps fit an SM)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Records sit at a 144-B stride in shared memory (128 B + 16 B of padding): the lanes of a warp read the
// same field of up to 8 neighbouring records without bank conflicts (at a 128-B stride they would all
// map to the same banks; ncu: 53% of the LDS wavefronts were conflicts at 2 M lookups).
constexpr int kRecStride = 144;

struct TileSmem {  // per warp
  unsigned char rec[2][kCap][kRecStride];  // [buffer]: the chunk's runs of interval records, packed
  uint2 meta[2][32];                // [buffer][slot]: {record index of klo, offset | length << 8 | wide << 16}
  uint32_t src[kCap];               // record index (in XR) of each staged record of the chunk being staged
};

__host__ __device__ inline size_t tile_table_bytes(int total) { return (xs_table_smem(total) + 127) & ~size_t(127); }
__host__ __device__ inline size_t tile_smem(int total) {
  return tile_table_bytes(total) + sizeof(TileSmem) * kTileWarps;
}

// One interval record from shared memory (its v0.x = E[k+1], ..., y at double 12).  Plain loads through
// a pointer into the extern __shared__ array: they compile to LDS and stay after the cp.async wait.
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

__device__ __forceinline__ long long smem_bits(const unsigned char *a) { return *reinterpret_cast<const long long *>(a); }

// Shared-memory loads by 32-bit address, not volatile (the compiler may schedule them freely): every
// address is derived from the token the cp.async wait returns, so none can move above the wait.
__device__ __forceinline__ long long lds64(uint32_t a) {
  long long v;
  asm("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_u2(uint32_t a) {
  uint2 v;
  asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
template <bool FAST>
__device__ __forceinline__ void lds_rec(uint32_t a, Rec &R) {
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(R.v0.x), "=d"(R.v0.y) : "r"(a));
  asm("ld.shared.v2.f64 {%0, %1}, [%2 + 16];" : "=d"(R.v1.x), "=d"(R.v1.y) : "r"(a));
  asm("ld.shared.v2.f64 {%0, %1}, [%2 + 32];" : "=d"(R.v2.x), "=d"(R.v2.y) : "r"(a));
  asm("ld.shared.v2.f64 {%0, %1}, [%2 + 48];" : "=d"(R.v3.x), "=d"(R.v3.y) : "r"(a));
  asm("ld.shared.v2.f64 {%0, %1}, [%2 + 64];" : "=d"(R.v4.x), "=d"(R.v4.y) : "r"(a));
  asm("ld.shared.v2.f64 {%0, %1}, [%2 + 80];" : "=d"(R.v5.x), "=d"(R.v5.y) : "r"(a));
  if (FAST) asm("ld.shared.f64 %0, [%1 + 96];" : "=d"(R.y) : "r"(a));
}

// Record index of lookup E for table entry e by the plain bisection over the nuclide's energies
// (= the index grid's interval; also for band grids: the absolute interval).  The
// unionized tile kernel's rare per-lookup paths use it: they have no per-lookup union index.
__device__ __forceinline__ uint32_t nuc_bisect_rec(const XsDev &X, uint2 e, double E) {
  const uint32_t base = (e.y / (uint32_t)X.ig_pitch) * (uint32_t)X.n_gp;
  int k = bisect<int>(X.Ed + base, E, 0, X.n_gp - 1);
  return base + (uint32_t)(k == X.n_gp - 1 ? k - 1 : k);
}

// The record index of lookup E (grid index ix) for entry e, per lookup: the literal search.
template <int GT, bool PREP>
__device__ __forceinline__ uint32_t lookup_rec(const XsDev &X, uint2 e, double E, uint32_t ix) {
  if (GT == GF_GRID_UNIONIZED && PREP) return nuc_bisect_rec(X, e, E);
  long long id = ix;
  if (GT == kGridNB) id = energy_index<kGridNB>(X, E);
  return e.x + interval<GT>(X, e, E, id);
}

// The grid type's literal search for the tile at energy E with grid index ix (union index / hash bin;
// kGridNB bins the energy itself).
template <int GT>
__device__ __forceinline__ uint32_t tile_k(const XsDev &X, uint2 e, double E, uint32_t ix) {
  if (GT == GF_GRID_UNIONIZED) return __ldg(X.IG + e.y + ix);  // (the index grid is clamped to n_gp - 2)
  long long ia = ix;
  if (GT == kGridNB) ia = energy_index<kGridNB>(X, E);
  return interval<GT>(X, e, E, ia);
}

// The runs of the next candidate nuclides (lane l: entry c0 + l): klo = K(Emin), khi = K(Emax).
struct RunSearch {
  uint32_t klo, khi;
};
template <int GT>
__device__ __forceinline__ RunSearch tile_search(const XsDev &X, const XsTables &T, int c0, int j1, double Emin,
                                                 double Emax, uint32_t imin, uint32_t imax) {
  const int j = c0 + (int)(threadIdx.x & 31);
  RunSearch r{0u, 0u};
  if (j < j1) {
    const uint2 e = tab_ent(T, j, true);
    r.klo = tile_k<GT>(X, e, Emin, imin);
    r.khi = tile_k<GT>(X, e, Emax, imax);
  }
  return r;
}

// Stages the runs of entries c0, c0 + 1, ... into buffer b: as many as fit kCap records (a prefix of the
// 32 candidates, at least one: a run longer than kCap is cut to kCap records and marked wide).  Returns
// the number of entries staged.  All 32 lanes call it; every lane commits one cp.async group per call
// (possibly empty), so the groups of the two buffers complete in order.
__device__ __forceinline__ int tile_stage(const XsDev &X, const XsTables &T, TileSmem &S, int b, int c0, int j1,
                                          RunSearch r) {
  const int lane = threadIdx.x & 31;
  const bool valid = c0 + lane < j1;
  uint32_t cnt = valid ? r.khi - r.klo + 1u : 0u;
  const uint32_t wide = cnt > (uint32_t)kCap ? 1u : 0u;
  cnt = min(cnt, (uint32_t)kCap);
  uint32_t incl = cnt;  // inclusive warp scan of the run lengths
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const bool fits = valid && incl <= (uint32_t)kCap;  // a prefix of the lanes (every valid run has >= 1 record)
  const int nsel = __popc(__ballot_sync(0xffffffffu, fits));
  const uint32_t total = __shfl_sync(0xffffffffu, incl, nsel > 0 ? nsel - 1 : 0);
  if (fits) {
    const uint2 e = tab_ent(T, c0 + lane, true);
    const uint32_t kb = e.x + r.klo, off = incl - cnt;
    S.meta[b][lane] = make_uint2(kb, off | (cnt << 8) | (wide << 16));
    for (uint32_t k = 0; k < cnt; k++) S.src[off + k] = kb + k;
  }
  __syncwarp();
  // the warp copies the chunk's records cooperatively, 16 B per cp.async (8 per record; a bulk copy
  // takes uniform operands, so per-lane bulk copies serialise through an elect loop)
  for (uint32_t q = lane; q < total * 8u; q += 32) {
    const uint32_t rr = q >> 3, part = q & 7u;
    const double *src = X.XR + (size_t)S.src[rr] * 16 + 2 * part;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(S.rec[b][rr] + 16 * part)), "l"(src)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  return nsel;
}

// #{m < nbd : boundary m <= E}, the boundaries being the first doubles of the records at `rec` (kRecStride
// stride, sorted): a branch-free binary search whose steps depend on nbd only (warp-uniform).  Bit
// patterns of non-negative doubles order as signed 64-bit integers.
__device__ __forceinline__ uint32_t run_count(uint32_t rec, uint32_t nbd, long long eb) {
  uint32_t c = 0;
  if (nbd == 0) return 0;
  for (uint32_t step = 1u << (31 - __clz(nbd)); step; step >>= 1)
    if (c + step <= nbd && eb >= lds64(rec + kRecStride * (c + step - 1))) c += step;
  return c;
}

template <int GT, bool FAST, bool PREP>
__device__ __forceinline__ void tile_loop(const XsDev &X, const XsTables &T, TileSmem &S,
                                          const double (&E)[kL], const uint32_t (&ix)[kL], int j0, int j1,
                                          double Emin, double Emax, uint32_t imin, uint32_t imax,
                                          double (&m)[kL][5]) {
  long long eb[kL];
#pragma unroll
  for (int i = 0; i < kL; i++) eb[i] = __double_as_longlong(E[i]);
  const uint32_t csa = smem_u32(T.pk) + 8u;  // concentration of table entry j: csa + 16 j (PK layout)
  __syncwarp();  // the previous tile's readers of S are done
  // prologue: stage chunks 0 and 1, search the candidates after them
  int cs0 = j0, cn0, cs1, cn1 = 0, nxt;
  {
    RunSearch r = tile_search<GT>(X, T, j0, j1, Emin, Emax, imin, imax);
    cn0 = tile_stage(X, T, S, 0, j0, j1, r);
    cs1 = j0 + cn0;
    if (cs1 < j1) {
      r = tile_search<GT>(X, T, cs1, j1, Emin, Emax, imin, imax);
      cn1 = tile_stage(X, T, S, 1, cs1, j1, r);
    }
    nxt = cs1 + cn1;
  }
  RunSearch pend = tile_search<GT>(X, T, nxt, j1, Emin, Emax, imin, imax);
  int b = 0;
  while (cs0 < j1) {
    uint32_t tok;  // 0, produced after the wait: the chunk's shared addresses depend on it
    if (cn1 > 0)  // the next chunk's group was committed after this one's: let it stay in flight
      asm volatile("cp.async.wait_group 1;\n mov.u32 %0, 0;" : "=r"(tok) :: "memory");
    else
      asm volatile("cp.async.wait_group 0;\n mov.u32 %0, 0;" : "=r"(tok) :: "memory");
    __syncwarp();
    const uint32_t mb = smem_u32(&S.meta[b][0]) + tok, rb = smem_u32(&S.rec[b][0][0]) + tok;
    // the concentration by a 32-bit shared address (through the generic table pointer ptxas re-derived
    // the shared window, S2UR + ULEA, in every iteration)
#pragma unroll kTileUnroll
    for (int s = 0; s < cn0; s++) {
      const int jj = cs0 + s;
      const uint32_t my = lds_u32(mb + 8u * (uint32_t)s + 4u);
      const double conc = lds_f64(csa + 16u * (uint32_t)jj);
      const uint32_t off = my & 0xFFu, cnt = (my >> 8) & 0xFFu;
      const bool wide = (my >> 16) != 0u;
      const uint32_t ra = rb + kRecStride * off;  // shared address of the run's first record
      const uint32_t nbd = cnt - 1u;  // staged boundaries A[klo + 1 .. klo + cnt - 1]
      // lookup 0 by a binary search over the run; the thread's other lookups (a much narrower range)
      // against the next three boundaries: c_i = ca + [E_i >= bx] + [E_i >= by] while E_i < bz.  A run of
      // one record (nbd = 0, warp-uniform; about half the runs of a dense batch) needs none of it, a run of
      // two one compare per lookup.
      const long long kInf = 0x7FF0000000000000ll;  // (+inf: no boundary)
      uint32_t ca = 0u, cd = 0u;
      long long bx = kInf, by = kInf;
      bool slow = false, strad = false;
      if (nbd == 1u) {  // two records, one boundary (the next most common run): c_i = [E_i >= b1]
        const long long b1 = lds64(ra);  // (boundary m is the first double of staged record m)
        ca = eb[0] >= b1 ? 1u : 0u;
        cd = eb[kL - 1] >= b1 ? 1u : 0u;
        bx = ca ? kInf : b1;
        strad = __any_sync(0xffffffffu, ca != cd);
      } else if (nbd != 0u) {
        ca = run_count(ra, nbd, eb[0]);
        bx = ca < nbd ? lds64(ra + kRecStride * ca) : kInf;
        by = ca + 1u < nbd ? lds64(ra + kRecStride * (ca + 1u)) : kInf;
        const long long bz = ca + 2u < nbd ? lds64(ra + kRecStride * (ca + 2u)) : kInf;
        cd = ca + (eb[kL - 1] >= bx ? 1u : 0u) + (eb[kL - 1] >= by ? 1u : 0u);
        // common case: no lookup of the warp beyond a cut run, and no thread's lookups span more than two
        // boundaries (E_3 < bz)
        slow = __any_sync(0xffffffffu, (wide && cd == nbd) || eb[kL - 1] >= bz);
        strad = __any_sync(0xffffffffu, ca != cd);
      }
      Rec P;
      if (!slow) {
        const uint32_t sa = ra;
        uint32_t cP = ca;
        lds_rec<FAST>(ra + kRecStride * ca, P);
        if (!strad) {  // no thread straddles: the 4 chains interleave
#pragma unroll
          for (int i = 0; i < kL; i++) accumulate_rec<FAST>(P, E[i], conc, m[i]);
        } else {
          accumulate_rec<FAST>(P, E[0], conc, m[0]);
#pragma unroll
          for (int i = 1; i < kL; i++) {
            // lanes whose lookup i is past their boundary reload (predicated LDS; ptxas spills if this
            // is a branch around plain loads)
            const uint32_t c = (i == kL - 1) ? cd : ca + (eb[i] >= bx ? 1u : 0u) + (eb[i] >= by ? 1u : 0u);
            reload_rec_smem_if(sa + kRecStride * c, c != cP, P);
            cP = c;
            accumulate_rec<FAST>(P, E[i], conc, m[i]);
          }
        }
      } else {  // three boundaries inside some thread's lookups, or a lookup beyond a cut run: per lookup
#pragma unroll
        for (int i = 0; i < kL; i++) {
          const uint32_t c = run_count(ra, nbd, eb[i]);
          if (!(wide && c == nbd)) {
            lds_rec<FAST>(ra + kRecStride * c, P);
          } else {  // beyond the staged part of a cut run: the literal search
            load_rec<FAST>(X, lookup_rec<GT, PREP>(X, tab_ent(T, jj, true), E[i], ix[i]), P);
          }
          accumulate_rec<FAST>(P, E[i], conc, m[i]);
        }
      }
    }
    __syncwarp();  // every lane is done with buffer b
    int cn2 = 0;
    if (nxt < j1) {
      cn2 = tile_stage(X, T, S, b, nxt, j1, pend);
      pend = tile_search<GT>(X, T, nxt + cn2, j1, Emin, Emax, imin, imax);
    }
    cs0 = cs1;
    cn0 = cn1;
    cs1 = nxt;
    cn1 = cn2;
    nxt += cn2;
    b ^= 1;
  }
}

// One-by-one path: lookups of a tile that straddles a material boundary or the batch end, or with
// energies outside the tile path's domain.  The literal per-lookup search (interval<GT>).
template <int GT, bool FAST, bool PREP>
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
    for (int j = j0; j < j1; j++) {
      Rec P;
      const uint2 ej = tab_ent(T, j, true);
      const uint32_t rec = lookup_rec<GT, PREP>(X, ej, E[i], ix[i]);
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

__device__ __forceinline__ bool ok_energies(const double (&E)[kL]) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < kL; i++) ok = ok && __double_as_longlong(E[i]) >= 0 && E[i] <= 2.0;
  return ok;
}

__device__ __forceinline__ long long warp_max64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}
__device__ __forceinline__ long long warp_min64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// The union indices of lo and hi (two-level search), out of line: only the passes of the <= 13 tiles
// across a material boundary need it in the tile kernel, whose loop registers it must not cost.
__device__ __noinline__ uint32_t union_index(const uint32_t *ubin, const double *U, long long n_union, double E) {
  XsDev X;  // (the two-level search reads ubin, U and n_union only)
  X.ubin = ubin;
  X.U = U;
  X.n_union = n_union;
  return (uint32_t)energy_index<GF_GRID_UNIONIZED>(X, E);
}
__device__ __forceinline__ uint2 union_range(const XsDev &X, double lo, double hi) {
  return make_uint2(union_index(X.ubin, X.U, X.n_union, lo), union_index(X.ubin, X.U, X.n_union, hi));
}

#ifndef GF_TILE_MINB
#define GF_TILE_MINB 4
#endif

// One lane of a tile with odd energies (caller states outside [+0, 2], hash lookups on a bin edge): the
// group kernel's pipelined loop if its 4 lookups share a material, else one by one.
template <int GT, bool FAST, bool PREP>
__device__ __forceinline__ void odd_lane(const XsDev &X, const XsTables &T, const uint32_t *ms, uint32_t p0,
                                      uint32_t nl, double (&E)[kL], uint32_t (&ix)[kL], double (&m)[kL][5],
                                      uint32_t &perm) {
  int lm0 = 0, lm1 = 0;
#pragma unroll
  for (int mm = 1; mm < kMats; mm++) {
    if (p0 >= ms[mm]) lm0 = mm;
    if (p0 + nl - 1 >= ms[mm]) lm1 = mm;
  }
  const bool fast = FAST && (GT == GF_GRID_HASH || (GT == GF_GRID_UNIONIZED && !PREP)) && nl == kL && ok_energies(E);  // (unionized: no per-lookup index)
  if (fast && lm0 == lm1) {
    local_sort(E, ix, perm);
    const int j0 = T.off[lm0], j1 = T.off[lm0 + 1];
    if (j1 > j0) group_loop<GT, FAST>(X, T, E, ix, j0, j1, m);
  } else {
    lookups_one_by_one<GT, FAST, PREP>(X, T, ms, p0, nl, E, ix, m);
  }
}

// The 4 sorted lookups of lane position p0 (nl of them; missing ones repeat the last, or E = 0 if none).
template <int GT, bool PREP>
__device__ __forceinline__ void load_tile_lookups(const double *__restrict__ Es, const uint32_t *__restrict__ ixs,
                                                  uint32_t p0, uint32_t nl, double (&E)[kL], uint32_t (&ix)[kL]) {
  if (nl == kL) {
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(E[0]), "=d"(E[1]), "=d"(E[2]), "=d"(E[3]) : "l"(Es + p0));
    if (GT == GF_GRID_HASH || (GT == GF_GRID_UNIONIZED && !PREP)) {
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
      ix[i] = (nl && (GT == GF_GRID_HASH || (GT == GF_GRID_UNIONIZED && !PREP))) ? ixs[p] : 0u;
    }
  }
}

// ix: the per-lookup grid index from idx_prep (union index / hash bin); unused for kGridNB.
template <int GT, bool FAST, bool PREP>
__global__ void __launch_bounds__(kTileTpb, GF_TILE_MINB)
    xs_lookup_tile(XsDev X, uint32_t n, const double *__restrict__ Es, const uint32_t *__restrict__ ixs,
                   const uint32_t *__restrict__ idx, const uint32_t *__restrict__ mstart, OutSpec out,
                   unsigned long long *__restrict__ vsum, uint32_t *__restrict__ work) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t ms[kMats + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  TileSmem &S = reinterpret_cast<TileSmem *>(smem + tile_table_bytes(X.total))[warp];
  if (threadIdx.x <= kMats) ms[threadIdx.x] = __ldg(mstart + threadIdx.x);
  const XsTables T = stage_xs_tables<true, GT == kGridNB>(X, smem);  // (its __syncthreads publishes ms)
  n = min(n, ms[kMats]);  // lookups kept by the sort (band grids keep their band's)
  uint32_t vacc = 0;
  const uint32_t ntiles = (n + 32 * kL - 1) / (32 * kL);
  double du = 0.0;
  if (GT == GF_GRID_HASH) du = __ddiv_rn(1.0, (double)X.bins);
  // dynamic tile scheduling: a warp takes the next work item when it finishes one.  The tiles across a
  // material boundary or at the batch end (<= 13: one pass per material, the longest tiles) are handed
  // out first, then the rest in sorted order (the 321-nuclide fuel first), so long tiles start early.
  __shared__ uint32_t s_odd[kMats + 1];
  __shared__ int s_nodd;
  if (threadIdx.x == 0) {
    int no = 0;
    for (int mm = 1; mm <= kMats; mm++) {
      const uint32_t b = mm < kMats ? ms[mm] : n;  // (ms is non-decreasing: the list comes out sorted)
      const uint32_t tb = b / (32 * kL);
      if (b % (32 * kL) != 0u && tb < ntiles && (no == 0 || s_odd[no - 1] != tb)) s_odd[no++] = tb;
    }
    s_nodd = no;
  }
  __syncthreads();
  const int nodd = GF_ODD_FIRST ? s_nodd : 0;
  for (uint32_t w = next_tile(work); w < ntiles; w = next_tile(work)) {
    uint32_t t;
    if (w < (uint32_t)nodd) {
      t = s_odd[w];
    } else {  // the (w - nodd)-th tile not in the list
      t = w - (uint32_t)nodd;
      for (int q = 0; q < nodd; q++)
        if (s_odd[q] <= t) t++;
    }
    const uint32_t P = t * 32 * kL;
    const uint32_t p0 = P + lane * kL;
    const uint32_t nl = p0 < n ? min((uint32_t)kL, n - p0) : 0u;
    const uint32_t plast = min(P + 32 * kL, n) - 1;
    int mat0 = 0, mat1 = 0;
#pragma unroll
    for (int mm = 1; mm < kMats; mm++) {
      if (P >= ms[mm]) mat0 = mm;
      if (plast >= ms[mm]) mat1 = mm;
    }
    // tile path: energies in [+0, 2] (hash grid: strictly inside the bin).  A tile across a material
    // boundary (or the batch end) runs one pass per material: the pass's lookups are the active ones,
    // the others (and missing ones) take a copy of an active energy of their lane -- computed and
    // discarded -- so every pass is an ordinary tile over one material's nuclides.
    double E[kL];
    uint32_t ix[kL];
    bool ok = FAST;
    load_tile_lookups<GT, PREP>(Es, ixs, p0, nl, E, ix);
    // unionized: the tile's energy range and its union indices (tile_prep), for every pass
    long long tlo = 0x7FF0000000000000ll, thi = (long long)0x8000000000000000ull;
    uint2 tu = make_uint2(0u, 0u);
    if (GT == GF_GRID_UNIONIZED && PREP) {
#pragma unroll
      for (int i = 0; i < kL; i++) {
        if ((uint32_t)i >= nl) continue;
        const long long b = __double_as_longlong(E[i]);
        tlo = b < tlo ? b : tlo;
        thi = b > thi ? b : thi;
      }
      tlo = warp_min64(tlo);
      thi = warp_max64(thi);
      tu = __ldg(reinterpret_cast<const uint2 *>(ixs) + t);
    }
#pragma unroll
    for (int i = 0; i < kL; i++) {
      if ((uint32_t)i >= nl) continue;
      const long long bits = __double_as_longlong(E[i]);
      ok = ok && bits >= 0 && E[i] <= 2.0;
      if (GT == GF_GRID_HASH) {
        const double lo = __dmul_rn((double)ix[i], du);
        const double hi = (int)ix[i] >= X.bins - 1 ? 1.0 / 0.0 : __dmul_rn((double)(ix[i] + 1), du);
        ok = ok && lo < E[i] && E[i] < hi;
      }
    }
    if (__all_sync(0xffffffffu, ok)) {
      for (int mt = mat0; mt <= mat1; mt++) {
        uint32_t act = 0;  // bit i: lookup i of this lane is in the pass (material segment [ms[mt], ms[mt+1]))
        const uint32_t sb = ms[mt], se = mt + 1 < kMats ? ms[mt + 1] : n;
#pragma unroll
        for (int i = 0; i < kL; i++) act |= ((uint32_t)i < nl && p0 + i >= sb && p0 + i < se) ? (1u << i) : 0u;
        if (!__any_sync(0xffffffffu, act != 0u)) continue;
        if (mt != mat0) load_tile_lookups<GT, PREP>(Es, ixs, p0, nl, E, ix);  // (not kept live across passes)
        // stand-in for inactive lookups: the lane's first active lookup, else the warp's smallest active energy
        long long a0 = 0x7FF0000000000000ll;
        uint32_t x0 = 0;
#pragma unroll
        for (int i = kL - 1; i >= 0; i--)
          if (act & (1u << i)) { a0 = __double_as_longlong(E[i]); x0 = ix[i]; }
        const long long wmin = warp_min64(a0);
        const uint32_t wx = __shfl_sync(0xffffffffu, x0, __ffs(__ballot_sync(0xffffffffu, a0 == wmin)) - 1);
        if (act == 0u) { a0 = wmin; x0 = wx; }
#pragma unroll
        for (int i = 0; i < kL; i++)
          if (!(act & (1u << i))) { E[i] = __longlong_as_double(a0); ix[i] = x0; }
        uint32_t perm = 0x76543210u;
        local_sort(E, ix, perm);
        double m[kL][5];
#pragma unroll
        for (int i = 0; i < kL; i++)
#pragma unroll
          for (int c = 0; c < 5; c++) m[i][c] = 0.0;
        double Emin, Emax;
        uint32_t imin, imax;
        if (GT == GF_GRID_UNIONIZED && PREP && mat0 == mat1 && P + 32 * kL <= n) {  // a full tile in one material:
          // the tile's range, its union indices from the sort (sampled batches) or tile_prep
          Emin = __longlong_as_double(tlo);
          Emax = __longlong_as_double(thi);
          imin = tu.x;
          imax = tu.y;
        } else if (GT == GF_GRID_UNIONIZED && PREP) {  // a pass of a tile across a material boundary (or the
          // batch's last, partial tile): its own range
          Emin = __longlong_as_double(warp_min64(__double_as_longlong(E[0])));
          Emax = __longlong_as_double(warp_max64(__double_as_longlong(E[kL - 1])));
          const uint2 u = union_range(X, Emin, Emax);
          imin = u.x;
          imax = u.y;
        } else {
          Emin = __longlong_as_double(warp_min64(__double_as_longlong(E[0])));
          Emax = __longlong_as_double(warp_max64(__double_as_longlong(E[kL - 1])));
          imin = __reduce_min_sync(0xffffffffu, ix[0]);
          imax = __reduce_max_sync(0xffffffffu, ix[kL - 1]);
        }
        const int j0 = T.off[mt], j1 = T.off[mt + 1];
        if (j1 > j0) tile_loop<GT, FAST, PREP>(X, T, S, E, ix, j0, j1, Emin, Emax, imin, imax, m);
#pragma unroll
        for (int i = 0; i < kL; i++) {  // slot i holds lookup q; the pass finishes its active lookups
          const uint32_t q = (perm >> (4 * i)) & 15u;
          if (act & (1u << q)) {
            vacc += argmax5_plus1(m[i]);
            if (out.any()) write_out<5>(out, idx[p0 + q], m[i]);
          }
        }
      }
    } else if (nl) {  // odd energies (caller states): each lane on its own
      double m[kL][5];
#pragma unroll
      for (int i = 0; i < kL; i++)
#pragma unroll
        for (int c = 0; c < 5; c++) m[i][c] = 0.0;
      uint32_t perm = 0x76543210u;
      odd_lane<GT, FAST, PREP>(X, T, ms, p0, nl, E, ix, m, perm);
#pragma unroll
      for (uint32_t i = 0; i < (uint32_t)kL; i++) {
        if (i < nl) {
          vacc += argmax5_plus1(m[i]);
          if (out.any()) write_out<5>(out, idx[p0 + ((perm >> (4 * i)) & 15u)], m[i]);
        }
      }
    }
  }
  hash_epilogue(vacc, vsum);
}

// A3 for the unionized tile kernel, per tile instead of per lookup: tix[t] = {u(Emin), u(Emax)}, the union
// indices (two-level search) of the smallest and largest energy of sorted tile t (positions
// [128 t, 128 t + 128) below n).  One warp per tile; replaces idx_prep (one search per lookup).
__global__ void __launch_bounds__(256) tile_prep(XsDev X, uint32_t n, const double *__restrict__ Es,
                                                 const uint32_t *__restrict__ mstart, uint2 *__restrict__ tix) {
  n = min(n, __ldg(mstart + kMats));
  const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t P = t * 32 * kL;
  if (P >= n) return;  // (warp-uniform)
  long long lo = 0x7FF0000000000000ll, hi = (long long)0x8000000000000000ull;
#pragma unroll
  for (int i = 0; i < kL; i++) {
    const uint32_t p = P + lane * kL + i;
    if (p < n) {
      const long long b = __double_as_longlong(__ldg(Es + p));
      lo = b < lo ? b : lo;
      hi = b > hi ? b : hi;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long a = __shfl_xor_sync(0xffffffffu, lo, o), c = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = c > hi ? c : hi;
  }
  if (lane < 2) {
    const uint32_t u = (uint32_t)energy_index<GF_GRID_UNIONIZED>(X, __longlong_as_double(lane ? hi : lo));
    const uint32_t v = __shfl_sync(0x3u, u, 1);
    if (lane == 0) tix[t] = make_uint2(u, v);
  }
}

template <int GT, bool FAST, bool PREP>
static cudaError_t launch_tile_p(const XsDev &X, uint32_t n, const SortScratch &S, const OutSpec &out,
                               unsigned long long *vsum, cudaStream_t st, bool tile_prep_on) {
  const size_t smem = tile_smem(X.total);
  int blocks_per_sm = 0;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(xs_lookup_tile<GT, FAST, PREP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, xs_lookup_tile<GT, FAST, PREP>, kTileTpb, smem)) !=
      cudaSuccess)
    return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t ntiles = (n + 32 * kL - 1) / (32 * kL);
  const uint32_t grid =
      max(1u, min((ntiles + kTileWarps - 1) / kTileWarps, (uint32_t)(sms * max(blocks_per_sm, 1))));
  if (GT == GF_GRID_UNIONIZED && PREP) {
    // per-tile union indices (S.us holds uint2 per tile): written by the sort's scatter for sampled
    // batches (TixSpec, launch_gt), else by tile_prep (the exact tile extremes, one warp per tile)
    if (tile_prep_on) {
      tile_prep<<<nblk((long long)ntiles * 32, 256), 256, 0, st>>>(X, n, S.Es, S.mstart, reinterpret_cast<uint2 *>(S.us));
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  } else if (GT != kGridNB) {  // per-lookup hash bins (the bin-interior check)
    idx_prep<GT><<<nblk(((long long)n + 3) / 4, 256), 256, 0, st>>>(X, n, S.Es, S.mstart, S.us);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if ((e = cudaMemsetAsync(S.work, 0, sizeof(uint32_t), st)) != cudaSuccess) return e;
  xs_lookup_tile<GT, FAST, PREP><<<grid, kTileTpb, smem, st>>>(X, n, S.Es, S.us, S.idx, S.mstart, out, vsum, S.work);
  return cudaGetLastError();
}

template <int GT, bool FAST>
static cudaError_t launch_tile(const XsDev &X, uint32_t n, const SortScratch &S, const OutSpec &out,
                               unsigned long long *vsum, cudaStream_t st, bool tile_prep_on) {
  if constexpr (GT == GF_GRID_UNIONIZED) {
    if (n >= X.prep_min) return launch_tile_p<GT, FAST, true>(X, n, S, out, vsum, st, tile_prep_on);
  }
  return launch_tile_p<GT, FAST, false>(X, n, S, out, vsum, st, false);
}
