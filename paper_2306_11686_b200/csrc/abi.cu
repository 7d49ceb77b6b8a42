// abi.cu -- the C ABI declared in include/gf_xs.h: validation, memory layout, launches.
//
// Host-side responsibilities only: argument checks (synchronous, before anything is enqueued),
// carving the caller's buffers into arrays, uploading the built-in / custom
// material tables, and enqueueing the kernels of xs_grid.cu / xs_lookup.cu / rs.cu.  No arithmetic
// of the method runs here.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "gf_internal.cuh"

using namespace gf;

// ------------------------------------------------------------------------------------------ errors
static thread_local std::string t_err;

static gf_status fail(gf_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return s;
}

#define GF_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t _e = (call);                                                                   \
    if (_e != cudaSuccess) return fail(GF_E_CUDA, "%s: %s", #call, cudaGetErrorString(_e));    \
  } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) return;
    ok = (prev == dev) || (cudaSetDevice(dev) == cudaSuccess);
  }
  ~DeviceGuard() {
    if (ok && prev >= 0) cudaSetDevice(prev);
  }
};

// ------------------------------------------------------------------------------------------ tables
// Hoogenboom-Martin compositions (SURVEY.md:552-558, R-MATS), typed here for the product.
static const int32_t kFuelSmall[34] = {58, 59, 60, 61, 40, 42, 43, 44, 45, 46, 1,  2,  3,  7,  8,  9,  10,
                                       29, 57, 47, 48, 0,  62, 15, 33, 34, 52, 53, 54, 55, 56, 18, 23, 41};
static const int32_t kClad[5] = {63, 64, 65, 66, 67};
static const int32_t kWater[4] = {24, 41, 4, 5};
static const int32_t kSteel27[27] = {19, 20, 21, 22, 35, 36, 37, 38, 39, 25, 27, 28, 29, 30,
                                     31, 32, 26, 49, 50, 51, 11, 12, 13, 14, 6,  16, 17};
static const int32_t kWaterSteel[21] = {24, 41, 4, 5, 19, 20, 21, 22, 35, 36, 37, 38, 39, 25, 27, 28, 29, 30, 31, 32, 26};
static const int32_t kWaterClad[9] = {24, 41, 4, 5, 63, 64, 65, 66, 67};

// CSR material tables: off[13], nuc[total].
static gf_status build_tables(const gf_xs_params *p, std::vector<int32_t> &off, std::vector<int32_t> &nuc) {
  off.assign(kMats + 1, 0);
  nuc.clear();
  const int n_iso = p->n_isotopes;
  if (!p->num_nucs) {
    if (p->mats) return fail(GF_E_INVAL, "mats given without num_nucs");
    if (n_iso != 68 && n_iso != 355)
      return fail(GF_E_INVAL, "built-in material tables exist for n_isotopes 68 or 355 (got %d)", n_iso);
    auto add = [&](const int32_t *a, int k) { nuc.insert(nuc.end(), a, a + k); };
    add(kFuelSmall, 34);
    if (n_iso == 355)
      for (int i = 68; i < 355; i++) nuc.push_back(i);
    off[1] = (int)nuc.size();
    add(kClad, 5); off[2] = (int)nuc.size();
    add(kWater, 4); off[3] = (int)nuc.size();
    add(kWater, 4); off[4] = (int)nuc.size();
    add(kSteel27, 27); off[5] = (int)nuc.size();
    for (int m = 5; m <= 9; m++) { add(kWaterSteel, 21); off[m + 1] = (int)nuc.size(); }
    for (int m = 10; m <= 11; m++) { add(kWaterClad, 9); off[m + 1] = (int)nuc.size(); }
    return GF_OK;
  }
  if (!p->mats || p->max_num_nucs < 1) return fail(GF_E_INVAL, "custom tables need mats and max_num_nucs >= 1");
  for (int m = 0; m < kMats; m++) {
    int k = p->num_nucs[m];
    if (k < 0 || k > p->max_num_nucs) return fail(GF_E_INVAL, "num_nucs[%d] = %d outside [0, max_num_nucs]", m, k);
    for (int j = 0; j < k; j++) {
      int v = p->mats[(size_t)m * p->max_num_nucs + j];
      if (v < 0 || v >= n_iso) return fail(GF_E_INVAL, "mats[%d][%d] = %d is not a nuclide id", m, j, v);
      nuc.push_back(v);
    }
    off[m + 1] = (int)nuc.size();
  }
  return GF_OK;
}

// ------------------------------------------------------------------------------------------ layout
static inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  // XS
  size_t G, Ed, Rd, XR, flags, U, IG, HG, ubin, NB;
  int nb_pitch;
  size_t k0, binfo;  // NEXT-2 band grid: k0 / cnt / first [3][n_iso] u32, band info 16 B
  int band_cap;      // in-band points per nuclide the layout holds
  long long ig_pitch;
  int hg_pitch;
  // RS
  size_t pole, pole_l, win, K0RS, poff, woff;
  // both
  size_t thr, moff, mnuc, mconc;
  size_t total_bytes, scratch_bytes;
};

// In-band points per nuclide the layout provisions: LCG gridpoint energies are iid U[0, 1), so the
// count is Binomial(n_gp, 1/W); mean + 12 sd + 64 (checked at init, GF_E_UNSUPPORTED if exceeded).
static int band_capacity(const gf_xs_params *p) {
  if (p->n_bands <= 1) return (int)p->n_gridpoints;
  const double n = (double)p->n_gridpoints, w = 1.0 / p->n_bands;
  const double c = n * w + 12.0 * sqrt(n * w * (1.0 - w)) + 64.0;
  return (int)std::min(n, std::ceil(c));
}

static gf_status validate(const gf_xs_params *p) {
  if (!p) return fail(GF_E_INVAL, "params is NULL");
  if (p->abi_version != GF_XS_ABI_VERSION)
    return fail(GF_E_INVAL, "abi_version %u != %u", p->abi_version, GF_XS_ABI_VERSION);
  if (p->bench != GF_XSBENCH && p->bench != GF_RSBENCH) return fail(GF_E_INVAL, "bench %d", p->bench);
  if (p->n_isotopes < 1) return fail(GF_E_INVAL, "n_isotopes %d < 1", p->n_isotopes);
  if (p->bench == GF_XSBENCH) {
    if (p->n_gridpoints < 2) return fail(GF_E_INVAL, "n_gridpoints %lld < 2", (long long)p->n_gridpoints);
    if (p->n_gridpoints > kMaxGp)
      return fail(GF_E_UNSUPPORTED, "n_gridpoints %lld > %d", (long long)p->n_gridpoints, kMaxGp);
    if (p->n_bands < 1 || p->band < 0 || p->band >= p->n_bands)
      return fail(GF_E_INVAL, "band %d of n_bands %d", p->band, p->n_bands);
    if (p->n_bands > 1 && p->grid_type != GF_GRID_UNIONIZED)
      return fail(GF_E_INVAL, "energy bands shard the unionized grid only (grid_type %d)", p->grid_type);
    if (p->grid_type == GF_GRID_UNIONIZED && (p->n_bands > 1 ? band_capacity(p) + 2 > 65535
                                                              : p->n_gridpoints > kMaxGp16))
      return fail(GF_E_UNSUPPORTED, "unionized grid with %d points per nuclide per band (u16 index grid): "
                  "use more energy bands (n_bands), or the hash or nuclide grid", band_capacity(p));
    if (p->grid_type < 0 || p->grid_type > 2) return fail(GF_E_INVAL, "grid_type %d", p->grid_type);
    if (p->grid_type == GF_GRID_HASH && p->hash_bins < 1) return fail(GF_E_INVAL, "hash_bins %d < 1", p->hash_bins);
    if ((long long)p->n_isotopes * p->n_gridpoints >= (1ll << 31))
      return fail(GF_E_UNSUPPORTED, "n_isotopes * n_gridpoints >= 2^31");
    if (p->grid_type == GF_GRID_UNIONIZED &&
        (double)p->n_isotopes * (double)(p->n_isotopes * (double)band_capacity(p) + 66) >= 4294967296.0)
      return fail(GF_E_UNSUPPORTED, "index grid larger than 2^32 entries");
  } else {
    if (p->numL != 4) return fail(GF_E_INVAL, "numL must be 4 (got %d)", p->numL);
    if (p->doppler != 0 && p->doppler != 1) return fail(GF_E_INVAL, "doppler must be 0 or 1 (got %d)", p->doppler);
    if (p->avg_n_poles < 1 || p->avg_n_windows < 1) return fail(GF_E_INVAL, "avg_n_poles / avg_n_windows must be >= 1");
    if ((long long)p->avg_n_poles * p->n_isotopes >= (1ll << 28)) return fail(GF_E_UNSUPPORTED, "too many poles");
  }
  return GF_OK;
}

static gf_status plan(const gf_xs_params *p, int total, Layout &L) {
  memset(&L, 0, sizeof L);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += al(bytes);
    return at;
  };
  if (p->bench == GF_XSBENCH) {
    const size_t npts = (size_t)p->n_isotopes * (size_t)p->n_gridpoints;
    L.G = take(npts * 48);
    L.Ed = take(npts * 8);
    L.Rd = take(npts * 8);
    L.flags = take(16);
    // interval records (+ the tile kernel's slot overrun); nuclide grids have them where the tile kernel can
    // run on them (n_gp < 65536: the per-nuclide bin brackets find its runs)
    if (p->grid_type != GF_GRID_NUCLIDE || p->n_gridpoints < 65536) L.XR = take(npts * 128 + 256);
    if (p->grid_type == GF_GRID_NUCLIDE && p->n_gridpoints < 65536) {  // sorted batches search NB brackets
      L.nb_pitch = ((1 << kNbLog2) + 1 + 63) & ~63;
      L.NB = take((size_t)p->n_isotopes * L.nb_pitch * 2);
    }
    if (p->grid_type == GF_GRID_UNIONIZED) {
      // whole grid: all n_iso n_gp energies; band: <= band_cap per nuclide plus the two sentinels
      L.band_cap = band_capacity(p);
      const size_t nu = p->n_bands > 1 ? (size_t)p->n_isotopes * L.band_cap + 2 : npts;
      L.ig_pitch = (long long)((nu + 63) & ~size_t(63));
      L.U = take(nu * 8);
      L.IG = take((size_t)p->n_isotopes * (size_t)L.ig_pitch * 2);
      L.ubin = take((size_t)(kUBins + 1) * 4);
      if (p->n_bands <= 1 && p->n_gridpoints < 65536) {
        L.nb_pitch = ((1 << kNbLog2) + 1 + 63) & ~63;
        L.NB = take((size_t)p->n_isotopes * L.nb_pitch * 2);
      }
      L.scratch_bytes = al(npts * 8);
      if (p->n_bands > 1) {
        L.k0 = take((size_t)p->n_isotopes * 12);
        L.binfo = take(16);
        L.scratch_bytes = std::max(L.scratch_bytes, al((size_t)p->n_isotopes * L.band_cap * 16));
      }
    } else {
      L.scratch_bytes = 256;
    }
    if (p->n_gridpoints > kMaxSortGp) L.scratch_bytes = std::max(L.scratch_bytes, al(npts * 24));  // big_* sort
    if (p->grid_type == GF_GRID_HASH) {
      L.hg_pitch = (p->hash_bins + 63) & ~63;
      L.HG = take((size_t)p->n_isotopes * (size_t)L.hg_pitch * (p->n_gridpoints > kMaxGp16 ? 4 : 2));
    }
  } else {
    const size_t n = (size_t)p->n_isotopes;
    const size_t tp = (size_t)p->avg_n_poles * n, tw = (size_t)p->avg_n_windows * n;
    L.pole = take(tp * 64);
    L.pole_l = take(tp * 4);
    L.win = take(tw * 32);
    L.K0RS = take(n * 4 * 8);
    L.poff = take((n + 1) * 4);
    L.woff = take((n + 1) * 4);
    L.scratch_bytes = al(2 * n * 4);
  }
  L.thr = take(kThrBytes);  // T[12] doubles, the integer thresholds S[12] (u64), the sampling tables
  L.moff = take(16 * 4);
  L.mnuc = take((size_t)(total > 0 ? total : 1) * 4);
  L.mconc = take((size_t)(total > 0 ? total : 1) * 8);
  L.total_bytes = o;
  return GF_OK;
}

// Sorted-path kernel choice, read once per grid here (never on the lookup path).  The environment
// overrides exist for A/B measurements only; every choice gives identical results.
//   GF_XS_KERNEL   = tile | tilenb | group | thread | warp   (default: auto)
//   GF_XS_TILE_MIN = smallest batch of the warp-tile kernel in auto mode (default kTileMinN)
//   GF_XS_GROUP_MIN = smallest batch of the group kernel in auto mode (default kGroupMinN)
//   GF_XS_NB       = 0: sparse batches search the index grid instead of the NB brackets
// tools/ab_batch_n.py (gpurun_out/r02w): the tile kernel wins from ~2 M lookups (C3 2.125 M: 0.75 ms vs
// group 0.96, thread 1.17; C4 21.25 M: 4.2 vs 8.1 / 12.0), one lookup per thread below (C3 1 M: 0.68 vs
// tile 1.02); the group kernel never leads by more than noise (C2 17 M: 1.383 vs 1.387) -- A/B only.
constexpr uint32_t kTileMinN = 2000000u;
constexpr uint32_t kGroupMinN = 0xFFFFFFFFu;
static void kernel_choice(XsDev &X) {
  static_assert(kKernTile == GF_KERN_TILE && kKernWarpSearch == GF_KERN_WARP_SEARCH, "kernel ids");
  X.kern = kKernAuto;
  if (const char *s = getenv("GF_XS_KERNEL")) {
    const std::string v(s);
    if (v == "tile") X.kern = kKernTile;
    else if (v == "tilenb") X.kern = kKernTileNB;
    else if (v == "group") X.kern = kKernGroup;
    else if (v == "thread") X.kern = kKernThread;
    else if (v == "warp") X.kern = kKernWarpSearch;
  }
  X.tile_min = kTileMinN;
  if (const char *m = getenv("GF_XS_TILE_MIN")) X.tile_min = (uint32_t)strtoul(m, nullptr, 10);
  X.group_min = kGroupMinN;
  if ((X.grid_type == GF_GRID_HASH && X.n_gp > 65536) || (X.grid_type == GF_GRID_UNIONIZED && X.n_gp > 262144)) {
    // XL hash and XXL unionized grids: a tile's runs (~n_gp x the tile's energy width per nuclide)
    // outgrow the staging buffers, and the group kernel wins from 2 M lookups (gpurun_out/r02ak, C6 XL
    // hash 17 M: group 15.7 ms, tile 17.4, thread 19.9; r02ax, C8 XXL in 16 bands: group 25.1 ms, tile 48.7;
    // the XL unionized bands of C7 stay on the tile kernel: 12.1 vs group 15.0 ms)
    X.tile_min = 0xFFFFFFFFu;
    X.group_min = kTileMinN;
  }
  X.prep_min = 8u << 20;
  if (const char *m = getenv("GF_XS_GROUP_MIN")) X.group_min = (uint32_t)strtoul(m, nullptr, 10);
  const char *nb = getenv("GF_XS_NB");
  X.nb_on = !(nb && nb[0] == '0');
}

// ------------------------------------------------------------------------------------------ handle
struct ArrView {
  const void *ptr = nullptr;
  size_t bytes = 0;
  int64_t pitch = 0;
};

struct gf_xs_grid {
  gf_xs_params p;
  int fastdiv_ok = 0;  // the grid admits the exact reciprocal division (no zero-width interval)
  int device = 0;
  int total = 0;
  XsDev xs{};
  RsDev rs{};
  ArrView arr[32];
  // host-IO pipeline objects (created on first GF_HOST_IO call; calls serialise on io_mu)
  std::mutex io_mu;
  bool io_ready = false;
  cudaStream_t io_s[3] = {};
  cudaEvent_t io_ev[7] = {};
  ~gf_xs_grid() {
    if (!io_ready) return;
    DeviceGuard dg(device);
    for (auto s : io_s) cudaStreamDestroy(s);
    for (auto e : io_ev) cudaEventDestroy(e);
  }
};

extern "C" {

const char *gf_xs_last_error(void) { return t_err.c_str(); }

const char *gf_xs_version(void) {
  static char v[96];
  snprintf(v, sizeof v, "gf_xs abi %u sm_100a nvcc %d.%d", GF_XS_ABI_VERSION, __CUDACC_VER_MAJOR__,
           __CUDACC_VER_MINOR__);
  return v;
}

gf_status gf_xs_default_params(int32_t bench, gf_xs_params *p) {
  if (!p) return fail(GF_E_INVAL, "params is NULL");
  memset(p, 0, sizeof *p);
  p->abi_version = GF_XS_ABI_VERSION;
  p->bench = bench;
  p->n_isotopes = 355;
  p->n_gridpoints = 11303;
  p->grid_type = GF_GRID_UNIONIZED;
  p->hash_bins = 10000;
  p->avg_n_poles = 1000;
  p->avg_n_windows = 100;
  p->numL = 4;
  p->doppler = 1;
  p->n_bands = 1;
  p->band = 0;
  p->init_seed = 42;
  if (bench != GF_XSBENCH && bench != GF_RSBENCH) return fail(GF_E_INVAL, "bench %d", bench);
  return GF_OK;
}

gf_status gf_xs_grid_bytes(const gf_xs_params *p, size_t *grid_bytes, size_t *init_scratch_bytes) {
  try {
    gf_status s = validate(p);
    if (s != GF_OK) return s;
    std::vector<int32_t> off, nuc;
    if ((s = build_tables(p, off, nuc)) != GF_OK) return s;
    if ((int)nuc.size() > kMaxTable) return fail(GF_E_UNSUPPORTED, "material tables larger than %d entries", kMaxTable);
    Layout L;
    plan(p, (int)nuc.size(), L);
    if (grid_bytes) *grid_bytes = L.total_bytes;
    if (init_scratch_bytes) *init_scratch_bytes = L.scratch_bytes;
    return GF_OK;
  } catch (...) {
    return fail(GF_E_NOMEM, "host allocation failed");
  }
}

gf_status gf_xs_grid_init(const gf_xs_params *p, int device, void *grid_mem, size_t grid_bytes, void *scratch,
                          size_t scratch_bytes, gf_stream_t stream, gf_xs_grid **out) {
  try {
    if (!out) return fail(GF_E_INVAL, "out is NULL");
    *out = nullptr;
    gf_status s = validate(p);
    if (s != GF_OK) return s;
    std::vector<int32_t> off, nuc;
    if ((s = build_tables(p, off, nuc)) != GF_OK) return s;
    const int total = (int)nuc.size();
    if (total > kMaxTable) return fail(GF_E_UNSUPPORTED, "material tables larger than %d entries", kMaxTable);
    Layout L;
    plan(p, total, L);
    if (!grid_mem || grid_bytes < L.total_bytes)
      return fail(GF_E_NOMEM, "grid buffer %zu B < required %zu B", grid_bytes, L.total_bytes);
    if (!scratch || scratch_bytes < L.scratch_bytes)
      return fail(GF_E_NOMEM, "init scratch %zu B < required %zu B", scratch_bytes, L.scratch_bytes);
    if (((uintptr_t)grid_mem & 255) || ((uintptr_t)scratch & 255))
      return fail(GF_E_INVAL, "grid and scratch buffers must be 256-byte aligned");
    int ndev = 0;
    GF_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(GF_E_INVAL, "device %d of %d", device, ndev);
    DeviceGuard dg(device);
    if (!dg.ok) return fail(GF_E_CUDA, "cannot make device %d current", device);
    cudaPointerAttributes pa;
    GF_CUDA(cudaPointerGetAttributes(&pa, grid_mem));
    if (pa.type != cudaMemoryTypeDevice && pa.type != cudaMemoryTypeManaged)
      return fail(GF_E_INVAL, "grid_mem is not device memory");
    int major = 0, minor = 0;
    GF_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    GF_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10 || minor != 0)
      return fail(GF_E_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a only", device, major, minor);

    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    char *base = static_cast<char *>(grid_mem);
    gf_xs_grid *g = new gf_xs_grid();
    g->p = *p;
    g->p.num_nucs = nullptr;
    g->p.mats = nullptr;
    g->device = device;
    g->total = total;
    double *thr = reinterpret_cast<double *>(base + L.thr);
    int32_t *moff = reinterpret_cast<int32_t *>(base + L.moff);
    int32_t *mnuc = reinterpret_cast<int32_t *>(base + L.mnuc);
    double *mconc = reinterpret_cast<double *>(base + L.mconc);
    // Tables are uploaded synchronously from host vectors that die with this call.
    cudaError_t ce = cudaMemcpyAsync(moff, off.data(), sizeof(int32_t) * off.size(), cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess && total)
      ce = cudaMemcpyAsync(mnuc, nuc.data(), sizeof(int32_t) * total, cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    if (ce == cudaSuccess) ce = launch_tables(nullptr, thr, st);
    auto put = [&](int w, const void *ptr, size_t bytes, int64_t pitch) { g->arr[w] = ArrView{ptr, bytes, pitch}; };
    put(GF_ARR_THRESHOLDS, thr, 12 * 8, 12);
    put(GF_ARR_MAT_OFFSETS, moff, 13 * 4, 13);
    put(GF_ARR_MAT_NUCS, mnuc, (size_t)total * 4, total);
    put(GF_ARR_CONCS, mconc, (size_t)total * 8, total);
    if (ce == cudaSuccess && p->bench == GF_XSBENCH) {
      XsDev &X = g->xs;
      X.n_iso = p->n_isotopes;
      X.n_gp = (int)p->n_gridpoints;
      X.grid_type = p->grid_type;
      X.bins = p->hash_bins;
      X.n_union = (long long)X.n_iso * X.n_gp;
      X.ig_pitch = L.ig_pitch;
      X.hg_pitch = L.hg_pitch;
      X.hg32 = X.n_gp > kMaxGp16 ? 1 : 0;
      X.total = total;
      double *G = reinterpret_cast<double *>(base + L.G);
      double *Ed = reinterpret_cast<double *>(base + L.Ed);
      double *Rd = reinterpret_cast<double *>(base + L.Rd);
      int *zero_width = reinterpret_cast<int *>(base + L.flags);
      double *XR = L.XR ? reinterpret_cast<double *>(base + L.XR) : nullptr;
      double *U = X.grid_type == GF_GRID_UNIONIZED ? reinterpret_cast<double *>(base + L.U) : nullptr;
      uint16_t *IG = X.grid_type == GF_GRID_UNIONIZED ? reinterpret_cast<uint16_t *>(base + L.IG) : nullptr;
      uint16_t *HG = X.grid_type == GF_GRID_HASH ? reinterpret_cast<uint16_t *>(base + L.HG) : nullptr;
      uint32_t *ubin = X.grid_type == GF_GRID_UNIONIZED ? reinterpret_cast<uint32_t *>(base + L.ubin) : nullptr;
      X.G = G; X.Ed = Ed; X.Rd = Rd; X.XR = XR; X.U = U; X.IG = IG; X.HG = HG; X.ubin = ubin;
      uint16_t *NB = (X.grid_type != GF_GRID_HASH && L.nb_pitch) ? reinterpret_cast<uint16_t *>(base + L.NB)
                                                                   : nullptr;
      X.NB = NB;
      X.nb_pitch = L.nb_pitch;
      X.thr = thr; X.moff = moff; X.mnuc = mnuc; X.mconc = mconc;
      kernel_choice(X);
      const bool banded = X.grid_type == GF_GRID_UNIONIZED && p->n_bands > 1;
      X.k0 = banded ? reinterpret_cast<uint32_t *>(base + L.k0) : nullptr;
      const double inf = 1.0 / 0.0;
      X.band_lo = (banded && p->band > 0) ? (double)p->band / (double)p->n_bands : -inf;
      X.band_hi = (banded && p->band < p->n_bands - 1) ? (double)(p->band + 1) / (double)p->n_bands : inf;
      const size_t npts = (size_t)X.n_iso * X.n_gp;
      put(GF_ARR_NUCLIDE_GRID, G, npts * 48, X.n_gp);
      put(GF_ARR_ENERGY, Ed, npts * 8, X.n_gp);
      if (IG) put(GF_ARR_INDEX_GRID, IG, (size_t)X.n_iso * X.ig_pitch * 2, X.ig_pitch);
      if (HG) put(GF_ARR_HASH_GRID, HG, (size_t)X.n_iso * X.hg_pitch * (X.hg32 ? 4 : 2), X.hg_pitch);
      if (ubin) put(GF_ARR_UNION_BINS, ubin, (size_t)(kUBins + 1) * 4, kUBins + 1);
      put(GF_ARR_RECIP_WIDTH, Rd, npts * 8, X.n_gp);
      if (XR) put(GF_ARR_INTERVALS, XR, npts * 128, X.n_gp);
      if (NB) put(GF_ARR_NUCLIDE_BINS, NB, (size_t)X.n_iso * X.nb_pitch * 2, X.nb_pitch);
      ce = launch_xs_grid(X, G, Ed, Rd, XR, zero_width, U, IG, HG, ubin, mconc, p->init_seed,
                          static_cast<double *>(scratch), st);
      if (ce == cudaSuccess && banded) {  // NEXT-2: the band's U (sync: its length sizes the index grid)
        uint32_t *binfo = reinterpret_cast<uint32_t *>(base + L.binfo);
        uint32_t *kk = const_cast<uint32_t *>(X.k0);
        ce = launch_band_union(X, L.band_cap, kk, kk + X.n_iso, U, binfo, static_cast<double *>(scratch), st);
        uint32_t info[4] = {0, 0, 0, 0};
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(info, binfo, 16, cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        if (ce == cudaSuccess && info[1]) {
          delete g;
          return fail(GF_E_UNSUPPORTED, "a nuclide has more than %d points in band %d of %d (layout bound)",
                      L.band_cap, p->band, p->n_bands);
        }
        X.n_union = (long long)info[0] + 2;
        if (ce == cudaSuccess) ce = launch_band_index(X, U, IG, ubin, st);
      }
      if (ce == cudaSuccess && NB) ce = launch_nb_build(X, NB, st);
      if (U) put(GF_ARR_UNIONIZED, U, (size_t)X.n_union * 8, (int64_t)X.n_union);
      // the exact reciprocal division is used only if no interval has zero (or underflowing) width
      int zw = 1;
      if (ce == cudaSuccess) ce = cudaMemcpyAsync(&zw, zero_width, sizeof(int), cudaMemcpyDeviceToHost, st);
      if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
      X.fastdiv = (zw == 0) ? 1 : 0;
      g->fastdiv_ok = X.fastdiv;
    } else if (ce == cudaSuccess) {
      RsDev &R = g->rs;
      const int n = p->n_isotopes;
      const size_t tp = (size_t)p->avg_n_poles * n, tw = (size_t)p->avg_n_windows * n;
      R.n_nuc = n;
      R.total = total;
      R.doppler = p->doppler;
      double *pole = reinterpret_cast<double *>(base + L.pole);
      int32_t *pole_l = reinterpret_cast<int32_t *>(base + L.pole_l);
      double4 *win = reinterpret_cast<double4 *>(base + L.win);
      double *K0RS = reinterpret_cast<double *>(base + L.K0RS);
      int32_t *poff = reinterpret_cast<int32_t *>(base + L.poff);
      int32_t *woff = reinterpret_cast<int32_t *>(base + L.woff);
      R.pole = pole; R.pole_l = pole_l; R.win = win; R.K0RS = K0RS; R.poff = poff; R.woff = woff;
      R.thr = thr; R.moff = moff; R.mnuc = mnuc; R.mconc = mconc;
      put(GF_ARR_RS_POLES, pole, tp * 64, 8);
      put(GF_ARR_RS_POLE_L, pole_l, tp * 4, 1);
      put(GF_ARR_RS_WINDOWS, win, tw * 32, 4);
      put(GF_ARR_RS_K0RS, K0RS, (size_t)n * 32, 4);
      put(GF_ARR_RS_POLE_OFF, poff, (size_t)(n + 1) * 4, n + 1);
      put(GF_ARR_RS_WIN_OFF, woff, (size_t)(n + 1) * 4, n + 1);
      ce = launch_rs_data(R, p->avg_n_poles, p->avg_n_windows, p->init_seed, pole, pole_l, win, K0RS, poff, woff,
                          mconc, static_cast<int32_t *>(scratch), st);
    }
    if (ce != cudaSuccess) {
      delete g;
      return fail(GF_E_CUDA, "grid init: %s", cudaGetErrorString(ce));
    }
    *out = g;
    return GF_OK;
  } catch (...) {
    return fail(GF_E_NOMEM, "host allocation failed");
  }
}

gf_status gf_xs_grid_free(gf_xs_grid *g) {
  delete g;
  return GF_OK;
}

gf_status gf_xs_grid_array(const gf_xs_grid *g, int32_t which, const void **ptr, size_t *bytes, int64_t *pitch_out) {
  if (!g || !ptr) return fail(GF_E_INVAL, "grid or ptr is NULL");
  if (which < 0 || which >= 32 || !g->arr[which].ptr) return fail(GF_E_INVAL, "grid has no array %d", which);
  *ptr = g->arr[which].ptr;
  if (bytes) *bytes = g->arr[which].bytes;
  if (pitch_out) *pitch_out = g->arr[which].pitch;
  return GF_OK;
}

// ------------------------------------------------------------------------------------------ lookups
// Scratch of one lookup slot.  Device-resident calls use one slot sized for the whole batch.  Host-IO
// calls (GF_HOST_IO) are pipelined in chunks of kIoChunk lookups over two slots and three streams:
// chunk c's host->device copy, chunk c-1's lookup and chunk c-2's device->host copy overlap (PCIe is
// full duplex).  Each chunk is sorted and looked up on its own; results are identical.  4 M-lookup
// chunks (C3 e2e, hash only: 2^21 2.0e9, 2^22 2.37e9, 2^23 2.47e9 lookups/s; with the macro output
// 1.18 / 1.10 / 0.99e9): a chunk at or above the group kernel's 4 M threshold.
#ifndef GF_IO_CHUNK_LOG2
#define GF_IO_CHUNK_LOG2 22
#endif
constexpr uint64_t kIoChunk = 1ull << GF_IO_CHUNK_LOG2;

struct SlotLayout {
  size_t counts, cursor, btot, mstart, Es, idx, us, work, Et, idxt, rk, segcnt, h_macro, h_E, h_mat, bytes;
};
struct BatchLayout {
  SlotLayout slot;
  int slots;
  SlotLayout full;  // host-IO, sorted, energies, no per-lookup output: one whole-batch slot (counts overlap
  bool has_full;    // the chunked H2D; one sort and one lookup pass over the whole batch), aliasing the slots
  size_t h_vsum, total;
};

static void plan_slot(const gf_xs_grid *g, uint64_t m, uint32_t flags, bool want_macro, bool energies,
                      SlotLayout &L);

// whole: plan the whole-batch host-I/O slot too (host-I/O energies, sorted, no per-lookup outputs);
// otherwise the chunked pipeline's two chunk slots only, whose size is bounded by the chunk.
static void plan_batch(const gf_xs_grid *g, uint64_t n, uint32_t flags, bool want_macro, bool energies,
                       BatchLayout &B, bool whole = false) {
  memset(&B, 0, sizeof B);
  const bool host_io = (flags & GF_HOST_IO) != 0;
  const uint64_t m = host_io ? (n < kIoChunk ? n : kIoChunk) : n;
  plan_slot(g, m, flags, want_macro, energies, B.slot);
  B.slots = host_io ? 2 : 1;
  size_t end = B.slots * B.slot.bytes;
  if (whole && host_io && energies && !want_macro && (flags & GF_SORT_LOCALITY)) {
    plan_slot(g, n, flags, false, true, B.full);
    B.has_full = true;
    end = std::max(end, B.full.bytes);
  }
  B.h_vsum = end;
  B.total = B.h_vsum + (host_io ? 256 : 0);
}

static void plan_slot(const gf_xs_grid *g, uint64_t m, uint32_t flags, bool want_macro, bool energies,
                      SlotLayout &L) {
  const bool host_io = (flags & GF_HOST_IO) != 0;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += al(bytes);
    return at;
  };
  const int ch = g->p.bench == GF_XSBENCH ? 5 : 4;
  if (flags & GF_SORT_LOCALITY) {
    const size_t hw = sort_hist_words(m);
    L.counts = take(sizeof(uint32_t) * hw);
    L.cursor = take(sizeof(uint32_t) * hw);
    L.btot = take(sizeof(uint32_t) * (hw / kScanBlk + 1));
    L.mstart = take(sizeof(uint32_t) * 16);
    L.Es = take(sizeof(double) * m);
    L.idx = take(sizeof(uint32_t) * m);
    L.us = take(sizeof(uint32_t) * m);
    L.work = take(256);
    if (g->p.bench == GF_XSBENCH && g->p.n_bands > 1) {  // band grids: the compacted in-band lookups (sort.cu)
      L.Et = take(sizeof(uint64_t) * m);
      L.idxt = take(sizeof(uint32_t) * m);
      L.rk = take(sizeof(uint32_t) * m);
      L.segcnt = take(sizeof(uint32_t) * (m / 512 + 1));
    }
  }
  if (host_io) {
    if (want_macro) L.h_macro = take(sizeof(double) * ch * m);
    if (energies) {
      L.h_E = take(sizeof(double) * m);
      L.h_mat = take(m);
    }
  }
  L.bytes = al(o > 0 ? o : 256);
}

gf_status gf_xs_batch_bytes(const gf_xs_grid *g, uint64_t n_lookups, uint32_t flags, size_t *scratch_bytes) {
  if (!g || !scratch_bytes) return fail(GF_E_INVAL, "grid or scratch_bytes is NULL");
  BatchLayout B;
  plan_batch(g, n_lookups, flags, true, true, B);  // upper bound over the optional parts (chunked host I/O)
  *scratch_bytes = B.total;
  return GF_OK;
}

gf_status gf_xs_batch_bytes_whole(const gf_xs_grid *g, uint64_t n_lookups, uint32_t flags, size_t *scratch_bytes) {
  if (!g || !scratch_bytes) return fail(GF_E_INVAL, "grid or scratch_bytes is NULL");
  BatchLayout Bc, Bw;
  plan_batch(g, n_lookups, flags, true, true, Bc);
  plan_batch(g, n_lookups, flags, false, true, Bw, true);
  *scratch_bytes = std::max(Bc.total, Bw.total);
  return GF_OK;
}

static SortScratch slot_sort(char *base, const SlotLayout &L) {
  SortScratch S{};
  S.counts = reinterpret_cast<uint32_t *>(base + L.counts);
  S.cursor = reinterpret_cast<uint32_t *>(base + L.cursor);
  S.btot = reinterpret_cast<uint32_t *>(base + L.btot);
  S.mstart = reinterpret_cast<uint32_t *>(base + L.mstart);
  S.Es = reinterpret_cast<double *>(base + L.Es);
  S.idx = reinterpret_cast<uint32_t *>(base + L.idx);
  S.us = reinterpret_cast<uint32_t *>(base + L.us);
  S.work = reinterpret_cast<uint32_t *>(base + L.work);
  S.Et = L.Et ? reinterpret_cast<double *>(base + L.Et) : nullptr;
  S.idxt = L.idxt ? reinterpret_cast<uint32_t *>(base + L.idxt) : nullptr;
  S.rk = L.rk ? reinterpret_cast<uint32_t *>(base + L.rk) : nullptr;
  S.segcnt = L.segcnt ? reinterpret_cast<uint32_t *>(base + L.segcnt) : nullptr;
  return S;
}

static cudaError_t launch_lookup(const gf_xs_grid *g, uint64_t first, uint32_t n, uint64_t seed, const double *dE,
                                 const uint8_t *dmat, bool sort, const SortScratch &S, double *dmacro,
                                 unsigned long long *dvsum, cudaStream_t st, cudaEvent_t ev_mid) {
  return g->p.bench == GF_XSBENCH
             ? launch_xs_lookup(g->xs, first, n, seed, dE, dmat, sort, S, out_macro(dmacro, 5), dvsum, st, ev_mid)
             : launch_rs_lookup(g->rs, first, n, seed, dE, dmat, sort, S, out_macro(dmacro, 4), dvsum, st, ev_mid);
}

// Internal streams / events of the host-IO pipeline (created on first use, per grid).
static gf_status io_setup(gf_xs_grid *g) {
  if (g->io_ready) return GF_OK;
  for (int i = 0; i < 3; i++) GF_CUDA(cudaStreamCreateWithFlags(&g->io_s[i], cudaStreamNonBlocking));
  for (int i = 0; i < 7; i++) GF_CUDA(cudaEventCreateWithFlags(&g->io_ev[i], cudaEventDisableTiming));
  g->io_ready = true;
  return GF_OK;
}

static gf_status run_host_io(const gf_xs_grid *gc, uint64_t first, uint64_t n, uint64_t seed, const double *E,
                             const uint8_t *mat, bool sort, double *macro_out, uint64_t *vsum, char *sc,
                             const BatchLayout &B, cudaStream_t st) {
  gf_xs_grid *g = const_cast<gf_xs_grid *>(gc);  // the pipeline objects are the only mutable state
  std::lock_guard<std::mutex> lock(g->io_mu);
  gf_status s = io_setup(g);
  if (s != GF_OK) return s;
  cudaStream_t sin = g->io_s[0], scomp = g->io_s[1], sout = g->io_s[2];
  cudaEvent_t start = g->io_ev[0], *h2d = g->io_ev + 1, *comp = g->io_ev + 3, *d2h = g->io_ev + 5;
  const int ch = g->p.bench == GF_XSBENCH ? 5 : 4;
  const bool energies = E != nullptr;
  unsigned long long *dvsum = reinterpret_cast<unsigned long long *>(sc + B.h_vsum);
  GF_CUDA(cudaEventRecord(start, st));  // ordered after the caller's prior work on `stream`
  GF_CUDA(cudaStreamWaitEvent(sin, start, 0));
  GF_CUDA(cudaStreamWaitEvent(scomp, start, 0));
  GF_CUDA(cudaMemsetAsync(dvsum, 0, 8, scomp));
  if (energies && sort && !macro_out && B.has_full) {
    // whole-batch mode: the chunks' host->device copies overlap the counting pass of the locality sort;
    // then one scatter and one lookup pass over the whole batch (full sort locality, the group kernel)
    const SlotLayout &L = B.full;
    SortScratch S = slot_sort(sc, L);
    S.counted = true;
    double *dE = reinterpret_cast<double *>(sc + L.h_E);
    uint8_t *dmat = reinterpret_cast<uint8_t *>(sc + L.h_mat);
    const double *thr = g->p.bench == GF_XSBENCH ? g->xs.thr : g->rs.thr;
    cudaError_t ce = launch_sort_zero((uint32_t)n, S, scomp);
    if (ce != cudaSuccess) return fail(GF_E_CUDA, "sort: %s", cudaGetErrorString(ce));
    for (uint64_t off = 0; off < n; off += kIoChunk) {
      const uint64_t cn = (n - off < kIoChunk) ? n - off : kIoChunk;
      GF_CUDA(cudaMemcpyAsync(dE + off, E + off, sizeof(double) * cn, cudaMemcpyHostToDevice, sin));
      GF_CUDA(cudaMemcpyAsync(dmat + off, mat + off, cn, cudaMemcpyHostToDevice, sin));
      GF_CUDA(cudaEventRecord(h2d[0], sin));
      GF_CUDA(cudaStreamWaitEvent(scomp, h2d[0], 0));
      ce = launch_sort_count((uint32_t)n, (uint32_t)cn, dE + off, dmat + off, thr, S, dvsum, scomp);
      if (ce != cudaSuccess) return fail(GF_E_CUDA, "sort count: %s", cudaGetErrorString(ce));
    }
    ce = launch_lookup(g, first, (uint32_t)n, seed, dE, dmat, true, S, nullptr, dvsum, scomp, nullptr);
    if (ce != cudaSuccess) return fail(GF_E_CUDA, "lookup launch: %s", cudaGetErrorString(ce));
    uint64_t add = 0;
    GF_CUDA(cudaMemcpyAsync(&add, dvsum, 8, cudaMemcpyDeviceToHost, scomp));
    GF_CUDA(cudaStreamSynchronize(scomp));
    if (add & kInvalidInputBit) return fail(GF_E_INVAL, "invalid caller inputs: material id > 11 or non-finite energy");
    *vsum += add;
    return GF_OK;
  }
  const uint64_t nch = (n + kIoChunk - 1) / kIoChunk;
  for (uint64_t c = 0; c < nch; c++) {
    const int k = (int)(c & 1);
    const uint64_t off = c * kIoChunk, cn = (n - off < kIoChunk) ? n - off : kIoChunk;
    char *base = sc + k * B.slot.bytes;
    const SlotLayout &L = B.slot;
    if (c >= 2) GF_CUDA(cudaStreamWaitEvent(sin, d2h[k], 0));  // slot k free (chunk c-2 copied out)
    const double *dE = nullptr;
    const uint8_t *dmat = nullptr;
    if (energies) {
      GF_CUDA(cudaMemcpyAsync(base + L.h_E, E + off, sizeof(double) * cn, cudaMemcpyHostToDevice, sin));
      GF_CUDA(cudaMemcpyAsync(base + L.h_mat, mat + off, cn, cudaMemcpyHostToDevice, sin));
      dE = reinterpret_cast<const double *>(base + L.h_E);
      dmat = reinterpret_cast<const uint8_t *>(base + L.h_mat);
    }
    GF_CUDA(cudaEventRecord(h2d[k], sin));
    GF_CUDA(cudaStreamWaitEvent(scomp, h2d[k], 0));
    double *dmacro = macro_out ? reinterpret_cast<double *>(base + L.h_macro) : nullptr;
    cudaError_t ce = launch_lookup(g, first + off, (uint32_t)cn, seed, dE, dmat, sort, slot_sort(base, L), dmacro,
                                   dvsum, scomp, nullptr);
    if (ce != cudaSuccess) return fail(GF_E_CUDA, "lookup launch: %s", cudaGetErrorString(ce));
    GF_CUDA(cudaEventRecord(comp[k], scomp));
    GF_CUDA(cudaStreamWaitEvent(sout, comp[k], 0));
    if (macro_out)
      GF_CUDA(cudaMemcpyAsync(macro_out + off * ch, dmacro, sizeof(double) * ch * cn, cudaMemcpyDeviceToHost, sout));
    GF_CUDA(cudaEventRecord(d2h[k], sout));
  }
  uint64_t add = 0;
  GF_CUDA(cudaMemcpyAsync(&add, dvsum, 8, cudaMemcpyDeviceToHost, scomp));
  GF_CUDA(cudaStreamSynchronize(scomp));
  GF_CUDA(cudaStreamSynchronize(sout));
  if (add & kInvalidInputBit) return fail(GF_E_INVAL, "invalid caller inputs: material id > 11 or non-finite energy");
  *vsum += add;
  return GF_OK;
}

static gf_status run_lookup(const gf_xs_grid *g, uint64_t first, uint64_t n, uint64_t seed, const double *E,
                            const uint8_t *mat, uint32_t flags, double *macro_out, uint64_t *vsum, void *scratch,
                            size_t scratch_bytes, gf_stream_t stream, const gf_stage_events *ev = nullptr) {
  if (!g) return fail(GF_E_INVAL, "grid is NULL");
  if (!vsum) return fail(GF_E_INVAL, "vsum is NULL");
  if (flags & GF_HISTORY) return fail(GF_E_UNSUPPORTED, "history-based mode is gf_xs_history_batch");
  if (flags & ~(uint32_t)(GF_SORT_LOCALITY | GF_HISTORY | GF_HOST_IO)) return fail(GF_E_INVAL, "unknown flags 0x%x", flags);
  if (n >= (1ull << 32)) return fail(GF_E_INVAL, "n = %llu >= 2^32: split the job into batches", (unsigned long long)n);
  const bool energies = E != nullptr;
  if (energies && !mat) return fail(GF_E_INVAL, "mat is NULL");
  if (g->p.bench == GF_XSBENCH && g->p.n_bands > 1 && (energies || !(flags & GF_SORT_LOCALITY) || (flags & GF_HOST_IO)))
    return fail(GF_E_UNSUPPORTED, "energy-band grids serve sorted, device-resident event lookups only");
  const bool host_io = (flags & GF_HOST_IO) != 0;
  BatchLayout B;
  plan_batch(g, n, flags, macro_out != nullptr, energies, B, true);  // the whole-batch host-I/O mode if it fits,
  if (B.has_full && scratch_bytes < B.total)                        // else the chunked pipeline
    plan_batch(g, n, flags, macro_out != nullptr, energies, B, false);
  if (n && (!scratch || scratch_bytes < B.total))
    return fail(GF_E_NOMEM, "scratch %zu B < required %zu B", scratch_bytes, B.total);
  if (n && ((uintptr_t)scratch & 255)) return fail(GF_E_INVAL, "scratch must be 256-byte aligned");
  if (n == 0) return GF_OK;
  DeviceGuard dg(g->device);
  if (!dg.ok) return fail(GF_E_CUDA, "cannot make device %d current", g->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char *sc = static_cast<char *>(scratch);
  const bool sort = (flags & GF_SORT_LOCALITY) != 0;
  if (host_io) return run_host_io(g, first, n, seed, E, mat, sort, macro_out, vsum, sc, B, st);

  unsigned long long *dvsum = reinterpret_cast<unsigned long long *>(vsum);
  cudaEvent_t ev_mid = ev ? static_cast<cudaEvent_t>(ev->before_lookup) : nullptr;
  if (ev && ev->before_sort) GF_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev->before_sort), st));
  cudaError_t ce = launch_lookup(g, first, (uint32_t)n, seed, E, mat, sort, slot_sort(sc, B.slot), macro_out, dvsum,
                                 st, ev_mid);
  if (ce != cudaSuccess) return fail(GF_E_CUDA, "lookup launch: %s", cudaGetErrorString(ce));
  if (ev && ev->after_lookup) GF_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev->after_lookup), st));
  return GF_OK;
}

gf_status gf_xs_lookup_batch(const gf_xs_grid *g, uint64_t first, uint64_t n, uint64_t starting_seed, uint32_t flags,
                             double *d_macro_out, uint64_t *d_vsum, void *scratch, size_t scratch_bytes,
                             gf_stream_t stream) {
  try {
    return run_lookup(g, first, n, starting_seed, nullptr, nullptr, flags, d_macro_out, d_vsum, scratch,
                      scratch_bytes, stream);
  } catch (...) {
    return fail(GF_E_NOMEM, "host allocation failed");
  }
}

gf_status gf_xs_lookup_batch_ev(const gf_xs_grid *g, uint64_t first, uint64_t n, uint64_t starting_seed,
                                uint32_t flags, double *d_macro_out, uint64_t *d_vsum, void *scratch,
                                size_t scratch_bytes, gf_stream_t stream, const gf_stage_events *ev) {
  try {
    return run_lookup(g, first, n, starting_seed, nullptr, nullptr, flags, d_macro_out, d_vsum, scratch,
                      scratch_bytes, stream, ev);
  } catch (...) {
    return fail(GF_E_NOMEM, "host allocation failed");
  }
}

gf_status gf_xs_lookup_energies(const gf_xs_grid *g, const double *E, const uint8_t *mat, uint64_t n, uint32_t flags,
                                double *macro_out, uint64_t *vsum, void *scratch, size_t scratch_bytes,
                                gf_stream_t stream) {
  try {
    if (!E && n) return fail(GF_E_INVAL, "E is NULL");
    static const double kDummy = 0.0;
    static const uint8_t kDummyMat = 0;
    return run_lookup(g, 0, n, 0, E ? E : &kDummy, mat ? mat : (n ? nullptr : &kDummyMat), flags, macro_out, vsum,
                      scratch, scratch_bytes, stream);
  } catch (...) {
    return fail(GF_E_NOMEM, "host allocation failed");
  }
}

gf_status gf_xs_lookup_energies_async(const gf_xs_grid *g, const double *E_host, const uint8_t *mat_host, uint64_t n,
                                      uint32_t flags, uint64_t *d_vsum, void *scratch, size_t scratch_bytes,
                                      gf_stream_t stream) {
  if (!g || !d_vsum || (n && (!E_host || !mat_host))) return fail(GF_E_INVAL, "grid, d_vsum, E or mat is NULL");
  if (flags != GF_SORT_LOCALITY) return fail(GF_E_INVAL, "flags must be GF_SORT_LOCALITY");
  if (n >= (1ull << 32)) return fail(GF_E_INVAL, "n %llu >= 2^32", (unsigned long long)n);
  if (g->p.bench == GF_XSBENCH && g->p.n_bands > 1) return fail(GF_E_INVAL, "band grids take sampled lookups only");
  if (n == 0) return GF_OK;
  DeviceGuard dg(g->device);
  BatchLayout B;
  plan_batch(g, n, GF_SORT_LOCALITY | GF_HOST_IO, false, true, B, true);  // the whole-batch slot
  const SlotLayout &L = B.full;
  if (!scratch || scratch_bytes < L.bytes)
    return fail(GF_E_NOMEM, "scratch %zu B < required %zu B", scratch_bytes, L.bytes);
  char *sc = static_cast<char *>(scratch);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double *dE = reinterpret_cast<double *>(sc + L.h_E);
  uint8_t *dmat = reinterpret_cast<uint8_t *>(sc + L.h_mat);
  GF_CUDA(cudaMemcpyAsync(dE, E_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  GF_CUDA(cudaMemcpyAsync(dmat, mat_host, n, cudaMemcpyHostToDevice, st));
  const cudaError_t ce = launch_lookup(g, 0, (uint32_t)n, 0, dE, dmat, true, slot_sort(sc, L), nullptr,
                                       reinterpret_cast<unsigned long long *>(d_vsum), st, nullptr);
  if (ce != cudaSuccess) return fail(GF_E_CUDA, "lookup launch: %s", cudaGetErrorString(ce));
  return GF_OK;
}

// ------------------------------------------------------------------------------------------ history (NEXT-1)
// Waves scratch: per particle the LCG state (8 B), this wave's E (8 B) and material (1 B), the
// feedback byte of the previous wave, then one sort slot for n_particles lookups.
struct HistLayout {
  size_t state, Ep, matp, fb, slot, total;
  BatchLayout B;
};

static void plan_history(const gf_xs_grid *g, uint64_t np, uint32_t flags, HistLayout &H) {
  memset(&H, 0, sizeof H);
  const bool waves = (flags & (GF_HIST_WAVES | GF_SORT_LOCALITY)) != 0;
  if (!waves) {
    H.total = 256;
    return;
  }
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += al(bytes);
    return at;
  };
  H.state = take(8 * np);
  H.Ep = take(8 * np);
  H.matp = take(np);
  H.fb = take(np);
  plan_batch(g, np, flags & GF_SORT_LOCALITY, true, true, H.B);
  H.slot = take(H.B.slot.bytes);
  H.total = o;
}

gf_status gf_xs_history_bytes(const gf_xs_grid *g, uint64_t n_particles, uint32_t flags, size_t *scratch_bytes) {
  if (!g || !scratch_bytes) return fail(GF_E_INVAL, "grid or scratch_bytes is NULL");
  HistLayout H;
  plan_history(g, n_particles, flags, H);
  *scratch_bytes = H.total;
  return GF_OK;
}

gf_status gf_xs_history_batch(const gf_xs_grid *g, uint64_t first_particle, uint64_t n_particles,
                              int32_t lookups_per_particle, uint64_t starting_seed, uint32_t flags,
                              double *d_macro_out, uint64_t *d_vsum, void *scratch, size_t scratch_bytes,
                              gf_stream_t stream) {
  try {
    if (!g) return fail(GF_E_INVAL, "grid is NULL");
    if (!d_vsum) return fail(GF_E_INVAL, "vsum is NULL");
    if (flags & ~(uint32_t)(GF_SORT_LOCALITY | GF_HIST_WAVES)) return fail(GF_E_INVAL, "unknown flags 0x%x", flags);
    if (g->p.bench == GF_XSBENCH && g->p.n_bands > 1)
      return fail(GF_E_UNSUPPORTED, "history mode on an energy-band grid (a particle's lookups cross bands)");
    const int L = lookups_per_particle;
    if (L < 1 || L > (1 << 20)) return fail(GF_E_INVAL, "lookups_per_particle = %d outside [1, 2^20]", L);
    if (n_particles >= (1ull << 32)) return fail(GF_E_INVAL, "n_particles >= 2^32: split the job");
    HistLayout H;
    plan_history(g, n_particles, flags, H);
    if (n_particles && (!scratch || scratch_bytes < H.total))
      return fail(GF_E_NOMEM, "scratch %zu B < required %zu B", scratch_bytes, H.total);
    if (n_particles && ((uintptr_t)scratch & 255)) return fail(GF_E_INVAL, "scratch must be 256-byte aligned");
    if (n_particles == 0) return GF_OK;
    DeviceGuard dg(g->device);
    if (!dg.ok) return fail(GF_E_CUDA, "cannot make device %d current", g->device);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    unsigned long long *dvsum = reinterpret_cast<unsigned long long *>(d_vsum);
    const uint32_t np = (uint32_t)n_particles;
    const bool xs = g->p.bench == GF_XSBENCH;
    const int ch = xs ? 5 : 4;
    cudaError_t ce;
    if (!(flags & (GF_HIST_WAVES | GF_SORT_LOCALITY))) {
      ce = xs ? launch_xs_history_direct(g->xs, first_particle, np, L, starting_seed, d_macro_out, dvsum, st)
              : launch_rs_history_direct(g->rs, first_particle, np, L, starting_seed, d_macro_out, dvsum, st);
      if (ce != cudaSuccess) return fail(GF_E_CUDA, "history launch: %s", cudaGetErrorString(ce));
      return GF_OK;
    }
    char *sc = static_cast<char *>(scratch);
    uint64_t *state = reinterpret_cast<uint64_t *>(sc + H.state);
    double *Ep = reinterpret_cast<double *>(sc + H.Ep);
    uint8_t *matp = reinterpret_cast<uint8_t *>(sc + H.matp);
    uint8_t *fb = reinterpret_cast<uint8_t *>(sc + H.fb);
    const SortScratch S = slot_sort(sc + H.slot, H.B.slot);
    const bool sort = (flags & GF_SORT_LOCALITY) != 0;
    const uint64_t stride = (uint64_t)L * (xs ? 8ull : 2ull);
    const double *thr = xs ? g->xs.thr : g->rs.thr;
    for (int i = 0; i < L; i++) {
      ce = launch_hist_sample(g->p.bench, first_particle, np, starting_seed, stride, i, thr, state, fb, Ep, matp, st);
      if (ce != cudaSuccess) return fail(GF_E_CUDA, "history sample launch: %s", cudaGetErrorString(ce));
      // the last wave's feedback is never read
      OutSpec out{d_macro_out ? d_macro_out + (size_t)i * ch : nullptr, (uint32_t)(L * ch), i + 1 < L ? fb : nullptr,
                  xs ? 1.0 : 0.0};
      ce = xs ? launch_xs_lookup(g->xs, 0, np, 0, Ep, matp, sort, S, out, dvsum, st)
              : launch_rs_lookup(g->rs, 0, np, 0, Ep, matp, sort, S, out, dvsum, st);
      if (ce != cudaSuccess) return fail(GF_E_CUDA, "history wave launch: %s", cudaGetErrorString(ce));
    }
    return GF_OK;
  } catch (...) {
    return fail(GF_E_NOMEM, "host allocation failed");
  }
}

gf_status gf_xs_selftest_div(const double *d_a, const double *d_b, double *d_out, double *d_ref, uint64_t n,
                             gf_stream_t stream) {
  if (!d_a || !d_b || !d_out || !d_ref) return fail(GF_E_INVAL, "NULL pointer");
  if (n >= (1ull << 31)) return fail(GF_E_INVAL, "n too large");
  if (n == 0) return GF_OK;
  cudaError_t ce = launch_div_selftest(d_a, d_b, d_out, d_ref, (int)n, reinterpret_cast<cudaStream_t>(stream));
  if (ce != cudaSuccess) return fail(GF_E_CUDA, "selftest launch: %s", cudaGetErrorString(ce));
  return GF_OK;
}

gf_status gf_xs_debug_set_kernel(gf_xs_grid *g, int32_t kern, uint64_t tile_min, int32_t nb_on) {
  if (!g) return fail(GF_E_INVAL, "grid is NULL");
  if (g->p.bench != GF_XSBENCH) return fail(GF_E_INVAL, "kernel choice applies to XSBench grids");
  if (kern < GF_KERN_AUTO || kern > GF_KERN_WARP_SEARCH || kern == 3) return fail(GF_E_INVAL, "unknown kernel %d", kern);
  if (tile_min >= (1ull << 32)) return fail(GF_E_INVAL, "tile_min %llu >= 2^32", (unsigned long long)tile_min);
  g->xs.kern = kern;
  if (tile_min) g->xs.tile_min = (uint32_t)tile_min;
  g->xs.nb_on = nb_on ? 1 : 0;
  return GF_OK;
}

gf_status gf_xs_debug_set_division(gf_xs_grid *g, int32_t ieee) {
  if (!g) return fail(GF_E_INVAL, "grid is NULL");
  if (g->p.bench != GF_XSBENCH) return fail(GF_E_INVAL, "division choice applies to XSBench grids");
  g->xs.fastdiv = ieee ? 0 : g->fastdiv_ok;
  return GF_OK;
}

gf_status gf_xs_debug_set_prep_min(gf_xs_grid *g, uint64_t n) {
  if (!g) return fail(GF_E_INVAL, "grid is NULL");
  if (g->p.bench != GF_XSBENCH) return fail(GF_E_INVAL, "applies to XSBench grids");
  g->xs.prep_min = n >= (1ull << 32) ? 0xFFFFFFFFu : (uint32_t)n;
  return GF_OK;
}

gf_status gf_xs_kernel_for(const gf_xs_grid *g, uint64_t n, uint32_t flags, int32_t *kern) {
  if (!g || !kern) return fail(GF_E_INVAL, "grid or kern is NULL");
  *kern = -1;
  if (g->p.bench != GF_XSBENCH || !(flags & GF_SORT_LOCALITY)) return GF_OK;  // RS / unsorted: one kernel each
  const XsDev &X = g->xs;
  if (X.grid_type == GF_GRID_NUCLIDE) {
    const bool tile = X.XR && X.NB && (X.kern == kKernTile || X.kern == kKernTileNB ||
                                       (X.kern == kKernAuto && n >= X.tile_min));
    *kern = tile ? GF_KERN_TILE_NB
                 : (X.NB && X.nb_on && X.kern != kKernWarpSearch) ? GF_KERN_THREAD
                 : (X.kern == kKernThread ? GF_KERN_THREAD : GF_KERN_WARP_SEARCH);
    return GF_OK;
  }
  *kern = X.kern != kKernAuto ? X.kern : (n >= X.tile_min ? GF_KERN_TILE : n >= X.group_min ? GF_KERN_GROUP : GF_KERN_THREAD);
  return GF_OK;
}

gf_status gf_xs_grid_info(const gf_xs_grid *g, int32_t *fastdiv) {
  if (!g) return fail(GF_E_INVAL, "grid is NULL");
  if (fastdiv) *fastdiv = g->p.bench == GF_XSBENCH ? g->xs.fastdiv : 0;
  return GF_OK;
}

gf_status gf_xs_verify(uint64_t raw_sum, uint64_t expected, uint64_t *hash) {
  if (!hash) return fail(GF_E_INVAL, "hash is NULL");
  if (raw_sum & kInvalidInputBit)
    return fail(GF_E_INVAL, "raw sum carries the invalid-input flag (bit 63): a caller lookup had a material "
                "id > 11 or a non-finite energy");
  *hash = raw_sum % GF_HASH_MODULUS;
  if (expected != UINT64_MAX && *hash != expected)
    return fail(GF_E_MISMATCH, "hash %llu != expected %llu", (unsigned long long)*hash, (unsigned long long)expected);
  return GF_OK;
}

}  // extern "C"
