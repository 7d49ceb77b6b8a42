// pagerank.cu -- NEXT-4: the page-rank propagation step on sm_100a (include/gf_pr.h; readings
// R-PR-GRAPH / R-PR-STEP).  Independent of oracle/.
//
// Graph build (init, untimed): pr_degrees (degrees, in-degree counts by atomics) -> three-kernel scan
// -> pr_fill (each edge claims a slot of its destination row; key = u << 6 | j) -> pr_order (each row
// sorted by key, i.e. by (source, draw) -- the order the reading fixes, so sums are bit-exact).
// Step: pr_contrib (r[u] / d_u, coalesced) then pr_gather: 4 lanes per destination row, each lane
// loading every 4th in-edge, the row's contributions combined in row order by a serial walk over the
// group's lanes (shuffles) -- coalesced index loads, independent gathers in flight, the reading's
// left-to-right sum.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <new>
#include <string>

#include "gf_internal.cuh"
#include "gf_pr.h"

namespace gf {

#ifndef GF_PR_L2HINT
#define GF_PR_L2HINT 1  // P1 2.488 -> 2.438 ms (an evict_last store of c in pr_contrib: no further gain)
#endif
constexpr int kPrTpb = 256;
constexpr int kPrScan = 1024;

__global__ void __launch_bounds__(kPrTpb) pr_degrees(uint32_t n, int D, uint64_t seed, int32_t *__restrict__ outdeg,
                                                     uint32_t *__restrict__ indeg) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  uint64_t s = lcg_skip(seed, 2ull * (uint64_t)D * u);
  int d = 1 + (int)__dmul_rn(lcg_draw(s), (double)(2 * D - 1));
  d = d > 2 * D - 1 ? 2 * D - 1 : d;
  outdeg[u] = d;
  for (int j = 0; j < d; j++) {
    long long v = (long long)__dmul_rn(lcg_draw(s), (double)n);
    v = v > (long long)n - 1 ? (long long)n - 1 : v;
    atomicAdd(indeg + v, 1u);
  }
}

// exclusive scan: per CTA of kPrScan, CTA totals, then the totals' prefix added back
__global__ void __launch_bounds__(kPrScan) pr_scan_local(const uint32_t *__restrict__ in, uint32_t *__restrict__ out,
                                                         uint32_t *__restrict__ tot, uint32_t n) {
  __shared__ uint32_t ws[32];
  const uint32_t i = blockIdx.x * kPrScan + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t c = i < n ? in[i] : 0u;
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t v = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    ws[lane] = v;
  }
  __syncthreads();
  if (i < n) out[i] = x - c + (w > 0 ? ws[w - 1] : 0u);
  if (threadIdx.x == kPrScan - 1) tot[blockIdx.x] = ws[31];
}

// one CTA: exclusive scan of up to kPrScan * 64 CTA totals in place; total into *sum
__global__ void __launch_bounds__(kPrScan) pr_scan_totals(uint32_t *__restrict__ tot, uint32_t nb,
                                                          uint32_t *__restrict__ sum) {
  __shared__ uint32_t ws[32];
  constexpr int kPer = 64;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t v[kPer], s = 0;
#pragma unroll
  for (int q = 0; q < kPer; q++) {
    const uint32_t i = threadIdx.x * kPer + q;
    v[q] = i < nb ? tot[i] : 0u;
    s += v[q];
  }
  uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    ws[lane] = t;
  }
  __syncthreads();
  uint32_t run = x - s + (w > 0 ? ws[w - 1] : 0u);
#pragma unroll
  for (int q = 0; q < kPer; q++) {
    const uint32_t i = threadIdx.x * kPer + q;
    if (i < nb) tot[i] = run;
    run += v[q];
  }
  if (threadIdx.x == kPrScan - 1) *sum = run;
}

__global__ void __launch_bounds__(kPrScan) pr_scan_add(uint32_t *__restrict__ out, const uint32_t *__restrict__ tot,
                                                       uint32_t n, const uint32_t *__restrict__ sum,
                                                       uint32_t *__restrict__ cursor) {
  const uint32_t i = blockIdx.x * kPrScan + threadIdx.x;
  if (i < n) {
    out[i] += tot[blockIdx.x];
    cursor[i] = out[i];
  }
  if (i == n) out[n] = *sum;
}

__global__ void __launch_bounds__(kPrTpb) pr_fill(uint32_t n, int D, uint64_t seed, uint32_t *__restrict__ cursor,
                                                  uint32_t *__restrict__ key) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  uint64_t s = lcg_skip(seed, 2ull * (uint64_t)D * u);
  int d = 1 + (int)__dmul_rn(lcg_draw(s), (double)(2 * D - 1));
  d = d > 2 * D - 1 ? 2 * D - 1 : d;
  for (int j = 0; j < d; j++) {
    long long v = (long long)__dmul_rn(lcg_draw(s), (double)n);
    v = v > (long long)n - 1 ? (long long)n - 1 : v;
    key[atomicAdd(cursor + v, 1u)] = (u << 6) | (uint32_t)j;
  }
}

// Each row sorted by key (source, draw): insertion sort (rows average D entries); col = key >> 6.
__global__ void __launch_bounds__(kPrTpb) pr_order(uint32_t n, const uint32_t *__restrict__ rowptr,
                                                   uint32_t *__restrict__ key) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const uint32_t a = rowptr[v], b = rowptr[v + 1];
  for (uint32_t i = a + 1; i < b; i++) {
    const uint32_t x = key[i];
    uint32_t j = i;
    while (j > a && key[j - 1] > x) {
      key[j] = key[j - 1];
      j--;
    }
    key[j] = x;
  }
  for (uint32_t i = a; i < b; i++) key[i] >>= 6;
}

__global__ void __launch_bounds__(kPrTpb) pr_contrib(uint32_t n, const double *__restrict__ r,
                                                     const int32_t *__restrict__ outdeg, double *__restrict__ c) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  c[u] = __ddiv_rn(r[u], (double)outdeg[u]);
}

// kG lanes per row; lane q of the group loads in-edges a + q, a + q + kG, ...; the row's sum is
// accumulated in row order by walking the group's lanes in turn (one shuffle per edge step).
#ifndef GF_PR_G
#define GF_PR_G 4
#endif
constexpr int kG = GF_PR_G;  // lanes per destination row
#ifndef GF_PR_UNI
#define GF_PR_UNI 1
#endif
#ifndef GF_PR_UNR
#define GF_PR_UNR 4
#endif
constexpr int kPrUnr = GF_PR_UNR;
// GF_PR_L2HINT: L2 eviction priorities -- the contribution array (134 MB at 2^24 nodes, about the L2's
// size) evict_last, the streamed in-edge indices evict_first -- so the random 8-B gathers hit L2 more
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_hint_f64(const double *p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_hint_u32(const uint32_t *p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

__global__ void __launch_bounds__(kPrTpb) pr_gather(uint32_t n, const uint32_t *__restrict__ rowptr,
                                                    const uint32_t *__restrict__ col, const double *__restrict__ c,
                                                    double *__restrict__ out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t v = t / kG;
  const int q = (int)(t % kG);
  const bool live = v < n;
  const uint32_t a = live ? __ldg(rowptr + v) : 0u, b = live ? __ldg(rowptr + v + 1) : 0u;
  double s = 0.0;
#if GF_PR_UNI
  // warp-uniform trip count (the warp's longest row): converged full-mask shuffles, no per-round
  // convergence checks (MATCH/VOTE) from a per-group mask
  const uint32_t len = __reduce_max_sync(0xffffffffu, b - a);
#if GF_PR_L2HINT
  const uint64_t pl = l2_policy_last(), pf = l2_policy_first();
#endif
#pragma unroll kPrUnr
  for (uint32_t j = 0; j < len; j += kG) {
    const uint32_t e = a + j + q;
#if GF_PR_L2HINT
    const double x = e < b ? ld_hint_f64(c + ld_hint_u32(col + e, pf), pl) : 0.0;
#else
    const double x = e < b ? __ldg(c + __ldg(col + e)) : 0.0;
#endif
#pragma unroll
    for (int k = 0; k < kG; k++) {
      const double y = __shfl_sync(0xffffffffu, x, k, kG);
      if (a + j + k < b) s = __dadd_rn(s, y);  // every lane keeps the same running sum
    }
  }
#else
  const unsigned gmask = (unsigned)((1ull << kG) - 1) << ((threadIdx.x & 31) & ~(kG - 1));  // this row's lanes
  // rounds of kG edges: every lane fetches its edge of the round, then the group adds them in order
  for (uint32_t e0 = a; e0 < b; e0 += kG) {
    const uint32_t e = e0 + q;
    const double x = e < b ? __ldg(c + __ldg(col + e)) : 0.0;
#pragma unroll
    for (int k = 0; k < kG; k++) {
      const double y = __shfl_sync(gmask, x, k, kG);
      if (e0 + k < b) s = __dadd_rn(s, y);  // every lane keeps the same running sum
    }
  }
#endif
  if (live && q == 0) {
    const double base = __ddiv_rn(__dsub_rn(1.0, 0.85), (double)n);
    out[v] = __dadd_rn(base, __dmul_rn(0.85, s));
  }
}

}  // namespace gf

using namespace gf;

namespace {
thread_local std::string t_err;
gf_pr_status fail(gf_pr_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return s;
}
inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }
inline unsigned nb(long long n, int b) { return (unsigned)((n + b - 1) / b); }
}  // namespace

struct gf_pr_graph {
  int device;
  uint32_t n;
  uint32_t nnz;
  const uint32_t *rowptr;
  const uint32_t *col;
  const int32_t *outdeg;
};

extern "C" {

const char *gf_pr_last_error(void) { return t_err.c_str(); }

gf_pr_status gf_pr_graph_bytes(int64_t n, int32_t D, size_t *graph_bytes, size_t *scratch_bytes) {
  if (!graph_bytes || !scratch_bytes) return fail(GF_PR_E_INVAL, "NULL output");
  if (n < 1 || n >= (1ll << 26)) return fail(GF_PR_E_INVAL, "n_nodes %lld outside [1, 2^26)", (long long)n);
  if (D < 1 || D > 32) return fail(GF_PR_E_INVAL, "avg_degree %d outside [1, 32]", D);
  const size_t nnz_max = (size_t)n * (2 * D - 1);
  *graph_bytes = al((n + 1) * 4) + al(nnz_max * 4) + al(n * 4);
  *scratch_bytes = al(n * 4) + al(n * 4) + al(((n + kPrScan - 1) / kPrScan) * 4) + 256;
  return GF_PR_OK;
}

gf_pr_status gf_pr_graph_init(int64_t n, int32_t D, uint64_t seed, int device, void *graph_mem, size_t graph_bytes,
                              void *scratch, size_t scratch_bytes, gf_pr_stream_t stream, gf_pr_graph **out) {
  size_t gb = 0, sb = 0;
  gf_pr_status st = gf_pr_graph_bytes(n, D, &gb, &sb);
  if (st != GF_PR_OK) return st;
  if (!out || !graph_mem || !scratch) return fail(GF_PR_E_INVAL, "NULL argument");
  if (graph_bytes < gb || scratch_bytes < sb) return fail(GF_PR_E_NOMEM, "buffers smaller than gf_pr_graph_bytes");
  if (((uintptr_t)graph_mem & 255) || ((uintptr_t)scratch & 255)) return fail(GF_PR_E_INVAL, "buffers must be 256-B aligned");
  if (((n + kPrScan - 1) / kPrScan) > (int64_t)kPrScan * 64) return fail(GF_PR_E_INVAL, "n too large for the scan");
  int cur = 0;
  cudaGetDevice(&cur);
  if (cudaSetDevice(device) != cudaSuccess) return fail(GF_PR_E_CUDA, "cannot make device %d current", device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char *g = static_cast<char *>(graph_mem), *sc = static_cast<char *>(scratch);
  const size_t nnz_max = (size_t)n * (2 * D - 1);
  uint32_t *rowptr = reinterpret_cast<uint32_t *>(g);
  uint32_t *col = reinterpret_cast<uint32_t *>(g + al((n + 1) * 4));
  int32_t *outdeg = reinterpret_cast<int32_t *>(g + al((n + 1) * 4) + al(nnz_max * 4));
  uint32_t *indeg = reinterpret_cast<uint32_t *>(sc);
  uint32_t *cursor = reinterpret_cast<uint32_t *>(sc + al(n * 4));
  uint32_t *tot = reinterpret_cast<uint32_t *>(sc + 2 * al(n * 4));
  uint32_t *sum = reinterpret_cast<uint32_t *>(sc + 2 * al(n * 4) + al(((n + kPrScan - 1) / kPrScan) * 4));
  const uint32_t un = (uint32_t)n, nblocks = (uint32_t)((n + kPrScan - 1) / kPrScan);
  cudaError_t ce = cudaMemsetAsync(indeg, 0, n * 4, s);
  if (ce == cudaSuccess) {
    pr_degrees<<<nb(n, kPrTpb), kPrTpb, 0, s>>>(un, D, seed, outdeg, indeg);
    pr_scan_local<<<nblocks, kPrScan, 0, s>>>(indeg, rowptr, tot, un);
    pr_scan_totals<<<1, kPrScan, 0, s>>>(tot, nblocks, sum);
    pr_scan_add<<<nb(n + 1, kPrScan), kPrScan, 0, s>>>(rowptr, tot, un, sum, cursor);
    pr_fill<<<nb(n, kPrTpb), kPrTpb, 0, s>>>(un, D, seed, cursor, col);
    pr_order<<<nb(n, kPrTpb), kPrTpb, 0, s>>>(un, rowptr, col);
    ce = cudaGetLastError();
  }
  uint32_t nnz = 0;
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(&nnz, sum, 4, cudaMemcpyDeviceToHost, s);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  cudaSetDevice(cur);
  if (ce != cudaSuccess) return fail(GF_PR_E_CUDA, "graph init: %s", cudaGetErrorString(ce));
  gf_pr_graph *h = new (std::nothrow) gf_pr_graph{device, un, nnz, rowptr, col, outdeg};
  if (!h) return fail(GF_PR_E_NOMEM, "host allocation failed");
  *out = h;
  return GF_PR_OK;
}

gf_pr_status gf_pr_graph_free(gf_pr_graph *g) {
  delete g;
  return GF_PR_OK;
}

gf_pr_status gf_pr_graph_info(const gf_pr_graph *g, int64_t *n_edges, const uint32_t **rowptr, const uint32_t **col,
                              const int32_t **outdeg) {
  if (!g) return fail(GF_PR_E_INVAL, "graph is NULL");
  if (n_edges) *n_edges = g->nnz;
  if (rowptr) *rowptr = g->rowptr;
  if (col) *col = g->col;
  if (outdeg) *outdeg = g->outdeg;
  return GF_PR_OK;
}

gf_pr_status gf_pr_propagate(const gf_pr_graph *g, const double *d_in, double *d_out, double *d_contrib,
                             gf_pr_stream_t stream) {
  if (!g || !d_in || !d_out || !d_contrib) return fail(GF_PR_E_INVAL, "NULL argument");
  if (d_in == d_out) return fail(GF_PR_E_INVAL, "d_in and d_out alias");
  int cur = 0;
  cudaGetDevice(&cur);
  if (cudaSetDevice(g->device) != cudaSuccess) return fail(GF_PR_E_CUDA, "cannot make device current");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  pr_contrib<<<nb(g->n, kPrTpb), kPrTpb, 0, s>>>(g->n, d_in, g->outdeg, d_contrib);
  pr_gather<<<nb((long long)g->n * kG, kPrTpb), kPrTpb, 0, s>>>(g->n, g->rowptr, g->col, d_contrib, d_out);
  const cudaError_t ce = cudaGetLastError();
  cudaSetDevice(cur);
  if (ce != cudaSuccess) return fail(GF_PR_E_CUDA, "propagate launch: %s", cudaGetErrorString(ce));
  return GF_PR_OK;
}

}  // extern "C"
