// amg.cu -- NEXT-4: the AMGmk relax kernel on sm_100a (include/gf_amg.h; readings R-AMG-MAT /
// R-AMG-RELAX).  Independent of oracle/.
//
// Matrix build: every row's offset has a closed form -- the entries per row are cx(x) cy(y) cz(z)
// (2 at a face, 3 inside, 1 on a length-1 axis), so the prefix over the rows before (x, y, z) is
// Px(x) Sy Sz-planes etc. -- and each thread writes its row without atomics or scans.
// Relax: kLanes lanes per row; lane q loads entries q+1, q+1+kLanes, ... of the row (coalesced
// column / value loads, independent u gathers in flight), and the group subtracts the products in
// row order through shuffles (the reading's left-to-right sum).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <new>
#include <string>

#include "gf_amg.h"

namespace gfamg {

constexpr int kTpb = 256;
#ifndef GF_AMG_LANES
#define GF_AMG_LANES 2
#endif
constexpr int kLanes = GF_AMG_LANES;
#ifndef GF_AMG_UNR
#define GF_AMG_UNR 4
#endif
constexpr int kUnr = GF_AMG_UNR;  // row-loop unroll (loads of several rounds in flight)

__host__ __device__ inline long long axis_count(long long k, long long m) {
  return m == 1 ? 1 : ((k == 0 || k == m - 1) ? 2 : 3);
}
// sum of axis_count over k' < k
__host__ __device__ inline long long axis_prefix(long long k, long long m) {
  if (m == 1) return k;  // (k is 0 or 1)
  return k == 0 ? 0 : 2 + 3 * (k - 1) - (k == m ? 1 : 0);  // k == m: the last cell counts 2
}

__host__ __device__ inline long long row_offset(long long x, long long y, long long z, long long nx, long long ny,
                                                long long nz) {
  const long long Sx = axis_prefix(nx, nx), Sy = axis_prefix(ny, ny);
  return axis_prefix(z, nz) * Sx * Sy + axis_count(z, nz) * (axis_prefix(y, ny) * Sx + axis_count(y, ny) * axis_prefix(x, nx));
}

__global__ void __launch_bounds__(kTpb) amg_build(int nx, int ny, int nz, uint32_t *__restrict__ rowptr,
                                                  uint32_t *__restrict__ col, double *__restrict__ val) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = (long long)nx * ny * nz;
  if (i >= n) return;
  const int x = (int)(i % nx), y = (int)((i / nx) % ny), z = (int)(i / ((long long)nx * ny));
  long long e = row_offset(x, y, z, nx, ny, nz);
  rowptr[i] = (uint32_t)e;
  if (i == n - 1) rowptr[n] = (uint32_t)(e + axis_count(x, nx) * axis_count(y, ny) * axis_count(z, nz));
  col[e] = (uint32_t)i;
  val[e++] = 26.0;
  for (int dz = -1; dz <= 1; dz++)
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++) {
        if (!dx && !dy && !dz) continue;
        const int X = x + dx, Y = y + dy, Z = z + dz;
        if (X >= 0 && X < nx && Y >= 0 && Y < ny && Z >= 0 && Z < nz) {
          col[e] = (uint32_t)(X + (long long)nx * (Y + (long long)ny * Z));
          val[e++] = -1.0;
        }
      }
}

__global__ void __launch_bounds__(kTpb) amg_relax(uint32_t n, const uint32_t *__restrict__ rowptr,
                                                  const uint32_t *__restrict__ col, const double *__restrict__ val,
                                                  const double *__restrict__ f, const double *__restrict__ u,
                                                  double *__restrict__ out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t i = t / kLanes;
  const int q = (int)(t % kLanes);
  const bool live = i < n;
  const uint32_t a = live ? __ldg(rowptr + i) : 0u, b = live ? __ldg(rowptr + i + 1) : 0u;
  // warp-uniform trip count (the longest row of the warp): the shuffles then run converged on the full
  // mask (a per-group mask and trip count make the compiler re-check convergence with MATCH/VOTE every
  // round, which saturated the ADU pipe: DESIGN.md Sec. 7)
  const uint32_t len = __reduce_max_sync(0xffffffffu, b - a);
  double res = live ? __ldg(f + i) : 0.0;
#pragma unroll kUnr
  for (uint32_t j = 1; j < len; j += kLanes) {  // (entry a is the diagonal)
    const uint32_t e = a + j + q;
    const double p = e < b ? __dmul_rn(__ldg(val + e), __ldg(u + __ldg(col + e))) : 0.0;
    if (kLanes == 1) {
      res = __dsub_rn(res, p);
      continue;
    }
#pragma unroll
    for (int k = 0; k < kLanes; k++) {
      const double y = __shfl_sync(0xffffffffu, p, k, kLanes);
      if (a + j + k < b) res = __dsub_rn(res, y);
    }
  }
  if (live && q == 0) out[i] = __ddiv_rn(res, __ldg(val + a));
}

// CSR-stream variant (GF_AMG_STREAM=1): a CTA owns kRows consecutive rows; its threads first form
// every product val[e] u[col[e]] of the CTA's contiguous nonzero range with fully coalesced loads into
// shared memory, then each thread subtracts its row's products in order (same operations, same order).
#ifndef GF_AMG_STREAM
#define GF_AMG_STREAM 0
#endif
#ifndef GF_AMG_SU
#define GF_AMG_SU 4
#endif
constexpr int kSU = GF_AMG_SU;  // products in flight per thread
constexpr int kRows = 128;
constexpr int kMaxRow = 27;
__global__ void __launch_bounds__(kRows) amg_relax_stream(uint32_t n, const uint32_t *__restrict__ rowptr,
                                                         const uint32_t *__restrict__ col,
                                                         const double *__restrict__ val,
                                                         const double *__restrict__ f, const double *__restrict__ u,
                                                         double *__restrict__ out) {
  __shared__ double prod[kRows * kMaxRow];
  const uint32_t r0 = blockIdx.x * kRows;
  const uint32_t r1 = min(n, r0 + kRows);
  const uint32_t base = __ldg(rowptr + r0), end = __ldg(rowptr + r1);
  const uint32_t cnt = end - base;
  uint32_t k = threadIdx.x;
  for (; k + (kSU - 1) * kRows < cnt; k += kSU * kRows) {
    uint32_t c[kSU];
    double v[kSU];
#pragma unroll
    for (int j = 0; j < kSU; j++) c[j] = __ldg(col + base + k + j * kRows), v[j] = __ldg(val + base + k + j * kRows);
#pragma unroll
    for (int j = 0; j < kSU; j++) prod[k + j * kRows] = __dmul_rn(v[j], __ldg(u + c[j]));
  }
  for (; k < cnt; k += kRows) prod[k] = __dmul_rn(__ldg(val + base + k), __ldg(u + __ldg(col + base + k)));
  __syncthreads();
  const uint32_t i = r0 + threadIdx.x;
  if (i >= n) return;
  const uint32_t a = __ldg(rowptr + i) - base, b = __ldg(rowptr + i + 1) - base;
  double res = __ldg(f + i);
  for (uint32_t e = a + 1; e < b; e++) res = __dsub_rn(res, prod[e]);
  out[i] = __ddiv_rn(res, __ldg(val + base + a));
}

// Warp-stream variant (GF_AMG_STREAM=2): a warp owns 32 consecutive rows, one per lane.  Phase 1: the
// warp walks the rows' contiguous nonzero range 32 entries at a time (one line of col, two of val per
// load instruction) and stages every product val[e] u[col[e]] in its own SMEM slice; phase 2: each lane
// subtracts its row's products in order.  Same operations in the same order as amg_relax; no CTA sync.
constexpr int kWarpsW = 4;
__global__ void __launch_bounds__(32 * kWarpsW) amg_relax_warp(uint32_t n, const uint32_t *__restrict__ rowptr,
                                                              const uint32_t *__restrict__ col,
                                                              const double *__restrict__ val,
                                                              const double *__restrict__ f,
                                                              const double *__restrict__ u,
                                                              double *__restrict__ out) {
  __shared__ double prod[kWarpsW][32 * kMaxRow];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t r0 = (blockIdx.x * kWarpsW + w) * 32u;
  if (r0 >= n) return;  // (warp-uniform)
  const uint32_t r1 = min(n, r0 + 32u);
  const uint32_t base = __ldg(rowptr + r0), cnt = __ldg(rowptr + r1) - base;
  double *pw = prod[w];
  const uint32_t *cb = col + base;
  const double *vb = val + base;
  uint32_t k = lane;
  for (; k + 32 * (kSU - 1) < cnt; k += 32 * kSU) {
    uint32_t c[kSU];
    double v[kSU];
#pragma unroll
    for (int j = 0; j < kSU; j++) c[j] = __ldg(cb + k + 32 * j), v[j] = __ldg(vb + k + 32 * j);
#pragma unroll
    for (int j = 0; j < kSU; j++) pw[k + 32 * j] = __dmul_rn(v[j], __ldg(u + c[j]));
  }
  for (; k < cnt; k += 32) pw[k] = __dmul_rn(__ldg(vb + k), __ldg(u + __ldg(cb + k)));
  __syncwarp();
  const uint32_t i = r0 + lane;
  if (i >= n) return;
  const uint32_t a = __ldg(rowptr + i) - base, b = __ldg(rowptr + i + 1) - base;
  double res = __ldg(f + i);
  for (uint32_t e = a + 1; e < b; e++) res = __dsub_rn(res, pw[e]);
  out[i] = __ddiv_rn(res, __ldg(vb + a));
}

thread_local std::string t_err;
gf_amg_status fail(gf_amg_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return s;
}
inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace gfamg

using namespace gfamg;

struct gf_amg_matrix {
  int device;
  uint32_t n, nnz;
  const uint32_t *rowptr, *col;
  const double *val;
};

extern "C" {

const char *gf_amg_last_error(void) { return t_err.c_str(); }

gf_amg_status gf_amg_matrix_bytes(int32_t nx, int32_t ny, int32_t nz, size_t *bytes, int64_t *nnz) {
  if (!bytes || !nnz) return fail(GF_AMG_E_INVAL, "NULL output");
  if (nx < 1 || ny < 1 || nz < 1) return fail(GF_AMG_E_INVAL, "grid %d x %d x %d", nx, ny, nz);
  const long long n = (long long)nx * ny * nz;
  if (n >= (1ll << 27)) return fail(GF_AMG_E_INVAL, "n = %lld >= 2^27", n);
  const long long z = axis_prefix(nx, nx) * axis_prefix(ny, ny) * axis_prefix(nz, nz);
  *nnz = z;
  *bytes = al((n + 1) * 4) + al(z * 4) + al(z * 8);
  return GF_AMG_OK;
}

gf_amg_status gf_amg_matrix_init(int32_t nx, int32_t ny, int32_t nz, int device, void *mem, size_t bytes,
                                 gf_amg_stream_t stream, gf_amg_matrix **out) {
  size_t need = 0;
  int64_t nnz = 0;
  gf_amg_status st = gf_amg_matrix_bytes(nx, ny, nz, &need, &nnz);
  if (st != GF_AMG_OK) return st;
  if (!mem || !out) return fail(GF_AMG_E_INVAL, "NULL argument");
  if (bytes < need) return fail(GF_AMG_E_NOMEM, "buffer %zu B < %zu B", bytes, need);
  if ((uintptr_t)mem & 255) return fail(GF_AMG_E_INVAL, "buffer must be 256-B aligned");
  const long long n = (long long)nx * ny * nz;
  char *m = static_cast<char *>(mem);
  uint32_t *rowptr = reinterpret_cast<uint32_t *>(m);
  uint32_t *col = reinterpret_cast<uint32_t *>(m + al((n + 1) * 4));
  double *val = reinterpret_cast<double *>(m + al((n + 1) * 4) + al(nnz * 4));
  int cur = 0;
  cudaGetDevice(&cur);
  if (cudaSetDevice(device) != cudaSuccess) return fail(GF_AMG_E_CUDA, "cannot make device %d current", device);
  amg_build<<<(unsigned)((n + kTpb - 1) / kTpb), kTpb, 0, reinterpret_cast<cudaStream_t>(stream)>>>(nx, ny, nz, rowptr,
                                                                                                    col, val);
  const cudaError_t ce = cudaGetLastError();
  cudaSetDevice(cur);
  if (ce != cudaSuccess) return fail(GF_AMG_E_CUDA, "matrix build: %s", cudaGetErrorString(ce));
  gf_amg_matrix *A = new (std::nothrow) gf_amg_matrix{device, (uint32_t)n, (uint32_t)nnz, rowptr, col, val};
  if (!A) return fail(GF_AMG_E_NOMEM, "host allocation failed");
  *out = A;
  return GF_AMG_OK;
}

gf_amg_status gf_amg_matrix_free(gf_amg_matrix *A) {
  delete A;
  return GF_AMG_OK;
}

gf_amg_status gf_amg_matrix_info(const gf_amg_matrix *A, int64_t *n, int64_t *nnz, const uint32_t **rowptr,
                                 const uint32_t **col, const double **val) {
  if (!A) return fail(GF_AMG_E_INVAL, "matrix is NULL");
  if (n) *n = A->n;
  if (nnz) *nnz = A->nnz;
  if (rowptr) *rowptr = A->rowptr;
  if (col) *col = A->col;
  if (val) *val = A->val;
  return GF_AMG_OK;
}

gf_amg_status gf_amg_relax(const gf_amg_matrix *A, const double *d_f, const double *d_u, double *d_out,
                           gf_amg_stream_t stream) {
  if (!A || !d_f || !d_u || !d_out) return fail(GF_AMG_E_INVAL, "NULL argument");
  if (d_u == d_out) return fail(GF_AMG_E_INVAL, "d_u and d_out alias (Jacobi sweep)");
  int cur = 0;
  cudaGetDevice(&cur);
  if (cudaSetDevice(A->device) != cudaSuccess) return fail(GF_AMG_E_CUDA, "cannot make device current");
#if GF_AMG_STREAM == 2
  amg_relax_warp<<<(A->n + 32 * kWarpsW - 1) / (32 * kWarpsW), 32 * kWarpsW, 0,
                   reinterpret_cast<cudaStream_t>(stream)>>>(A->n, A->rowptr, A->col, A->val, d_f, d_u, d_out);
#elif GF_AMG_STREAM
  amg_relax_stream<<<(A->n + kRows - 1) / kRows, kRows, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      A->n, A->rowptr, A->col, A->val, d_f, d_u, d_out);
#else
  const long long threads = (long long)A->n * kLanes;
  amg_relax<<<(unsigned)((threads + kTpb - 1) / kTpb), kTpb, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      A->n, A->rowptr, A->col, A->val, d_f, d_u, d_out);
#endif
  const cudaError_t ce = cudaGetLastError();
  cudaSetDevice(cur);
  if (ce != cudaSuccess) return fail(GF_AMG_E_CUDA, "relax launch: %s", cudaGetErrorString(ce));
  return GF_AMG_OK;
}

}  // extern "C"
