// roofline_probe.cu -- measures the roofline denominators this path is judged against:
//   (1) FP64 pipe throughput of non-fused DADD / DMUL (the lookup may not contract to DFMA: R-FP),
//       and of IEEE __ddiv_rn (the per-micro-evaluation division);
//   (2) K6: the random 96-B gather bandwidth over a buffer >> L2:
//       records of 48 B at uniformly random 48-B-aligned offsets, 6 x 16-B loads per gather,
//       R independent gathers in flight per thread.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -fmad=false
#include <cuda_runtime.h>
#include <stdint.h>


__global__ void k_dadd(double *out, int iters, double a) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
      x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_dmul(double *out, int iters, double a) {
  double x0 = threadIdx.x + 1, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      x0 = __dmul_rn(x0, a); x1 = __dmul_rn(x1, a); x2 = __dmul_rn(x2, a); x3 = __dmul_rn(x3, a);
      x4 = __dmul_rn(x4, a); x5 = __dmul_rn(x5, a); x6 = __dmul_rn(x6, a); x7 = __dmul_rn(x7, a);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_ddiv(double *out, int iters, double a) {
  double x0 = threadIdx.x + 1.5, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 4; u++) {
      x0 = __ddiv_rn(a, x0); x1 = __ddiv_rn(a, x1); x2 = __ddiv_rn(a, x2); x3 = __ddiv_rn(a, x3);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

template <int R>
__global__ void k_gather(const double2 *__restrict__ buf, long long nrec, int per_thread, double *out, uint64_t salt) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (int it = 0; it < per_thread; it += R) {
    double2 v[R][6];
#pragma unroll
    for (int r = 0; r < R; r++) {
      // uniform record index in [0, nrec-1) by a multiply-high (no 64-bit modulo on the hot path)
      long long rec = (long long)__umul64hi(mix(tid * 1315423911ull + (uint64_t)(it + r) * 2654435761ull + salt),
                                            (uint64_t)(nrec - 1));
      const double2 *p = buf + rec * 3;  // 48-B record = 3 double2; a pair is 6 double2 (96 B)
#pragma unroll
      for (int k = 0; k < 6; k++) v[r][k] = __ldg(p + k);
    }
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
      for (int k = 0; k < 6; k++) acc += v[r][k].x + v[r][k].y;
  }
  if (acc == 12345.678) out[0] = acc;  // keep the loads alive
}

__global__ void k_copy(const double4 *__restrict__ a, double4 *__restrict__ b, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// Returns elapsed ms of one launch (after one warm-up), or a negative value on error.
static float time_it(void (*launch)(void *), void *ctx) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch(ctx);
  cudaEventRecord(a);
  launch(ctx);
  cudaEventRecord(b);
  if (cudaEventSynchronize(b) != cudaSuccess) return -1.f;
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms;
}

struct FpCtx { double *out; int blocks, threads, iters, which; };
static void launch_fp(void *c) {
  FpCtx *x = (FpCtx *)c;
  if (x->which == 0) k_dadd<<<x->blocks, x->threads>>>(x->out, x->iters, 1.0000001);
  else if (x->which == 1) k_dmul<<<x->blocks, x->threads>>>(x->out, x->iters, 0.9999999);
  else k_ddiv<<<x->blocks, x->threads>>>(x->out, x->iters, 1.0000001);
}

// ops/s (lane operations) of DADD (which=0), DMUL (1) or DDIV (2)
extern "C" double probe_fp64(int which) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  FpCtx c;
  c.threads = 512;
  c.blocks = sms * 4;
  c.iters = which == 2 ? 256 : 4096;
  c.which = which;
  cudaMalloc(&c.out, sizeof(double) * c.blocks * c.threads);
  float ms = time_it(launch_fp, &c);
  cudaFree(c.out);
  double per_thread = which == 2 ? 16.0 * c.iters : 64.0 * c.iters;
  return ms > 0 ? per_thread * c.blocks * c.threads / (ms * 1e-3) : -1.0;
}

struct GCtx { const double2 *buf; long long nrec; int blocks, threads, per, R; double *out; uint64_t salt; };
static void launch_g(void *v) {
  GCtx *c = (GCtx *)v;
  c->salt += 0x9e3779b97f4a7c15ull;
  switch (c->R) {
    case 1: k_gather<1><<<c->blocks, c->threads>>>(c->buf, c->nrec, c->per, c->out, c->salt); break;
    case 2: k_gather<2><<<c->blocks, c->threads>>>(c->buf, c->nrec, c->per, c->out, c->salt); break;
    case 4: k_gather<4><<<c->blocks, c->threads>>>(c->buf, c->nrec, c->per, c->out, c->salt); break;
    default: k_gather<8><<<c->blocks, c->threads>>>(c->buf, c->nrec, c->per, c->out, c->salt); break;
  }
}

// Useful-byte GB/s (96 B per gather) of random record-pair gathers over `bytes` of HBM.
extern "C" double probe_gather(long long bytes, int R, int threads, int blocks_per_sm) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  GCtx c;
  c.nrec = bytes / 48;
  if (cudaMalloc((void **)&c.buf, (size_t)c.nrec * 48) != cudaSuccess) return -1.0;
  cudaMemset((void *)c.buf, 0, (size_t)c.nrec * 48);
  cudaMalloc(&c.out, 8);
  c.threads = threads;
  c.blocks = sms * blocks_per_sm;
  c.per = 128;
  c.R = R;
  c.salt = 1;
  float ms = time_it(launch_g, &c);
  if (cudaGetLastError() != cudaSuccess) ms = -1.f;
  cudaFree((void *)c.buf);
  cudaFree(c.out);
  double gathers = (double)c.blocks * c.threads * c.per;
  return ms > 0 ? gathers * 96.0 / (ms * 1e-3) / 1e9 : -1.0;
}

struct CCtx { const double4 *a; double4 *b; long long n; int blocks; };
static void launch_c(void *v) {
  CCtx *c = (CCtx *)v;
  k_copy<<<c->blocks, 512>>>(c->a, c->b, c->n);
}

// Copy GB/s (read + write bytes) of `bytes` per buffer.
extern "C" double probe_copy(long long bytes) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  CCtx c;
  c.n = bytes / 32;
  if (cudaMalloc((void **)&c.a, bytes) != cudaSuccess) return -1.0;
  if (cudaMalloc((void **)&c.b, bytes) != cudaSuccess) return -1.0;
  cudaMemset((void *)c.a, 0, bytes);
  c.blocks = sms * 16;
  float ms = time_it(launch_c, &c);
  cudaFree((void *)c.a);
  cudaFree(c.b);
  return ms > 0 ? 2.0 * bytes / (ms * 1e-3) / 1e9 : -1.0;
}

extern "C" int probe_sm_count(void) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  return sms;
}

extern "C" int probe_l2_bytes(void) {
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  return l2;
}

extern "C" int probe_clock_khz(void) {
  int k = 0;
  cudaDeviceGetAttribute(&k, cudaDevAttrClockRate, 0);
  return k;
}
