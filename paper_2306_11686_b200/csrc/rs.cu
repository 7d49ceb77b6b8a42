// rs.cu -- RSBench (C5): device-side multipole data generation and the Doppler-broadened lookup
// (generator c.2 lines 594-603, kernel lines 605-632).
//
// Data generation consumes ONE LCG stream from init_seed in this order (R-RSGEN): concentrations,
// the n_poles increments, the n_windows increments, poles (8 doubles + 1 int each), windows
// (3 doubles each), K0RS.  Every element's stream position is known in closed form once the pole
// and window counts are scanned, so each is generated independently by skip-ahead.
//
// Lookup: per nuclide of the material, window w = (int)(E / (1.0/n_windows)), 4 phase factors
// from K0RS*sqrt(E) with the l-dependent atan corrections, background E*(T, A, F), then the poles
// in [start, end) (R-RSEND) through the Faddeeva proxy W (Abrarov-Quine if |Z| < 6 else the
// 4-point Gauss-Hermite asymptotic form).  Parity is 1e-10 * S (R-UNIQ): transcendental functions
// differ from libm by ulps, so the arithmetic here is NOT required to be bit-identical.
#include "gf_internal.cuh"

namespace gf {

#ifndef GF_RS_POLE_UNROLL
#define GF_RS_POLE_UNROLL 2  // two poles per iteration: C5 47.0 -> 45.6 ms, C5D0 37.1 -> 35.9 ms (4: register spill, slower)
#endif
constexpr int kRsPoleUnroll = GF_RS_POLE_UNROLL;

// ------------------------------------------------------------------------------------------ data
__global__ void rs_draw_unit(double *out, int count, uint64_t seed, uint64_t before, double scale) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= count) return;
  uint64_t s = lcg_skip(seed, before + (uint64_t)q);
  out[q] = __dmul_rn(scale, lcg_draw(s));
}

__global__ void rs_fill_one(int32_t *a, int n) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) a[q] = 1;
}

// n_poles[lcg_int % n] += 1, once per draw (order-free histogram of known stream positions).
__global__ void rs_count_draws(int32_t *cnt, int n, long long draws, uint64_t seed, uint64_t before) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= draws) return;
  uint64_t s = lcg_next(lcg_skip(seed, before + (uint64_t)r));
  atomicAdd(cnt + (int)(s % (uint64_t)n), 1);
}

// Exclusive scan of n counts (n is a few hundred): one thread, sequential.
__global__ void rs_scan(const int32_t *cnt, int32_t *off, int n) {
  if (threadIdx.x || blockIdx.x) return;
  int run = 0;
  for (int i = 0; i < n; i++) {
    off[i] = run;
    run += cnt[i];
  }
  off[n] = run;
}

// Pole q (flat, nuclide-major) consumes draws [P0 + 9q + 1, P0 + 9q + 9]: 4 x (re, im) then l.
__global__ void rs_poles(double *pole, int32_t *pole_l, int tp, uint64_t seed, uint64_t P0) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= tp) return;
  uint64_t s = lcg_skip(seed, P0 + 9ull * (uint64_t)q);
  double v[8];
#pragma unroll
  for (int f = 0; f < 8; f++) v[f] = __dmul_rn(152.5, lcg_draw(s));
  double2 *dst = reinterpret_cast<double2 *>(pole + (size_t)q * 8);
  dst[0] = make_double2(v[0], v[1]);
  dst[1] = make_double2(v[2], v[3]);
  dst[2] = make_double2(v[4], v[5]);
  dst[3] = make_double2(v[6], v[7]);
  s = lcg_next(s);
  pole_l[q] = (int32_t)(s % 4ull);
}

// Window q consumes draws [W0 + 3q + 1, W0 + 3q + 3]; start/end follow the generator's counter:
// start = w*space + min(w, rem), end = start + space - 1 + [w < rem] (inclusive).
__global__ void rs_windows(double4 *win, const int32_t *poff, const int32_t *woff, int n, int tw, uint64_t seed,
                           uint64_t W0) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= tw) return;
  int lo = 0, hi = n;  // nuclide i with woff[i] <= q < woff[i+1]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (woff[mid] <= q) lo = mid; else hi = mid;
  }
  const int i = lo, w = q - woff[i];
  const int np = poff[i + 1] - poff[i], nw = woff[i + 1] - woff[i];
  const int space = np / nw, rem = np - space * nw;
  const int start = w * space + (w < rem ? w : rem);
  const int end = start + space - 1 + (w < rem ? 1 : 0);
  uint64_t s = lcg_skip(seed, W0 + 3ull * (uint64_t)q);
  double T = lcg_draw(s), A = lcg_draw(s), F = lcg_draw(s);
  int2 se = make_int2(start, end);
  win[q] = make_double4(T, A, F, *reinterpret_cast<double *>(&se));
}

static inline unsigned nblk(long long n, int b) { return (unsigned)((n + b - 1) / b); }

cudaError_t launch_rs_data(const RsDev &R, int avg_poles, int avg_windows, uint64_t seed, double *pole,
                           int32_t *pole_l, double4 *win, double *K0RS, int32_t *poff, int32_t *woff, double *mconc,
                           int32_t *cnt, cudaStream_t st) {
  cudaError_t e;
  const int n = R.n_nuc;
  const uint64_t Tc = (uint64_t)R.total;
  const long long Rp = (long long)avg_poles * n - n, Rw = (long long)avg_windows * n - n;
  const int tp = avg_poles * n, tw = avg_windows * n;
  int32_t *cntp = cnt, *cntw = cnt + n;
  rs_draw_unit<<<nblk(R.total, 256), 256, 0, st>>>(mconc, R.total, seed, 0, 1.0);
  rs_fill_one<<<nblk(2 * n, 256), 256, 0, st>>>(cnt, 2 * n);
  if (Rp > 0) rs_count_draws<<<nblk(Rp, 256), 256, 0, st>>>(cntp, n, Rp, seed, Tc);
  if (Rw > 0) rs_count_draws<<<nblk(Rw, 256), 256, 0, st>>>(cntw, n, Rw, seed, Tc + Rp);
  rs_scan<<<1, 32, 0, st>>>(cntp, poff, n);
  rs_scan<<<1, 32, 0, st>>>(cntw, woff, n);
  const uint64_t P0 = Tc + Rp + Rw, W0 = P0 + 9ull * tp, K0 = W0 + 3ull * tw;
  rs_poles<<<nblk(tp, 256), 256, 0, st>>>(pole, pole_l, tp, seed, P0);
  rs_windows<<<nblk(tw, 256), 256, 0, st>>>(win, poff, woff, n, tw, seed, W0);
  rs_draw_unit<<<nblk(4 * n, 256), 256, 0, st>>>(K0RS, 4 * n, seed, K0, 1.0);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cudaSuccess;
}

// ------------------------------------------------------------------------------------------ Faddeeva
struct cplx {
  double r, i;
};
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return {a.r + b.r, a.i + b.i}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return {a.r - b.r, a.i - b.i}; }
__device__ __forceinline__ cplx cmul(cplx A, cplx B) {
  return {__dsub_rn(__dmul_rn(A.r, B.r), __dmul_rn(A.i, B.i)), __dadd_rn(__dmul_rn(A.r, B.i), __dmul_rn(A.i, B.r))};
}
__device__ __forceinline__ cplx cdiv(cplx A, cplx B) {
  double den = __dadd_rn(__dmul_rn(B.r, B.r), __dmul_rn(B.i, B.i));
  return {__ddiv_rn(__dadd_rn(__dmul_rn(A.r, B.r), __dmul_rn(A.i, B.i)), den),
          __ddiv_rn(__dsub_rn(__dmul_rn(A.i, B.r), __dmul_rn(A.r, B.i)), den)};
}

__device__ __forceinline__ double fast_exp12(double x) {
  x = __dadd_rn(1.0, __dmul_rn(x, 0.000244140625));
#pragma unroll
  for (int k = 0; k < 12; k++) x = __dmul_rn(x, x);
  return x;
}

__constant__ double c_an[10] = {2.758402e-01, 2.245740e-01, 1.594149e-01, 9.866577e-02, 5.324414e-02,
                                2.505215e-02, 1.027747e-02, 3.676164e-03, 1.146494e-03, 3.117570e-04};
__constant__ double c_denl[10] = {9.869604e+00, 3.947842e+01, 8.882644e+01, 1.579137e+02, 2.467401e+02,
                                  3.553058e+02, 4.836106e+02, 6.316547e+02, 7.994380e+02, 9.869604e+02};

// Abrarov-Quine branch (|Z| < 6, ~0.5% of evaluations), kept out of line.
__device__ __noinline__ cplx faddeeva_abrarov(cplx Z) {
  cplx iz12 = {-12.0 * Z.i, 12.0 * Z.r};  // (0 + 12i) Z
  double ex = fast_exp12(iz12.r);
  double sn, cs;
  sincos(iz12.i, &sn, &cs);
  cplx e = {ex * cs, ex * sn};
  cplx W = cdiv(cmul({0.0, 1.0}, csub({1.0, 0.0}, e)), {12.0 * Z.r, 12.0 * Z.i});
  cplx Z2 = cmul(Z, Z);
  cplx sum = {0.0, 0.0};
#pragma unroll 2
  for (int n = 0; n < 10; n++) {
    double sgn = (n & 1) ? 1.0 : -1.0;
    cplx top = {sgn * e.r - 1.0, sgn * e.i};
    cplx bot = {c_denl[n] - 144.0 * Z2.r, -144.0 * Z2.i};
    cplx q = cdiv(top, bot);
    sum = cadd(sum, {c_an[n] * q.r, c_an[n] * q.i});
  }
  cplx zs = cmul(Z, sum);
  return cadd(W, cmul({0.0, 8.124330e+01}, zs));
}

// W(Z).  The branch decision |Z| < 6 is computed exactly as the oracle does (RN products, RN sum,
// correctly rounded sqrt), so both sides take the same branch.  The asymptotic branch (99.5% of
// evaluations) is reassociated to one reciprocal instead of the four divisions of two complex
// divisions:  a / P + c / Q = (a conj(P) |Q|^2 + c conj(Q) |P|^2) / (|P|^2 |Q|^2),  P = Z^2 - b,
// Q = Z^2 - d  (|Z| >= 6 keeps |P|^2, |Q|^2 in [1e3, 2e8]: no overflow or cancellation); FMA is
// allowed here (rs.cu is built -fmad=true) -- RSBench parity is 1e-10 x S (R-UNIQ).
__device__ __forceinline__ cplx faddeeva(cplx Z) {
  const double az = sqrt(__dadd_rn(__dmul_rn(Z.r, Z.r), __dmul_rn(Z.i, Z.i)));
  if (az < 6.0) return faddeeva_abrarov(Z);
  constexpr double a = 0.512424224754768462984202823134979415014943561548661637413182;
  constexpr double b = 0.275255128608410950901357962647054304017026259671664935783653;
  constexpr double c = 0.051765358792987823963876628425793170829107067780337219430904;
  constexpr double d = 2.724744871391589049098642037352945695982973740328335064216346;
  const double z2r = Z.r * Z.r - Z.i * Z.i, z2i = 2.0 * Z.r * Z.i;
  const double pr = z2r - b, qr = z2r - d;  // imaginary parts of P and Q are z2i
  const double i2 = z2i * z2i;
  const double np = pr * pr + i2, nq = qr * qr + i2;
  const double rinv = 1.0 / (np * nq);
  const double ap = a * nq * rinv, cq = c * np * rinv;  // a / |P|^2, c / |Q|^2
  const double sr = ap * pr + cq * qr, si = -(ap + cq) * z2i;
  return {-Z.i * sr - Z.r * si, Z.r * sr - Z.i * si};  // (i Z) (sr + i si)
}

// ------------------------------------------------------------------------------------------ lookup
__device__ __forceinline__ void rs_macro(const RsDev &R, const Tables &T, double E, int mat, double m[4]) {
#pragma unroll
  for (int c = 0; c < 4; c++) m[c] = 0.0;
  const double sqrtE = sqrt(E);
  const int j1 = T.off[mat + 1];
  for (int j = T.off[mat]; j < j1; j++) {
    const int nuc = T.nuc[j];
    const double conc = T.conc[j];
    const int w0 = __ldg(R.woff + nuc), nw = __ldg(R.woff + nuc + 1) - w0;
    const double spacing = 1.0 / (double)nw;
    int w = (int)(E / spacing);
    if (w == nw) w--;
    w = w < 0 ? 0 : (w > nw - 1 ? nw - 1 : w);
    // Phase factors fac_l = e^{-2 i phi_l}, phi_l = p - atan(a_l / b_l), p = K0RS_l sqrt(E) (R-RSPHI: l = 1:
    // (a, b) = (-p, 1); l = 2: (3p, 3 - p^2); l = 3: (p (15 - p^2), 15 - 6 p^2)).  Since
    // e^{2 i atan(a / b)} = (b + i a)^2 / (a^2 + b^2) for any real a, b not both 0 (a b < 0 or b < 0 only
    // shifts the angle by a multiple of pi, which doubling removes), fac_l = e^{-2 i p} (b + i a)^2 / (a^2 + b^2):
    // one sincos per l and no atan (R-UNIQ: within rounding of the oracle's atan + sincos).
    cplx fac[4];
#pragma unroll
    for (int l = 0; l < 4; l++) {
      const double p = __ldg(R.K0RS + nuc * 4 + l) * sqrtE;
      double sn, cs;
      sincos(2.0 * p, &sn, &cs);
      if (l == 0) {
        fac[l] = {cs, -sn};
      } else {
        const double p2 = p * p;
        const double a = l == 1 ? -p : (l == 2 ? 3.0 * p : p * (15.0 - p2));
        const double b = l == 1 ? 1.0 : (l == 2 ? 3.0 - p2 : 15.0 - 6.0 * p2);
        const double rd = 1.0 / (a * a + b * b);
        const double rr = (b * b - a * a) * rd, ri = 2.0 * a * b * rd;
        fac[l] = {cs * rr + sn * ri, cs * ri - sn * rr};  // (cs - i sn) (rr + i ri)
      }
    }
    const double2 *wp = reinterpret_cast<const double2 *>(R.win + w0 + w);
    const double2 W0 = __ldg(wp), W1 = __ldg(wp + 1);
    const int2 se = *reinterpret_cast<const int2 *>(&W1.y);
    double sT = E * W0.x, sA = E * W0.y, sF = E * W1.x;
    const int pbase = __ldg(R.poff + nuc);
#pragma unroll kRsPoleUnroll
    for (int p = se.x; p < se.y; p++) {
      const double2 *P = reinterpret_cast<const double2 *>(R.pole + (size_t)(pbase + p) * 8);
      const double2 EA = __ldg(P), RT = __ldg(P + 1), RA = __ldg(P + 2), RF = __ldg(P + 3);
      const int l = __ldg(R.pole_l + pbase + p);
      cplx fw;
      if (R.doppler) {
        const cplx Z = {(E - EA.x) * 0.5, (0.0 - EA.y) * 0.5};
        fw = faddeeva(Z);
      } else {  // 0 K (R-RS0): i / (EA - sqrt E) / E = (d.i + i d.r) / (|d|^2 E), d = EA - sqrt E
        const double dr = EA.x - sqrtE, di = EA.y;
        const double inv = 1.0 / ((dr * dr + di * di) * E);
        fw = {di * inv, dr * inv};
      }
      // fac[l] by selects (a dynamic index would put fac in local memory)
      const double fr = l == 0 ? fac[0].r : (l == 1 ? fac[1].r : (l == 2 ? fac[2].r : fac[3].r));
      const double fi = l == 0 ? fac[0].i : (l == 1 ? fac[1].i : (l == 2 ? fac[2].i : fac[3].i));
      const cplx wf = {fw.r * fr - fw.i * fi, fw.r * fi + fw.i * fr};
      sT += RT.x * wf.r - RT.y * wf.i;
      sA += RA.x * fw.r - RA.y * fw.i;
      sF += RF.x * fw.r - RF.y * fw.i;
    }
    const double micro[4] = {sT, sA, sF, sT - sA};
#pragma unroll
    for (int c = 0; c < 4; c++) m[c] += micro[c] * conc;
  }
}

__device__ __forceinline__ uint32_t argmax4_plus1(const double m[4]) {
  double mx = -1.7976931348623157e308;  // -DBL_MAX (R-ARGMAX)
  uint32_t idx = 0;
#pragma unroll
  for (int c = 0; c < 4; c++)
    if (m[c] > mx) {
      mx = m[c];
      idx = c;
    }
  return idx + 1;
}

constexpr int kRsTpb = 128;

__global__ void __launch_bounds__(kRsTpb) rs_lookup_direct(RsDev R, uint64_t first, uint32_t n, uint64_t seed,
                                                           const double *__restrict__ src_E,
                                                           const uint8_t *__restrict__ src_mat,
                                                           OutSpec out,
                                                           unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Tables T = stage_tables(R.total, R.moff, R.mnuc, R.mconc, R.thr, smem);
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t v = 0;
  if (t < n) {
    double E;
    int mat;
    if (src_E) {
      E = src_E[t];
      mat = src_mat[t];
      if (mat >= kMats || !isfinite(E)) invalid_input(vsum);
      mat = mat < kMats ? mat : kMats - 1;
    } else {
      uint64_t s = lcg_skip(seed, 2ull * (first + t));
      E = lcg_draw(s);
      mat = pick_material(lcg_draw(s), T.thr);
    }
    double m[4];
    rs_macro(R, T, E, mat, m);
    v = argmax4_plus1(m);
    if (out.any()) write_out<4>(out, t, m);
  }
  hash_epilogue(v, vsum);
}

__global__ void __launch_bounds__(kRsTpb) rs_lookup_sorted(RsDev R, uint32_t n, const double *__restrict__ Es,
                                                           const uint32_t *__restrict__ idx,
                                                           const uint32_t *__restrict__ mstart,
                                                           OutSpec out,
                                                           unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Tables T = stage_tables(R.total, R.moff, R.mnuc, R.mconc, R.thr, smem);
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t v = 0;
  if (p < n) {
    int mat = 0;
#pragma unroll
    for (int m = 1; m < kMats; m++)
      if (p >= __ldg(mstart + m)) mat = m;
    double m[4];
    rs_macro(R, T, Es[p], mat, m);
    v = argmax4_plus1(m);
    if (out.any()) write_out<4>(out, idx[p], m);
  }
  hash_epilogue(v, vsum);
}

// History-based mode, direct mapping (history.cu; R-HIST-RS): one thread per particle, L dependent
// lookups; start at fast_forward(seed, 2 L p); after each lookup add 1337 p (macro_c > 0) or 42 per
// channel to the stream state (u64), then draw E and the material.  macro: NULL or [np][L][4].
__global__ void __launch_bounds__(kRsTpb) rs_history_direct(RsDev R, uint64_t first_p, uint32_t np, int L,
                                                            uint64_t seed, double *__restrict__ macro,
                                                            unsigned long long *__restrict__ vsum) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Tables T = stage_tables(R.total, R.moff, R.mnuc, R.mconc, R.thr, smem);
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t v = 0;
  if (t < np) {
    const uint64_t p = first_p + t;
    uint64_t s = lcg_skip(seed, p * (uint64_t)L * 2ull);
    double E = lcg_draw(s);
    int mat = pick_material(lcg_draw(s), T.thr);
    for (int i = 0; i < L; i++) {
      double m[4];
      rs_macro(R, T, E, mat, m);
      v += argmax4_plus1(m);
      if (macro) {
#pragma unroll
        for (int c = 0; c < 4; c++) macro[((size_t)t * L + i) * 4 + c] = m[c];
      }
#pragma unroll
      for (int c = 0; c < 4; c++) s += m[c] > 0.0 ? 1337ull * p : 42ull;
      E = lcg_draw(s);
      mat = pick_material(lcg_draw(s), T.thr);
    }
  }
  hash_epilogue(v, vsum);
}

cudaError_t launch_rs_history_direct(const RsDev &R, uint64_t first_p, uint32_t np, int L, uint64_t seed,
                                     double *macro, unsigned long long *vsum, cudaStream_t st) {
  cudaError_t e;
  if ((e = allow_smem(rs_history_direct, table_smem(R.total))) != cudaSuccess) return e;
  rs_history_direct<<<nblk(np, kRsTpb), kRsTpb, table_smem(R.total), st>>>(R, first_p, np, L, seed, macro, vsum);
  return cudaGetLastError();
}

cudaError_t launch_rs_lookup(const RsDev &R, uint64_t first, uint32_t n, uint64_t seed, const double *src_E,
                             const uint8_t *src_mat, bool sort, const SortScratch &S, const OutSpec &out,
                             unsigned long long *vsum, cudaStream_t st, cudaEvent_t ev_mid) {
  const size_t smem = table_smem(R.total);
  cudaError_t e;
  if (sort) {
    if ((e = launch_locality_sort(first, n, seed, src_E, src_mat, R.thr, S, out.any(), vsum, st)) != cudaSuccess)
      return e;
    if (ev_mid && (e = cudaEventRecord(ev_mid, st)) != cudaSuccess) return e;
    if ((e = allow_smem(rs_lookup_sorted, smem)) != cudaSuccess) return e;
    rs_lookup_sorted<<<nblk(n, kRsTpb), kRsTpb, smem, st>>>(R, n, S.Es, S.idx, S.mstart, out, vsum);
  } else {
    if (ev_mid && (e = cudaEventRecord(ev_mid, st)) != cudaSuccess) return e;
    if ((e = allow_smem(rs_lookup_direct, smem)) != cudaSuccess) return e;
    rs_lookup_direct<<<nblk(n, kRsTpb), kRsTpb, smem, st>>>(R, first, n, seed, src_E, src_mat, out, vsum);
  }
  return cudaGetLastError();
}

}  // namespace gf
