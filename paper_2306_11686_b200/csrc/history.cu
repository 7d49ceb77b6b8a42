// history.cu -- NEXT-1: history-based mode on sm_100a.
//
// "event-based lookup and history-based lookup".  In history mode each particle runs
// L dependent lookups; the next (E, material) of a particle depends on its previous macro xs through
// the LCG stream (readings R-HIST for XSBench -- skip ahead #{c : macro_c > 1.0} draws -- and
// R-HIST-RS for RSBench -- add 1337 p or 42 per channel by the sign of macro_c).
//
// Two device mappings, identical results:
//   * direct (flags without GF_HIST_WAVES / GF_SORT_LOCALITY): one thread per particle runs its L
//     lookups back to back -- the mapping GPU First gets from the OpenMP particle loop.
//     Every lookup is a random gather with a dependent search in front of it.
//   * waves (default in bench): step i of all particles is one event-style batch.  hist_sample
//     advances every particle's stream by the feedback of its step i-1 and draws (E, mat); the
//     batch then goes through the event path -- locality sort (A2), search, interpolation, hash --
//     whose epilogue writes the feedback count of each particle (OutSpec::fb).  The dependency is
//     per particle, between waves, so sorting across particles inside a wave is legal and the sorted
//     kernels' record sharing applies.  State between waves: the particle's LCG state (8 B) and one
//     feedback byte.
#include "gf_internal.cuh"

namespace gf {

// Wave `wave` of particles [first_p, first_p + np): stream state after the feedback of the previous
// wave, then E = draw, mat = pick_mat(draw).  Wave 0 starts at fast_forward(seed, p * stride).
__global__ void __launch_bounds__(256) hist_sample(int bench, uint64_t first_p, uint32_t np, uint64_t seed,
                                                   uint64_t stride, int wave, const double *__restrict__ thr,
                                                   uint64_t *__restrict__ state, const uint8_t *__restrict__ fb,
                                                   double *__restrict__ Ep, uint8_t *__restrict__ matp) {
  __shared__ double sT[kMats];
  if (threadIdx.x < kMats) sT[threadIdx.x] = thr[threadIdx.x];
  __syncthreads();
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= np) return;
  const uint64_t p = first_p + t;
  uint64_t s;
  if (wave == 0) {
    s = lcg_skip(seed, p * stride);
  } else {
    s = state[t];
    const uint32_t k = fb[t];
    if (bench == GF_XSBENCH) {
      for (uint32_t i = 0; i < k; i++) s = lcg_next(s);  // fast_forward(s, n_forward), n_forward <= 5
    } else {
      s += (uint64_t)k * (1337ull * p) + (uint64_t)(4u - k) * 42ull;  // u64 wraparound (R-HIST-RS)
    }
  }
  const double E = lcg_draw(s);
  const int mat = pick_material(lcg_draw(s), sT);
  state[t] = s;
  Ep[t] = E;
  matp[t] = (uint8_t)mat;
}

cudaError_t launch_hist_sample(int bench, uint64_t first_p, uint32_t np, uint64_t seed, uint64_t stride, int wave,
                               const double *thr, uint64_t *state, const uint8_t *fb, double *Ep, uint8_t *matp,
                               cudaStream_t st) {
  hist_sample<<<(np + 255) / 256, 256, 0, st>>>(bench, first_p, np, seed, stride, wave, thr, state, fb, Ep, matp);
  return cudaGetLastError();
}

}  // namespace gf
