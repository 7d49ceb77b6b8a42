/* gf_pr.h -- C ABI of the page-rank propagation step (NEXT-4).
 *
 * GPU First also maps the timed parallel regions of HeCBench's page-rank to the GPU: "an
 * implementation of the page-rank algorithm for graphs in which the propagation step is measured"
 * (Fig. 9c).  The paper states no generator or formula; this library follows the
 * readings R-PR-GRAPH / R-PR-STEP of DESIGN.md Sec. 3:
 *   graph  N nodes; node u draws from the 63-bit LCG stream s = fast_forward(seed, 2 D u): out-degree
 *          d_u = 1 + floor(U * (2 D - 1)), then d_u targets v = floor(U * N) (U = lcg_double, v clamped
 *          to N - 1).  Stored as in-edge CSR by destination, each row ordered by (source u, draw j).
 *   step   contrib[u] = r[u] / d_u;  r'[v] = (1 - 0.85) / N + 0.85 * sum_{in-edges in row order}
 *          contrib[u]; fp64, every operation rounded to nearest, sums left to right.
 *
 * Conventions as in gf_xs.h: the caller owns all device memory (sizes from gf_pr_graph_bytes);
 * argument errors return GF_PR_E_INVAL synchronously with a message (gf_pr_last_error); work is
 * enqueued on `stream`; there is no CPU fallback.  All functions are noexcept.
 */
#ifndef GF_PR_H
#define GF_PR_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { GF_PR_OK = 0, GF_PR_E_INVAL = 1, GF_PR_E_NOMEM = 2, GF_PR_E_CUDA = 3 } gf_pr_status;
typedef struct CUstream_st *gf_pr_stream_t;
typedef struct gf_pr_graph gf_pr_graph; /* opaque; immutable after init */

/* Sizes of the caller-owned graph buffer (rowptr u32 [N+1], col u32 [nnz_max], outdeg i32 [N]) and
 * of the init scratch.  nnz_max = N (2D - 1) bounds the edge count.  1 <= N < 2^26, 1 <= D <= 32.
 * Host-only. */
gf_pr_status gf_pr_graph_bytes(int64_t n_nodes, int32_t avg_degree, size_t *graph_bytes, size_t *scratch_bytes);

/* Builds the graph on `device` (degrees and targets from the LCG, in-degree count, scan, fill,
 * per-row ordering) into graph_mem.  Synchronises `stream` once to learn the edge count. */
gf_pr_status gf_pr_graph_init(int64_t n_nodes, int32_t avg_degree, uint64_t seed, int device, void *graph_mem,
                              size_t graph_bytes, void *scratch, size_t scratch_bytes, gf_pr_stream_t stream,
                              gf_pr_graph **out);
gf_pr_status gf_pr_graph_free(gf_pr_graph *g);

/* *n_edges = nnz; device views of rowptr (u32 [N+1]), col (u32 [nnz]) and outdeg (i32 [N]); any may be NULL. */
gf_pr_status gf_pr_graph_info(const gf_pr_graph *g, int64_t *n_edges, const uint32_t **rowptr,
                              const uint32_t **col, const int32_t **outdeg);

/* One propagation step: d_out[v] = R-PR-STEP(d_in).  d_contrib: device fp64 scratch [N].  d_in and
 * d_out (device fp64 [N]) must not alias.  Enqueued on `stream`. */
gf_pr_status gf_pr_propagate(const gf_pr_graph *g, const double *d_in, double *d_out, double *d_contrib,
                             gf_pr_stream_t stream);

const char *gf_pr_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* GF_PR_H */
