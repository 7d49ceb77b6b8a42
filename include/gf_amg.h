/* gf_amg.h -- C ABI of the AMGmk relax kernel (NEXT-4).
 *
 * GPU First maps "only the relax kernel of the original AMGmk proxy application" to the GPU
 * (Fig. 9c).  The paper states no matrix or sweep; readings R-AMG-MAT /
 * R-AMG-RELAX:
 *   matrix  the 27-point Laplacian on an nx x ny x nz grid (row i = x + nx (y + ny z)), CSR with the
 *           diagonal 26 first and the existing neighbours (-1) after it in increasing column order;
 *   relax   one Jacobi sweep u'[i] = (f[i] - sum_{jj > first} a[jj] u[col[jj]]) / a[first], fp64
 *           round to nearest, the row sum left to right starting from f[i].
 * Caller-owned device memory, synchronous argument checks (gf_amg_last_error), work enqueued on
 * `stream`; no CPU fallback.  All functions are noexcept.
 */
#ifndef GF_AMG_H
#define GF_AMG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { GF_AMG_OK = 0, GF_AMG_E_INVAL = 1, GF_AMG_E_NOMEM = 2, GF_AMG_E_CUDA = 3 } gf_amg_status;
typedef struct CUstream_st *gf_amg_stream_t;
typedef struct gf_amg_matrix gf_amg_matrix;

/* Bytes of the caller-owned matrix buffer (rowptr u32 [n+1], col u32 [nnz], val f64 [nnz]) and the
 * nonzero count.  1 <= nx, ny, nz and n = nx ny nz < 2^27.  Host-only. */
gf_amg_status gf_amg_matrix_bytes(int32_t nx, int32_t ny, int32_t nz, size_t *bytes, int64_t *nnz);

/* Builds the matrix on `device` into mem (each row written independently from its closed-form offset). */
gf_amg_status gf_amg_matrix_init(int32_t nx, int32_t ny, int32_t nz, int device, void *mem, size_t bytes,
                                 gf_amg_stream_t stream, gf_amg_matrix **out);
gf_amg_status gf_amg_matrix_free(gf_amg_matrix *A);

/* Device views (any may be NULL): rowptr u32 [n+1], col u32 [nnz], val f64 [nnz]; *n and *nnz. */
gf_amg_status gf_amg_matrix_info(const gf_amg_matrix *A, int64_t *n, int64_t *nnz, const uint32_t **rowptr,
                                 const uint32_t **col, const double **val);

/* One Jacobi relaxation sweep: d_out = R-AMG-RELAX(d_f, d_u); device fp64 [n] each, d_out must not
 * alias d_u.  Enqueued on `stream`. */
gf_amg_status gf_amg_relax(const gf_amg_matrix *A, const double *d_f, const double *d_u, double *d_out,
                           gf_amg_stream_t stream);

const char *gf_amg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* GF_AMG_H */
