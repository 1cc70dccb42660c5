/* Thin C shim over METIS_NodeND from the CUDA toolkit's libmetis_static.a.
 * Nested dissection is outside the reference; configs c2/c3
 * feed this permutation through SolverConfig.ordering (config.py:46-47,69-77). */
#include <stdint.h>
typedef int64_t idx_t;
extern int METIS_NodeND(idx_t *nvtxs, idx_t *xadj, idx_t *adjncy, idx_t *vwgt,
                        idx_t *options, idx_t *perm, idx_t *iperm);

/* perm[k] = original vertex at position k; iperm = inverse. Returns METIS status (1 = OK). */
int hy_metis_nodend(int64_t n, int64_t *xadj, int64_t *adjncy, int64_t *perm, int64_t *iperm) {
  idx_t nv = n;
  return METIS_NodeND(&nv, xadj, adjncy, 0, 0, perm, iperm);
}
