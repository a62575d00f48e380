// Dense SPD solve of the real-time tracking step (Eq. qp_rto):
// (Hs + tau I) d = -g with Hs = (H + H^T)/2 (DESIGN.md R-T1), by a blocked
// right-looking Cholesky factorization on the fp64 tensor cores in one
// cooperative launch, the forward substitution folded into it (the right-hand
// side rides as an extra bordered row), and a flag-chained backward
// substitution.  Host side of dense.cu; the C-ABI wrapper is in redhess.cu.
#pragma once

#include <cuda_runtime.h>

namespace rh {

struct DenseWs {
  double *A = nullptr;       // [nt 32][nt 32] row-major, lower tiles: the bordered matrix, then L
  double *Linv = nullptr;    // [nt][32][32] inverses of the diagonal tiles of L
  double *dbuf = nullptr;    // [nt 32] solution (padding entries 0)
  int *flags = nullptr;      // [cap] diagonal tile ready (== epoch)
  int *flags_d = nullptr;    // [cap] solution block ready (== epoch)
  int *fail = nullptr;       // [2]: [0] first non-positive pivot + 1 (0 = none), [1] ticket counter
  unsigned *bar = nullptr;   // grid barrier words
  int cap = 0;               // tiles per dimension the buffers hold
  int epoch = 0;
  int coop_per_sm = 0, nsm = 0;
};

// size the workspace for an n x n system (idempotent; grows only)
cudaError_t dense_ws_ensure(DenseWs &w, int n, int device);
void dense_ws_free(DenseWs &w);
// enqueue one factorization attempt with shift tau and the substitution;
// on success (no pivot <= 0) p[0..n) += alpha d when p != nullptr.
// Read w.fail[0] after the stream completes: 0 = success.
cudaError_t dense_spd_attempt(DenseWs &w, int n, const double *H, long long ldh, const double *g, double tau,
                              double *p, double alpha, cudaStream_t st, int *launches);

}  // namespace rh
