// Full Arnoldi (Eq. (2)), the method the paper compares
// against ("Arnoldi", l.72, l.358, Table 1 l.262-264): an orthonormal basis by
// classical Gram-Schmidt with one reorthogonalisation (CGS2).  Per step
// (0-based column c):
//
//   K1     w = A w_hat_{c-1}                              (stored in V[:, c])
//   pass 1 w <- w / beta_{c-1};  g = V_c^T w             (K6 tall GEMV, 1 pass)
//   pass 2 w <- w - V_c h1;      g = V_c^T w  (h2)       (1 pass)
//   pass 3 w <- w - V_c h2;      ||w||^2                 (1 pass)
//   K_{.,c-1} = h1 + h2,  K_{c,c-1} = ||w||  (stored unnormalised, beta_c = ||w||)
//
// i.e. three streaming passes over V_c per step against Algorithm 1's one
// (l.72: "up to twice as fast"; here 3x the GEMV bytes because of the
// reorthogonalisation a stable fp64 Arnoldi needs).  Breakdown as G-5.
// fab_compress(FAB_NONE) then gives FOM, Eq. (4).
#include <math.h>

#include "fab_internal.cuh"

namespace fab {

int launch_tall_gemv(fab_ctx* c, int ncols, const double* p, double scal, int use_state_scal,
                     const double* t_old, double* t_new, cudaStream_t st, int* nparts_out);
int launch_pass_reduce(fab_ctx* c, int nparts, int ncols, double* out, cudaStream_t st);
int enqueue_k1(fab_ctx* c, int col, int nw, double* z, bool need_z, cudaStream_t st, int64_t* launches,
               int* nparts, double* step_sums = nullptr);

__global__ void k_arn_reset(DevState* st, int m) {
  st->breakdown = 0;
  st->m_eff = m;
  st->err = 0;
  st->lsqr_done = 0;
  st->scal = -1.0;   // pass 0: t = b
}

// after pass 0 (t = b): beta_0 = ||b|| = gamma_b
__global__ void k_arn_first(const double* red, int m, double* beta, DevState* st) {
  for (int j = 1 + threadIdx.x; j <= m + 1; j += blockDim.x) beta[j] = 1.0;
  if (threadIdx.x == 0) {
    const double b0 = sqrt(red[1]);
    beta[0] = b0;
    st->gamma = b0;
    st->scal = -1.0 / b0;          // pass 1 of step 1: t = A b / ||b|| = A v_1
    if (!(b0 > 0.0)) {
      st->breakdown = 1;
      st->m_eff = 0;
      st->lsqr_done = 1;
    }
  }
}

// phase 1: h1 = g (coefficients of the normalised v_j: g_j / beta_j);
// phase 2: h2, K(:, c-1) = h1 + h2.  Next pass: t <- t - V h (pvec = -h_j/beta_j).
__global__ void k_arn_coef(int c, int phase, const double* red, const double* beta, double* H, int ldH,
                           double* pvec, double* h1, DevState* st) {
  if (st->breakdown) return;
  for (int j = threadIdx.x; j < c; j += blockDim.x) {
    const double h = red[j] / beta[j];
    if (phase == 1) {
      h1[j] = h;
    } else {
      H[j + (int64_t)(c - 1) * ldH] = h1[j] + h;
    }
    pvec[j] = -h / beta[j];
  }
  if (threadIdx.x == 0) st->scal = -1.0;
}

// after pass 3: K_{c,c-1} = beta_c = ||w||; breakdown test (G-5)
__global__ void k_arn_norm(int c, const double* red, double* beta, double* H, int ldH, int final_step,
                           DevState* st) {
  if (st->breakdown || threadIdx.x != 0) return;
  const double nrm = sqrt(red[c]);
  beta[c] = nrm;
  H[c + (int64_t)(c - 1) * ldH] = nrm;
  if (!(nrm > st->thresh)) {
    st->breakdown = 1;
    st->m_eff = c;
    st->lsqr_done = 1;
  } else {
    if (final_step) st->m_eff = c;
    st->scal = -1.0 / nrm;         // pass 1 of the next step: t = A w_hat_c / beta_c
  }
}

static int enqueue_arnoldi_all(fab_ctx* c, int m, cudaStream_t st, int64_t* launches) {
  double* pvec = svec(c, 22);
  double* h1 = svec(c, 21);
  double* red = c->red;
  int G = 0;
  k_arn_reset<<<1, 1, 0, st>>>(c->st_d, m);
  ++*launches;
  FAB_CUDA(cudaMemsetAsync(c->H, 0, (size_t)c->ldH * m * sizeof(double), st));
  FAB_CUDA(cudaMemsetAsync(pvec, 0, sizeof(double) * kSmall, st));
  // pass 0 over [b]: ||b||^2 (t = b into the scratch vector)
  FAB_TRY(launch_tall_gemv(c, 1, pvec, 0.0, 1, c->V, c->vec, st, &G));
  FAB_TRY(launch_pass_reduce(c, G, 1, red, st));
  k_arn_first<<<1, kThreads, 0, st>>>(red, c->m_max, c->beta, c->st_d);
  *launches += 3;
  for (int col = 1; col <= m; ++col) {
    double* w = c->V + (int64_t)col * c->ld;
    int nparts = 0;
    FAB_TRY(enqueue_k1(c, col, 1, w, true, st, launches, &nparts));
    for (int phase = 1; phase <= 3; ++phase) {
      if (phase == 1) FAB_CUDA(cudaMemsetAsync(pvec, 0, sizeof(double) * col, st));   // pass 1: t = w / beta_{c-1}
      FAB_TRY(launch_tall_gemv(c, col, pvec, 0.0, 1, w, w, st, &G));
      FAB_TRY(launch_pass_reduce(c, G, col, red, st));
      *launches += 2;
      if (phase < 3)
        k_arn_coef<<<1, kThreads, 0, st>>>(col, phase, red, c->beta, c->H, c->ldH, pvec, h1, c->st_d);
      else
        k_arn_norm<<<1, 32, 0, st>>>(col, red, c->beta, c->H, c->ldH, col == m ? 1 : 0, c->st_d);
      ++*launches;
    }
  }
  return FAB_OK;
}

int run_basis_arnoldi(fab_ctx* c, int m) {
  if (!comm_graphable(c)) {   // loopback ranks: eager
    int64_t launches = 0;
    FAB_TRY(enqueue_arnoldi_all(c, m, c->stream, &launches));
    c->info.launches_basis = launches;
    return FAB_OK;
  }
  if (!(c->gexec_arn && c->g_arn_m == m)) {
    if (c->gexec_arn) {
      cudaGraphExecDestroy(c->gexec_arn);
      c->gexec_arn = nullptr;
    }
    int64_t launches = 0;
    cudaStream_t st = c->cap;
    FAB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_arnoldi_all(c, m, st, &launches);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(st, &graph);
    if (rc != FAB_OK) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    FAB_CUDA(e);
    FAB_CUDA(cudaGraphInstantiate(&c->gexec_arn, graph, 0));
    cudaGraphDestroy(graph);
    c->g_arn_m = m;
    c->g_arn_launches = launches;
  }
  FAB_CUDA(cudaGraphLaunch(c->gexec_arn, c->stream));
  c->info.launches_basis = c->g_arn_launches;
  return FAB_OK;
}

}  // namespace fab
