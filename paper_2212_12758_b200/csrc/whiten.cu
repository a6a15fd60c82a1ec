// Algorithm 2 with whitening (§5.1.3 l.395, conclusion
// l.457-458): build the truncated basis (Algorithm 2, fused sketch) while
// monitoring the sketch Theta V_i = Q_i R_i; the first time
// ||R_i||_1 ||R_i^{-1}||_1 > cond_max (l.395: 1000; reading R-5), whiten
//
//     V_i <- V_i R_i^{-1},   underline-H_{i-1} <- R_i underline-H_{i-1} R_{i-1}^{-1}
//
// and continue "as in Algorithm 1, using the same sketch matrix Theta" (l.106).
//
// Device work per Algorithm 2 step c (after K1 and K2 produce beta_{c-1}):
//   the sketch of column c-1 is reduced from K3's fused partials and
//   appended to an incremental QR (one CTA: Gram-Schmidt against Q, the new
//   column of R and of R^{-1}, running max column 1-norms -> cond_1 exactly).
// The host reads the trigger flag once per step (this path trades a host
// round trip per step for the data-dependent switch; the pure Algorithm 2
// and Algorithm 1 paths stay graph-captured).  The whitening itself is one
// in-place pass over V_i (k_whiten_cols, O(n i^2) flops, 2 x 8 n i bytes);
// column 0 keeps b (v~_1 = b / (||b|| R_11): only beta_0 changes).
#include <math.h>

#include "fab_internal.cuh"

namespace fab {

int enqueue_basis_prologue(fab_ctx* c, int m, bool fused, cudaStream_t st, int64_t* launches);
int enqueue_k1(fab_ctx* c, int col, int nw, double* z, bool need_z, cudaStream_t st, int64_t* launches,
               int* nparts, double* step_sums = nullptr);
int enqueue_scalar(fab_ctx* c, int col, int nw, int nparts, int final_step, cudaStream_t st, int64_t* launches);
int enqueue_k3(fab_ctx* c, int col, int nw, bool fused, cudaStream_t st, int64_t* launches, int nparts_k2,
               const double* sums);
int enqueue_col_sketch_reduce(fab_ctx* c, int col, double* p, cudaStream_t st, int64_t* launches);
int enqueue_sgs_column(fab_ctx* c, int col, int m, cudaStream_t st, int64_t* launches);

struct WhitenBufs {
  double *Q, *R, *Ri, *T1;   // Q: s x (m+1) (ld s); R, Ri, T1: (m+1) x (m+1) (ld m+1)
  int ldr;
};

static WhitenBufs whiten_bufs(fab_ctx* c) {
  WhitenBufs w;
  const size_t s = (size_t)(c->s_max > 0 ? c->s_max : 1), m1 = (size_t)c->m_max + 1;
  w.Q = c->wbuf;
  w.R = w.Q + s * m1;
  w.Ri = w.R + m1 * m1;
  w.T1 = w.Ri + m1 * m1;
  w.ldr = (int)m1;
  return w;
}

static size_t whiten_bytes(const fab_ctx* c) {
  const size_t s = (size_t)(c->s_max > 0 ? c->s_max : 1), m1 = (size_t)c->m_max + 1;
  return (s * m1 + 3 * m1 * m1) * sizeof(double);
}

__device__ double wsum1(double v, double* red) {
  double a[1] = {v}, o[1];
  block_sum<1>(a, red, o);
  __shared__ double bc;
  if (threadIdx.x == 0) bc = o[0];
  __syncthreads();
  return bc;
}

// Append column j of Theta V (p = Theta w_hat_j / beta_j) to Q R; update the
// column of R^{-1} and the running max column 1-norms (scratch[1], [2]);
// trigger when their product exceeds cond_max and j >= 1.
__global__ void k_wh_qr_step(int j, int s, const double* __restrict__ praw, const double* beta, double* Q,
                             double* R, double* Ri, int ldr, double cond_max, DevState* st) {
  __shared__ double red[kWarps];
  __shared__ double rr[kMaxM + 1];
  __shared__ double xs[kMaxM + 1];
  if (st->breakdown) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double bs = 1.0 / beta[j];
  // (the loops below issue their loads 8 at a time; every sum keeps its order)
  for (int l = warp; l < j; l += kWarps) {            // r_l = q_l^T p
    const double* ql = Q + (int64_t)l * s;
    double a = 0.0;
    for (int q0 = lane; q0 < s; q0 += 32 * 8) {
      double x[8], y[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = q0 + 32 * u;
        x[u] = q < s ? ql[q] : 0.0;
        y[u] = q < s ? praw[q] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (q0 + 32 * u < s) a = fma(x[u], y[u] * bs, a);
    }
    a = warp_sum(a);
    if (lane == 0) rr[l] = a;
  }
  __syncthreads();
  double a = 0.0;
  for (int q = threadIdx.x; q < s; q += blockDim.x) {
    double v = praw[q] * bs;
    for (int l0 = 0; l0 < j; l0 += 8) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = l0 + u < j ? Q[(int64_t)(l0 + u) * s + q] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (l0 + u < j) v = fma(-x[u], rr[l0 + u], v);
    }
    Q[(int64_t)j * s + q] = v;
    a = fma(v, v, a);
  }
  const double rjj = sqrt(wsum1(a, red));
  for (int q = threadIdx.x; q < s; q += blockDim.x) Q[(int64_t)j * s + q] /= rjj;
  if (threadIdx.x == 0) rr[j] = rjj;
  __syncthreads();
  for (int l = threadIdx.x; l <= j; l += blockDim.x) R[l + (int64_t)j * ldr] = rr[l];
  // new column of R^{-1}: x_j = 1/r_jj, x_l = -(1/r_jj) sum_{t=l}^{j-1} Ri[l,t] r_t
  for (int l = threadIdx.x; l < j; l += blockDim.x) {
    double acc = 0.0;
    for (int t0 = l; t0 < j; t0 += 8) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = t0 + u < j ? Ri[l + (int64_t)(t0 + u) * ldr] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (t0 + u < j) acc = fma(x[u], rr[t0 + u], acc);
    }
    xs[l] = -acc / rjj;
  }
  if (threadIdx.x == 0) xs[j] = 1.0 / rjj;
  __syncthreads();
  for (int l = threadIdx.x; l <= j; l += blockDim.x) Ri[l + (int64_t)j * ldr] = xs[l];
  double ar = 0.0, ai = 0.0;
  for (int l = threadIdx.x; l <= j; l += blockDim.x) {
    ar += fabs(rr[l]);
    ai += fabs(xs[l]);
  }
  const double nr = wsum1(ar, red);
  const double ni = wsum1(ai, red);
  if (threadIdx.x == 0) {
    if (j == 0) {
      st->scratch[1] = nr;
      st->scratch[2] = ni;
    } else {
      st->scratch[1] = fmax(st->scratch[1], nr);
      st->scratch[2] = fmax(st->scratch[2], ni);
    }
    st->scratch[3] = st->scratch[1] * st->scratch[2];   // cond_1(R_{j+1})
    st->scratch[4] = (j >= 1 && st->scratch[3] > cond_max) ? 1.0 : 0.0;
  }
}

// V_i <- V_i R_i^{-1} in place for columns 1..i-1 (column 0 keeps b):
// new column t = sum_{l <= t} (w_hat_l / beta_l) Ri[l, t].  A CTA stages 64
// rows x i columns in shared memory; thread (row, group) computes the columns
// t = group + 4 u of its row.  Launched with i * 64 * 8 bytes of dynamic smem.
__global__ void __launch_bounds__(256) k_whiten_cols(double* V, int64_t ld, int64_t n, int i, const double* Ri,
                                                     int ldr, const double* beta, int rows) {
  extern __shared__ double tile[];   // [i][rows]
  const int ngrp = blockDim.x / rows;
  const int row = threadIdx.x % rows, grp = threadIdx.x / rows;
  for (int64_t r0 = (int64_t)blockIdx.x * rows; r0 < n; r0 += (int64_t)gridDim.x * rows) {
    const int64_t r = r0 + row;
    for (int l = grp; l < i; l += ngrp) tile[l * rows + row] = r < n ? V[(int64_t)l * ld + r] / beta[l] : 0.0;
    __syncthreads();
    if (r < n) {
      for (int t = 1 + grp; t < i; t += ngrp) {
        double acc = 0.0;
        for (int l = 0; l <= t; ++l) acc = fma(tile[l * rows + row], Ri[l + (int64_t)t * ldr], acc);
        V[(int64_t)t * ld + r] = acc;
      }
    }
    __syncthreads();
  }
}

// underline-H_{i-1} <- R_i underline-H_{i-1} R_{i-1}^{-1} (i x (i-1)); beta_0 <-
// beta_0 R_00 (= gamma, V^+ b = gamma e_1), beta_j <- 1; SV[:, :i] <- Q_i
__global__ void k_wh_finish(int i, int s, double* H, int ldH, const double* R, const double* Ri, int ldr,
                            double* T1, const double* Q, double* SV, double* beta, int m_max, DevState* st) {
  // T1 = H Ri_{i-1}
  for (int e = threadIdx.x; e < i * (i - 1); e += blockDim.x) {
    const int a = e % i, b = e / i;
    double acc = 0.0;
    for (int t = 0; t <= b; ++t) acc = fma(H[a + (int64_t)t * ldH], Ri[t + (int64_t)b * ldr], acc);
    T1[a + (int64_t)b * ldr] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < i * (i - 1); e += blockDim.x) {
    const int a = e % i, b = e / i;
    double acc = 0.0;
    for (int t = a; t < i; ++t) acc = fma(R[a + (int64_t)t * ldr], T1[t + (int64_t)b * ldr], acc);
    H[a + (int64_t)b * ldH] = acc;
  }
  for (int64_t e = threadIdx.x; e < (int64_t)s * i; e += blockDim.x) SV[e] = Q[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    beta[0] *= R[0];
    st->gamma = beta[0];
  }
  for (int j = 1 + threadIdx.x; j <= m_max + 1; j += blockDim.x) beta[j] = 1.0;
}

__global__ void k_wh_reset(DevState* st) {
  st->scratch[1] = st->scratch[2] = st->scratch[3] = st->scratch[4] = 0.0;
  st->lsqr_done = 0;
}

int run_basis_whiten(fab_ctx* c, int m, int k, double cond_max, int* whitened_at, double* cond_at) {
  *whitened_at = 0;
  *cond_at = 0.0;
  if (!c->wbuf) {
    if (cudaMalloc(&c->wbuf, whiten_bytes(c)) != cudaSuccess) {
      cudaGetLastError();
      return FAB_ENOMEM;
    }
  }
  WhitenBufs wb = whiten_bufs(c);
  cudaStream_t st = c->stream;
  int64_t launches = 0;
  double* praw = svec(c, 20);
  FAB_TRY(enqueue_basis_prologue(c, m, true, st, &launches));
  k_wh_reset<<<1, 1, 0, st>>>(c->st_d);
  FAB_CHECK_LAUNCH();
  ++launches;
  int iw = 0;
  for (int col = 1; col <= m; ++col) {
    const int nw = col < k ? col : k;
    int nparts = 0;
    FAB_TRY(enqueue_k1(c, col, nw, c->vec, false, st, &launches, &nparts));
    FAB_TRY(enqueue_scalar(c, col, nw, nparts, 0, st, &launches));          // beta_{col-1}
    FAB_TRY(enqueue_col_sketch_reduce(c, col - 1, praw, st, &launches));    // Theta w_hat_{col-1} (K3 partials)
    k_wh_qr_step<<<1, kThreads, 0, st>>>(col - 1, c->s, praw, c->beta, wb.Q, wb.R, wb.Ri, wb.ldr, cond_max,
                                         c->st_d);
    FAB_CHECK_LAUNCH();
    ++launches;
    if (col - 1 >= 1) {
      FAB_CUDA(cudaMemcpyAsync(c->st_h, c->st_d, sizeof(DevState), cudaMemcpyDeviceToHost, st));
      FAB_CUDA(cudaStreamSynchronize(st));
      if (c->st_h->breakdown) break;
      if (c->st_h->scratch[4] != 0.0) {
        iw = col;                       // V_i = columns 0 .. col-1
        *cond_at = c->st_h->scratch[3];
        break;
      }
    }
    FAB_TRY(enqueue_k3(c, col, nw, true, st, &launches, 0, nullptr));
  }
  if (iw == 0) {
    // no trigger: the plain Algorithm 2 basis (final lagged norm, Theta V)
    FAB_TRY(enqueue_scalar(c, m + 1, 0, 0, 1, st, &launches));
    FAB_TRY(sketch_finalize(c, m + 1, st));
    ++launches;
  } else {
    int rows = 64;
    while (rows > 8 && (size_t)iw * rows * sizeof(double) > 200 * 1024) rows /= 2;
    const size_t smem = (size_t)iw * rows * sizeof(double);
    FAB_CUDA(set_max_dyn_smem((const void*)k_whiten_cols, (int)smem));
    const int64_t blocks = (c->n + rows - 1) / rows;
    const int grid = (int)(blocks < 4 * c->num_sms ? blocks : 4 * c->num_sms);
    k_whiten_cols<<<grid, 256, smem, st>>>(c->V, c->ld, c->n, iw, wb.Ri, wb.ldr, c->beta, rows);
    FAB_CHECK_LAUNCH();
    k_wh_finish<<<1, kThreads, 0, st>>>(iw, c->s, c->H, c->ldH, wb.R, wb.Ri, wb.ldr, wb.T1, wb.Q, c->SV, c->beta,
                                        c->m_max, c->st_d);
    FAB_CHECK_LAUNCH();
    launches += 2;
    for (int col = iw; col <= m; ++col) FAB_TRY(enqueue_sgs_column(c, col, m, st, &launches));
    *whitened_at = iw;
  }
  c->info.launches_basis = launches;
  return FAB_OK;
}

}  // namespace fab
