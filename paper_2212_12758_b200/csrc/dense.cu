// Small dense linear algebra on the device (m <= 1024, s <= 768):
//
//   dense_qr_sketch   Householder QR of Theta V_m (s x m) with R_ii >= 0 and
//                     Q^T (Theta v_{m+1}) -- the Blendenpik preconditioner
//                      and the sketch-and-solve factor
//                     (Remark 2, l.249-251).  Cooperative kernel, one warp per
//                     trailing column, one grid barrier per reflector.
//   dense_tri_inverse R^{-1} by back substitution, one CTA per column.
//   dense_fe1         c = f(alpha C_m + sigma I) e_1 (l.195, l.207, l.226):
//                     exp: [13/13] Pade with scaling and squaring;
//                     sqrt / invsqrt: scaled product-form Denman-Beavers
//                     iteration (X -> sqrt, Z -> inverse sqrt), determinant
//                     scaling from log|det| of Gauss-Jordan pivots;
//                     poly: Horner-free Krylov sum p_0 e_1 + p_1 X e_1 + ...
//   The paper uses MATLAB expm / sqrtm (l.356); these are the device
//   counterparts (reading G-19).
#include <cooperative_groups.h>
#include <math.h>

#include "fab_internal.cuh"

namespace cg = cooperative_groups;

namespace fab {

// ---------------------------------------------------------------------------
// Householder QR (cooperative).  A: rows x ncols_total, lda = rows.  Factors
// the first nf columns; later columns are only transformed.  diag[j] = R_jj.
// ---------------------------------------------------------------------------
constexpr int kQrNQ = 24;   // rows <= 768

__global__ void __launch_bounds__(kThreads)
k_qr_coop(double* A, int rows, int nf, int ntot, double* diag) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int tw = (gridDim.x * blockDim.x) >> 5;
  for (int j = 0; j < nf; ++j) {
    const double* colj = A + (int64_t)j * rows;
    double x[kQrNQ];
    double sig = 0.0;
#pragma unroll
    for (int q = 0; q < kQrNQ; ++q) {
      const int i = lane + 32 * q;
      x[q] = (i > j && i < rows) ? colj[i] : 0.0;
      sig = fma(x[q], x[q], sig);
    }
    sig = warp_sum(sig);
    const double x0 = colj[j];
    double beta, mu, v0;
    if (sig == 0.0) {
      beta = (x0 >= 0.0) ? 0.0 : 2.0;
      mu = fabs(x0);
      v0 = 1.0;
    } else {
      mu = sqrt(x0 * x0 + sig);
      v0 = (x0 <= 0.0) ? (x0 - mu) : (-sig / (x0 + mu));
      beta = 2.0 * v0 * v0 / (sig + v0 * v0);
    }
    const double iv0 = 1.0 / v0;
    if (beta != 0.0) {
      for (int jj = j + 1 + gw; jj < ntot; jj += tw) {
        double* col = A + (int64_t)jj * rows;
        double w = 0.0;
#pragma unroll
        for (int q = 0; q < kQrNQ; ++q) {
          const int i = lane + 32 * q;
          if (i > j && i < rows) w = fma(x[q] * iv0, col[i], w);
        }
        const double cj = col[j];
        w = warp_sum(w) + cj;
        const double bw = beta * w;
        __syncwarp();
        if (lane == 0) col[j] = cj - bw;
#pragma unroll
        for (int q = 0; q < kQrNQ; ++q) {
          const int i = lane + 32 * q;
          if (i > j && i < rows) col[i] = fma(-bw, x[q] * iv0, col[i]);
        }
      }
    }
    if (gw == 0 && lane == 0) diag[j] = mu;
    grid.sync();
  }
}

__global__ void k_qr_extract(const double* A, int rows, int m, const double* diag, double* R, double* qtb) {
  const int64_t total = (int64_t)m * m;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % m), col = (int)(i / m);
    R[i] = (r < col) ? A[r + (int64_t)col * rows] : (r == col ? diag[r] : 0.0);
  }
  if (qtb)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
      qtb[i] = A[i + (int64_t)m * rows];
}

static int coop_grid(fab_ctx* c, const void* fn, int want) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, 0);
  if (occ < 1) occ = 1;
  int mx = occ * c->num_sms;
  if (want > mx) want = mx;
  if (want < 1) want = 1;
  return want;
}

double* qr_work(fab_ctx* c);   // abi.cu

// QR of the rows x ntot matrix already in the QR work area (lda = rows):
// R of its first m columns; qtb = Q^T column m when ntot > m (else NULL).
int dense_qr_work(fab_ctx* c, int m, int rows, int ntot, double* R, double* qtb, cudaStream_t st) {
  if (rows > 32 * kQrNQ) return FAB_EINVAL;
  double* A = qr_work(c);
  double* diag = svec(c, 10);
  int nf = m;
  void* args[] = {&A, &rows, &nf, &ntot, &diag};
  const int grid = coop_grid(c, (const void*)k_qr_coop, (ntot + kWarps - 1) / kWarps);
  FAB_CUDA(cudaLaunchCooperativeKernel((const void*)k_qr_coop, grid, kThreads, args, 0, st));
  ++c->nlaunch;
  k_qr_extract<<<(m * m + kThreads - 1) / kThreads, kThreads, 0, st>>>(A, rows, m, diag, R, ntot > m ? qtb : nullptr);
  FAB_CHECK_LAUNCH();
  return FAB_OK;
}

int dense_qr_sketch(fab_ctx* c, int m, double* R, double* qtb, cudaStream_t st) {
  const int s = c->s;
  if (s > 32 * kQrNQ) return FAB_EINVAL;
  FAB_CUDA(cudaMemcpyAsync(qr_work(c), c->SV, (size_t)s * (m + 1) * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return dense_qr_work(c, m, s, m + 1, R, qtb, st);
}

// ---------------------------------------------------------------------------
// R^{-1} for upper triangular R (column-major m x m): CTA j solves R x = e_j
// by column-oriented back substitution (x_i = 0 for i > j).
// ---------------------------------------------------------------------------
// Column l of R (and its diagonal) is loaded one step ahead, so a step waits
// on shared memory and barriers only, not on an L2 round trip (m <= 1024:
// 8 rows per thread at kTriThreads = 128).  Same operations in the same order.
constexpr int kTriThreads = 128;
__global__ void __launch_bounds__(kTriThreads) k_tri_inverse(const double* R, int m, double* Rinv) {
  extern __shared__ double b[];
  constexpr int kPer = (kMaxM + kTriThreads - 1) / kTriThreads;
  const int j = blockIdx.x;
  for (int i = threadIdx.x; i < m; i += kTriThreads) b[i] = (i == j) ? 1.0 : 0.0;
  double rc[kPer], rn[kPer], dg, dn = 0.0;
  auto load_col = [&](int l, double (&r)[kPer], double& d) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int i = threadIdx.x + kTriThreads * u;
      r[u] = (l >= 0 && i < l) ? R[i + (int64_t)l * m] : 0.0;
    }
    d = l >= 0 ? R[l + (int64_t)l * m] : 1.0;
  };
  load_col(j, rc, dg);
  __syncthreads();
  for (int l = j; l >= 0; --l) {
    load_col(l - 1, rn, dn);   // next column, in flight during this step
    const double xl = b[l] / dg;
    __syncthreads();
    if (threadIdx.x == 0) b[l] = xl;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int i = threadIdx.x + kTriThreads * u;
      if (i < l) b[i] = fma(-rc[u], xl, b[i]);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPer; ++u) rc[u] = rn[u];
    dg = dn;
  }
  for (int i = threadIdx.x; i < m; i += kTriThreads) Rinv[i + (int64_t)j * m] = (i <= j) ? b[i] : 0.0;
}

int dense_tri_inverse(fab_ctx* c, const double* R, int m, double* Rinv, cudaStream_t st) {
  k_tri_inverse<<<m, kTriThreads, m * sizeof(double), st>>>(R, m, Rinv);
  FAB_CHECK_LAUNCH();
  return FAB_OK;
}

// ---------------------------------------------------------------------------
// GEMM: D = alpha A B + beta C + gamma I   (m x m, column-major, ld = m).
// D may alias C (each output element is read once, then written, by one thread).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_gemm(int m, const double* __restrict__ A, const double* __restrict__ B, double alpha, double beta,
       const double* C, double gamma, double* D) {
  __shared__ double As[32][33];
  __shared__ double Bs[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int row0 = blockIdx.x * 32, col0 = blockIdx.y * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k0 = 0; k0 < m; k0 += 32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kk = ty + 8 * i;
      const int r = row0 + tx, kA = k0 + kk;
      As[kk][tx] = (r < m && kA < m) ? A[r + (int64_t)kA * m] : 0.0;
      const int kB = k0 + tx, cB = col0 + kk;
      Bs[tx][kk] = (kB < m && cB < m) ? B[kB + (int64_t)cB * m] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const double a = As[kk][tx];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = fma(a, Bs[kk][ty + 8 * i], acc[i]);
    }
    __syncthreads();
  }
  const int r = row0 + tx;
  if (r < m) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int col = col0 + ty + 8 * i;
      if (col < m) {
        const int64_t o = r + (int64_t)col * m;
        double v = alpha * acc[i];
        if (beta != 0.0) v = fma(beta, C[o], v);
        if (r == col) v += gamma;
        D[o] = v;
      }
    }
  }
}

static int gemm(fab_ctx* c, int m, const double* A, const double* B, double alpha, double beta,
                const double* C, double gamma, double* D, cudaStream_t st) {
  dim3 g((m + 31) / 32, (m + 31) / 32);
  k_gemm<<<g, 256, 0, st>>>(m, A, B, alpha, beta, C, gamma, D);
  FAB_CHECK_LAUNCH();
  return FAB_OK;
}

// D = a1 X1 + a2 X2 + a3 X3 + a0 I (null pointers skipped); D may alias any Xi
__global__ void k_lincomb(int m, double a1, const double* X1, double a2, const double* X2, double a3,
                          const double* X3, double a0, double* D) {
  const int64_t total = (int64_t)m * m;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % m), col = (int)(i / m);
    double v = (r == col) ? a0 : 0.0;
    if (X1) v = fma(a1, X1[i], v);
    if (X2) v = fma(a2, X2[i], v);
    if (X3) v = fma(a3, X3[i], v);
    D[i] = v;
  }
}

static int lincomb(fab_ctx* c, int m, double a1, const double* X1, double a2, const double* X2, double a3,
                   const double* X3, double a0, double* D, cudaStream_t st) {
  const int64_t total = (int64_t)m * m;
  int g = (int)((total + kThreads - 1) / kThreads);
  if (g > 1024) g = 1024;
  k_lincomb<<<g, kThreads, 0, st>>>(m, a1, X1, a2, X2, a3, X3, a0, D);
  FAB_CHECK_LAUNCH();
  return FAB_OK;
}

// out[0] = ||X||_1 (max column abs sum), out[1] = ||X - I||_F, out[2] = any non-finite
// ||X||_1 (max column abs sum), ||X - I||_F and a non-finite flag.  One CTA
// of 1024 threads: warp w takes columns w, w+32, ... with the lanes over the
// rows (coalesced), per-column partials in shared memory, then thread 0
// reduces them in column order (deterministic).
constexpr int kStatsThreads = 1024;
__global__ void __launch_bounds__(kStatsThreads) k_mat_stats(const double* X, int m, double* out) {
  __shared__ double cabs[kMaxM], cdev[kMaxM];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int b = 0;
  for (int col = warp; col < m; col += kStatsThreads / 32) {
    double a = 0.0, fs = 0.0;
    for (int r = lane; r < m; r += 32) {
      const double v = X[r + (int64_t)col * m];
      if (!isfinite(v)) b = 1;
      a += fabs(v);
      const double d = v - (r == col ? 1.0 : 0.0);
      fs = fma(d, d, fs);
    }
    a = warp_sum(a);
    fs = warp_sum(fs);
    if (lane == 0) {
      cabs[col] = a;
      cdev[col] = fs;
    }
  }
  if (b) bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    double M = 0.0, S = 0.0;
    for (int col = 0; col < m; ++col) {
      M = fmax(M, cabs[col]);
      S += cdev[col];
    }
    out[0] = M;
    out[1] = sqrt(S);
    out[2] = bad ? 1.0 : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Gauss-Jordan with partial pivoting (cooperative): solves A X = B in place
// (B <- X), A destroyed.  One warp per column of [A(:, k+1:) | B]; one grid
// barrier per pivot.  out[0] = sum log|pivot| (log|det A|), out[1] = 1 if a
// zero pivot was met.
// ---------------------------------------------------------------------------
constexpr int kGjNQ = kMaxM / 32;

__global__ void __launch_bounds__(kThreads)
k_gj_coop(double* A, double* B, int m, int nrhs, double* out) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int tw = (gridDim.x * blockDim.x) >> 5;
  double logdet = 0.0;
  int singular = 0;
  const int nq = (m + 31) >> 5;
  for (int k = 0; k < m; ++k) {
    const double* colk = A + (int64_t)k * m;
    double cv[kGjNQ];
    double best = -1.0;
    int bi = m;
#pragma unroll
    for (int q = 0; q < kGjNQ; ++q) {
      const int i = lane + 32 * q;
      cv[q] = (q < nq && i < m) ? colk[i] : 0.0;
      if (q < nq && i >= k && i < m) {
        const double a = fabs(cv[q]);
        if (a > best) {
          best = a;
          bi = i;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    const int p = bi;
    const double piv = colk[p];
    const double ck = colk[k];
    if (!(best > 0.0)) singular = 1;
    logdet += log(fabs(piv));
    const double ipiv = 1.0 / piv;
    // columns k+1..m-1 of A, then all of B
    const int ncol = (m - k - 1) + nrhs;
    for (int t = gw; t < ncol; t += tw) {
      double* col = (t < m - k - 1) ? (A + (int64_t)(k + 1 + t) * m) : (B + (int64_t)(t - (m - k - 1)) * m);
      const double ap = col[p], ak = col[k];
      const double rr = ap * ipiv;   // new row k value
      __syncwarp();
#pragma unroll
      for (int q = 0; q < kGjNQ; ++q) {
        const int i = lane + 32 * q;
        if (q < nq && i < m) {
          double nv;
          if (i == k)
            nv = rr;
          else if (i == p)
            nv = fma(-ck, rr, ak);   // old row k moves to row p
          else
            nv = fma(-cv[q], rr, col[i]);
          col[i] = nv;
        }
      }
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = logdet;
    out[1] = singular ? 1.0 : 0.0;
  }
}

// Gauss-Jordan with partial pivoting on ONE thread-block cluster of kGjCl
// CTAs: the columns of [A | B] are dealt round-robin to the CTAs and live in
// their shared memory for the whole elimination (m <= ~330: 2m/8 columns of
// m doubles per CTA).  Pivot step k: the owner of column k searches the
// pivot and publishes the column in a double-buffered broadcast slot; ONE
// cluster barrier; every CTA reads it through distributed shared memory and
// updates its own columns.  No global-memory traffic and no grid-wide
// barrier inside the elimination (the cooperative k_gj_coop pays one grid
// sync and a global round trip per pivot).  Same arithmetic per element as
// k_gj_coop (swap rows k, p and eliminate), same tie rule for the pivot.
constexpr int kGjCl = 8;
constexpr int kGjClMaxM = 330;
constexpr int kGjRows = (kGjClMaxM + 31) / 32;   // rows per lane in the unrolled update
constexpr int kGjThreads = 512;                  // 16 warps per CTA: the update is issue-bound
constexpr int kGjWarps = kGjThreads / 32;

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void __launch_bounds__(kGjThreads, 1) k_gj_cluster(const double* __restrict__ A, double* B, int m,
                                                            int nrhs, double* out) {
  namespace cgx = cooperative_groups;
  cgx::cluster_group cl = cgx::this_cluster();
  extern __shared__ double sm[];
  const int q = (int)cl.block_rank();
  const int ntot = m + nrhs;
  const int nloc = (ntot - q + kGjCl - 1) / kGjCl;   // columns j = q + kGjCl * l
  const int nmax = (ntot + kGjCl - 1) / kGjCl;       // same layout in every CTA (DSMEM offsets)
  double* cols = sm;                                 // [nmax][m]
  double* bc = cols + (size_t)nmax * m;              // [2][m + 2]: column, then pivot index
  double* pc = bc + 2 * (m + 2);                     // local copy of the broadcast column
  __shared__ double red_log[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int l = 0; l < nloc; ++l) {
    const int j = q + kGjCl * l;
    const double* src = j < m ? A + (int64_t)j * m : B + (int64_t)(j - m) * m;
    for (int i = tid; i < m; i += blockDim.x) cols[(size_t)l * m + i] = src[i];
  }
  double logdet = 0.0;
  int singular = 0;
  __syncthreads();
  cluster_barrier();
  for (int k = 0; k < m; ++k) {
    const int owner = k % kGjCl, lk = k / kGjCl;
    double* slot = bc + (size_t)(k & 1) * (m + 2);
    if (q == owner && warp == 0) {
      const double* ck = cols + (size_t)lk * m;
      double best = -1.0;
      int bi = m;
      double av[kGjRows];
#pragma unroll
      for (int r = 0; r < kGjRows; ++r) {
        const int i = k + lane + 32 * r;
        av[r] = i < m ? fabs(ck[i]) : -1.0;
      }
#pragma unroll
      for (int r = 0; r < kGjRows; ++r) {   // ascending i per lane, as the strided loop
        if (av[r] > best) {
          best = av[r];
          bi = k + lane + 32 * r;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      for (int i = lane; i < m; i += 32) slot[i] = ck[i];
      if (lane == 0) slot[m] = (double)bi;
    }
    cluster_barrier();
    const double* rs = cl.map_shared_rank(slot, owner);
    for (int i = tid; i <= m; i += blockDim.x) pc[i] = rs[i];
    __syncthreads();
    const int p = (int)pc[m];
    const double piv = pc[p], ckk = pc[k];
    if (!(fabs(piv) > 0.0)) singular = 1;
    if (q == owner && tid == 0) logdet += log(fabs(piv));
    const double ipiv = 1.0 / piv;
    // columns j > k of A and every column of B (j >= m).  Each lane holds
    // rows lane + 32 r (r < kGjRows) of the pivot column in registers and
    // issues all its loads of a column before the FMAs (the row loop is
    // fully unrolled: shared-memory latency is paid once per column, not
    // once per row).  Same arithmetic per element as before.
    double pr[kGjRows];
#pragma unroll
    for (int r = 0; r < kGjRows; ++r) {
      const int i = lane + 32 * r;
      pr[r] = i < m ? pc[i] : 0.0;
    }
    for (int l = warp; l < nloc; l += kGjWarps) {
      const int j = q + kGjCl * l;
      if (j <= k) continue;
      double* col = cols + (size_t)l * m;
      const double ap = col[p], ak = col[k];
      const double rr = ap * ipiv;
      __syncwarp();
      double cv[kGjRows];
#pragma unroll
      for (int r = 0; r < kGjRows; ++r) {
        const int i = lane + 32 * r;
        cv[r] = i < m ? col[i] : 0.0;
      }
      // every row as a generic row (branch-free), then rows k and p rewritten
      // by their lanes: row k <- rr, row p <- a_kj - a_kk rr (the swap)
#pragma unroll
      for (int r = 0; r < kGjRows; ++r) {
        const int i = lane + 32 * r;
        if (i < m) col[i] = fma(-pr[r], rr, cv[r]);
      }
      __syncwarp();
      if (lane == (k & 31)) col[k] = rr;
      if (p != k && lane == (p & 31)) col[p] = fma(-ckk, rr, ak);
    }
    __syncthreads();
  }
  for (int l = 0; l < nloc; ++l) {
    const int j = q + kGjCl * l;
    if (j < m) continue;
    double* dst = B + (int64_t)(j - m) * m;
    for (int i = tid; i < m; i += blockDim.x) dst[i] = cols[(size_t)l * m + i];
  }
  // log|det| and the singular flag: per-CTA (owner) sums, reduced on rank 0
  if (tid == 0) {
    pc[0] = logdet;
    pc[1] = singular ? 1.0 : 0.0;
  }
  __syncthreads();
  cluster_barrier();
  if (q == 0 && tid == 0) {
    double lsum = 0.0, sg = 0.0;
    for (int r = 0; r < kGjCl; ++r) {
      const double* o = cl.map_shared_rank(pc, r);
      lsum += o[0];
      sg = fmax(sg, o[1]);
    }
    out[0] = lsum;
    out[1] = sg;
  }
  cluster_barrier();   // keep every CTA's shared memory alive until rank 0 has read it
  (void)red_log;
}

// In-place Gauss-Jordan inverse on one cluster (the Denman-Beavers M^{-1}):
// only the m columns of A are stored -- at pivot step k column k turns into
// column k of the running inverse (-c'/piv, 1/piv at row k) while every other
// column takes the usual elimination -- and the row interchanges are undone
// as a column permutation when the result is written.  Versus [A | I]: half
// the shared memory and 2/3 of the update work; rows are handled in pairs
// (double2 shared-memory accesses, column stride rounded up to even).  Same
// pivot rule as k_gj_cluster.
constexpr int kGjPairs = (kGjClMaxM + 63) / 64;   // row pairs per lane

__global__ void __launch_bounds__(kGjThreads, 1) k_gj_inv_cluster(const double* __restrict__ A, double* Ainv,
                                                                  int m, double* out) {
  namespace cgx = cooperative_groups;
  cgx::cluster_group cl = cgx::this_cluster();
  extern __shared__ __align__(16) double sm[];
  __shared__ int pk[kGjClMaxM];
  __shared__ int posof[kGjClMaxM];
  const int q = (int)cl.block_rank();
  const int mp = (m + 1) & ~1;
  const int nloc = (m - q + kGjCl - 1) / kGjCl;   // columns j = q + kGjCl * l
  const int nmax = (m + kGjCl - 1) / kGjCl;
  double* cols = sm;                              // [nmax][mp]
  double* bc = cols + (size_t)nmax * mp;          // [2][mp + 2]: column, then pivot index at [mp]
  double* pc = bc + 2 * (mp + 2);                 // local copy of the broadcast column
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int l = 0; l < nloc; ++l) {
    const int j = q + kGjCl * l;
    for (int i = tid; i < mp; i += blockDim.x) cols[(size_t)l * mp + i] = i < m ? A[(int64_t)j * m + i] : 0.0;
  }
  double logdet = 0.0;
  int singular = 0;
  // pivot search of column kk (rows >= kk, the first largest |a|) by one warp
  // of its owner, published with the pivot row in slot kk & 1
  auto search_publish = [&](int kk) {
    const double* ck = cols + (size_t)(kk / kGjCl) * mp;
    double* slot = bc + (size_t)(kk & 1) * (mp + 2);
    double best = -1.0;
    int bi = m;
    double av[kGjRows];
#pragma unroll
    for (int r = 0; r < kGjRows; ++r) {
      const int i = kk + lane + 32 * r;
      av[r] = i < m ? fabs(ck[i]) : -1.0;
    }
#pragma unroll
    for (int r = 0; r < kGjRows; ++r) {
      if (av[r] > best) {
        best = av[r];
        bi = kk + lane + 32 * r;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    const double2* c2 = reinterpret_cast<const double2*>(ck);
    double2* s2 = reinterpret_cast<double2*>(slot);
    for (int i = lane; i < mp / 2; i += 32) s2[i] = c2[i];
    if (lane == 0) slot[mp] = (double)bi;
  };
  __syncthreads();
  if (q == 0 && warp == 0) search_publish(0);
  cluster_barrier();
  for (int k = 0; k < m; ++k) {
    const int owner = k % kGjCl;
    const double* slot = bc + (size_t)(k & 1) * (mp + 2);
    {
      const double2* rs = reinterpret_cast<const double2*>(cl.map_shared_rank(slot, owner));
      double2* p2 = reinterpret_cast<double2*>(pc);
      for (int i = tid; i <= mp / 2; i += blockDim.x) p2[i] = rs[i];   // pair mp/2 holds the pivot index
    }
    __syncthreads();
    const int p = (int)pc[mp];
    const double piv = pc[p], ckk = pc[k];
    if (!(fabs(piv) > 0.0)) singular = 1;
    if (q == owner && tid == 0) logdet += log(fabs(piv));
    if (tid == 0) pk[k] = p;
    const double ipiv = 1.0 / piv;
    double2 pr[kGjPairs];
    const double2* p2 = reinterpret_cast<const double2*>(pc);
#pragma unroll
    for (int r = 0; r < kGjPairs; ++r) {
      const int i2 = lane + 32 * r;
      pr[r] = 2 * i2 < mp ? p2[i2] : make_double2(0.0, 0.0);
    }
    auto update_col = [&](int l) {
      const int j = q + kGjCl * l;
      double* col = cols + (size_t)l * mp;
      double2* c2 = reinterpret_cast<double2*>(col);
      if (j == k) {
        // the pivot column becomes column k of the inverse: -c'/piv, 1/piv at row k
#pragma unroll
        for (int r = 0; r < kGjPairs; ++r) {
          const int i2 = lane + 32 * r;
          if (2 * i2 < mp) c2[i2] = make_double2(-pr[r].x * ipiv, -pr[r].y * ipiv);
        }
        __syncwarp();
        if (lane == 0) {
          col[k] = ipiv;
          if (p != k) col[p] = -ckk * ipiv;
        }
      } else {
        const double ap = col[p], ak = col[k];
        const double rr = ap * ipiv;
        __syncwarp();
        double2 cv[kGjPairs];
#pragma unroll
        for (int r = 0; r < kGjPairs; ++r) {
          const int i2 = lane + 32 * r;
          cv[r] = 2 * i2 < mp ? c2[i2] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int r = 0; r < kGjPairs; ++r) {
          const int i2 = lane + 32 * r;
          if (2 * i2 < mp) c2[i2] = make_double2(fma(-pr[r].x, rr, cv[r].x), fma(-pr[r].y, rr, cv[r].y));
        }
        __syncwarp();
        if (lane == 0) {   // row k <- rr, row p <- a_kj - a_kk rr (the interchange)
          col[k] = rr;
          if (p != k) col[p] = fma(-ckk, rr, ak);
        }
      }
      __syncwarp();
    };
    // look-ahead: the owner of column k+1 updates it first (warp 0), searches
    // its pivot and publishes it into the other slot while the remaining
    // warps (and CTAs) update the other columns -- the search and the publish
    // leave the per-pivot critical path.  The other slot was last read at
    // step k-1, before the previous cluster barrier.
    const int nk = k + 1;
    if (nk < m && q == nk % kGjCl) {
      const int ln = nk / kGjCl;
      if (warp == 0) {
        update_col(ln);
        search_publish(nk);
      } else {
        for (int l = warp - 1; l < nloc; l += kGjWarps - 1)
          if (l != ln) update_col(l);
      }
    } else {
      for (int l = warp; l < nloc; l += kGjWarps) update_col(l);
    }
    __syncthreads();
    cluster_barrier();
  }
  // undo the row interchanges as column interchanges (in reverse order):
  // stored column s is column posof[s] of A^{-1}
  if (tid == 0) {
    int* colat = reinterpret_cast<int*>(pc);   // pc is free now
    for (int s2 = 0; s2 < m; ++s2) {
      posof[s2] = s2;
      colat[s2] = s2;
    }
    for (int k = m - 1; k >= 0; --k) {
      const int p = pk[k];
      if (p == k) continue;
      const int a = colat[k], b = colat[p];
      colat[k] = b;
      colat[p] = a;
      posof[a] = p;
      posof[b] = k;
    }
  }
  __syncthreads();
  for (int l = 0; l < nloc; ++l) {
    const int j = q + kGjCl * l;
    double* dst = Ainv + (int64_t)posof[j] * m;
    for (int i = tid; i < m; i += blockDim.x) dst[i] = cols[(size_t)l * mp + i];
  }
  __syncthreads();
  if (tid == 0) {
    bc[0] = logdet;
    bc[1] = singular ? 1.0 : 0.0;
  }
  __syncthreads();
  cluster_barrier();
  if (q == 0 && tid == 0) {
    double lsum = 0.0, sg = 0.0;
    for (int r = 0; r < kGjCl; ++r) {
      const double* o = cl.map_shared_rank(bc, r);
      lsum += o[0];
      sg = fmax(sg, o[1]);
    }
    out[0] = lsum;
    out[1] = sg;
  }
  cluster_barrier();
}

static size_t gj_inv_smem(int m) {
  const int mp = (m + 1) & ~1;
  const int nmax = (m + kGjCl - 1) / kGjCl;
  return ((size_t)nmax * mp + 3 * ((size_t)mp + 2)) * sizeof(double);
}

static size_t gj_cluster_smem(int m, int nrhs) {
  const int nloc = (m + nrhs + kGjCl - 1) / kGjCl;
  return ((size_t)nloc * m + 3 * ((size_t)m + 2)) * sizeof(double);
}

// solve A X = B; A is copied to a scratch so the input survives
static int gj_solve(fab_ctx* c, int m, const double* A, double* Awork, double* B, int nrhs, double* out,
                    cudaStream_t st) {
  const size_t smem = gj_cluster_smem(m, nrhs);
  if (m <= kGjClMaxM && smem <= 226 * 1024) {
    FAB_CUDA(ensure_dyn_smem((const void*)k_gj_cluster, 226 * 1024));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kGjCl, 1, 1);
    cfg.blockDim = dim3(kGjThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kGjCl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FAB_CUDA(cudaLaunchKernelEx(&cfg, k_gj_cluster, A, B, m, nrhs, out));
    ++c->nlaunch;
    return FAB_OK;
  }
  FAB_CUDA(cudaMemcpyAsync(Awork, A, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  int mm = m, nr = nrhs;
  void* args[] = {&Awork, &B, &mm, &nr, &out};
  const int grid = coop_grid(c, (const void*)k_gj_coop, (m + nrhs + kWarps - 1) / kWarps);
  FAB_CUDA(cudaLaunchCooperativeKernel((const void*)k_gj_coop, grid, kThreads, args, 0, st));
  ++c->nlaunch;
  return FAB_OK;
}

// A^{-1} (out[0] = log|det A|, out[1] = 1 if singular): the in-place cluster
// inverse when it fits, else the general solve against I
static int gj_inverse(fab_ctx* c, int m, const double* A, double* Awork, double* Ainv, double* out,
                      cudaStream_t st);

static int gj_inverse(fab_ctx* c, int m, const double* A, double* Awork, double* Ainv, double* out,
                      cudaStream_t st) {
  const size_t smem = gj_inv_smem(m);
  if (m > kGjClMaxM || smem > 226 * 1024) {
    FAB_TRY(lincomb(c, m, 0, nullptr, 0, nullptr, 0, nullptr, 1.0, Ainv, st));   // I
    return gj_solve(c, m, A, Awork, Ainv, m, out, st);
  }
  FAB_CUDA(ensure_dyn_smem((const void*)k_gj_inv_cluster, 226 * 1024));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kGjCl, 1, 1);
  cfg.blockDim = dim3(kGjThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kGjCl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FAB_CUDA(cudaLaunchKernelEx(&cfg, k_gj_inv_cluster, A, Ainv, m, out));
  ++c->nlaunch;
  return FAB_OK;
}

__global__ void k_gemv_e(const double* X, int m, const double* u, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int j = 0; j < m; ++j) a = fma(X[i + (int64_t)j * m], u[j], a);
    out[i] = a;
  }
}
__global__ void k_axpy_small(int m, double a, const double* x, double* y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) y[i] = fma(a, x[i], y[i]);
}
__global__ void k_unit(int m, double a, double* y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) y[i] = (i == 0) ? a : 0.0;
}

static int read_stats(fab_ctx* c, const double* X, int m, double* h, cudaStream_t st) {
  double* d = svec(c, 11);
  k_mat_stats<<<1, kStatsThreads, 0, st>>>(X, m, d);
  FAB_CHECK_LAUNCH();
  FAB_CUDA(cudaMemcpyAsync(h, d, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  FAB_CUDA(cudaStreamSynchronize(st));
  return FAB_OK;
}

// 1-norms of up to 4 matrices (one CTA each, fixed order)
struct Mats4 {
  const double* p[4];
};
__global__ void k_norm1_multi(Mats4 M, int m, double scale0, double* out) {
  __shared__ double smax[kThreads];
  const double* X = M.p[blockIdx.x];
  double mx = 0.0;
  for (int col = threadIdx.x; col < m; col += blockDim.x) {
    double a = 0.0;
    for (int r = 0; r < m; ++r) a += fabs(X[r + (int64_t)col * m]);
    mx = fmax(mx, a);
  }
  smax[threadIdx.x] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double M2 = 0.0;
    for (int t = 0; t < (int)blockDim.x; ++t) M2 = fmax(M2, smax[t]);
    out[blockIdx.x] = M2;
  }
}

// out = || |s X|^p ||_1 computed exactly as max_j (1^T |s X|^p)_j (row-vector
// powers; all entries are non-negative).  One CTA; warp per column.
__global__ void k_abs_power_norm(const double* X, int m, double s, int p, double* out) {
  __shared__ double v[kMaxM], w[kMaxM];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < m; i += blockDim.x) v[i] = 1.0;
  __syncthreads();
  for (int it = 0; it < p; ++it) {
    for (int j = warp; j < m; j += nw) {
      double a = 0.0;
      for (int i = lane; i < m; i += 32) a = fma(v[i], fabs(s * X[i + (int64_t)j * m]), a);
      a = warp_sum(a);
      if (lane == 0) w[j] = a;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) v[i] = w[i];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int i = 0; i < m; ++i) mx = fmax(mx, v[i]);
    out[0] = mx;
  }
}

// exp by the scaling and squaring algorithm of Al-Mohy & Higham (2009) --
// the algorithm of MATLAB's expm that the paper used -- with
// the [13/13] Pade approximant: s from eta_5 = min(max(d6, d8), max(d8, d10)),
// d_k = ||X^k||_1^{1/k} (exact norms of the powers, cheap on the device),
// theta_13 = 4.25, plus the ell(2^-s X, 13) correction that prevents
// overscaling of nonnormal matrices.
static int expm_e1(fab_ctx* c, int m, const double* X0, double* c_out, int* iters, cudaStream_t st) {
  static const double b[14] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                               1187353796428800.0,  129060195264000.0,   10559470521600.0,
                               670442572800.0,      33522128640.0,       1323241920.0,
                               40840800.0,          960960.0,            16380.0,
                               182.0,               1.0};
  double* X = dmat(c, 5);
  double* X2 = dmat(c, 6);
  double* X4 = dmat(c, 7);
  double* X6 = dmat(c, 8);
  double* T = dmat(c, 9);
  double* U = dmat(c, 10);
  double* Vp = dmat(c, 11);
  double* P = dmat(c, 12);
  double* W = dmat(c, 13);
  double h[3];
  FAB_TRY(read_stats(c, X0, m, h, st));
  if (h[2] != 0.0) return FAB_EDOMAIN;
  const double theta13 = 4.25;
  const double u = ldexp(1.0, -53);
  const double c27 = 8.829961602018678e-36;   // |c_27| = (13!)^2 / (26! 27!)
  int s = 0;
  if (h[0] > 0.0) {
    FAB_TRY(gemm(c, m, X0, X0, 1.0, 0.0, nullptr, 0.0, X2, st));
    FAB_TRY(gemm(c, m, X2, X2, 1.0, 0.0, nullptr, 0.0, X4, st));
    FAB_TRY(gemm(c, m, X4, X2, 1.0, 0.0, nullptr, 0.0, X6, st));
    FAB_TRY(gemm(c, m, X4, X4, 1.0, 0.0, nullptr, 0.0, T, st));    // X^8
    FAB_TRY(gemm(c, m, X4, X6, 1.0, 0.0, nullptr, 0.0, U, st));    // X^10
    double* nd = svec(c, 17);
    Mats4 M4{{X4, X6, T, U}};
    k_norm1_multi<<<4, kThreads, 0, st>>>(M4, m, 1.0, nd);
    FAB_CHECK_LAUNCH();
    double hn[4];
    FAB_CUDA(cudaMemcpyAsync(hn, nd, sizeof(hn), cudaMemcpyDeviceToHost, st));
    FAB_CUDA(cudaStreamSynchronize(st));
    const double d6 = pow(hn[1], 1.0 / 6), d8 = pow(hn[2], 1.0 / 8), d10 = pow(hn[3], 1.0 / 10);
    double eta5 = fmin(fmax(d6, d8), fmax(d8, d10));
    if (!isfinite(eta5)) eta5 = h[0];            // powers overflowed: fall back to ||X||_1
    if (eta5 > 0.0) s = (int)ceil(log2(eta5 / theta13));
    if (s < 0) s = 0;
    // ell(2^-s X, 13)
    const double sc = ldexp(1.0, -s);
    k_abs_power_norm<<<1, kThreads, 0, st>>>(X0, m, sc, 27, nd);
    FAB_CHECK_LAUNCH();
    double pn;
    FAB_CUDA(cudaMemcpyAsync(&pn, nd, sizeof(double), cudaMemcpyDeviceToHost, st));
    FAB_CUDA(cudaStreamSynchronize(st));
    if (pn > 0.0 && isfinite(pn)) {
      const double alpha = c27 * pn / (h[0] * sc);
      const int ell = (int)ceil(log2(alpha / u) / 26.0);
      if (ell > 0) s += ell;
    }
  }
  const double sc = ldexp(1.0, -s);
  FAB_TRY(lincomb(c, m, sc, X0, 0, nullptr, 0, nullptr, 0.0, X, st));
  FAB_TRY(gemm(c, m, X, X, 1.0, 0.0, nullptr, 0.0, X2, st));
  FAB_TRY(gemm(c, m, X2, X2, 1.0, 0.0, nullptr, 0.0, X4, st));
  FAB_TRY(gemm(c, m, X4, X2, 1.0, 0.0, nullptr, 0.0, X6, st));
  // U = X [X6 (b13 X6 + b11 X4 + b9 X2) + b7 X6 + b5 X4 + b3 X2 + b1 I]
  FAB_TRY(lincomb(c, m, b[13], X6, b[11], X4, b[9], X2, 0.0, T, st));
  FAB_TRY(gemm(c, m, X6, T, 1.0, 0.0, nullptr, 0.0, W, st));
  FAB_TRY(lincomb(c, m, 1.0, W, b[7], X6, b[5], X4, b[1], T, st));
  FAB_TRY(lincomb(c, m, 1.0, T, b[3], X2, 0, nullptr, 0.0, T, st));
  FAB_TRY(gemm(c, m, X, T, 1.0, 0.0, nullptr, 0.0, U, st));
  // V = X6 (b12 X6 + b10 X4 + b8 X2) + b6 X6 + b4 X4 + b2 X2 + b0 I
  FAB_TRY(lincomb(c, m, b[12], X6, b[10], X4, b[8], X2, 0.0, T, st));
  FAB_TRY(gemm(c, m, X6, T, 1.0, 0.0, nullptr, 0.0, W, st));
  FAB_TRY(lincomb(c, m, 1.0, W, b[6], X6, b[4], X4, b[0], Vp, st));
  FAB_TRY(lincomb(c, m, 1.0, Vp, b[2], X2, 0, nullptr, 0.0, Vp, st));
  // (V - U) R = (V + U)
  FAB_TRY(lincomb(c, m, 1.0, Vp, -1.0, U, 0, nullptr, 0.0, P, st));
  FAB_TRY(lincomb(c, m, 1.0, Vp, 1.0, U, 0, nullptr, 0.0, T, st));
  double* gout = svec(c, 12);
  FAB_TRY(gj_solve(c, m, P, W, T, m, gout, st));
  double gh[2];
  FAB_CUDA(cudaMemcpyAsync(gh, gout, sizeof(gh), cudaMemcpyDeviceToHost, st));
  FAB_CUDA(cudaStreamSynchronize(st));
  if (gh[1] != 0.0 || !isfinite(gh[0])) return FAB_ESINGULAR;
  // square s times (the last squaring only needs the first column)
  double* cur = T;
  double* nxt = X2;
  *iters = s;
  for (int i = 0; i < s; ++i) {
    if (i == s - 1) {
      k_gemv_e<<<(m + 127) / 128, 128, 0, st>>>(cur, m, cur, c_out);   // cur * cur[:,0]
      FAB_CHECK_LAUNCH();
      return FAB_OK;
    }
    FAB_TRY(gemm(c, m, cur, cur, 1.0, 0.0, nullptr, 0.0, nxt, st));
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  FAB_CUDA(cudaMemcpyAsync(c_out, cur, m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return FAB_OK;
}

// sqrt / inverse sqrt by the scaled product-form Denman-Beavers iteration:
//   M_0 = X, Y_0 = X, Z_0 = I
//   mu_k = |det M_k|^{-1/(2m)}  (while ||M_k - I||_F > 1e-2, else 1)
//   Y_{k+1} = mu/2 Y_k (I + mu^-2 M_k^-1),  Z_{k+1} = mu/2 Z_k (I + mu^-2 M_k^-1)
//   M_{k+1} = 1/2 I + mu^2/4 M_k + mu^-2/4 M_k^-1
// Y -> X^{1/2}, Z -> X^{-1/2}, M -> I.
// Coupled Newton-Schulz iteration for the principal square root (Higham,
// Functions of Matrices, 2008, eq. (6.35)): with A' = X / ||X||_1,
//   Y_0 = A', Z_0 = I,  T_k = (3I - Z_k Y_k)/2,  Y_{k+1} = Y_k T_k,  Z_{k+1} = T_k Z_k
// Y_k -> A'^{1/2}, Z_k -> A'^{-1/2} quadratically when ||I - A'|| < 1 --
// three m x m GEMMs per step and no inverse, where Denman-Beavers needs a
// Gauss-Jordan inverse (a 2-us-per-pivot chain on the cluster) every step.
// Convergence is monitored as ||T_k - I||_F; a step that doubles its smallest
// value so far, a non-finite value or 60 steps mean the matrix is outside the basin
// (eigenvalues far from the positive real interval, e.g. c4-like or a
// negative eigenvalue): *ok = false and the caller runs Denman-Beavers,
// which also reports EDOMAIN.  Same principal root, different rounding.
static int ns_e1(fab_ctx* c, int m, const double* X0, int want_inv, double* c_out, int* iters, cudaStream_t st,
                 bool* ok) {
  *ok = false;
  double* Y = dmat(c, 6);
  double* Z = dmat(c, 7);
  double* T = dmat(c, 10);
  double* Y2 = dmat(c, 11);
  double* Z2 = dmat(c, 12);
  double h[3];
  FAB_TRY(read_stats(c, X0, m, h, st));
  if (h[2] != 0.0 || !(h[0] > 0.0) || !isfinite(h[0])) return FAB_OK;
  const double sc = h[0];
  FAB_TRY(lincomb(c, m, 1.0 / sc, X0, 0, nullptr, 0, nullptr, 0.0, Y, st));   // Y_0 = X / ||X||_1
  FAB_TRY(lincomb(c, m, 0, nullptr, 0, nullptr, 0, nullptr, 1.0, Z, st));      // Z_0 = I
  bool extra = false;
  double emin = INFINITY;
  for (int it = 0; it < 60; ++it) {
    FAB_TRY(gemm(c, m, Z, Y, -0.5, 0.0, nullptr, 1.5, T, st));                // T = (3I - Z Y) / 2
    FAB_TRY(read_stats(c, T, m, h, st));
    const double e = h[1];                                                    // ||T - I||_F
    if (h[2] != 0.0 || !isfinite(e) || e > 2.0 * emin) return FAB_OK;         // outside the basin
    emin = fmin(emin, e);
    FAB_TRY(gemm(c, m, Y, T, 1.0, 0.0, nullptr, 0.0, Y2, st));
    FAB_TRY(gemm(c, m, T, Z, 1.0, 0.0, nullptr, 0.0, Z2, st));
    double* t = Y;
    Y = Y2;
    Y2 = t;
    t = Z;
    Z = Z2;
    Z2 = t;
    *iters = it + 1;
    if (extra) break;
    if (e <= 1e-13 * sqrt((double)m)) extra = true;   // one more step after convergence
  }
  if (!extra) return FAB_OK;
  // c = f(X) e_1: sqrt(X) = sqrt(sc) Y, X^{-1/2} = Z / sqrt(sc)
  const int g = (m + 127) / 128;
  k_unit<<<g, 128, 0, st>>>(m, 0.0, c_out);
  k_axpy_small<<<g, 128, 0, st>>>(m, want_inv ? 1.0 / sqrt(sc) : sqrt(sc), want_inv ? Z : Y, c_out);
  FAB_CHECK_LAUNCH();
  *ok = true;
  return FAB_OK;
}

static int db_e1(fab_ctx* c, int m, const double* X0, int want_inv, double* c_out, int* iters,
                 cudaStream_t st) {
  double* M = dmat(c, 5);
  double* Y = dmat(c, 6);
  double* Z = dmat(c, 7);
  double* Mi = dmat(c, 8);
  double* Wk = dmat(c, 9);
  double* T = dmat(c, 10);
  double* Y2 = dmat(c, 11);
  double* Z2 = dmat(c, 12);
  double* gout = svec(c, 12);
  FAB_CUDA(cudaMemcpyAsync(M, X0, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  FAB_CUDA(cudaMemcpyAsync(Y, X0, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  FAB_TRY(lincomb(c, m, 0, nullptr, 0, nullptr, 0, nullptr, 1.0, Z, st));
  double h[3];
  FAB_TRY(read_stats(c, M, m, h, st));
  if (h[2] != 0.0) return FAB_EDOMAIN;
  double err = h[1];
  bool extra_done = false;
  const int maxit = 100;
  for (int it = 0; it < maxit; ++it) {
    FAB_TRY(gj_inverse(c, m, M, Wk, Mi, gout, st));
    double gh[2];
    FAB_CUDA(cudaMemcpyAsync(gh, gout, sizeof(gh), cudaMemcpyDeviceToHost, st));
    FAB_CUDA(cudaStreamSynchronize(st));
    if (gh[1] != 0.0 || !isfinite(gh[0])) return FAB_EDOMAIN;
    double mu = 1.0;
    if (err > 1e-2) mu = exp(-gh[0] / (2.0 * m));
    const double imu2 = 1.0 / (mu * mu);
    FAB_TRY(lincomb(c, m, imu2, Mi, 0, nullptr, 0, nullptr, 1.0, T, st));   // I + mu^-2 M^-1
    // only the wanted factor is carried (the iteration itself runs on M)
    double* t;
    if (want_inv) {
      FAB_TRY(gemm(c, m, Z, T, 0.5 * mu, 0.0, nullptr, 0.0, Z2, st));
      t = Z; Z = Z2; Z2 = t;
    } else {
      FAB_TRY(gemm(c, m, Y, T, 0.5 * mu, 0.0, nullptr, 0.0, Y2, st));
      t = Y; Y = Y2; Y2 = t;
    }
    FAB_TRY(lincomb(c, m, 0.25 * mu * mu, M, 0.25 * imu2, Mi, 0, nullptr, 0.5, M, st));
    FAB_TRY(read_stats(c, M, m, h, st));
    if (h[2] != 0.0) return FAB_EDOMAIN;
    err = h[1];
    *iters = it + 1;
    if (extra_done) break;
    if (err <= 1e-12 * sqrt((double)m)) extra_done = true;   // one more step after convergence
  }
  if (!extra_done) return FAB_ENOCONV;
  FAB_CUDA(cudaMemcpyAsync(c_out, want_inv ? Z : Y, m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return FAB_OK;
}

static int poly_e1(fab_ctx* c, int m, const double* X, double* c_out, cudaStream_t st) {
  double* u = svec(c, 13);
  double* u2 = svec(c, 14);
  const int g = (m + 127) / 128;
  k_unit<<<g, 128, 0, st>>>(m, 1.0, u);
  k_unit<<<g, 128, 0, st>>>(m, c->npoly > 0 ? c->poly[0] : 0.0, c_out);
  for (int i = 1; i < c->npoly; ++i) {
    k_gemv_e<<<g, 128, 0, st>>>(X, m, u, u2);
    k_axpy_small<<<g, 128, 0, st>>>(m, c->poly[i], u2, c_out);
    double* t = u;
    u = u2;
    u2 = t;
  }
  FAB_CHECK_LAUNCH();
  return FAB_OK;
}

int dense_fe1(fab_ctx* c, int f, double alpha, double sigma, double* c_out, int* iters) {
  const int m = c->m_eff;
  cudaStream_t st = c->stream;
  const double* C = dmat(c, 0);
  double* X = dmat(c, 4);
  *iters = 0;
  FAB_TRY(lincomb(c, m, alpha, C, 0, nullptr, 0, nullptr, sigma, X, st));   // alpha C + sigma I
  switch (f) {
    case FAB_EXP:
      return expm_e1(c, m, X, c_out, iters, st);
    case FAB_SQRT:
    case FAB_INVSQRT: {
      const int inv = (f == FAB_INVSQRT) ? 1 : 0;
      const char* e = getenv("FAB_DENSE_DB");   // "1": Denman-Beavers only (A/B)
      if (!(e && e[0] == '1')) {
        bool ok = false;
        FAB_TRY(ns_e1(c, m, X, inv, c_out, iters, st, &ok));
        if (ok) return FAB_OK;
      }
      *iters = 0;
      return db_e1(c, m, X, inv, c_out, iters, st);
    }
    case FAB_POLY:
      return poly_e1(c, m, X, c_out, st);
    default:
      return FAB_EINVAL;
  }
}

}  // namespace fab
