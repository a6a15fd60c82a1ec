// Blendenpik-LSQR evaluated through the Gram matrix of the basis
// (fab_compress mode FAB_BLENDENPIK_GRAM; a B200-specific alternative to the
// per-iteration passes of lsqr.cu, not in the paper).
//
// LSQR on M = V_m R^{-1} with right-hand side c = v_{m+1} (PAPER.md l.174-184,
// Eq. (7)) touches the n-dimensional vectors only through M p, M^T u and
// norms.  Every u of the Golub-Kahan recurrence lies in span{M R^m, c}:
// u = M a + g c, so with
//     K = M^T M = R^{-T} D G_WW D R^{-1},  h = M^T c = R^{-T} D G_Wm / beta_m,
//     s = ||c||^2 = G_mm / beta_m^2,       G = V_hat^T V_hat ((m+1) x (m+1)),
// (V_hat = the stored columns w_hat_0..w_hat_m, D = diag(1/beta_j)) the whole
// iteration runs in R^m: ||u||^2 = a^T K a + 2 g a^T h + g^2 s and
// M^T u = K a + g h.  In exact arithmetic the iterates are LSQR's; the n x m
// work collapses into ONE pass over V_{m+1} (the Gram matrix, a tall-skinny
// SYRK: n (m+1)^2 / 2 fp64 FMAs, compute-bound) instead of L + 1 streaming
// passes.  Rounding: G carries ~eps ||v_i|| ||v_j|| absolute error, which K
// amplifies by ||R^{-1}||^2 ~ cond(R)^2 / m; fab_compress therefore uses it
// only when cond(R) <= kGramCondMax and otherwise runs the explicit passes
// (fab_info.gram_used says which).
#include <stdlib.h>

#include "fab_internal.cuh"

namespace fab {

constexpr int kGB = 8;          // 8 x 8 block of G per thread
constexpr int kGBS = 10;        // shared-memory stride of an 8-column block (doubles)
constexpr int kGRows = 32;      // rows per chunk
constexpr int kGThreadsMax = 352;   // 186 registers per thread at one CTA per SM

// Upper-triangular 8 x 8 blocks (I <= J) of an (nc x nc) Gram matrix, block b
// of group gi handled by thread b - gi * per_group.  Partials per CTA:
// part[cta][nc * nc] (column-major, upper blocks written, the rest untouched).
// Row chunks of kGRows rows are staged ROW-major in shared memory (a thread's
// 8 columns of a row are 64 contiguous bytes: 4 x LDS.128, different blocks
// hit different banks) in two buffers: the next chunk's global loads are
// issued into registers before this chunk's FMAs and stored after them.
__global__ void __launch_bounds__(kGThreadsMax, 1)
k_gram(const double* __restrict__ V, int64_t ld, int64_t n, int nc, int ngroups, int per_group,
       double* __restrict__ part) {
  extern __shared__ __align__(16) double tile[];   // [2][kGRows][str]
  const int nbk = (nc + kGB - 1) / kGB;
  const int nblocks = nbk * (nbk + 1) / 2;
  // row layout: 8-column block J at J * kGBS doubles (80 B apart, so the 8
  // threads of a quarter-warp reading 8 different blocks hit 8 different
  // 16-B bank groups; 64 B apart they would collide 4-way)
  const int str = nbk * kGBS + 2;
  const int group = blockIdx.x % ngroups;
  const int cta_in_group = blockIdx.x / ngroups;
  const int ctas_per_group = gridDim.x / ngroups;
  const int b = group * per_group + threadIdx.x;
  int I = 0, J = 0;
  const bool active = threadIdx.x < per_group && b < nblocks;
  if (active) {
    int rem = b;
    while (rem >= nbk - I) {
      rem -= nbk - I;
      ++I;
    }
    J = I + rem;
  }
  double acc[kGB][kGB];
#pragma unroll
  for (int u = 0; u < kGB; ++u)
#pragma unroll
    for (int v = 0; v < kGB; ++v) acc[u][v] = 0.0;
  const int64_t nchunks = (n + kGRows - 1) / kGRows;
  // chunk loads: cp.async (LDGSTS) 8-B copies straight into the other buffer,
  // transposing column-major V into the row-major tile; out-of-range rows and
  // the padding columns are zero-filled (src-size 0)
  const int nel = nbk * kGB * kGRows;
  auto load_chunk = [&](int64_t ch2, double* T) {
    const int64_t r0 = ch2 * kGRows;
    for (int e = threadIdx.x; e < nel; e += blockDim.x) {
      const int j = e / kGRows, r = e - j * kGRows;
      const bool ok = j < nc && r0 + r < n;
      const double* src = ok ? V + (int64_t)j * ld + r0 + r : V;
      const uint32_t dst =
          static_cast<uint32_t>(__cvta_generic_to_shared(T + r * str + (j / kGB) * kGBS + (j % kGB)));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t ch = cta_in_group;
  int buf = 0;
  if (ch < nchunks) load_chunk(ch, tile);
  for (; ch < nchunks; ch += ctas_per_group) {
    const int64_t nx = ch + ctas_per_group;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();                                     // chunk ch landed; buffer buf^1 is free
    if (nx < nchunks) load_chunk(nx, tile + (size_t)(buf ^ 1) * kGRows * str);   // in flight during the FMAs
    const double* T = tile + (size_t)buf * kGRows * str;
    if (active) {
      // software-pipelined: row r+1's eight 16-B loads are issued before row
      // r's 64 FMAs, so the FMAs never wait on shared memory
      double2 fi[kGB / 2], fj[kGB / 2];
      {
        const double2* pi = reinterpret_cast<const double2*>(T + I * kGBS);
        const double2* pj = reinterpret_cast<const double2*>(T + J * kGBS);
#pragma unroll
        for (int u = 0; u < kGB / 2; ++u) {
          fi[u] = pi[u];
          fj[u] = pj[u];
        }
      }
#pragma unroll 1
      for (int r = 0; r < kGRows; ++r) {
        double xi[kGB], xj[kGB];
#pragma unroll
        for (int u = 0; u < kGB / 2; ++u) {
          xi[2 * u] = fi[u].x;
          xi[2 * u + 1] = fi[u].y;
          xj[2 * u] = fj[u].x;
          xj[2 * u + 1] = fj[u].y;
        }
        if (r + 1 < kGRows) {
          const double2* pi = reinterpret_cast<const double2*>(T + (r + 1) * str + I * kGBS);
          const double2* pj = reinterpret_cast<const double2*>(T + (r + 1) * str + J * kGBS);
#pragma unroll
          for (int u = 0; u < kGB / 2; ++u) {
            fi[u] = pi[u];
            fj[u] = pj[u];
          }
        }
#pragma unroll
        for (int u = 0; u < kGB; ++u)
#pragma unroll
          for (int v = 0; v < kGB; ++v) acc[u][v] = fma(xi[u], xj[v], acc[u][v]);
      }
    }
    buf ^= 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (active) {
    double* P = part + (int64_t)blockIdx.x * nc * nc;
#pragma unroll
    for (int u = 0; u < kGB; ++u)
#pragma unroll
      for (int v = 0; v < kGB; ++v) {
        const int ci = I * kGB + u, cj = J * kGB + v;
        if (ci < nc && cj < nc) P[ci + (int64_t)cj * nc] = acc[u][v];
      }
  }
}

// fp64 tensor-core variant (mma.sync m8n8k4 f64, DMMA): a warp owns a 4 x 4
// tile of 8 x 8 blocks (TI <= TJ over the 4-block tiles of the upper
// triangle), 32 accumulators per thread; per k-step of 4 rows it loads one
// A/B fragment per block row / column (the same fragment serves as A for
// block row X and as B for block column X: A[i][k] = B[k][i] = x[k][8X+i])
// and issues 16 DMMAs -- 8 shared-memory loads per 4096 FMAs per warp instead
// of 16 loads per 64 FMAs per thread in k_gram.  Warp tiles are dealt to
// kGmWarps-warp groups; a CTA of group g sweeps every row chunk for its tiles.
constexpr int kGmT = 4;          // blocks per warp-tile side
constexpr int kGmWarps = 16;     // warps (tiles) per CTA group

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__host__ __device__ inline int gm_tile_str(int nbk) {
  // row stride of the staged tile (doubles): 8-column blocks kGBS apart, then
  // padded to 8 mod 16 so the 4 rows of a fragment load hit 2 disjoint
  // halves of the banks
  int s = nbk * kGBS;
  while (s % 16 != 8) ++s;
  return s;
}

__global__ void __launch_bounds__(kGmWarps * 32, 1)
k_gram_mma(const double* __restrict__ V, int64_t ld, int64_t n, int nc, int ngroups, double* __restrict__ part) {
  extern __shared__ __align__(16) double tile[];   // [2][kGRows][str]
  const int nbk = (nc + kGB - 1) / kGB;
  const int nwt = (nbk + kGmT - 1) / kGmT;
  const int ntiles = nwt * (nwt + 1) / 2;
  const int str = gm_tile_str(nbk);
  const int group = blockIdx.x % ngroups;
  const int cta_in_group = blockIdx.x / ngroups;
  const int ctas_per_group = gridDim.x / ngroups;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wt = group * kGmWarps + warp;
  const bool active = wt < ntiles;
  int TI = 0, TJ = 0;
  if (active) {
    int rem = wt;
    while (rem >= nwt - TI) {
      rem -= nwt - TI;
      ++TI;
    }
    TJ = TI + rem;
  }
  double acc[kGmT][kGmT][2];
#pragma unroll
  for (int a = 0; a < kGmT; ++a)
#pragma unroll
    for (int b = 0; b < kGmT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int64_t nchunks = (n + kGRows - 1) / kGRows;
  const int ncol_pad = nbk * kGB;
  const int nel = ncol_pad * kGRows;
  auto load_chunk = [&](int64_t ch2, double* T) {
    const int64_t r0 = ch2 * kGRows;
    for (int e = threadIdx.x; e < nel; e += blockDim.x) {
      const int j = e / kGRows, r = e - j * kGRows;
      const bool ok = j < nc && r0 + r < n;
      const double* src = ok ? V + (int64_t)j * ld + r0 + r : V;
      const uint32_t dst =
          static_cast<uint32_t>(__cvta_generic_to_shared(T + r * str + (j / kGB) * kGBS + (j % kGB)));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // this lane's fragment offset inside a 4-row k-step: row (lane & 3), column (lane >> 2)
  const int foff = (lane & 3) * str + (lane >> 2);
  int64_t ch = cta_in_group;
  int buf = 0;
  if (ch < nchunks) load_chunk(ch, tile);
  for (; ch < nchunks; ch += ctas_per_group) {
    const int64_t nx = ch + ctas_per_group;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (nx < nchunks) load_chunk(nx, tile + (size_t)(buf ^ 1) * kGRows * str);
    const double* T = tile + (size_t)buf * kGRows * str;
    if (active) {
#pragma unroll 2
      for (int ks = 0; ks < kGRows / 4; ++ks) {
        const double* Tk = T + (4 * ks) * str + foff;
        double fa[kGmT], fb[kGmT];
#pragma unroll
        for (int a = 0; a < kGmT; ++a) {
          const int bi = TI * kGmT + a, bj = TJ * kGmT + a;
          fa[a] = bi < nbk ? Tk[bi * kGBS] : 0.0;
          fb[a] = bj < nbk ? Tk[bj * kGBS] : 0.0;
        }
#pragma unroll
        for (int a = 0; a < kGmT; ++a)
#pragma unroll
          for (int b = 0; b < kGmT; ++b) dmma(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
      }
    }
    buf ^= 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (active) {
    double* P = part + (int64_t)blockIdx.x * nc * nc;
#pragma unroll
    for (int a = 0; a < kGmT; ++a)
#pragma unroll
      for (int b = 0; b < kGmT; ++b) {
        const int I = TI * kGmT + a, J = TJ * kGmT + b;
        if (I > J || J >= nbk) continue;
        const int ci = I * kGB + (lane >> 2);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cj = J * kGB + 2 * (lane & 3) + h;
          if (ci < nc && cj < nc) P[ci + (int64_t)cj * nc] = acc[a][b][h];
        }
      }
  }
}

// G from the k_gram_mma partials: the group owning block (I, J) is that of
// its warp tile (I / 4, J / 4)
__global__ void k_gram_mma_reduce(const double* part, int nc, int ngroups, int nctas, double* G) {
  const int64_t total = (int64_t)nc * nc;
  const int nbk = (nc + kGB - 1) / kGB;
  const int nwt = (nbk + kGmT - 1) / kGmT;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int ci = (int)(e % nc), cj = (int)(e / nc);
    const int I = ci / kGB, J = cj / kGB;
    if (I > J) continue;
    const int TI = I / kGmT, TJ = J / kGmT;
    const int wt = TI * nwt - TI * (TI - 1) / 2 + (TJ - TI);
    const int g = wt / kGmWarps;
    double a = 0.0;
    for (int c = g; c < nctas; c += ngroups) a += part[(int64_t)c * total + e];
    G[ci + (int64_t)cj * nc] = a;
    G[cj + (int64_t)ci * nc] = a;
  }
}

// G = sum over the CTAs holding each block (fixed order), mirrored to the
// lower triangle
__global__ void k_gram_reduce(const double* part, int nc, int ngroups, int nctas, double* G) {
  const int64_t total = (int64_t)nc * nc;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int ci = (int)(e % nc), cj = (int)(e / nc);
    if (ci > cj) continue;
    // the group holding block (ci/8, cj/8)
    const int nbk = (nc + kGB - 1) / kGB;
    const int I = ci / kGB, J = cj / kGB;
    const int bidx = I * nbk - I * (I - 1) / 2 + (J - I);
    const int per_group = (nbk * (nbk + 1) / 2 + ngroups - 1) / ngroups;
    const int g = bidx / per_group;
    double a = 0.0;
    for (int c = g; c < nctas; c += ngroups) a += part[(int64_t)c * total + e];
    G[ci + (int64_t)cj * nc] = a;
    G[cj + (int64_t)ci * nc] = a;
  }
}

// LSQR (Paige-Saunders, x_0 = 0) in the coordinates u = M a + g c, one CTA.
// Rinv: R^{-1} (upper, column-major), RinvT its transpose; bcol = beta_0..m.
// Same MATLAB-style stopping test as the streaming LSQR (lsqr.cu); x -> L.x.
struct GramVecs {
  double *a, *v, *w, *x, *t1, *t2, *Ka, *h;
};

__device__ void gram_kmul(const double* G, int nc, const double* Rinv, const double* RinvT, const double* bcol,
                          int m, const double* in, double* out, double* t1, double* t2) {
  // t1 = D R^{-1} in
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < m; i += nw) {
    double a = 0.0;
    for (int j = i + lane; j < m; j += 32) a = fma(RinvT[j + (int64_t)i * m], in[j], a);   // row i of R^{-1}
    a = warp_sum(a);
    if (lane == 0) t1[i] = a / bcol[i];
  }
  __syncthreads();
  // t2 = D G_WW t1
  for (int i = warp; i < m; i += nw) {
    double a = 0.0;
    for (int j = lane; j < m; j += 32) a = fma(G[i + (int64_t)j * nc], t1[j], a);
    a = warp_sum(a);
    if (lane == 0) t2[i] = a / bcol[i];
  }
  __syncthreads();
  // out = R^{-T} t2  (row i of R^{-T} = column i of R^{-1}, entries 0..i)
  for (int i = warp; i < m; i += nw) {
    double a = 0.0;
    for (int j = lane; j <= i; j += 32) a = fma(Rinv[j + (int64_t)i * m], t2[j], a);
    a = warp_sum(a);
    if (lane == 0) out[i] = a;
  }
  __syncthreads();
}

__device__ double gram_dot(const double* x, const double* y, int m, double* red) {
  double a = 0.0;
  for (int j = threadIdx.x; j < m; j += blockDim.x) a = fma(x[j], y[j], a);
  double v1[1] = {a}, o1[1];
  block_sum<1>(v1, red, o1);
  __shared__ double bc;
  if (threadIdx.x == 0) bc = o1[0];
  __syncthreads();
  return bc;
}

__global__ void __launch_bounds__(1024) k_gram_lsqr(const double* G, int m, const double* Rinv, const double* RinvT,
                                                    const double* bcol, GramVecs L, int fixed, int maxit, double tol,
                                                    DevState* st) {
  __shared__ double red[32];
  const int nc = m + 1;
  const double bm = bcol[m];
  // h = M^T c = R^{-T} D G_Wm / beta_m
  for (int i = threadIdx.x; i < m; i += blockDim.x) L.t2[i] = G[i + (int64_t)m * nc] / bcol[i] / bm;
  __syncthreads();
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = warp; i < m; i += nw) {
      double a = 0.0;
      for (int j = lane; j <= i; j += 32) a = fma(Rinv[j + (int64_t)i * m], L.t2[j], a);
      a = warp_sum(a);
      if (lane == 0) L.h[i] = a;
    }
  }
  __syncthreads();
  const double s = G[m + (int64_t)m * nc] / (bm * bm);
  double beta = sqrt(s);
  double g = 1.0 / beta;                                   // u_1 = c / beta_1
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    L.a[i] = 0.0;
    L.v[i] = L.h[i] * g;                                   // M^T u_1
    L.x[i] = 0.0;
  }
  __syncthreads();
  double alpha = sqrt(gram_dot(L.v, L.v, m, red));
  const double ia0 = alpha > 0 ? 1.0 / alpha : 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    L.v[i] *= ia0;
    L.w[i] = L.v[i];
  }
  __syncthreads();
  const double bnorm = beta;
  double phibar = beta, rhobar = alpha, anorm2 = 0.0;
  int it = 0, done = (alpha == 0.0) ? 1 : 0;
  double rnorm = bnorm, arnorm = alpha, anorm = 0.0;
  while (!done && it < maxit) {
    // u <- M v - alpha u:  a <- v - alpha a, g <- -alpha g
    for (int i = threadIdx.x; i < m; i += blockDim.x) L.a[i] = L.v[i] - alpha * L.a[i];
    g = -alpha * g;
    __syncthreads();
    gram_kmul(G, nc, Rinv, RinvT, bcol, m, L.a, L.Ka, L.t1, L.t2);
    const double aka = gram_dot(L.a, L.Ka, m, red);
    const double ah = gram_dot(L.a, L.h, m, red);
    const double b2 = aka + 2.0 * g * ah + g * g * s;
    const double alpha_old = alpha;
    beta = sqrt(b2 > 0.0 ? b2 : 0.0);
    const double ib = beta > 0 ? 1.0 / beta : 0.0;
    g *= ib;
    // v <- M^T u - beta v = (K a + g_old h) / beta - beta v
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      L.a[i] *= ib;
      L.v[i] = fma(L.Ka[i], ib, g * L.h[i]) - beta * L.v[i];
    }
    __syncthreads();
    alpha = sqrt(gram_dot(L.v, L.v, m, red));
    const double rho = hypot(rhobar, beta);
    if (!(rho > 0.0)) break;
    const double cs = rhobar / rho, sn = beta / rho;
    const double theta = sn * alpha;
    rhobar = -cs * alpha;
    const double phi = cs * phibar;
    phibar = sn * phibar;
    const double ia = alpha > 0 ? 1.0 / alpha : 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      const double vn = L.v[i] * ia;
      L.x[i] = fma(phi / rho, L.w[i], L.x[i]);
      L.w[i] = fma(-(theta / rho), L.w[i], vn);
      L.v[i] = vn;
    }
    __syncthreads();
    anorm2 += alpha_old * alpha_old + beta * beta;
    anorm = sqrt(anorm2);
    rnorm = phibar;
    arnorm = phibar * alpha * fabs(cs);
    ++it;
    if (alpha == 0.0 || beta == 0.0) done = 1;
    if (!fixed && (rnorm <= tol * bnorm || (rnorm > 0 && arnorm <= tol * anorm * rnorm))) done = 1;
  }
  if (threadIdx.x == 0) {
    st->lsqr_iters = it;
    st->lsqr_done = done;
    st->rnorm = rnorm;
    st->arnorm = arnorm;
    st->anorm = anorm;
  }
}

static size_t gram_smem(int nc) {
  const int nbk = (nc + kGB - 1) / kGB;
  return (size_t)2 * kGRows * (nbk * kGBS + 2) * sizeof(double);
}

// G = V_hat^T V_hat of the stored columns 0..m (nc = m+1) into G (nc x nc,
// column-major); uses c->wbuf-style scratch for the per-CTA partials.
static int gram_pass_mma(fab_ctx* c, int nc, double* G, cudaStream_t st) {
  const int nbk = (nc + kGB - 1) / kGB;
  const int nwt = (nbk + kGmT - 1) / kGmT;
  const int ntiles = nwt * (nwt + 1) / 2;
  const int ngroups = (ntiles + kGmWarps - 1) / kGmWarps;
  int grid = c->num_sms / ngroups * ngroups;
  if (grid < ngroups) grid = ngroups;
  const size_t need = (size_t)grid * nc * nc * sizeof(double);
  if (c->gram_part_bytes < need) {
    if (c->gram_part) cudaFree(c->gram_part);
    c->gram_part = nullptr;
    c->gram_part_bytes = 0;
    FAB_CUDA(cudaMalloc(&c->gram_part, need));
    c->gram_part_bytes = need;
  }
  const size_t smem = (size_t)2 * kGRows * gm_tile_str(nbk) * sizeof(double);
  FAB_CUDA(ensure_dyn_smem((const void*)k_gram_mma, 200 * 1024));
  k_gram_mma<<<grid, kGmWarps * 32, smem, st>>>(c->V, c->ld, c->n, nc, ngroups, c->gram_part);
  FAB_CHECK_LAUNCH();
  k_gram_mma_reduce<<<(nc * nc + 255) / 256, 256, 0, st>>>(c->gram_part, nc, ngroups, grid, G);
  FAB_CHECK_LAUNCH();
  return FAB_OK;
}

int gram_pass(fab_ctx* c, int nc, double* G, cudaStream_t st) {
  // the DMMA variant is opt-in (FAB_GRAM_MMA=1): measured at c3 51 ms vs
  // 36.7 ms for the DFMA k_gram (two CTA groups each stage every row chunk,
  // and the m8n8k4 f64 path does not outrun the FP64 FMA pipe here)
  const char* e = getenv("FAB_GRAM_MMA");
  if (e && e[0] == '1') return gram_pass_mma(c, nc, G, st);
  const int nbk = (nc + kGB - 1) / kGB;
  const int nblocks = nbk * (nbk + 1) / 2;
  const int ngroups = (nblocks + kGThreadsMax - 1) / kGThreadsMax;
  const int per_group = (nblocks + ngroups - 1) / ngroups;
  const int threads = (per_group + 31) / 32 * 32;
  int grid = c->num_sms;
  grid = grid / ngroups * ngroups;
  if (grid < ngroups) grid = ngroups;
  const size_t need = (size_t)grid * nc * nc * sizeof(double);
  if (c->gram_part_bytes < need) {
    if (c->gram_part) cudaFree(c->gram_part);
    c->gram_part = nullptr;
    c->gram_part_bytes = 0;
    FAB_CUDA(cudaMalloc(&c->gram_part, need));
    c->gram_part_bytes = need;
  }
  FAB_CUDA(ensure_dyn_smem((const void*)k_gram, 200 * 1024));
  k_gram<<<grid, threads, gram_smem(nc), st>>>(c->V, c->ld, c->n, nc, ngroups, per_group, c->gram_part);
  FAB_CHECK_LAUNCH();
  k_gram_reduce<<<(nc * nc + 255) / 256, 256, 0, st>>>(c->gram_part, nc, ngroups, grid, G);
  FAB_CHECK_LAUNCH();
  return FAB_OK;
}

int gram_lsqr(fab_ctx* c, int m, const double* G, const double* Rinv, const double* RinvT, double* x, int fixed,
              int maxit, double tol, cudaStream_t st) {
  GramVecs L{svec(c, 17), svec(c, 18), svec(c, 19), x, svec(c, 20), svec(c, 21), svec(c, 22), svec(c, 23)};
  k_gram_lsqr<<<1, 1024, 0, st>>>(G, m, Rinv, RinvT, c->beta, L, fixed, maxit, tol, c->st_d);
  FAB_CHECK_LAUNCH();
  return FAB_OK;
}

}  // namespace fab
