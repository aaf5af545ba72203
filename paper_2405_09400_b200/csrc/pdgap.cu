// pdgap.cu — primal-dual gap of the current state (App. A.2.2).
//
//   E = <c, pi> + eps KL(pi | mu (x) nu) of the last sweep's plans: the solve
//       kernel leaves E_J / h^2 per composite cell (sweep.cu primal_terms);
//       E = h^2 sum_J E_J + eps |mu| |nu|.
//   D = D(alpha†, beta†) with alpha† stitched from the
//       last A and B potentials along the comb tree of reading R15 and beta†
//       its exact global Y-response; the exp-term of D then vanishes and
//       D = eps (<a†, mu> + <b†, nu>) (nat units a = alpha / eps).
//   transport_cost = <c, pi> from the plan moments of the last sweep (R13).
//
// All in fp64 except the exponentials of the Y-response (fp32 ex2 of
// differences to the running maximum, which are <= 0).  Deterministic:
// partial sums per block in fixed order.  Diagnostic path, not timed.
#include <algorithm>
#include <cmath>

#include "ctx.cuh"

namespace dd {
namespace {

constexpr double kLn2 = 0.69314718055994531;
constexpr double kLog2e = 1.4426950408889634;

// Global-gauge nat potential of both partitions at every pixel:
// a(k) = ln2 A2(kappa) + (|D|^2 + 2 D.kappa) / eps', D = K - G.
__global__ void k_anat(const float* __restrict__ alA, const int* __restrict__ gA, const CompCell* __restrict__ cA,
                       const float* __restrict__ alB, const int* __restrict__ gB, const CompCell* __restrict__ cB,
                       int N1, int N2, int s, int na2, int nb2, double eps_p, double* __restrict__ aA,
                       double* __restrict__ aB) {
  const long long NN = (long long)N1 * N2;
  for (long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x; pix < NN;
       pix += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(pix / N2), c = (int)(pix - (long long)r * N2);
    {
      const int J = (r / (2 * s)) * na2 + c / (2 * s);
      const CompCell cc = cA[J];
      const double D1 = cc.r0 - gA[2 * J], D2 = cc.c0 - gA[2 * J + 1];
      const double k1 = r - cc.r0, k2 = c - cc.c0;
      aA[pix] = kLn2 * (double)alA[pix] + (D1 * D1 + D2 * D2 + 2.0 * (D1 * k1 + D2 * k2)) / eps_p;
    }
    {
      const int J = ((r / s + 1) / 2) * nb2 + (c / s + 1) / 2;
      const CompCell cc = cB[J];
      const double D1 = cc.r0 - gB[2 * J], D2 = cc.c0 - gB[2 * J + 1];
      const double k1 = r - cc.r0, k2 = c - cc.c0;
      aB[pix] = kLn2 * (double)alB[pix] + (D1 * D1 + D2 * D2 + 2.0 * (D1 * k1 + D2 * k2)) / eps_p;
    }
  }
}

__device__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// mu-weighted mean over basic cell (i1, i2) of (pv - pu); one warp.
__device__ double wmean_diff(const double* pv, const double* pu, const float* mu, int N2, int s, int i1, int i2) {
  const int lane = threadIdx.x & 31;
  double sw = 0.0, sd = 0.0;
  for (int t = lane; t < s * s; t += 32) {
    const long long pix = (long long)(i1 * s + t / s) * N2 + i2 * s + t % s;
    const double m = mu[pix];
    sw += m;
    sd += m * (pv[pix] - pu[pix]);
  }
  return warp_sum(sd) / warp_sum(sw);
}

// Offset increment of each A-cell along the comb tree (reading R15).
__global__ void k_stitch_inc(const double* __restrict__ aA, const double* __restrict__ aB,
                             const float* __restrict__ mu, int N2, int s, int na1, int na2, double* __restrict__ inc) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= na1 * na2) return;
  const int a1 = warp / na2, a2 = warp % na2;
  double d = 0.0;
  if (a2 > 0)        // A(a1, a2-1) -> B(a1, a2) -> A(a1, a2)
    d = wmean_diff(aB, aA, mu, N2, s, 2 * a1, 2 * a2 - 1) + wmean_diff(aA, aB, mu, N2, s, 2 * a1, 2 * a2);
  else if (a1 > 0)   // A(a1-1, 0) -> B(a1, 0) -> A(a1, 0)
    d = wmean_diff(aB, aA, mu, N2, s, 2 * a1 - 1, 0) + wmean_diff(aA, aB, mu, N2, s, 2 * a1, 0);
  if ((threadIdx.x & 31) == 0) inc[warp] = d;
}

// Prefix sums along the comb: column 0 first, then every row.
__global__ void k_stitch_scan(double* __restrict__ inc, int na1, int na2) {
  if (threadIdx.x == 0)
    for (int a1 = 1; a1 < na1; ++a1) inc[a1 * na2] += inc[(a1 - 1) * na2];
  __syncthreads();
  for (int a1 = threadIdx.x; a1 < na1; a1 += blockDim.x)
    for (int a2 = 1; a2 < na2; ++a2) inc[a1 * na2 + a2] += inc[a1 * na2 + a2 - 1];
}

// a† = a_A - off; g = a† + ln mu (input of the Y-response); partial sums of
// mu a† and of mu per block.
__global__ void k_adag(const double* __restrict__ aA, const double* __restrict__ off, const float* __restrict__ mu,
                       int N1, int N2, int s, int na2, double* __restrict__ g, double* __restrict__ part) {
  const long long NN = (long long)N1 * N2;
  double sa = 0.0, sm = 0.0;
  for (long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x; pix < NN;
       pix += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(pix / N2), c = (int)(pix - (long long)r * N2);
    const double a = aA[pix] - off[(r / (2 * s)) * na2 + c / (2 * s)];
    const double m = mu[pix];
    g[pix] = m > 0.0 ? a + log(m) : -INFINITY;
    sa += m * a;
    sm += m;
  }
  __shared__ double sh[2][32];
  sa = warp_sum(sa);
  sm = warp_sum(sm);
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = sa;
    sh[1][threadIdx.x >> 5] = sm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0.0, tm = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      ta += sh[0][w];
      tm += sh[1][w];
    }
    part[2 * blockIdx.x] = ta;
    part[2 * blockIdx.x + 1] = tm;
  }
}

// One separable LSE stage of the exact Y-response (global, dense):
//   out[y * R + x] = LSE_z [ in[x * M + z] - (z - y)^2 / eps' ]   (nat units)
// for x < R (one block per x), y, z < M; written transposed so the next stage
// reads rows.  fp64 terms, fp32 exponentials of (term - max) <= 0.
__global__ void k_lse_stage(const double* __restrict__ in, double* __restrict__ out, int R, int M, double inv_eps) {
  extern __shared__ double row[];
  const int x = blockIdx.x;
  for (int z = threadIdx.x; z < M; z += blockDim.x) row[z] = in[(long long)x * M + z];
  __syncthreads();
  for (int y = threadIdx.x; y < M; y += blockDim.x) {
    double m = -INFINITY;
    for (int z = 0; z < M; ++z) {
      const double d = (double)(z - y);
      m = fmax(m, row[z] - d * d * inv_eps);
    }
    float sum = 0.f;
    if (m > -INFINITY)
      for (int z = 0; z < M; ++z) {
        const double d = (double)(z - y);
        const float t = (float)((row[z] - d * d * inv_eps - m) * kLog2e);
        sum += exp2f(t);
      }
    out[(long long)y * R + x] = m + log((double)sum);
  }
}

// b(y) = -T2(y); partial sums of nu b over nu > 0 and of nu per block.
__global__ void k_dual_nu(const double* __restrict__ T2, const double* __restrict__ nu, long long NN,
                          double* __restrict__ part) {
  double sb = 0.0, sn = 0.0;
  for (long long y = blockIdx.x * (long long)blockDim.x + threadIdx.x; y < NN; y += (long long)gridDim.x * blockDim.x) {
    const double v = nu[y];
    if (v > 0.0) {
      sb += v * -T2[y];
      sn += v;
    }
  }
  __shared__ double sh[2][32];
  sb = warp_sum(sb);
  sn = warp_sum(sn);
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = sb;
    sh[1][threadIdx.x >> 5] = sn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tb = 0.0, tn = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      tb += sh[0][w];
      tn += sh[1][w];
    }
    part[2 * blockIdx.x] = tb;
    part[2 * blockIdx.x + 1] = tn;
  }
}

// Fixed-order final reductions: out[0] = sum ecell, out[1] = sum_i <c, pi_i>/h^2
// (G0 - 2 G1 + M2), out[2..5] = sums of the two partial arrays.
__global__ void k_pd_final(const double* __restrict__ ecell, int ncells, const double* __restrict__ mom, int I,
                           const double* __restrict__ pa, const double* __restrict__ pb, int nparts,
                           double* __restrict__ out) {
  __shared__ double sh[6][32];
  double v[6] = {0, 0, 0, 0, 0, 0};
  for (int j = threadIdx.x; j < ncells; j += blockDim.x) v[0] += ecell[j];
  for (int i = threadIdx.x; i < I; i += blockDim.x) v[1] += mom[6 * i + 3] - 2.0 * mom[6 * i + 4] + mom[6 * i + 5];
  for (int k = threadIdx.x; k < nparts; k += blockDim.x) {
    v[2] += pa[2 * k];
    v[3] += pa[2 * k + 1];
    v[4] += pb[2 * k];
    v[5] += pb[2 * k + 1];
  }
  for (int q = 0; q < 6; ++q) {
    const double t = warp_sum(v[q]);
    if ((threadIdx.x & 31) == 0) sh[q][threadIdx.x >> 5] = t;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[threadIdx.x][w];
    out[threadIdx.x] = t;
  }
}

}  // namespace

dd_status pd_gap_impl(dd_ctx* c, double* primal, double* dual, double* rel_gap, double* transport) {
  const long long NN = (long long)c->N1 * c->N2;
  const int s = c->s;
  const int na1 = (c->n1 + 1) / 2, na2 = (c->n2 + 1) / 2, nb2 = c->n2 / 2 + 1;
  const int nparts = 256;
  // scratch: aA, aB (later g, T), inc [na1 na2], partial sums 2 x [2 nparts], out [8]
  const size_t need = 2 * (size_t)NN + (size_t)na1 * na2 + 4 * nparts + 8;
  if (!c->d_pd) DD_CUDA(cudaMallocAsync(&c->d_pd, need * sizeof(double), c->stream));
  double* aA = c->d_pd;
  double* aB = aA + NN;
  double* inc = aB + NN;
  double* pa = inc + (size_t)na1 * na2;
  double* pb = pa + 2 * nparts;
  double* out = pb + 2 * nparts;
  cudaStream_t st = c->stream;
  k_anat<<<nparts, 256, 0, st>>>(c->d_alpha[0], c->d_gauge[0], c->d_cells[0], c->d_alpha[1], c->d_gauge[1],
                                 c->d_cells[1], c->N1, c->N2, s, na2, nb2, c->eps_p, aA, aB);
  DD_CUDA(cudaGetLastError());
  k_stitch_inc<<<(na1 * na2 * 32 + 255) / 256, 256, 0, st>>>(aA, aB, c->d_mu, c->N2, s, na1, na2, inc);
  DD_CUDA(cudaGetLastError());
  k_stitch_scan<<<1, 256, 0, st>>>(inc, na1, na2);
  DD_CUDA(cudaGetLastError());
  double* g = aB;   // aB is no longer needed
  k_adag<<<nparts, 256, 0, st>>>(aA, inc, c->d_mu, c->N1, c->N2, s, na2, g, pa);
  DD_CUDA(cudaGetLastError());
  // stage 1 (x = x1, z = x2, y = y2): aA[y2 * N1 + x1] = LSE_x2 [g - (x2 - y2)^2 / eps'];
  // stage 2 (x = y2, z = x1, y = y1): g[y1 * N2 + y2] = LSE_x1 [aA - (x1 - y1)^2 / eps'] = -b(y).
  const double inv_eps = 1.0 / c->eps_p;
  const size_t sh1 = (size_t)c->N2 * 8, sh2 = (size_t)c->N1 * 8, shm = std::max(sh1, sh2);
  if (shm > 48 * 1024)
    DD_CUDA(cudaFuncSetAttribute(k_lse_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  k_lse_stage<<<c->N1, 256, sh1, st>>>(g, aA, c->N1, c->N2, inv_eps);
  DD_CUDA(cudaGetLastError());
  k_lse_stage<<<c->N2, 256, sh2, st>>>(aA, g, c->N2, c->N1, inv_eps);
  DD_CUDA(cudaGetLastError());
  k_dual_nu<<<nparts, 256, 0, st>>>(g, c->d_nu, NN, pb);
  DD_CUDA(cudaGetLastError());
  k_pd_final<<<1, 256, 0, st>>>(c->d_ecell, c->ncells[c->last_part], c->d_mom, c->I, pa, pb, nparts, out);
  DD_CUDA(cudaGetLastError());
  double h[6];
  DD_CUDA(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, st));
  DD_CUDA(cudaStreamSynchronize(st));
  const double h2 = c->h * c->h, eps = c->eps;
  const double E = h2 * h[0] + eps * h[3] * h[5];   // + eps |mu| |nu|
  const double D = eps * (h[2] + h[4]);
  if (primal) *primal = E;
  if (dual) *dual = D;
  if (rel_gap) *rel_gap = (E - D) / D;
  if (transport) *transport = h2 * h[1];
  return DD_OK;
}

}  // namespace dd
