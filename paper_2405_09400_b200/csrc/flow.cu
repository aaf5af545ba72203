#include <cstdio>
#include <cstdlib>
// flow.cu — flow update steps 1 and 3 (§5.1) and the
// flow-related C-ABI entry points.
//
// Step 1 (F1): edge costs c_bar_ij = <c, pi_hat_ij - pi_hat_ii> (Eq. edge-cost
// PAPER.md:419-421) with the product gluing candidate
// pi_hat_ij = mu_j/m_j (x) nu_i/m_i, where pi_i is the last
// sweep's plan on X_i and nu_i = P_Y pi_i (reading R13).  Closed form through
// moments about the cell centre z_i:
//   m_i c_bar_ij = M0 W_ij - G0 - 2 M1 . (xbar_j - z_i) + 2 G1,
//   W_ij = E_{mu_j}|x - z_i|^2 = V_j + |xbar_j - z_i|^2,
// the |y|^2 terms cancelling exactly.  One thread per basic cell, no plan is
// instantiated (this sidesteps the memory bottleneck noted at PAPER.md:927).
// Step 3 (F3): nu_hat_j = sum_{i in N(j)} (w_ij / q_i) nu_i (Lemma, Eq.
// flow-update-cell-marginals PAPER.md:453-456), bounding-box merge + truncate
// + minimal box, one CTA per changed cell.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "ctx.cuh"

namespace dd {

long long* mcf_info_ptr(void* ws, int I);

namespace {

__device__ __forceinline__ int nbr_cell(int i, int a, int n1, int n2) {
  const int i1 = i / n2, i2 = i - (i / n2) * n2;
  switch (a) {
    case 0: return i;
    case 1: return i1 > 0 ? i - n2 : -1;
    case 2: return i1 + 1 < n1 ? i + n2 : -1;
    case 3: return i2 > 0 ? i - 1 : -1;
    default: return i2 + 1 < n2 ? i + 1 : -1;
  }
}

// Static mu moments of each basic cell: xbar_i (pixel coords) and
// V_i = E_{mu_i/m_i} |x - xbar_i|^2.
__global__ void k_mu_moments(const double* __restrict__ mu, int N2, int s, int n2, int I,
                             double* __restrict__ xbar, double* __restrict__ var) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= I) return;
  const int i1 = i / n2, i2 = i - i1 * n2;
  double m = 0, a = 0, b = 0;
  for (int r = 0; r < s; ++r)
    for (int c = 0; c < s; ++c) {
      const double v = mu[(long long)(i1 * s + r) * N2 + i2 * s + c];
      m += v;
      a += v * (i1 * s + r);
      b += v * (i2 * s + c);
    }
  a /= m;
  b /= m;
  double vv = 0;
  for (int r = 0; r < s; ++r)
    for (int c = 0; c < s; ++c) {
      const double v = mu[(long long)(i1 * s + r) * N2 + i2 * s + c];
      const double d1 = i1 * s + r - a, d2 = i2 * s + c - b;
      vv += v * (d1 * d1 + d2 * d2);
    }
  xbar[2 * i] = a;
  xbar[2 * i + 1] = b;
  var[i] = vv / m;
}

__global__ void k_flow_costs(const double* __restrict__ mom, const double* __restrict__ xbar,
                             const double* __restrict__ var, const double* __restrict__ m, int n1, int n2, int s,
                             double* __restrict__ cbar, long long* __restrict__ C) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n1 * n2) return;
  const int i1 = i / n2, i2 = i - i1 * n2;
  const double z1 = i1 * s + 0.5 * (s - 1), z2 = i2 * s + 0.5 * (s - 1);
  const double M0 = mom[6 * i], M1a = mom[6 * i + 1], M1b = mom[6 * i + 2];
  const double G0 = mom[6 * i + 3], G1 = mom[6 * i + 4];
  cbar[5 * i] = 0.0;
  C[5 * i] = 0;
  for (int a = 1; a < 5; ++a) {
    const int j = nbr_cell(i, a, n1, n2);
    if (j < 0) {
      cbar[5 * i + a] = nan("");
      C[5 * i + a] = 0;
      continue;
    }
    const double x1 = xbar[2 * j] - z1, x2 = xbar[2 * j + 1] - z2;
    const double W = var[j] + x1 * x1 + x2 * x2;
    const double cb = (M0 * W - G0 - 2.0 * (M1a * x1 + M1b * x2) + 2.0 * G1) / m[i];
    cbar[5 * i + a] = cb;
    C[5 * i + a] = __double2ll_rn(cb * 1024.0);   // reading R11: round half even
  }
}

// F3: one CTA per target cell j writes its new box into the spare pool
// (bump-allocated); unchanged cells (w_jj = q_j) are copied.  The weighted
// sum is accumulated in place in the output pool on the hull of the
// contributing boxes (fixed order: self, from up, down, left, right; explicit
// _rn operations), truncated, and compacted to the minimal box.
__global__ void k_apply_flow(const long long* __restrict__ w, const long long* __restrict__ q, int n1, int n2,
                             const double* __restrict__ pool, const long long* __restrict__ pos,
                             const int* __restrict__ off, const int* __restrict__ ext, double* __restrict__ pool_new,
                             long long* __restrict__ pos_new, int* __restrict__ off_new, int* __restrict__ ext_new,
                             unsigned long long* __restrict__ ctr, long long cap, double tau,
                             unsigned long long* __restrict__ counters, double* __restrict__ dropped, int j0) {
  extern __shared__ __align__(16) double rowbuf[];
  __shared__ int src[5];
  __shared__ double frac[5];
  __shared__ int nsrc;
  __shared__ int bnd[4];
  __shared__ long long base;
  __shared__ int mm[4];
  __shared__ double dsum[32];
  const int j = j0 + blockIdx.x, tid = threadIdx.x, T = blockDim.x;
  if (w[5LL * j] == q[j]) {   // no inflow from a neighbour: nu_j unchanged
    const long long len = (long long)ext[2 * j] * ext[2 * j + 1];
    if (tid == 0) {
      long long b = (long long)atomicAdd(ctr, (unsigned long long)len);
      if (b + len > cap) { b = -1; atomicAdd(&counters[1], 1ull); }
      base = b;
    }
    __syncthreads();
    if (base < 0) return;
    for (long long t = tid; t < len; t += T) pool_new[base + t] = pool[pos[j] + t];
    if (tid == 0) {
      pos_new[j] = base;
      off_new[2 * j] = off[2 * j];
      off_new[2 * j + 1] = off[2 * j + 1];
      ext_new[2 * j] = ext[2 * j];
      ext_new[2 * j + 1] = ext[2 * j + 1];
    }
    return;
  }
  if (tid == 0) {
    int k = 0;
    if (w[5LL * j] > 0) { src[k] = j; frac[k] = (double)w[5LL * j] / (double)q[j]; ++k; }
    // from up (its 'down' arc 2), down ('up' 1), left ('right' 4), right ('left' 3)
    const int srcs[4] = {nbr_cell(j, 1, n1, n2), nbr_cell(j, 2, n1, n2), nbr_cell(j, 3, n1, n2),
                         nbr_cell(j, 4, n1, n2)};
    const int arcs[4] = {2, 1, 4, 3};
    for (int t = 0; t < 4; ++t) {
      const int i = srcs[t];
      if (i < 0) continue;
      const long long wij = w[5LL * i + arcs[t]];
      if (wij > 0) { src[k] = i; frac[k] = (double)wij / (double)q[i]; ++k; }
    }
    nsrc = k;
    int L1 = 1 << 30, L2 = 1 << 30, U1 = -1, U2 = -1;
    for (int t = 0; t < k; ++t) {
      const int i = src[t];
      L1 = min(L1, off[2 * i]);
      L2 = min(L2, off[2 * i + 1]);
      U1 = max(U1, off[2 * i] + ext[2 * i]);
      U2 = max(U2, off[2 * i + 1] + ext[2 * i + 1]);
    }
    bnd[0] = L1; bnd[1] = L2; bnd[2] = U1 - L1; bnd[3] = U2 - L2;
    const long long A = (long long)bnd[2] * bnd[3];
    long long b = (long long)atomicAdd(ctr, (unsigned long long)A);
    if (b + A > cap) { b = -1; atomicAdd(&counters[1], 1ull); }
    base = b;
    mm[0] = 1 << 30; mm[1] = -1; mm[2] = 1 << 30; mm[3] = -1;
  }
  __syncthreads();
  if (base < 0) return;
  const int L1 = bnd[0], L2 = bnd[1], b1 = bnd[2], b2 = bnd[3];
  double* acc = pool_new + base;
  for (int t = tid; t < b1 * b2; t += T) acc[t] = 0.0;
  __syncthreads();
  for (int k = 0; k < nsrc; ++k) {
    const int i = src[k];
    const double f = frac[k];
    const int r0 = off[2 * i] - L1, c0 = off[2 * i + 1] - L2, e1 = ext[2 * i], e2 = ext[2 * i + 1];
    const double* d = pool + pos[i];
    for (int t = tid; t < e1 * e2; t += T) {
      const int r = t / e2, c = t - r * e2;
      double* a = &acc[(r0 + r) * b2 + c0 + c];
      *a = __dadd_rn(*a, __dmul_rn(f, d[t]));
    }
    __syncthreads();
  }
  double dr = 0.0;
  for (int t = tid; t < b1 * b2; t += T) {
    const double v = acc[t];
    const int r = t / b2, c = t - r * b2;
    if (v >= tau) {
      atomicMin(&mm[0], r); atomicMax(&mm[1], r); atomicMin(&mm[2], c); atomicMax(&mm[3], c);
    } else if (v > 0.0) {
      dr += v;
    }
  }
  for (int o = 16; o > 0; o >>= 1) dr += __shfl_xor_sync(0xffffffffu, dr, o);
  if ((tid & 31) == 0) dsum[tid >> 5] = dr;
  __syncthreads();
  if (mm[1] < mm[0]) {
    if (tid == 0) atomicAdd(&counters[1], 1ull);
    return;
  }
  const int e1 = mm[1] - mm[0] + 1, e2 = mm[3] - mm[2] + 1;
  // in-place compaction to the minimal box, one row at a time through shared memory
  for (int r = 0; r < e1; ++r) {
    for (int c = tid; c < e2; c += T) {
      const double v = acc[(mm[0] + r) * b2 + mm[2] + c];
      rowbuf[c] = v >= tau ? v : 0.0;
    }
    __syncthreads();
    for (int c = tid; c < e2; c += T) acc[r * e2 + c] = rowbuf[c];
    __syncthreads();
  }
  if (tid == 0) {
    pos_new[j] = base;
    off_new[2 * j] = L1 + mm[0];
    off_new[2 * j + 1] = L2 + mm[2];
    ext_new[2 * j] = e1;
    ext_new[2 * j + 1] = e2;
    double s = 0;
    for (int k = 0; k < (int)(T >> 5); ++k) s += dsum[k];
    atomicAdd(dropped, s);
    atomicAdd(&counters[0], 1ull);
  }
}

// ---- gluing edge candidates (Def. glued-plan
// PAPER.md:531-541, Remark eps-gamma PAPER.md:543-559) ----------------------
// gamma_ij in Pi(mu_i/m_i, mu_j/m_j) is the entropic OT plan for |x - x'|^2
// with regularisation eps_g (pixel^2 units), computed once per problem (it
// depends on mu only): one warp per (cell i, arc a), fp64 log-domain Sinkhorn
// with eps-scaling (factor 4 per stage, 20 iterations per stage, then to an
// L1 marginal error <= tol).  Stored per pixel x of X_i (row-major) as the
// moments of its disintegration gamma~(. | x) about the cell centre z_i:
// b = E[x'] - z_i (2) and delta = E|x' - z_i|^2 (1).
constexpr int kGamWarps = 4;   // warps per block of k_gamma
__global__ void k_gamma(const double* __restrict__ mu, int N2, int s, int n1, int n2, const double* __restrict__ m,
                        double eps_g, double tol, int max_iter, double* __restrict__ gam,
                        unsigned long long* __restrict__ nonconv) {
  __shared__ double sh[kGamWarps][6][64];   // la, lb, fa, fb, pb, tmp
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const long long wid = (long long)blockIdx.x * kGamWarps + wl;
  const int I = n1 * n2;
  if (wid >= 4LL * I) return;
  const int i = (int)(wid / 4), a = 1 + (int)(wid % 4);
  const int j = nbr_cell(i, a, n1, n2);
  const int P = s * s;
  double* out = gam + (size_t)(4LL * i + (a - 1)) * P * 3;
  if (j < 0) {
    for (int p = lane; p < P; p += 32) out[3 * p] = out[3 * p + 1] = out[3 * p + 2] = 0.0;
    return;
  }
  double* la = sh[wl][0];
  double* lb = sh[wl][1];
  double* fa = sh[wl][2];
  double* fb = sh[wl][3];
  double* pb = sh[wl][4];
  const int i1 = i / n2, i2 = i % n2, j1 = j / n2, j2 = j % n2;
  for (int p = lane; p < P; p += 32) {
    la[p] = log(mu[(long long)(i1 * s + p / s) * N2 + i2 * s + p % s] / m[i]);
    const double vb = mu[(long long)(j1 * s + p / s) * N2 + j2 * s + p % s] / m[j];
    lb[p] = log(vb);
    pb[p] = vb;
    fa[p] = 0.0;
    fb[p] = 0.0;
  }
  __syncwarp();
  // D(p, q) = |x_p - x'_q|^2 in pixels (x' = x + (j - i) s offset)
  const int dy = (j1 - i1) * s, dx = (j2 - i2) * s;
  auto D = [&](int p, int q) {
    const double d1 = (double)(q / s + dy - p / s), d2 = (double)(q % s + dx - p % s);
    return d1 * d1 + d2 * d2;
  };
  double dmax = 0.0;
  for (int p = 0; p < P; ++p)
    for (int q = lane; q < P; q += 32) dmax = fmax(dmax, D(p, q));
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  double e = fmax(dmax, eps_g), prev = e;
  bool done = false;
  int iters_left = max_iter;
  while (!done) {
    const bool last = e <= eps_g;
    if (last) e = eps_g;
    for (int p = lane; p < P; p += 32) { fa[p] *= prev / e; fb[p] *= prev / e; }
    __syncwarp();
    prev = e;
    const double ie = 1.0 / e;
    for (int it = 0; it < (last ? iters_left : 20); ++it) {
      for (int q = lane; q < P; q += 32) {   // Y-side (second marginal) update
        double mx = -INFINITY;
        for (int p = 0; p < P; ++p) mx = fmax(mx, fa[p] + la[p] - D(p, q) * ie);
        double sm = 0.0;
        for (int p = 0; p < P; ++p) sm += exp(fa[p] + la[p] - D(p, q) * ie - mx);
        fb[q] = -(mx + log(sm));
      }
      __syncwarp();
      for (int p = lane; p < P; p += 32) {   // X-side update
        double mx = -INFINITY;
        for (int q = 0; q < P; ++q) mx = fmax(mx, fb[q] + lb[q] - D(p, q) * ie);
        double sm = 0.0;
        for (int q = 0; q < P; ++q) sm += exp(fb[q] + lb[q] - D(p, q) * ie - mx);
        fa[p] = -(mx + log(sm));
      }
      __syncwarp();
      if (last && (it % 10 == 9 || it == iters_left - 1)) {
        double err = 0.0;   // L1 error of the second marginal
        for (int q = lane; q < P; q += 32) {
          double cs = 0.0;
          for (int p = 0; p < P; ++p) cs += exp(fa[p] + fb[q] + la[p] + lb[q] - D(p, q) * ie);
          err += fabs(cs - pb[q]);
        }
        for (int o = 16; o > 0; o >>= 1) err += __shfl_xor_sync(0xffffffffu, err, o);
        if (err <= tol) break;
        if (it == iters_left - 1 && lane == 0) atomicAdd(nonconv, 1ull);
      }
    }
    if (last) done = true;
    else e *= 0.25;
  }
  // moments of gamma~(. | x_p) about the cell centre z_i
  const double zc = 0.5 * (double)(s - 1);
  for (int p = lane; p < P; p += 32) {
    double w = 0.0, b1 = 0.0, b2 = 0.0, dd = 0.0;
    for (int q = 0; q < P; ++q) {
      const double g = exp(fa[p] + fb[q] + lb[q] - D(p, q) / prev);
      const double y1 = (double)(q / s + dy) - zc, y2 = (double)(q % s + dx) - zc;
      w += g;
      b1 += g * y1;
      b2 += g * y2;
      dd += g * (y1 * y1 + y2 * y2);
    }
    out[3 * p] = b1 / w;
    out[3 * p + 1] = b2 / w;
    out[3 * p + 2] = dd / w;
  }
}

// Edge costs with gluing candidates (reading R26): for i != j,
//   m_i c_bar_ij = sum_{x in X_i} PX(x) [(delta(x) - |u|^2) - 2 (b(x) - u) . (u + E[y - x | x])],
// u = x - z_i, from the per-pixel records of the last sweep (PX, E[y - x | x])
// and the static gamma tables; the product candidate is the special case
// b = xbar_j - z_i, delta = V_j + |xbar_j - z_i|^2.
__global__ void k_flow_costs_glued(const double* __restrict__ pxm, const double* __restrict__ gam,
                                   const double* __restrict__ m, int N2, int n1, int n2, int s,
                                   double* __restrict__ cbar, long long* __restrict__ C) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n1 * n2) return;
  const int i1 = i / n2, i2 = i - i1 * n2, P = s * s;
  const double zc = 0.5 * (double)(s - 1);
  cbar[5 * i] = 0.0;
  C[5 * i] = 0;
  for (int a = 1; a < 5; ++a) {
    if (nbr_cell(i, a, n1, n2) < 0) {
      cbar[5 * i + a] = nan("");
      C[5 * i + a] = 0;
      continue;
    }
    const double* g = gam + (size_t)(4LL * i + (a - 1)) * P * 3;
    double acc = 0.0;
    for (int p = 0; p < P; ++p) {
      const long long pix = (long long)(i1 * s + p / s) * N2 + i2 * s + p % s;
      const double px = pxm[3 * pix], e1 = pxm[3 * pix + 1], e2 = pxm[3 * pix + 2];
      const double u1 = (double)(p / s) - zc, u2 = (double)(p % s) - zc;
      const double b1 = g[3 * p], b2 = g[3 * p + 1], dl = g[3 * p + 2];
      acc += px * ((dl - (u1 * u1 + u2 * u2)) - 2.0 * ((b1 - u1) * (u1 + e1) + (b2 - u2) * (u2 + e2)));
    }
    const double cb = acc / m[i];
    cbar[5 * i + a] = cb;
    C[5 * i + a] = __double2ll_rn(cb * 1024.0);   // reading R11: round half even
  }
}

__global__ void k_check_flow(const long long* __restrict__ w, const long long* __restrict__ q, int n1, int n2,
                             unsigned long long* __restrict__ bad) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n1 * n2) return;
  long long out = 0, in = 0;
  for (int a = 0; a < 5; ++a) {
    const long long v = w[5LL * j + a];
    if (v < 0) atomicAdd(bad, 1ull);
    if (nbr_cell(j, a, n1, n2) < 0 && v != 0) atomicAdd(bad, 1ull);
    out += v;
  }
  in += w[5LL * j];
  const int srcs[4] = {nbr_cell(j, 1, n1, n2), nbr_cell(j, 2, n1, n2), nbr_cell(j, 3, n1, n2), nbr_cell(j, 4, n1, n2)};
  const int arcs[4] = {2, 1, 4, 3};
  for (int t = 0; t < 4; ++t)
    if (srcs[t] >= 0) in += w[5LL * srcs[t] + arcs[t]];
  if (out != q[j] || in != q[j]) atomicAdd(bad, 1ull);
}

}  // namespace

dd_status flow_init_static(dd_ctx* c) {
  const int I = c->I;
  auto alloc = [&](void** p, size_t bytes) -> dd_status {
    keep_device_pool(c->device);
    cudaError_t e = cudaMallocAsync(p, bytes + 16, c->stream);
    if (e != cudaSuccess) {
      c->err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
      return DD_ERR_OOM;
    }
    return DD_OK;
  };
  dd_status s;
  if ((s = alloc((void**)&c->d_xbar, (size_t)I * 16))) return s;
  if ((s = alloc((void**)&c->d_var, (size_t)I * 8))) return s;
  if ((s = alloc((void**)&c->d_cbar, (size_t)I * 40))) return s;
  if ((s = alloc((void**)&c->d_C, (size_t)I * 40))) return s;
  if ((s = alloc((void**)&c->d_w, (size_t)I * 40))) return s;
  if ((s = alloc((void**)&c->d_flow_info, 64 * 8))) return s;
  // d_scratch still holds mu (fp64) from init
  k_mu_moments<<<(I + 127) / 128, 128, 0, c->stream>>>(c->d_scratch, c->N2, c->s, c->n2, I, c->d_xbar, c->d_var);
  DD_CUDA(cudaGetLastError());
  return DD_OK;
}

static dd_status apply_w(dd_ctx* c, unsigned long long* d_counters, double* d_dropped) {
  const int I = c->I;
  const int cur = c->cur, spare = 1 - c->cur;
  const size_t smem = (size_t)std::max(c->N1, c->N2) * 8;
  if (smem > 48 * 1024)   // per-device attribute: set on every launch
    DD_CUDA(cudaFuncSetAttribute(k_apply_flow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DD_CUDA(cudaMemsetAsync(c->d_poolctr + spare, 0, 8, c->stream));
  // owned rows only (stripe mode: their neighbours' rows must be current)
  (void)I;
  k_apply_flow<<<(c->re - c->rb) * c->n2, 128, smem, c->stream>>>(
      (const long long*)c->d_w, (const long long*)c->d_q, c->n1, c->n2, c->d_pool[cur], c->d_pos[cur],
      c->d_off[cur], c->d_ext[cur], c->d_pool[spare], c->d_pos[spare], c->d_off[spare], c->d_ext[spare],
      c->d_poolctr + spare, c->pool_cap, c->opt.trunc, d_counters, d_dropped, c->rb * c->n2);
  DD_CUDA(cudaGetLastError());
  c->cur = spare;   // the new state (failures are reported by counters[1])
  return DD_OK;
}

dd_status flow_costs_impl(dd_ctx* c) {
  if (c->candidate == 1) {
    if (!c->d_gam) {
      c->err = "gluing candidates selected but the gamma tables are missing";
      return DD_ERR_PRECOND;
    }
    k_flow_costs_glued<<<(c->I + 127) / 128, 128, 0, c->stream>>>(c->d_pxm, c->d_gam, c->d_m, c->N2, c->n1, c->n2,
                                                                 c->s, c->d_cbar, (long long*)c->d_C);
  } else {
    k_flow_costs<<<(c->I + 127) / 128, 128, 0, c->stream>>>(c->d_mom, c->d_xbar, c->d_var, c->d_m, c->n1, c->n2,
                                                           c->s, c->d_cbar, (long long*)c->d_C);
  }
  DD_CUDA(cudaGetLastError());
  return DD_OK;
}

dd_status flow_update_impl(dd_ctx* c, dd_flow_stats* stats) {
  ++c->n_flows;
  dd_status s;
  {
    NvtxRange nv("dd:flow edge costs");
    s = flow_costs_impl(c);
  }
  if (s) return s;
  {
    NvtxRange nv("dd:min-cost flow");
    s = mcf_solve_device(c->n1, c->n2, c->d_q, c->d_C, c->d_w, &c->d_mcf, &c->mcf_bytes, 1, c->stream, c->err);
  }
  if (s) return s;
  unsigned long long* ctr = (unsigned long long*)c->d_flow_info;   // [0] changed, [1] failed
  double* dropped = (double*)(c->d_flow_info + 8);
  DD_CUDA(cudaMemsetAsync(c->d_flow_info, 0, 64 * 8, c->stream));
  s = apply_w(c, ctr, dropped);
  if (s) return s;
  if (stats) {
    long long info[16];
    unsigned long long cnt[2];
    DD_CUDA(cudaMemcpyAsync(info, mcf_info_ptr(c->d_mcf, c->I), sizeof(info), cudaMemcpyDeviceToHost, c->stream));
    DD_CUDA(cudaMemcpyAsync(cnt, ctr, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
    DD_CUDA(cudaStreamSynchronize(c->stream));
    stats->objective = info[0];
    stats->stationary = (int32_t)info[1];
    stats->certificate = (int32_t)info[2];
    stats->refines = (int32_t)info[3];
    stats->rounds = (int32_t)info[4];
    stats->label_rounds = (int32_t)info[5];
    stats->changed_cells = (int64_t)cnt[0];
    stats->solver_ms = info[12] * 1e-6;
    if (getenv("DD_MCF_TIMERS"))
      fprintf(stderr, "mcf timers (ms): refine %.1f update %.1f phase %.1f wait %.1f total %.1f local_rounds %lld\n",
              info[8] * 1e-6, info[9] * 1e-6, info[10] * 1e-6, info[11] * 1e-6, info[12] * 1e-6, info[7]);
    if (info[6]) {
      c->err = "min-cost flow did not converge (round cap)";
      return DD_ERR_NUMERIC;
    }
    if (cnt[1]) {
      c->err = "flow apply: pool capacity exceeded or a cell annihilated (state invalid)";
      return DD_ERR_NUMERIC;
    }
  }
  return DD_OK;
}

}  // namespace dd

using namespace dd;

extern "C" {

dd_status flow_edge_costs(dd_ctx* c, double* cbar, int64_t* C, int64_t* q) {
  if (!c) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  dd_status s = flow_costs_impl(c);
  if (s) return s;
  if (cbar) DD_CUDA(cudaMemcpyAsync(cbar, c->d_cbar, (size_t)c->I * 40, cudaMemcpyDeviceToHost, c->stream));
  if (C) DD_CUDA(cudaMemcpyAsync(C, c->d_C, (size_t)c->I * 40, cudaMemcpyDeviceToHost, c->stream));
  if (q) DD_CUDA(cudaMemcpyAsync(q, c->d_q, (size_t)c->I * 8, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  return DD_OK;
}

dd_status flow_apply(dd_ctx* c, const int64_t* w) {
  if (!c || !w) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  DD_CUDA(cudaMemcpyAsync(c->d_w, w, (size_t)c->I * 40, cudaMemcpyHostToDevice, c->stream));
  unsigned long long* ctr = (unsigned long long*)c->d_flow_info;
  double* dropped = (double*)(c->d_flow_info + 8);
  DD_CUDA(cudaMemsetAsync(c->d_flow_info, 0, 64 * 8, c->stream));
  k_check_flow<<<(c->I + 127) / 128, 128, 0, c->stream>>>((const long long*)c->d_w, (const long long*)c->d_q, c->n1,
                                                         c->n2, ctr + 2);
  DD_CUDA(cudaGetLastError());
  unsigned long long bad = 0;
  DD_CUDA(cudaMemcpyAsync(&bad, ctr + 2, 8, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  if (bad) {
    c->err = "w violates the divergence constraints (PAPER.md:350-354)";
    return DD_ERR_PRECOND;
  }
  dd_status s = apply_w(c, ctr, dropped);
  if (s) return s;
  unsigned long long cnt[2];
  DD_CUDA(cudaMemcpyAsync(cnt, ctr, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  if (cnt[1]) {
    c->err = "flow apply: pool capacity exceeded or a cell annihilated (state invalid)";
    return DD_ERR_NUMERIC;
  }
  return DD_OK;
}

dd_status flow_set_candidate(dd_ctx* c, int32_t candidate, double eps_gamma_p) {
  if (!c || (candidate != 0 && candidate != 1) || (candidate == 1 && !(eps_gamma_p > 0))) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  c->candidate = candidate;
  if (candidate == 0) return DD_OK;
  const long long NN = (long long)c->N1 * c->N2;
  const int P = c->s * c->s;
  if (!c->d_pxm) {
    DD_CUDA(cudaMallocAsync(&c->d_pxm, NN * 24, c->stream));
    DD_CUDA(cudaMemsetAsync(c->d_pxm, 0, NN * 24, c->stream));
  }
  if (!c->d_gam || c->eps_gamma_p != eps_gamma_p) {
    if (!c->d_gam) DD_CUDA(cudaMallocAsync(&c->d_gam, (size_t)c->I * 4 * P * 3 * 8, c->stream));
    c->eps_gamma_p = eps_gamma_p;
    if (P > 64) {
      c->err = "gluing candidates need cell_size <= 8";
      return DD_ERR_ARG;
    }
    unsigned long long* nc = (unsigned long long*)(c->d_flow_info + 32);
    DD_CUDA(cudaMemsetAsync(nc, 0, 8, c->stream));
    const long long warps = 4LL * c->I;
    k_gamma<<<(unsigned)((warps + kGamWarps - 1) / kGamWarps), 32 * kGamWarps, 0, c->stream>>>(
        c->d_mu64, c->N2, c->s, c->n1, c->n2, c->d_m, eps_gamma_p, 1e-12, 20000, c->d_gam, nc);
    DD_CUDA(cudaGetLastError());
    unsigned long long hnc = 0;
    DD_CUDA(cudaMemcpyAsync(&hnc, nc, 8, cudaMemcpyDeviceToHost, c->stream));
    DD_CUDA(cudaStreamSynchronize(c->stream));
    if (hnc) {
      c->err = "gamma_ij Sinkhorn did not reach its tolerance for " + std::to_string(hnc) + " arcs";
      return DD_ERR_NUMERIC;
    }
  }
  return DD_OK;
}

dd_status flow_edge_costs_device(dd_ctx* c, double* d_cbar, int64_t* d_C) {
  if (!c) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  dd_status s = flow_costs_impl(c);
  if (s) return s;
  if (d_cbar) DD_CUDA(cudaMemcpyAsync(d_cbar, c->d_cbar, (size_t)c->I * 40, cudaMemcpyDeviceToDevice, c->stream));
  if (d_C) DD_CUDA(cudaMemcpyAsync(d_C, c->d_C, (size_t)c->I * 40, cudaMemcpyDeviceToDevice, c->stream));
  return DD_OK;
}

dd_status flow_solve(dd_ctx* c, const int64_t* d_C, int64_t* d_w, dd_flow_stats* stats) {
  if (!c || !d_C) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  DD_CUDA(cudaMemcpyAsync(c->d_C, d_C, (size_t)c->I * 40, cudaMemcpyDeviceToDevice, c->stream));
  dd_status s = mcf_solve_device(c->n1, c->n2, c->d_q, c->d_C, c->d_w, &c->d_mcf, &c->mcf_bytes, 1, c->stream, c->err);
  if (s) return s;
  if (d_w) DD_CUDA(cudaMemcpyAsync(d_w, c->d_w, (size_t)c->I * 40, cudaMemcpyDeviceToDevice, c->stream));
  if (stats) {
    long long info[16];
    DD_CUDA(cudaMemcpyAsync(info, mcf_info_ptr(c->d_mcf, c->I), sizeof(info), cudaMemcpyDeviceToHost, c->stream));
    DD_CUDA(cudaStreamSynchronize(c->stream));
    stats->objective = info[0];
    stats->stationary = (int32_t)info[1];
    stats->certificate = (int32_t)info[2];
    stats->refines = (int32_t)info[3];
    stats->rounds = (int32_t)info[4];
    stats->label_rounds = (int32_t)info[5];
    stats->changed_cells = 0;
    stats->solver_ms = info[12] * 1e-6;
    if (info[6]) {
      c->err = "min-cost flow did not converge (round cap)";
      return DD_ERR_NUMERIC;
    }
  }
  return DD_OK;
}

dd_status flow_apply_device(dd_ctx* c, const int64_t* d_w) {
  if (!c || !d_w) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  DD_CUDA(cudaMemcpyAsync(c->d_w, d_w, (size_t)c->I * 40, cudaMemcpyDeviceToDevice, c->stream));
  unsigned long long* ctr = (unsigned long long*)c->d_flow_info;
  double* dropped = (double*)(c->d_flow_info + 8);
  DD_CUDA(cudaMemsetAsync(c->d_flow_info, 0, 64 * 8, c->stream));
  return apply_w(c, ctr, dropped);
}

dd_status dd_mincost_flow(int32_t n1, int32_t n2, const int64_t* q, const int64_t* C, int64_t* w, int64_t* objective,
                          dd_flow_stats* stats, int32_t device, void* stream) {
  if (n1 <= 0 || n2 <= 0 || !q || !C || !w) return DD_ERR_ARG;
  const int I = n1 * n2;
  for (int i = 0; i < I; ++i) {
    if (q[i] <= 0) return DD_ERR_ARG;
    for (int a = 1; a < 5; ++a)
      if (C[5 * i + a] >= (1LL << 40) || C[5 * i + a] <= -(1LL << 40)) return DD_ERR_ARG;
  }
  if (cudaSetDevice(device) != cudaSuccess) return DD_ERR_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t *dq = nullptr, *dC = nullptr, *dw = nullptr;
  void* ws = nullptr;
  size_t wsb = 0;
  std::string err;
  dd_status s = DD_OK;
  keep_device_pool(device);
  if (cudaMallocAsync(&dq, I * 8, st) || cudaMallocAsync(&dC, I * 40, st) || cudaMallocAsync(&dw, I * 40, st)) {
    s = DD_ERR_OOM;
  } else {
    cudaMemcpyAsync(dq, q, I * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dC, C, I * 40, cudaMemcpyHostToDevice, st);
    s = mcf_solve_device(n1, n2, dq, dC, dw, &ws, &wsb, 0, st, err);
    if (s == DD_OK) {
      long long info[16];
      cudaMemcpyAsync(w, dw, I * 40, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(info, mcf_info_ptr(ws, I), sizeof(info), cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) {
        s = DD_ERR_CUDA;
      } else {
        if (objective) *objective = info[0];
        if (stats) {
          stats->objective = info[0];
          stats->stationary = (int32_t)info[1];
          stats->certificate = (int32_t)info[2];
          stats->refines = (int32_t)info[3];
          stats->rounds = (int32_t)info[4];
          stats->label_rounds = (int32_t)info[5];
          stats->changed_cells = 0;
          stats->solver_ms = info[12] * 1e-6;
        }
        if (info[6]) s = DD_ERR_NUMERIC;
        if (getenv("DD_MCF_TIMERS"))
          fprintf(stderr, "mcf timers (ms): refine %.1f update %.1f phase %.1f wait %.1f total %.1f local_rounds %lld\n",
                  info[8] * 1e-6, info[9] * 1e-6, info[10] * 1e-6, info[11] * 1e-6, info[12] * 1e-6, info[7]);
      }
    }
  }
  if (dq) cudaFreeAsync(dq, st);
  if (dC) cudaFreeAsync(dC, st);
  if (dw) cudaFreeAsync(dw, st);
  if (ws) cudaFreeAsync(ws, st);
  cudaStreamSynchronize(st);
  if (s != DD_OK) {
    if (err.empty()) err = s == DD_ERR_NUMERIC ? "min-cost flow did not finish within the round cap"
                                                : std::string("CUDA: ") + cudaGetErrorString(cudaGetLastError());
    set_global_error(err);
  }
  return s;
}

}  // extern "C"
