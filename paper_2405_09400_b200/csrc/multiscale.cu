// multiscale.cu — SURVEY 8(f) row f3: multiscale domain decomposition
// (App. A.2.1 "Multi-scale and eps-scaling"; the
// coarse-to-fine strategy of [BoSch2020, Section 6.4] that the paper uses,
// PAPER.md:1205).  The paper gives no procedure, so this follows DESIGN.md
// readings R23-R25 (the same readings as oracle/multiscale.py):
//   R23 layers N_l = N / 2^(L-1-l) with the same cell size s; mu_l, nu_l are
//       2x2 block sums of the next finer layer (k_coarsen; exact on dyadic
//       inputs);
//   R24 eps = eps' h_l^2 on every layer (eps' of the finest problem), each
//       layer runs the hybrid scheme (Alg. 3) until both
//       sweep-entry errors / ||mu|| <= conv (reading R14) or a cycle cap;
//   R25 refinement (k_refine): for a fine basic cell i' inside coarse basic
//       cell i and a fine pixel y' inside coarse pixel y,
//           nu_i'(y') = (nu_i(y) * (m_i' / m_i)) * (nu(y') / nu_l(y)),
//       in this order in fp64 (_rn: bit-identical to the oracle), then
//       truncate + minimal box (a5).  The coarsest layer starts from the
//       product coupling nu_i = m_i nu (k_product).
// Every step runs in the kernels below or in the sweep / flow kernels; the
// host code only sequences layers and reads the convergence statistics.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.cuh"

namespace dd {
long long* mcf_info_ptr(void* ws, int I);
namespace {

// out (N1/2 x N2/2) = 2x2 block sums of a (R23)
__global__ void k_coarsen(const double* __restrict__ a, int N1, int N2, double* __restrict__ out) {
  const long long n = (long long)(N1 / 2) * (N2 / 2);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(t / (N2 / 2)), c = (int)(t % (N2 / 2));
    const double* p = a + (long long)(2 * r) * N2 + 2 * c;
    out[t] = (p[0] + p[1]) + (p[N2] + p[N2 + 1]);
  }
}

// ry(y') = nu(y') / nu_l(parent(y')), 0 where the coarse pixel is empty (R25)
__global__ void k_ratio(const double* __restrict__ nu_f, const double* __restrict__ nu_c, int N1, int N2,
                        double* __restrict__ ry) {
  const long long n = (long long)N1 * N2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(t / N2), c = (int)(t % N2);
    const double p = nu_c[(long long)(r / 2) * (N2 / 2) + c / 2];
    ry[t] = p > 0.0 ? __ddiv_rn(nu_f[t], p) : 0.0;
  }
}

// Truncate at tau + minimal box (a5) of the box [R0, R0 + E1) x [C0, C0 + E2)
// whose values val(rr, cc) the functor gives, written compactly to the pool
// (bump allocation); one CTA.  The values are evaluated twice (bounds, write)
// with the same operations, hence identically.
template <typename F>
__device__ void emit_box(const F& val, const int R0, const int C0, const int E1, const int E2, const double tau,
                         const int j, double* __restrict__ pool, long long* __restrict__ pos, int* __restrict__ off,
                         int* __restrict__ ext, unsigned long long* __restrict__ ctr, const long long cap,
                         double* __restrict__ dropped, unsigned long long* __restrict__ fail) {
  __shared__ int mm[4];
  __shared__ double dsum[32];
  __shared__ long long base;
  const int tid = threadIdx.x, T = blockDim.x;
  if (tid == 0) { mm[0] = 1 << 30; mm[1] = -1; mm[2] = 1 << 30; mm[3] = -1; }
  __syncthreads();
  double dr = 0.0;
  for (int t = tid; t < E1 * E2; t += T) {
    const int rr = t / E2, cc = t - rr * E2;
    const double v = val(rr, cc);
    if (v >= tau) {
      atomicMin(&mm[0], rr); atomicMax(&mm[1], rr); atomicMin(&mm[2], cc); atomicMax(&mm[3], cc);
    } else if (v > 0.0) {
      dr += v;
    }
  }
  for (int o = 16; o > 0; o >>= 1) dr += __shfl_xor_sync(0xffffffffu, dr, o);
  if ((tid & 31) == 0) dsum[tid >> 5] = dr;
  __syncthreads();
  if (mm[1] < mm[0]) {   // annihilated cell
    if (tid == 0) atomicAdd(fail, 1ull);
    __syncthreads();
    return;
  }
  const int e1 = mm[1] - mm[0] + 1, e2 = mm[3] - mm[2] + 1;
  if (tid == 0) {
    long long b = (long long)atomicAdd(ctr, (unsigned long long)e1 * e2);
    if (b + (long long)e1 * e2 > cap) { b = -1; atomicAdd(fail, 1ull); }
    base = b;
    double s = 0.0;
    for (int k = 0; k < (T >> 5); ++k) s += dsum[k];
    atomicAdd(dropped, s);
  }
  __syncthreads();
  if (base >= 0) {
    for (int t = tid; t < e1 * e2; t += T) {
      const int rr = mm[0] + t / e2, cc = mm[2] + t % e2;
      const double v = val(rr, cc);
      pool[base + t] = v >= tau ? v : 0.0;
    }
    if (tid == 0) {
      pos[j] = base;
      off[2 * j] = R0 + mm[0];
      off[2 * j + 1] = C0 + mm[2];
      ext[2 * j] = e1;
      ext[2 * j + 1] = e2;
    }
  }
  __syncthreads();
}

// Product coupling nu_i = m_i nu on the box [L1, L1 + B1) x [L2, L2 + B2) of
// supp(nu); one CTA per basic cell.
__global__ void k_product(const double* __restrict__ nu, int N2, int L1, int L2, int B1, int B2,
                          const double* __restrict__ m, double tau, double* __restrict__ pool,
                          long long* __restrict__ pos, int* __restrict__ off, int* __restrict__ ext,
                          unsigned long long* __restrict__ ctr, long long cap, double* __restrict__ dropped,
                          unsigned long long* __restrict__ fail) {
  const int i = blockIdx.x;
  const double mi = m[i];
  auto val = [&](int rr, int cc) { return __dmul_rn(mi, nu[(long long)(L1 + rr) * N2 + L2 + cc]); };
  emit_box(val, L1, L2, B1, B2, tau, i, pool, pos, off, ext, ctr, cap, dropped, fail);
}

// Refinement (R25): one CTA per coarse basic cell i, its four children in
// row-major order.
__global__ void k_refine(const double* __restrict__ pool_c, const long long* __restrict__ pos_c,
                         const int* __restrict__ off_c, const int* __restrict__ ext_c, const double* __restrict__ m_c,
                         const double* __restrict__ m_f, const double* __restrict__ ry, int n2c, int n2f, int N2f,
                         double tau, double* __restrict__ pool, long long* __restrict__ pos, int* __restrict__ off,
                         int* __restrict__ ext, unsigned long long* __restrict__ ctr, long long cap,
                         double* __restrict__ dropped, unsigned long long* __restrict__ fail) {
  const int i = blockIdx.x, i1 = i / n2c, i2 = i - (i / n2c) * n2c;
  const int e2 = ext_c[2 * i + 1];
  const int R0 = 2 * off_c[2 * i], C0 = 2 * off_c[2 * i + 1], E1 = 2 * ext_c[2 * i], E2 = 2 * e2;
  const double* d = pool_c + pos_c[i];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      const int j = (2 * i1 + a) * n2f + 2 * i2 + b;
      const double rx = __ddiv_rn(m_f[j], m_c[i]);
      auto val = [&](int rr, int cc) {
        return __dmul_rn(__dmul_rn(d[(rr >> 1) * e2 + (cc >> 1)], rx), ry[(long long)(R0 + rr) * N2f + C0 + cc]);
      };
      emit_box(val, R0, C0, E1, E2, tau, j, pool, pos, off, ext, ctr, cap, dropped, fail);
    }
}

// Warm start of the fine layer's partition A from the coarse layer's A
// potential (reading R25'): the physical potential alpha is kept, so in units
// of eps the fine a is fac = eps_c / eps_f times the coarse a at the parent
// pixel (4 when eps' is the same on both layers, R24; 1 with the paper's
// per-layer eps-scaling over a factor 4, R24').  Every fine A-cell lies inside one coarse A-cell (it is a
// coarse basic cell), so the coarse per-cell gauge constants stay constant
// over a fine cell.  The coarse value is taken back to the global gauge (up
// to its cell constant) as A + 2 w (K - g).kappa (the re-gauge of the sweep
// kernel), and the fine cell stores it with its gauge origin at its X-block
// corner (D = 0), minus the value at that corner.  One CTA per fine A-cell.
__global__ void k_alpha_refine(const float* __restrict__ alpha_c, const int* __restrict__ gauge_c, int N2c, int s,
                               const CompCell* __restrict__ cells_f, int N2f, float w, float fac,
                               float* __restrict__ alpha_f, int* __restrict__ gauge_f) {
  const CompCell cc = cells_f[blockIdx.x];
  const int ncolc = (N2c / s + 1) / 2;   // A-cell columns of the coarse grid
  auto coarse_value = [&](int r, int c) {   // fac x global-gauge coarse potential (log2 units) at fine pixel (r, c)
    const int rc = r >> 1, cl = c >> 1;
    const int K1 = rc - rc % (2 * s), K2 = cl - cl % (2 * s);
    const int Jc = (rc / (2 * s)) * ncolc + cl / (2 * s);
    const float a = alpha_c[(long long)rc * N2c + cl] +
                    2.f * w * ((float)(K1 - gauge_c[2 * Jc]) * (rc - K1) + (float)(K2 - gauge_c[2 * Jc + 1]) * (cl - K2));
    return fac * a;
  };
  const float ref = coarse_value(cc.r0, cc.c0);
  for (int t = threadIdx.x; t < cc.n1 * cc.n2; t += blockDim.x) {
    const int r = cc.r0 + t / cc.n2, c = cc.c0 + t % cc.n2;
    alpha_f[(long long)r * N2f + c] = coarse_value(r, c) - ref;
  }
  if (threadIdx.x == 0) {
    gauge_f[2 * blockIdx.x] = cc.r0;
    gauge_f[2 * blockIdx.x + 1] = cc.c0;
  }
}

void keep_device_pool_ms() {
  int dev = 0;
  cudaGetDevice(&dev);
  keep_device_pool(dev);
}

std::string cuda_msg(const char* what, cudaError_t e) { return std::string(what) + ": " + cudaGetErrorString(e); }

// Device buffers of one device-made initial coupling.
struct Staging {
  double* pool = nullptr;
  long long* pos = nullptr;
  int* off = nullptr;
  int* ext = nullptr;
  unsigned long long* ctr = nullptr;   // [0] used, [1] fail
  double* dropped = nullptr;
  cudaStream_t st = nullptr;            // the pool is stream-ordered (cudaMallocAsync)
  ~Staging() {
    for (void* p : {(void*)pool, (void*)pos, (void*)off, (void*)ext, (void*)ctr, (void*)dropped})
      if (p) cudaFreeAsync(p, st);
  }
  cudaError_t alloc(int I, long long cap, cudaStream_t stream) {
    cudaError_t e;
    st = stream;
    keep_device_pool_ms();
    if ((e = cudaMallocAsync(&pool, (size_t)cap * 8, st)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync(&pos, (size_t)I * 8, st)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync(&off, (size_t)I * 8, st)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync(&ext, (size_t)I * 8, st)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync(&ctr, 16, st)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync(&dropped, 8, st)) != cudaSuccess) return e;
    return cudaSuccess;
  }
};

// Finish a device-made coupling: read back the small metadata, make the ctx.
dd_status finish_staging(Staging& S, int I, const dd_problem* P, const dd_options* O, cudaStream_t st, dd_ctx** out,
                         std::string& err) {
  unsigned long long ctr[2] = {0, 0};
  std::vector<int> hoff(2 * (size_t)I), hext(2 * (size_t)I);
  cudaError_t e;
  if ((e = cudaMemcpyAsync(ctr, S.ctr, 16, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(hoff.data(), S.off, (size_t)I * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(hext.data(), S.ext, (size_t)I * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess) {
    err = cuda_msg("initial coupling", e);
    return DD_ERR_CUDA;
  }
  if (ctr[1]) {
    err = "initial coupling: a basic cell was annihilated by truncation or the staging pool overflowed";
    return DD_ERR_NUMERIC;
  }
  DevInit dev{S.pool, S.pos, S.off, S.ext, (long long)ctr[0], hoff.data(), hext.data()};
  dd_status s = init_with_device_coupling(P, O, dev, out);
  if (s != DD_OK) err = dd_last_error(nullptr);
  return s;
}

std::vector<double> basic_masses(const double* mu, int N1, int N2, int s) {
  const int n1 = N1 / s, n2 = N2 / s;
  std::vector<double> m((size_t)n1 * n2, 0.0);
  for (int r = 0; r < N1; ++r)
    for (int c = 0; c < N2; ++c) m[(size_t)(r / s) * n2 + c / s] += mu[(size_t)r * N2 + c];
  return m;
}

}  // namespace

// Product-coupling context (the coarsest layer's start).
static dd_status product_ctx(const dd_problem* P, const dd_options* O, dd_ctx** out, std::string& err) {
  const int N1 = P->N1, N2 = P->N2, s = P->cell_size;
  if (s <= 0 || N1 % s || N2 % s) {
    err = "cell_size must divide N1 and N2";
    return DD_ERR_ARG;
  }
  const int I = (N1 / s) * (N2 / s);
  int L1 = N1, L2 = N2, U1 = -1, U2 = -1;
  for (int r = 0; r < N1; ++r)
    for (int c = 0; c < N2; ++c)
      if (P->nu[(size_t)r * N2 + c] > 0) {
        L1 = std::min(L1, r); U1 = std::max(U1, r);
        L2 = std::min(L2, c); U2 = std::max(U2, c);
      }
  if (U1 < 0) {
    err = "nu is zero";
    return DD_ERR_PRECOND;
  }
  const int device = O ? O->device : 0;
  cudaStream_t st = O ? (cudaStream_t)O->stream : nullptr;
  if (cudaSetDevice(device) != cudaSuccess) {
    err = "no CUDA device available (libdomdec has no CPU fallback)";
    return DD_ERR_CUDA;
  }
  const std::vector<double> m = basic_masses(P->mu, N1, N2, s);
  const int B1 = U1 - L1 + 1, B2 = U2 - L2 + 1;
  const long long cap = (long long)I * B1 * B2;
  Staging S;
  double *dnu = nullptr, *dm = nullptr;
  cudaError_t e = S.alloc(I, cap, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&dnu, (size_t)N1 * N2 * 8, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&dm, (size_t)I * 8, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dnu, P->nu, (size_t)N1 * N2 * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dm, m.data(), (size_t)I * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(S.ctr, 0, 16, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(S.dropped, 0, 8, st);
  if (e == cudaSuccess) {
    const double tau = (O && O->trunc > 0) ? O->trunc : 1e-15;
    k_product<<<I, 128, 0, st>>>(dnu, N2, L1, L2, B1, B2, dm, tau, S.pool, S.pos, S.off, S.ext, S.ctr, cap,
                                 S.dropped, S.ctr + 1);
    e = cudaGetLastError();
  }
  dd_status res = DD_OK;
  if (e != cudaSuccess) {
    err = cuda_msg("product coupling", e);
    res = e == cudaErrorMemoryAllocation ? DD_ERR_OOM : DD_ERR_CUDA;
  } else {
    res = finish_staging(S, I, P, O, st, out, err);
  }
  cudaStreamSynchronize(st);
  if (dnu) cudaFreeAsync(dnu, st);
  if (dm) cudaFreeAsync(dm, st);
  return res;
}

static dd_status refine_ctx(dd_ctx* c, const dd_problem* P, const dd_options* O, dd_ctx** out, std::string& err) {
  const int N1 = P->N1, N2 = P->N2, s = P->cell_size;
  if (N1 != 2 * c->N1 || N2 != 2 * c->N2 || s != c->s) {
    err = "the fine problem must have twice the coarse grid and the same cell size";
    return DD_ERR_ARG;
  }
  if (cudaSetDevice(c->device) != cudaSuccess) {
    err = "cudaSetDevice failed";
    return DD_ERR_CUDA;
  }
  cudaStream_t st = c->stream;
  const int n1f = N1 / s, n2f = N2 / s, If = n1f * n2f, Ic = c->I;
  const long long NNf = (long long)N1 * N2, NNc = (long long)c->N1 * c->N2;
  // masses of the fine cells; their 2x2 sums must be the coarse masses (R23)
  DevTimer tm;
  const std::vector<double> mf = basic_masses(P->mu, N1, N2, s);
  std::vector<double> mc(Ic);
  std::vector<int> coff(2 * (size_t)Ic), cext(2 * (size_t)Ic);
  cudaError_t e = cudaMemcpyAsync(mc.data(), c->d_m, (size_t)Ic * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(coff.data(), c->d_off[c->cur], (size_t)Ic * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(cext.data(), c->d_ext[c->cur], (size_t)Ic * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    err = cuda_msg("refine: coarse state", e);
    return DD_ERR_CUDA;
  }
  for (int i = 0; i < Ic; ++i) {
    const int i1 = i / c->n2, i2 = i % c->n2;
    double sm = 0.0;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) sm += mf[(size_t)(2 * i1 + a) * n2f + 2 * i2 + b];
    if (std::fabs(sm - mc[i]) > 1e-12 * mc[i]) {
      err = "the fine mu does not coarsen to the coarse mu (R23)";
      return DD_ERR_PRECOND;
    }
  }
  long long cap = 0;
  for (int i = 0; i < Ic; ++i) cap += 16LL * cext[2 * i] * cext[2 * i + 1];
  tm.mark("refine: coarse readback");
  Staging S;
  double *dnuf = nullptr, *dnuc = nullptr, *dry = nullptr, *dmf = nullptr, *dl1 = nullptr;
  e = S.alloc(If, cap, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&dnuf, NNf * 8, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&dnuc, NNc * 8, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&dry, NNf * 8, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&dmf, (size_t)If * 8, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&dl1, 8, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dnuf, P->nu, NNf * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dmf, mf.data(), (size_t)If * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(S.ctr, 0, 16, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(S.dropped, 0, 8, st);
  dd_status res = DD_OK;
  if (e == cudaSuccess) {
    k_coarsen<<<592, 256, 0, st>>>(dnuf, N1, N2, dnuc);
    k_ratio<<<592, 256, 0, st>>>(dnuf, dnuc, N1, N2, dry);
    const double tau = c->opt.trunc;
    k_refine<<<Ic, 128, 0, st>>>(c->d_pool[c->cur], c->d_pos[c->cur], c->d_off[c->cur], c->d_ext[c->cur], c->d_m,
                                 dmf, dry, c->n2, n2f, N2, tau, S.pool, S.pos, S.off, S.ext, S.ctr, cap, S.dropped,
                                 S.ctr + 1);
    e = cudaGetLastError();
  }
  tm.mark("refine: staging + kernels");
  if (e == cudaSuccess) {
    // the fine nu must coarsen to the coarse one (R23), exactly for dyadic data
    std::vector<double> hc((size_t)NNc), hn((size_t)NNc);
    e = cudaMemcpyAsync(hc.data(), dnuc, NNc * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hn.data(), c->d_nu, NNc * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
      double l1 = 0.0, tot = 0.0;
      for (long long t = 0; t < NNc; ++t) { l1 += std::fabs(hc[t] - hn[t]); tot += hn[t]; }
      if (l1 > 1e-12 * tot) {
        err = "the fine nu does not coarsen to the coarse nu (R23)";
        res = DD_ERR_PRECOND;
      }
    }
  }
  if (e != cudaSuccess) {
    err = cuda_msg("refine", e);
    res = e == cudaErrorMemoryAllocation ? DD_ERR_OOM : DD_ERR_CUDA;
  } else if (res == DD_OK) {
    tm.mark("refine: nu check");
    res = finish_staging(S, If, P, O, st, out, err);
    tm.mark("refine: finish staging (init)");
    if (res == DD_OK && c->alpha_valid[0] && !c->stripe && !(*out)->stripe) {
      dd_ctx* f = *out;
      // potential in units of eps: x eps_c / eps_f = 4 eps'_c / eps'_f (R25', R24')
      k_alpha_refine<<<f->ncells[0], 64, 0, f->stream>>>(c->d_alpha[0], c->d_gauge[0], c->N2, s, f->d_cells[0], N2,
                                                        (float)(1.4426950408889634 / c->eps_p),
                                                        (float)(4.0 * c->eps_p / f->eps_p), f->d_alpha[0],
                                                        f->d_gauge[0]);
      if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(f->stream)) != cudaSuccess) {
        err = cuda_msg("refine: potential", e);
        res = DD_ERR_CUDA;
      } else {
        f->alpha_valid[0] = 1;
      }
    }
  }
  cudaStreamSynchronize(st);
  for (void* p : {(void*)dnuf, (void*)dnuc, (void*)dry, (void*)dmf, (void*)dl1})
    if (p) cudaFreeAsync(p, st);
  tm.mark("refine: alpha + frees");
  return res;
}

}  // namespace dd

using namespace dd;

extern "C" {

dd_status domdec_init_product(const dd_problem* problem, const dd_options* options, dd_ctx** out) {
  if (!out || !problem || !problem->mu || !problem->nu) return DD_ERR_ARG;
  *out = nullptr;
  std::string err;
  dd_status s = product_ctx(problem, options, out, err);
  if (s != DD_OK) set_global_error(err);
  return s;
}

dd_status domdec_refine(dd_ctx* coarse, const dd_problem* fine, const dd_options* options, dd_ctx** out) {
  if (!out || !coarse || !fine || !fine->mu || !fine->nu) return DD_ERR_ARG;
  *out = nullptr;
  std::string err;
  dd_status s = refine_ctx(coarse, fine, options, out, err);
  if (s != DD_OK) set_global_error(err);
  return s;
}

dd_status dd_multiscale_solve(const dd_problem* P, const dd_options* O, const dd_ms_options* ms, dd_ctx** out,
                              dd_ms_stats* stats) {
  using clk = std::chrono::steady_clock;
  if (!out || !P || !P->mu || !P->nu || !ms) return DD_ERR_ARG;
  *out = nullptr;
  const int L = ms->levels, s = P->cell_size;
  if (L < 1 || L > 16) {
    set_global_error("levels must be in [1, 16]");
    return DD_ERR_ARG;
  }
  const int f = 1 << (L - 1);
  if (P->N1 % (f * s) || P->N2 % (f * s) || P->N1 / f / s < 2 || P->N2 / f / s < 2) {
    set_global_error("N1, N2 must be multiples of 2^(levels-1) s with >= 2 coarsest basic cells per axis");
    return DD_ERR_ARG;
  }
  const auto t_start = clk::now();
  // layers (R23): 2x2 block sums on the device, coarsest first
  std::vector<std::vector<double>> mus(L), nus(L);
  const int device = O ? O->device : 0;
  cudaStream_t st = O ? (cudaStream_t)O->stream : nullptr;
  if (cudaSetDevice(device) != cudaSuccess) {
    set_global_error("no CUDA device available (libdomdec has no CPU fallback)");
    return DD_ERR_CUDA;
  }
  {
    const long long NN = (long long)P->N1 * P->N2;
    double *da = nullptr, *db = nullptr;
    keep_device_pool_ms();
    cudaError_t e = cudaMallocAsync(&da, NN * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&db, NN * 8, st);
    for (int which = 0; which < 2 && e == cudaSuccess; ++which) {
      std::vector<std::vector<double>>& dst = which ? nus : mus;
      const double* src = which ? P->nu : P->mu;
      dst[L - 1].assign(src, src + NN);
      e = cudaMemcpyAsync(da, src, NN * 8, cudaMemcpyHostToDevice, st);
      int N1 = P->N1, N2 = P->N2;
      for (int l = L - 2; l >= 0 && e == cudaSuccess; --l) {
        k_coarsen<<<592, 256, 0, st>>>(da, N1, N2, db);
        N1 /= 2;
        N2 /= 2;
        dst[l].resize((size_t)N1 * N2);
        e = cudaMemcpyAsync(dst[l].data(), db, (size_t)N1 * N2 * 8, cudaMemcpyDeviceToHost, st);
        std::swap(da, db);
      }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (da) cudaFreeAsync(da, st);
    if (db) cudaFreeAsync(db, st);
    cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_global_error(cuda_msg("multiscale layers", e));
      return DD_ERR_CUDA;
    }
  }
  const double eps_p = P->eps / (P->h * P->h);
  // R24': eps' stages of every layer, eps' F, eps' F / 2, ..., eps' (F = eps_scale)
  std::vector<double> stages{eps_p * std::max(1.0, ms->eps_scale)};
  while (stages.back() > eps_p * (1 + 1e-12)) stages.push_back(std::max(eps_p, stages.back() / 2));
  // Marginal-pool slot size of every layer from the FINAL eps' (R24'): the
  // larger eps' of the first stages only widens boxes for a cycle or two,
  // which the 2x initial-data term of the capacity covers; sizing from the
  // first stage's eps' doubled the pools at 2048^2 (~50 GB) and made layer
  // construction grow the memory pool.
  dd_options Os = O ? *O : dd_options{};
  if (!O) {
    Os.err = 1e-4;
    Os.max_iter = 2000;
    Os.trunc = 1e-15;
  }
  if (Os.slot_cap <= 0) {
    const int typ = 2 * s + 2 * (int)std::ceil(std::sqrt(eps_p * std::log(1e10))) + 12;
    Os.slot_cap = typ * typ;
  }
  dd_ms_stats S{};
  S.levels = L;
  dd_ctx* c = nullptr;
  std::string err;
  NvtxRange nv("dd:multiscale_solve");
  for (int l = 0; l < L; ++l) {
    const auto t0 = clk::now();
    char lname[32];
    snprintf(lname, sizeof(lname), "dd:layer %d", l);
    NvtxRange nvl(lname);
    dd_problem Q = *P;
    const int div = 1 << (L - 1 - l);
    Q.N1 = P->N1 / div;
    Q.N2 = P->N2 / div;
    Q.h = P->h * div;
    Q.eps = stages[0] * Q.h * Q.h;   // R24 / R24' (first stage)
    Q.mu = mus[l].data();
    Q.nu = nus[l].data();
    Q.init_off = nullptr; Q.init_ext = nullptr; Q.init_pos = nullptr; Q.init_data = nullptr;
    dd_ctx* next = nullptr;
    dd_status r = l == 0 ? product_ctx(&Q, &Os, &next, err) : refine_ctx(c, &Q, &Os, &next, err);
    DevTimer tmd;
    if (c) domdec_destroy(c);
    tmd.mark("multiscale: destroy coarse");
    c = next;
    if (r != DD_OK) {
      set_global_error(err);
      return r;
    }
    S.init_seconds[l] = std::chrono::duration<double>(clk::now() - t0).count();
    double smu = 0.0;
    for (double v : mus[l]) smu += v;
    S.N[l] = Q.N1;
    int cyc = 0;
    double emax = INFINITY;
    // one host read-back per cycle (device-resident sweep totals and flow
    // result, one synchronisation), flow updates timed with CUDA events
    cudaEvent_t ef0 = nullptr, ef1 = nullptr;
    cudaEventCreate(&ef0);
    cudaEventCreate(&ef1);
    auto fail = [&](const char* what, dd_status st) {
      set_global_error(std::string(what) + dd_last_error(c));
      cudaEventDestroy(ef0);
      cudaEventDestroy(ef1);
      domdec_destroy(c);
      return st;
    };
    int total = 0;
    for (size_t stage = 0; stage < stages.size(); ++stage) {
    if (stage > 0 && (r = domdec_set_eps(c, stages[stage] * Q.h * Q.h)) != DD_OK) return fail("multiscale eps: ", r);
    S.converged[l] = 0;
    // intermediate stages: eps_stage_cycles cycles each (0: until conv); the last stage until conv
    const int cap = (stage + 1 < stages.size() && ms->eps_stage_cycles > 0) ? ms->eps_stage_cycles : ms->max_cycles;
    for (cyc = 0; cyc < cap; ++cyc) {
      if ((r = domdec_sweep(c, DD_PART_A, nullptr)) != DD_OK || (r = domdec_sweep(c, DD_PART_B, nullptr)) != DD_OK)
        return fail("multiscale sweep: ", r);
      const bool doflow = ms->flow_every > 0 && (cyc % ms->flow_every) == ms->flow_every - 1;
      if (doflow) {
        cudaEventRecord(ef0, c->stream);
        if ((r = flow_update(c, nullptr)) != DD_OK) return fail("multiscale flow update: ", r);
        cudaEventRecord(ef1, c->stream);
      }
      SweepTotals ta{}, tb{};
      long long info[16] = {0};
      unsigned long long fcnt[2] = {0, 0};
      cudaMemcpyAsync(&ta, c->d_totals[0], sizeof(ta), cudaMemcpyDeviceToHost, c->stream);
      cudaMemcpyAsync(&tb, c->d_totals[1], sizeof(tb), cudaMemcpyDeviceToHost, c->stream);
      if (doflow) {
        cudaMemcpyAsync(info, mcf_info_ptr(c->d_mcf, c->I), sizeof(info), cudaMemcpyDeviceToHost, c->stream);
        cudaMemcpyAsync(fcnt, c->d_flow_info, sizeof(fcnt), cudaMemcpyDeviceToHost, c->stream);
      }
      if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
        c->err = cudaGetErrorString(cudaGetLastError());
        return fail("multiscale cycle: ", DD_ERR_CUDA);
      }
      if (ta.overflow || tb.overflow) {
        c->err = "box capacity exceeded or pool exhausted";
        return fail("multiscale sweep: ", DD_ERR_NUMERIC);
      }
      if (doflow) {
        float ms_f = 0.f;
        cudaEventElapsedTime(&ms_f, ef0, ef1);
        S.flow_seconds[l] += 1e-3 * ms_f;
        if (info[6] || fcnt[1]) {
          c->err = info[6] ? "min-cost flow did not converge" : "flow apply: pool exhausted";
          return fail("multiscale flow update: ", DD_ERR_NUMERIC);
        }
        S.flows[l] += info[1] ? 0 : 1;
      }
      // a non-finite error never counts as converged
      emax = (std::isfinite(ta.e0) && std::isfinite(tb.e0)) ? std::max(ta.e0, tb.e0) / smu : INFINITY;
      if (emax <= ms->conv) {
        S.converged[l] = 1;
        ++cyc;
        break;
      }
    }
    total += cyc;
    }   // stages
    cudaEventDestroy(ef0);
    cudaEventDestroy(ef1);
    S.cycles[l] = total;
    S.entry_error[l] = emax;
    S.seconds[l] = std::chrono::duration<double>(clk::now() - t0).count();
  }
  S.total_seconds = std::chrono::duration<double>(clk::now() - t_start).count();
  if (stats) *stats = S;
  *out = c;
  return DD_OK;
}

}  // extern "C"
