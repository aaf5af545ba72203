// api.cu — C-ABI entry points of libdomdec (include/domdec.h).
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.cuh"

using namespace dd;

static std::string g_last_error;   // errors with no ctx (init / standalone solver)
namespace dd {
void set_global_error(const std::string& m) { g_last_error = m; }
}  // namespace dd

// Context memory comes from the device's stream-ordered pool (cudaMallocAsync,
// freed with cudaFreeAsync): multiscale layers and tests create and destroy
// contexts of several GB.  The library allocates device memory from the device's stream-ordered pool
// only (cudaMallocAsync).  The pool keeps what it has mapped (release
// threshold = max) and is pre-grown once per process (DD_POOL_RESERVE_GB,
// default min(80 GB, free / 2): the 2048^2 multiscale solve peaks at
// ~67 GB): growing a pool maps physical memory, and
// growth in the middle of a multiscale solve cost 0.1-1 s per layer
// (profiles/r02_pool_timers.txt).
namespace dd {
void keep_device_pool(int dev) {
  static bool done[256] = {};
  if (dev < 0 || dev >= 256 || done[dev]) return;
  done[dev] = true;
  cudaMemPool_t mp;
  if (cudaDeviceGetDefaultMemPool(&mp, dev) != cudaSuccess) return;
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
  size_t fr = 0, tot = 0;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != dev) cudaSetDevice(dev);
  double gb = 80.0;
  if (const char* env = getenv("DD_POOL_RESERVE_GB")) gb = atof(env);
  if (gb > 0 && cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
    size_t want = std::min((size_t)(gb * (1ull << 30)), fr / 2);
    void* p = nullptr;
    if (want > 0 && cudaMallocAsync(&p, want, 0) == cudaSuccess) {
      cudaFreeAsync(p, 0);
      cudaStreamSynchronize(0);
    }
    cudaGetLastError();   // a reservation that does not fit is not an error
  }
  if (cur != dev) cudaSetDevice(cur);
}
}  // namespace dd

namespace {

__global__ void k_init_mu(const double* __restrict__ mu, float* __restrict__ muf, float* __restrict__ l2,
                          long long n) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < n) {
    const double v = mu[t];
    muf[t] = (float)v;
    l2[t] = v > 0.0 ? (float)log2(v) : kNeg;
  }
}

// Y-marginal of the stored state: scatter-add all boxes (diagnostic, fp64).
__global__ void k_scatter_boxes(const double* __restrict__ pool, const long long* __restrict__ pos,
                                const int* __restrict__ off, const int* __restrict__ ext, int N2,
                                double* __restrict__ acc, int i0) {
  const int i = i0 + blockIdx.x;
  const int r0 = off[2 * i], c0 = off[2 * i + 1], e1 = ext[2 * i], e2 = ext[2 * i + 1];
  const double* src = pool + pos[i];
  for (int t = threadIdx.x; t < e1 * e2; t += blockDim.x) {
    const int r = t / e2, c = t - r * e2;
    atomicAdd(&acc[(long long)(r0 + r) * N2 + c0 + c], src[t]);
  }
}

// Halo pack / unpack: one CTA per cell of the row; meta[3 k .. 3 k + 2] =
// (source element offset, destination element offset, length).
__global__ void k_copy_boxes(const double* __restrict__ src, double* __restrict__ dst,
                             const long long* __restrict__ meta) {
  const long long s0 = meta[3 * blockIdx.x], d0 = meta[3 * blockIdx.x + 1], len = meta[3 * blockIdx.x + 2];
  for (long long t = threadIdx.x; t < len; t += blockDim.x) dst[d0 + t] = src[s0 + t];
}

// Halo buffers (domdec_halo_pack): int64 total bytes, int32 off[n2][2],
// int32 ext[n2][2], then the fp64 boxes (head = 8 + 16 n2 bytes).  The
// metadata kernels run on one thread (n2 <= a few thousand cells) and build
// the per-cell copy list meta[3 k .. 3 k + 2] = (source element, destination
// element, length) for k_copy_boxes; no host round trip.
__global__ void k_halo_meta_pack(const long long* __restrict__ pos, const int* __restrict__ off,
                                 const int* __restrict__ ext, int i0, int n2, long long cap, char* __restrict__ buf,
                                 long long* __restrict__ meta) {
  if (threadIdx.x != 0) return;
  const long long head = 8 + 16LL * n2;
  int* ho = (int*)(buf + 8);
  int* he = ho + 2 * n2;
  long long at = 0;
  for (int k = 0; k < n2; ++k) {
    const int i = i0 + k;
    const long long len = (long long)ext[2 * i] * ext[2 * i + 1];
    ho[2 * k] = off[2 * i];
    ho[2 * k + 1] = off[2 * i + 1];
    he[2 * k] = ext[2 * i];
    he[2 * k + 1] = ext[2 * i + 1];
    meta[3 * k] = pos[i];
    meta[3 * k + 1] = head / 8 + at;
    meta[3 * k + 2] = len;
    at += len;
  }
  const long long total = head + 8 * at;
  *(long long*)buf = total;   // > cap: the receiver rejects the buffer
  if (total > cap)
    for (int k = 0; k < n2; ++k) meta[3 * k + 2] = 0;
}

__global__ void k_halo_meta_unpack(const char* __restrict__ buf, long long bytes, int i0, int n2, int N1, int N2,
                                   unsigned long long* __restrict__ poolctr, long long pool_cap,
                                   long long* __restrict__ pos, int* __restrict__ off, int* __restrict__ ext,
                                   long long* __restrict__ meta, unsigned long long* __restrict__ invalid) {
  if (threadIdx.x != 0) return;
  const long long head = 8 + 16LL * n2;
  const int* ho = (const int*)(buf + 8);
  const int* he = ho + 2 * n2;
  long long at = 0;
  bool ok = *(const long long*)buf <= bytes;
  for (int k = 0; k < n2 && ok; ++k) {
    ok = he[2 * k] >= 1 && he[2 * k + 1] >= 1 && ho[2 * k] >= 0 && ho[2 * k + 1] >= 0 &&
         ho[2 * k] + he[2 * k] <= N1 && ho[2 * k + 1] + he[2 * k + 1] <= N2;
    at += (long long)he[2 * k] * he[2 * k + 1];
  }
  ok = ok && head + 8 * at == *(const long long*)buf;
  long long base = -1;
  if (ok) {
    base = (long long)atomicAdd(poolctr, (unsigned long long)at);
    ok = base + at <= pool_cap;
  }
  if (!ok) {
    atomicAdd(invalid, 1ull);
    for (int k = 0; k < n2; ++k) meta[3 * k + 2] = 0;
    return;
  }
  at = 0;
  for (int k = 0; k < n2; ++k) {
    const int i = i0 + k;
    const long long len = (long long)he[2 * k] * he[2 * k + 1];
    meta[3 * k] = head / 8 + at;
    meta[3 * k + 1] = base + at;
    meta[3 * k + 2] = len;
    pos[i] = base + at;
    off[2 * i] = ho[2 * k];
    off[2 * i + 1] = ho[2 * k + 1];
    ext[2 * i] = he[2 * k];
    ext[2 * i + 1] = he[2 * k + 1];
    at += len;
  }
}

// Deterministic single-block reductions for the diagnostics.
__global__ void k_l1_diff(const double* __restrict__ a, const double* __restrict__ b, long long n,
                          double* __restrict__ out) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (long long t = threadIdx.x; t < n; t += blockDim.x) s += fabs(a[t] - b[t]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

__global__ void k_sum_stats(const CellStats* __restrict__ st, int n, double* __restrict__ out) {
  __shared__ double s0[256], s1[256];
  double a = 0.0, b = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    a += (double)st[t].e;
    b += (double)st[t].e0;
  }
  s0[threadIdx.x] = a;
  s1[threadIdx.x] = b;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s0[threadIdx.x] += s0[threadIdx.x + o];
      s1[threadIdx.x] += s1[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s0[0];
    out[1] = s1[0];
  }
}

std::vector<CompCell> build_partition(int n1, int n2, int s, int kind) {
  // Def. partitions; A = {2j, 2j+1}, B = {2j-1, 2j} clipped (R4)
  std::vector<std::vector<int>> rows, cols;
  if (kind == 0) {
    for (int j = 0; 2 * j < n1; ++j) {
      std::vector<int> r;
      for (int x : {2 * j, 2 * j + 1})
        if (x < n1) r.push_back(x);
      rows.push_back(r);
    }
    for (int j = 0; 2 * j < n2; ++j) {
      std::vector<int> r;
      for (int x : {2 * j, 2 * j + 1})
        if (x < n2) r.push_back(x);
      cols.push_back(r);
    }
  } else {
    for (int j = 0; j <= n1 / 2; ++j) {
      std::vector<int> r;
      for (int x : {2 * j - 1, 2 * j})
        if (x >= 0 && x < n1) r.push_back(x);
      if (!r.empty()) rows.push_back(r);
    }
    for (int j = 0; j <= n2 / 2; ++j) {
      std::vector<int> r;
      for (int x : {2 * j - 1, 2 * j})
        if (x >= 0 && x < n2) r.push_back(x);
      if (!r.empty()) cols.push_back(r);
    }
  }
  std::vector<CompCell> out;
  for (auto& rr : rows)
    for (auto& cc : cols) {
      CompCell c{};
      c.r0 = rr[0] * s;
      c.c0 = cc[0] * s;
      c.n1 = (int)rr.size() * s;
      c.n2 = (int)cc.size() * s;
      c.nmem = 0;
      for (size_t a = 0; a < rr.size(); ++a)
        for (size_t b = 0; b < cc.size(); ++b) {
          c.mem[c.nmem] = rr[a] * n2 + cc[b];
          c.quad[c.nmem] = ((int)a << 1) | (int)b;
          ++c.nmem;
        }
      for (int k = c.nmem; k < 4; ++k) {
        c.mem[k] = -1;
        c.quad[k] = 0;
      }
      out.push_back(c);
    }
  return out;
}

template <class T>
dd_status dalloc(dd_ctx* c, T** p, size_t n) {
  keep_device_pool(c->device);
  cudaError_t e = cudaMallocAsync((void**)p, n * sizeof(T) + 16, c->stream);
  if (e != cudaSuccess) {
    c->err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? DD_ERR_OOM : DD_ERR_CUDA;
  }
  return DD_OK;
}

void free_ctx(dd_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  // dalloc'd (stream-ordered pool) and cudaMalloc'd (flow / solver / diagnostics) memory
  void* pooled[] = {c->d_pos[0], c->d_pos[1], c->d_poolctr, c->d_scratch_huge, c->d_mu, c->d_log2mu, c->d_nu,
                    c->d_m, c->d_q, c->d_pool[0], c->d_pool[1], c->d_off[0], c->d_off[1], c->d_ext[0], c->d_ext[1],
                    c->d_cells[0], c->d_cells[1], c->d_alpha[0], c->d_alpha[1], c->d_gauge[0], c->d_gauge[1],
                    c->d_stats[0], c->d_stats[1], c->d_totals[0], c->d_totals[1], c->d_mom, c->d_scratch, c->d_red,
                    c->d_cls, c->d_cum, c->d_mu64, c->d_ecell, c->d_halo, c->d_xbar, c->d_var, c->d_cbar,
                    c->d_C, c->d_w, c->d_mcf, c->d_flow_info, c->d_pxm, c->d_gam, c->d_pd, c->d_hist};
  if (c->cyc_exec) cudaGraphExecDestroy(c->cyc_exec);
  for (void* p : pooled)
    if (p) cudaFreeAsync(p, c->stream);
  if (c->stream) cudaStreamSynchronize(c->stream);
  else cudaDeviceSynchronize();
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->aux) cudaStreamDestroy(c->aux);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  delete c;
}

}  // namespace

#define TRY(x)                     \
  do {                             \
    dd_status s_ = (x);            \
    if (s_ != DD_OK) return s_;    \
  } while (0)

// Per basic cell box mass (initial-coupling check of the device init path).
// A device-made coupling (multiscale refinement of a coarse state) carries the
// coarse state's truncation ledger (reading R9): every cell's mass defect
// m_i - ||nu_i|| is >= 0 after balancing and their sum is the total deficit,
// which the L1 Y-error bounds, so each cell must match m_i within 1e-6 m_i
// plus that L1 Y-error (slack).
__global__ void k_box_mass(const double* __restrict__ pool, const long long* __restrict__ pos,
                           const int* __restrict__ ext, const double* __restrict__ m, int I, double slack,
                           unsigned long long* __restrict__ bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= I) return;
  const long long len = (long long)ext[2 * i] * ext[2 * i + 1];
  double s = 0.0;
  bool ok = true;
  for (long long t = 0; t < len; ++t) {
    const double v = pool[pos[i] + t];
    ok = ok && v >= 0.0 && isfinite(v);
    s += v;
  }
  if (!ok || fabs(s - m[i]) > 1e-6 * m[i] + slack) atomicAdd(bad, 1ull);
}

// init_impl: P's initial coupling comes either from host arrays (the public
// domdec_init) or, with dev != NULL, from device arrays written by a kernel
// of the library (multiscale refinement, multiscale.cu); then P->init_* are
// ignored and the coupling is checked on the device.
static dd_status init_impl(const dd_problem* P, const dd_options* O, dd_ctx* c, const DevInit* dev = nullptr) {
  if (!P || !P->mu || !P->nu || (!dev && (!P->init_off || !P->init_ext || !P->init_pos || !P->init_data))) {
    c->err = "NULL problem pointer";
    return DD_ERR_ARG;
  }
  if (P->N1 <= 0 || P->N2 <= 0 || P->cell_size <= 0 || P->N1 % P->cell_size || P->N2 % P->cell_size) {
    c->err = "cell_size must be positive and divide N1 and N2";
    return DD_ERR_ARG;
  }
  if (P->cell_size != 1 && P->cell_size != 2 && P->cell_size != 4 && P->cell_size != 8) {
    c->err = "cell_size must be 1, 2, 4 or 8 in this build";
    return DD_ERR_ARG;
  }
  if (!(P->eps > 0) || !(P->h > 0)) {
    c->err = "eps and h must be > 0";
    return DD_ERR_ARG;
  }
  c->N1 = P->N1;
  c->N2 = P->N2;
  c->s = P->cell_size;
  c->n1 = c->N1 / c->s;
  c->n2 = c->N2 / c->s;
  c->I = c->n1 * c->n2;
  c->h = P->h;
  c->eps = P->eps;
  c->eps_p = P->eps / (P->h * P->h);
  c->eps_p_init = c->eps_p;
  c->E = P->mass_exponent;
  dd_options def{};
  def.err = 1e-4;
  def.max_iter = 2000;
  def.fixed_iter = 0;
  def.trunc = 1e-15;
  c->opt = O ? *O : def;
  if (!(c->opt.err > 0)) c->opt.err = 1e-4;
  if (c->opt.max_iter <= 0) c->opt.max_iter = 2000;
  if (c->opt.trunc < 0) {
    c->err = "trunc must be >= 0";
    return DD_ERR_ARG;
  }
  if (O == nullptr) c->opt.trunc = 1e-15;
  c->device = c->opt.device;
  // stripe mode: owned basic-cell rows [rb, re)
  if (c->opt.row_begin == 0 && c->opt.row_end == 0) {
    c->rb = 0;
    c->re = c->n1;
  } else {
    c->rb = c->opt.row_begin;
    c->re = c->opt.row_end;
    if (c->rb < 0 || c->re > c->n1 || c->rb >= c->re || (c->rb & 1) || ((c->re & 1) && c->re != c->n1)) {
      c->err = "row range must satisfy 0 <= row_begin < row_end <= n1 with even boundaries (A-cell rows)";
      return DD_ERR_ARG;
    }
  }
  c->stripe = !(c->rb == 0 && c->re == c->n1);
  const long long NN = (long long)c->N1 * c->N2;
  const int I = c->I, s = c->s;
  DevTimer tm;
  // ---- host validation (PAPER.md:233 m_i > 0; feasibility of pi^0) ----------
  std::vector<double> m(I, 0.0);
  double smu = 0, snu = 0;
  for (long long t = 0; t < NN; ++t) {
    if (!(P->mu[t] >= 0) || !(P->nu[t] >= 0) || !std::isfinite(P->mu[t]) || !std::isfinite(P->nu[t])) {
      c->err = "mu and nu must be finite and >= 0";
      return DD_ERR_PRECOND;
    }
    smu += P->mu[t];
    snu += P->nu[t];
    const int r = (int)(t / c->N2), cl = (int)(t % c->N2);
    m[(r / s) * c->n2 + cl / s] += P->mu[t];
  }
  for (int i = 0; i < I; ++i)
    if (!(m[i] > 0)) {
      c->err = "zero-mass basic cell " + std::to_string(i) + " (PAPER.md:233 requires m_i > 0)";
      return DD_ERR_PRECOND;
    }
  if (std::fabs(smu - snu) > 1e-6 * smu) {
    c->err = "sum(mu) != sum(nu)";
    return DD_ERR_PRECOND;
  }
  std::vector<double> acc(dev ? 0 : NN, 0.0);
  int maxext1 = 0, maxext2 = 0;
  long long maxbox = 0;
  const int* hoff = dev ? dev->h_off : P->init_off;
  const int* hext = dev ? dev->h_ext : P->init_ext;
  for (int i = 0; i < I; ++i) {
    const int r0 = hoff[2 * i], c0 = hoff[2 * i + 1];
    const int e1 = hext[2 * i], e2 = hext[2 * i + 1];
    if (e1 < 1 || e2 < 1 || r0 < 0 || c0 < 0 || r0 + e1 > c->N1 || c0 + e2 > c->N2 || (!dev && P->init_pos[i] < 0)) {
      c->err = "initial box " + std::to_string(i) + " outside the grid";
      return DD_ERR_PRECOND;
    }
    maxext1 = std::max(maxext1, e1);
    maxext2 = std::max(maxext2, e2);
    maxbox = std::max(maxbox, (long long)e1 * e2);
    if (dev) continue;   // values are checked on the device below
    double mass = 0;
    for (int a = 0; a < e1; ++a)
      for (int b = 0; b < e2; ++b) {
        const double v = P->init_data[P->init_pos[i] + (long long)a * e2 + b];
        if (!(v >= 0) || !std::isfinite(v)) {
          c->err = "initial box values must be finite and >= 0";
          return DD_ERR_PRECOND;
        }
        acc[(long long)(r0 + a) * c->N2 + c0 + b] += v;
        mass += v;
      }
    if (std::fabs(mass - m[i]) > 1e-6 * m[i]) {
      c->err = "initial ||nu_i|| != m_i for cell " + std::to_string(i);
      return DD_ERR_PRECOND;
    }
  }
  double l1 = 0;
  if (!dev)
    for (long long t = 0; t < NN; ++t) l1 += std::fabs(acc[t] - P->nu[t]);
  if (l1 > 1e-6 * snu) {
    c->err = "initial boxes do not reproduce nu (L1 = " + std::to_string(l1) + ")";
    return DD_ERR_PRECOND;
  }
  // ---- capacities -------------------------
  const double tail = std::sqrt(c->eps_p * std::log(1e10));   // radius where nu_i drops ~1e-10 of its peak
  int side = std::max(maxext1, maxext2);
  // variable-size pool (bump-allocated each sweep): average capacity per basic
  // cell from the eps blur, generous; the total is what matters
  side = std::max(side, 2 * s + 2 * (int)std::ceil(tail) + 12);
  long long init_total = 0;
  for (int i = 0; i < I; ++i) init_total += (long long)hext[2 * i] * hext[2 * i + 1];
  if (dev) init_total = std::max(init_total, dev->total);
  // a typical box side from the eps blur for every cell plus twice the
  // initial data (the largest initial box must not size every cell's share:
  // a refined multiscale layer has a few very wide boxes)
  const int typ = 2 * s + 2 * (int)std::ceil(tail) + 12;
  const long long per_cell = c->opt.slot_cap > 0 ? c->opt.slot_cap : (long long)typ * typ;
  c->pool_cap = (long long)I * per_cell + 2 * init_total;
  // ---- device --------------------------------------------------------------
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= c->device) {
    c->err = "no CUDA device available (libdomdec has no CPU fallback)";
    return DD_ERR_CUDA;
  }
  DD_CUDA(cudaSetDevice(c->device));
  c->stream = (cudaStream_t)c->opt.stream;   // NULL = legacy default stream
  cudaStream_t st = c->stream;
  tm.mark("init: host validation");
  TRY(dalloc(c, &c->d_mu, NN));
  TRY(dalloc(c, &c->d_log2mu, NN));
  TRY(dalloc(c, &c->d_nu, NN));
  TRY(dalloc(c, &c->d_mu64, NN));
  TRY(dalloc(c, &c->d_m, I));
  TRY(dalloc(c, &c->d_q, I));
  TRY(dalloc(c, &c->d_mom, (size_t)I * 6));
  DD_CUDA(cudaMemsetAsync(c->d_mom, 0, (size_t)I * 6 * 8, c->stream));
  TRY(dalloc(c, &c->d_scratch, NN));
  TRY(dalloc(c, &c->d_red, 64));
  TRY(dalloc(c, &c->d_cum, 1));
  TRY(dalloc(c, &c->d_poolctr, 2));
  {
    // size classes of the sweep (sweep.cu)
    int nsm = 148;
    DD_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
    const int maxcells = (c->n1 / 2 + 1) * (c->n2 / 2 + 1);
    cudaError_t e = sweep_classes(s, std::max(c->N1, c->N2), nsm, maxcells, &c->cls, &c->scratch_stride);
    if (e != cudaSuccess) {
      c->err = std::string("sweep size classes: ") + cudaGetErrorString(e);
      return DD_ERR_CUDA;
    }
    if (c->opt.comp_cap > 0)   // testing knob: route larger hulls to the global-scratch class
      for (int k = 0; k < kClasses - 1; ++k) c->cls.ccap[k] = std::min(c->cls.ccap[k], c->opt.comp_cap);
    // one global-scratch slot per huge-class CTA, or per cluster (the leader's)
    const int slots = c->cls.cl_size > 1 ? c->cls.cl_grid / c->cls.cl_size : c->cls.grid[kClasses - 1];
    TRY(dalloc(c, &c->d_scratch_huge, (size_t)slots * c->scratch_stride));
    DD_CUDA(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
    DD_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    DD_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  }
  tm.mark("init: classes + scratch");
  DD_CUDA(cudaMemsetAsync(c->d_cum, 0, sizeof(SweepTotals), c->stream));
  for (int b = 0; b < 2; ++b) {
    TRY(dalloc(c, &c->d_pool[b], (size_t)c->pool_cap));
    TRY(dalloc(c, &c->d_pos[b], (size_t)I));
    TRY(dalloc(c, &c->d_off[b], (size_t)I * 2));
    TRY(dalloc(c, &c->d_ext[b], (size_t)I * 2));
    {
      // stripe mode keeps the A-cells of the owned rows and the B-cells whose
      // lower row 2 b1 is owned (+ the last B row when the stripe ends the grid)
      std::vector<CompCell> all = build_partition(c->n1, c->n2, s, b), kept;
      for (const CompCell& cc : all) {
        const int row = cc.r0 / s;
        const int key = b == 0 ? row : 2 * ((row + 1) / 2);
        if ((key >= c->rb && key < c->re) || (b == 1 && c->re == c->n1 && key >= c->n1)) kept.push_back(cc);
      }
      c->h_cells[b] = kept;
    }
    c->ncells[b] = (int)c->h_cells[b].size();
    TRY(dalloc(c, &c->d_cells[b], c->ncells[b]));
    TRY(dalloc(c, &c->d_alpha[b], NN));
    TRY(dalloc(c, &c->d_gauge[b], (size_t)c->ncells[b] * 2));
    TRY(dalloc(c, &c->d_stats[b], c->ncells[b]));
    if (b == 1) TRY(dalloc(c, &c->d_cls, 16 + (size_t)kClasses * std::max(c->ncells[0], c->ncells[1])));
    if (b == 1) TRY(dalloc(c, &c->d_ecell, (size_t)std::max(c->ncells[0], c->ncells[1])));
    TRY(dalloc(c, &c->d_totals[b], 1));
    DD_CUDA(cudaMemcpyAsync(c->d_cells[b], c->h_cells[b].data(), sizeof(CompCell) * c->ncells[b],
                            cudaMemcpyHostToDevice, st));
    DD_CUDA(cudaMemsetAsync(c->d_totals[b], 0, sizeof(SweepTotals), st));
    DD_CUDA(cudaMemsetAsync(c->d_stats[b], 0, sizeof(CellStats) * c->ncells[b], st));
  }
  tm.mark("init: pools + cells");
  // mu / nu / masses / supplies
  DD_CUDA(cudaMemcpyAsync(c->d_nu, P->nu, NN * 8, cudaMemcpyHostToDevice, st));
  DD_CUDA(cudaMemcpyAsync(c->d_scratch, P->mu, NN * 8, cudaMemcpyHostToDevice, st));
  DD_CUDA(cudaMemcpyAsync(c->d_mu64, P->mu, NN * 8, cudaMemcpyHostToDevice, st));
  k_init_mu<<<(unsigned)((NN + 255) / 256), 256, 0, st>>>(c->d_scratch, c->d_mu, c->d_log2mu, NN);
  DD_CUDA(cudaGetLastError());
  std::vector<int64_t> q(I);
  const double scale = std::ldexp(1.0, c->E);
  for (int i = 0; i < I; ++i) q[i] = (int64_t)std::llrint(m[i] * scale);
  for (int i = 0; i < I; ++i)
    if (q[i] <= 0) {
      c->err = "mass_exponent too small: a supply q_i = rint(m_i 2^E) is 0";
      return DD_ERR_PRECOND;
    }
  DD_CUDA(cudaMemcpyAsync(c->d_m, m.data(), I * 8, cudaMemcpyHostToDevice, st));
  DD_CUDA(cudaMemcpyAsync(c->d_q, q.data(), I * 8, cudaMemcpyHostToDevice, st));
  // initial boxes -> pool[0]
  if (dev) {
    const unsigned long long ctr0[2] = {(unsigned long long)dev->total, 0ull};
    DD_CUDA(cudaMemcpyAsync(c->d_pool[0], dev->d_pool, (size_t)dev->total * 8, cudaMemcpyDeviceToDevice, st));
    DD_CUDA(cudaMemcpyAsync(c->d_pos[0], dev->d_pos, I * 8, cudaMemcpyDeviceToDevice, st));
    DD_CUDA(cudaMemcpyAsync(c->d_off[0], dev->d_off, I * 8, cudaMemcpyDeviceToDevice, st));
    DD_CUDA(cudaMemcpyAsync(c->d_ext[0], dev->d_ext, I * 8, cudaMemcpyDeviceToDevice, st));
    DD_CUDA(cudaMemcpyAsync(c->d_poolctr, ctr0, 16, cudaMemcpyHostToDevice, st));
    // feasibility of the device-made coupling: ||nu_i|| = m_i, sum_i nu_i = nu
    unsigned long long* bad = (unsigned long long*)(c->d_red + 16);
    DD_CUDA(cudaMemsetAsync(bad, 0, 8, st));
    DD_CUDA(cudaMemsetAsync(c->d_scratch, 0, NN * 8, st));
    k_scatter_boxes<<<I, 128, 0, st>>>(c->d_pool[0], c->d_pos[0], c->d_off[0], c->d_ext[0], c->N2, c->d_scratch, 0);
    DD_CUDA(cudaGetLastError());
    k_l1_diff<<<1, 1024, 0, st>>>(c->d_scratch, c->d_nu, NN, c->d_red + 8);
    DD_CUDA(cudaGetLastError());
    double dl1 = 0;
    DD_CUDA(cudaMemcpyAsync(&dl1, c->d_red + 8, 8, cudaMemcpyDeviceToHost, st));
    DD_CUDA(cudaStreamSynchronize(st));
    k_box_mass<<<(I + 127) / 128, 128, 0, st>>>(c->d_pool[0], c->d_pos[0], c->d_ext[0], c->d_m, I, dl1, bad);
    DD_CUDA(cudaGetLastError());
    unsigned long long nbad = 0;
    DD_CUDA(cudaMemcpyAsync(&nbad, bad, 8, cudaMemcpyDeviceToHost, st));
    DD_CUDA(cudaStreamSynchronize(st));
    if (nbad || !(dl1 <= 1e-6 * snu)) {
      c->err = "device-made initial coupling infeasible (" + std::to_string(nbad) + " cells, L1 = " +
               std::to_string(dl1) + ")";
      return DD_ERR_PRECOND;
    }
  } else {
    std::vector<double> pool((size_t)init_total);
    std::vector<long long> pos(I);
    long long at = 0;
    for (int i = 0; i < I; ++i) {
      const long long len = (long long)P->init_ext[2 * i] * P->init_ext[2 * i + 1];
      std::memcpy(&pool[at], P->init_data + P->init_pos[i], len * 8);
      pos[i] = at;
      at += len;
    }
    const unsigned long long ctr0[2] = {(unsigned long long)init_total, 0ull};
    DD_CUDA(cudaMemcpyAsync(c->d_pool[0], pool.data(), pool.size() * 8, cudaMemcpyHostToDevice, st));
    DD_CUDA(cudaMemcpyAsync(c->d_pos[0], pos.data(), I * 8, cudaMemcpyHostToDevice, st));
    DD_CUDA(cudaMemcpyAsync(c->d_poolctr, ctr0, 16, cudaMemcpyHostToDevice, st));
    DD_CUDA(cudaMemcpyAsync(c->d_off[0], P->init_off, I * 8, cudaMemcpyHostToDevice, st));
    DD_CUDA(cudaMemcpyAsync(c->d_ext[0], P->init_ext, I * 8, cudaMemcpyHostToDevice, st));
    DD_CUDA(cudaStreamSynchronize(st));   // host staging buffer goes out of scope
  }
  tm.mark("init: initial coupling");
  c->cur = 0;
  TRY(flow_init_static(c));
  DD_CUDA(cudaStreamSynchronize(st));
  tm.mark("init: flow static");
  return DD_OK;
}

namespace dd {
dd_status init_with_device_coupling(const dd_problem* P, const dd_options* O, const DevInit& dev, dd_ctx** out) {
  *out = nullptr;
  dd_ctx* c = new dd_ctx();
  dd_status s = init_impl(P, O, c, &dev);
  if (s != DD_OK) {
    g_last_error = c->err;
    free_ctx(c);
    return s;
  }
  *out = c;
  return DD_OK;
}
}  // namespace dd

extern "C" {

dd_status domdec_init(const dd_problem* problem, const dd_options* options, dd_ctx** out) {
  if (!out) {
    g_last_error = "out is NULL";
    return DD_ERR_ARG;
  }
  *out = nullptr;
  dd_ctx* c = new dd_ctx();
  dd_status s = init_impl(problem, options, c);
  if (s != DD_OK) {
    g_last_error = c->err;
    free_ctx(c);
    return s;
  }
  *out = c;
  return DD_OK;
}

dd_status domdec_sweep(dd_ctx* c, dd_partition part, dd_sweep_stats* stats) {
  if (!c || (part != DD_PART_A && part != DD_PART_B)) return DD_ERR_ARG;
  NvtxRange nv(part == DD_PART_A ? "dd:sweep A" : "dd:sweep B");
  DD_CUDA(cudaSetDevice(c->device));
  const int b = (int)part;
  SweepParams p{};
  p.N1 = c->N1;
  p.N2 = c->N2;
  p.s = c->s;
  p.w = (float)(1.4426950408889634 / c->eps_p);
  p.mu = c->d_mu;
  p.log2mu = c->d_log2mu;
  p.cells = c->d_cells[b];
  p.ncells = c->ncells[b];
  p.pool_in = c->d_pool[c->cur];
  p.pos_in = c->d_pos[c->cur];
  p.off_in = c->d_off[c->cur];
  p.ext_in = c->d_ext[c->cur];
  p.pool_out = c->d_pool[1 - c->cur];
  p.pos_out = c->d_pos[1 - c->cur];
  p.off_out = c->d_off[1 - c->cur];
  p.ext_out = c->d_ext[1 - c->cur];
  p.pool_ctr = c->d_poolctr + (1 - c->cur);
  p.pool_cap = c->pool_cap;
  p.scratch = c->d_scratch_huge;
  p.scratch_stride = c->scratch_stride;
  p.alpha = c->d_alpha[b];
  p.gauge = c->d_gauge[b];
  p.alpha_valid = c->alpha_valid[b];
  p.m = c->d_m;
  p.tol = (float)c->opt.err;
  p.max_iter = c->opt.max_iter;
  p.fixed_iter = c->opt.fixed_iter;
  p.tau = c->opt.trunc;
  p.stats = c->d_stats[b];
  p.totals = c->d_totals[b];
  p.cum = c->d_cum;
  p.mom = c->d_mom;
  p.pxm = c->candidate ? c->d_pxm : nullptr;
  p.nu = c->d_nu;
  p.ecell = c->opt.track_primal ? c->d_ecell : nullptr;
  p.eps_p = c->eps_p;
  DD_CUDA(cudaMemsetAsync(c->d_totals[b], 0, sizeof(SweepTotals), c->stream));
  p.cls_count = c->d_cls;
  p.cls_fetch = c->d_cls + kClasses;
  p.cls_list = c->d_cls + 16;
  DD_CUDA(launch_sweep(p, c->cls, c->stream, c->aux, c->ev_fork, c->ev_join));
  c->cur = 1 - c->cur;
  ++c->n_sweeps;
  c->alpha_valid[b] = 1;
  c->last_part = b;
  c->swept |= (1 << b);
  c->primal_valid = c->opt.track_primal != 0;
  if (stats) {
    SweepTotals t{};
    DD_CUDA(cudaMemcpyAsync(&t, c->d_totals[b], sizeof(t), cudaMemcpyDeviceToHost, c->stream));
    DD_CUDA(cudaStreamSynchronize(c->stream));
    stats->cells = (int64_t)t.cells;
    stats->nonconverged = (int64_t)t.nonconv;
    stats->iters_total = (int64_t)t.iters;
    stats->iters_max = t.iters_max;
    stats->overflow = (int32_t)t.overflow;
    stats->l1x_entry = t.e0;
    stats->l1x_final = t.e;
    stats->dropped_mass = t.dropped;
    stats->mufu_ops = (double)t.mufu;
    stats->bytes = (double)t.bytes;
    if (t.overflow) {
      c->err = "box capacity exceeded in " + std::to_string(t.overflow) + " composite cells (left unchanged)";
      return DD_ERR_NUMERIC;
    }
  }
  return DD_OK;
}

dd_status marginal_error(dd_ctx* c, double* l1_x, double* l1_y) {
  if (!c) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  const long long NN = (long long)c->N1 * c->N2;
  double hx = NAN, hy = NAN;
  if (c->last_part >= 0) {
    k_sum_stats<<<1, 256, 0, c->stream>>>(c->d_stats[c->last_part], c->ncells[c->last_part], c->d_red);
    DD_CUDA(cudaGetLastError());
    DD_CUDA(cudaMemcpyAsync(&hx, c->d_red, 8, cudaMemcpyDeviceToHost, c->stream));
  }
  DD_CUDA(cudaMemsetAsync(c->d_scratch, 0, NN * 8, c->stream));
  // owned rows only (stripe mode: a partial sum of the global Y-marginal)
  k_scatter_boxes<<<(c->re - c->rb) * c->n2, 128, 0, c->stream>>>(c->d_pool[c->cur], c->d_pos[c->cur],
                                                                  c->d_off[c->cur], c->d_ext[c->cur], c->N2,
                                                                  c->d_scratch, c->rb * c->n2);
  DD_CUDA(cudaGetLastError());
  k_l1_diff<<<1, 1024, 0, c->stream>>>(c->d_scratch, c->d_nu, NN, c->d_red + 8);
  DD_CUDA(cudaGetLastError());
  DD_CUDA(cudaMemcpyAsync(&hy, c->d_red + 8, 8, cudaMemcpyDeviceToHost, c->stream));
  unsigned long long invalid = 0;
  DD_CUDA(cudaMemcpyAsync(&invalid, &c->d_cum->invalid, 8, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  if (invalid) {
    c->err = "marginal pool exhausted in an earlier sweep: the state is invalid";
    return DD_ERR_NUMERIC;
  }
  if (l1_x) *l1_x = hx;
  if (l1_y) *l1_y = hy;
  return DD_OK;
}

dd_status domdec_export_cells(dd_ctx* c, int32_t* off, int32_t* ext, int64_t* pos, double* data,
                              int64_t data_cap, int64_t* data_len) {
  if (!c) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  const int I = c->I;
  std::vector<int> ho(2 * I), he(2 * I);
  DD_CUDA(cudaMemcpyAsync(ho.data(), c->d_off[c->cur], I * 8, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaMemcpyAsync(he.data(), c->d_ext[c->cur], I * 8, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < I; ++i)   // stripe mode: cells outside the owned rows are not current here
    if (i < c->rb * c->n2 || i >= c->re * c->n2) ho[2 * i] = ho[2 * i + 1] = he[2 * i] = he[2 * i + 1] = 0;
  int64_t total = 0;
  for (int i = 0; i < I; ++i) total += (int64_t)he[2 * i] * he[2 * i + 1];
  if (data_len) *data_len = total;
  if (off) std::memcpy(off, ho.data(), I * 8);
  if (ext) std::memcpy(ext, he.data(), I * 8);
  if (pos) {
    int64_t p = 0;
    for (int i = 0; i < I; ++i) {
      pos[i] = p;
      p += (int64_t)he[2 * i] * he[2 * i + 1];
    }
  }
  if (!data) return DD_OK;
  if (data_cap < total) {
    c->err = "data_cap too small";
    return DD_ERR_ARG;
  }
  unsigned long long used = 0;
  std::vector<long long> hp(I);
  DD_CUDA(cudaMemcpyAsync(&used, c->d_poolctr + c->cur, 8, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaMemcpyAsync(hp.data(), c->d_pos[c->cur], I * 8, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<double> pool((size_t)used + 1);
  DD_CUDA(cudaMemcpyAsync(pool.data(), c->d_pool[c->cur], used * 8, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  int64_t p = 0;
  for (int i = 0; i < I; ++i) {
    const int64_t len = (int64_t)he[2 * i] * he[2 * i + 1];
    if (len) std::memcpy(data + p, &pool[(size_t)hp[i]], len * 8);
    p += len;
  }
  return DD_OK;
}

dd_status domdec_export_alpha(dd_ctx* c, dd_partition part, double* alpha) {
  if (!c || !alpha || (part != DD_PART_A && part != DD_PART_B)) return DD_ERR_ARG;
  const int b = (int)part;
  if (!c->alpha_valid[b]) {
    c->err = "partition never swept";
    return DD_ERR_PRECOND;
  }
  DD_CUDA(cudaSetDevice(c->device));
  const long long NN = (long long)c->N1 * c->N2;
  std::vector<float> a(NN), mu(NN);
  std::vector<int> g(2 * c->ncells[b]);
  DD_CUDA(cudaMemcpyAsync(a.data(), c->d_alpha[b], NN * 4, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaMemcpyAsync(mu.data(), c->d_mu, NN * 4, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaMemcpyAsync(g.data(), c->d_gauge[b], g.size() * 4, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  // a(k) = ln2 * A2(kappa) + (|D|^2 + 2 D.kappa)/eps' with D = K - G;
  // then subtract the mu-weighted mean per composite cell.
  for (int J = 0; J < c->ncells[b]; ++J) {
    const CompCell& cc = c->h_cells[b][J];
    const double D1 = cc.r0 - g[2 * J], D2 = cc.c0 - g[2 * J + 1];
    double sw = 0, swa = 0;
    for (int k1 = 0; k1 < cc.n1; ++k1)
      for (int k2 = 0; k2 < cc.n2; ++k2) {
        const long long pix = (long long)(cc.r0 + k1) * c->N2 + cc.c0 + k2;
        const double v = 0.69314718055994531 * a[pix] + (D1 * D1 + D2 * D2 + 2 * (D1 * k1 + D2 * k2)) / c->eps_p;
        alpha[pix] = v;
        sw += mu[pix];
        swa += mu[pix] * v;
      }
    const double mean = swa / sw;
    for (int k1 = 0; k1 < cc.n1; ++k1)
      for (int k2 = 0; k2 < cc.n2; ++k2) alpha[(long long)(cc.r0 + k1) * c->N2 + cc.c0 + k2] -= mean;
  }
  return DD_OK;
}

dd_status domdec_import_alpha(dd_ctx* c, dd_partition part, const double* alpha) {
  if (!c || !alpha || (part != DD_PART_A && part != DD_PART_B)) return DD_ERR_ARG;
  const int b = (int)part;
  DD_CUDA(cudaSetDevice(c->device));
  const long long NN = (long long)c->N1 * c->N2;
  // every composite cell takes its gauge origin at its X-block corner (D = 0),
  // where the stored base-2 potential is a / ln 2 (the inverse of the export)
  std::vector<float> a(NN, 0.f);
  std::vector<int> g(2 * (size_t)c->ncells[b]);
  for (int J = 0; J < c->ncells[b]; ++J) {
    const CompCell& cc = c->h_cells[b][J];
    g[2 * J] = cc.r0;
    g[2 * J + 1] = cc.c0;
    for (int k1 = 0; k1 < cc.n1; ++k1)
      for (int k2 = 0; k2 < cc.n2; ++k2) {
        const long long pix = (long long)(cc.r0 + k1) * c->N2 + cc.c0 + k2;
        if (!std::isfinite(alpha[pix])) {
          c->err = "domdec_import_alpha: non-finite potential";
          return DD_ERR_ARG;
        }
        a[pix] = (float)(alpha[pix] * 1.4426950408889634);
      }
  }
  DD_CUDA(cudaMemcpyAsync(c->d_alpha[b], a.data(), NN * 4, cudaMemcpyHostToDevice, c->stream));
  DD_CUDA(cudaMemcpyAsync(c->d_gauge[b], g.data(), g.size() * 4, cudaMemcpyHostToDevice, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));   // host staging goes out of scope
  c->alpha_valid[b] = 1;
  if (c->cyc_exec) cudaGraphExecDestroy(c->cyc_exec);   // captured units baked alpha_valid
  c->cyc_exec = nullptr;
  c->cyc_G = 0;
  return DD_OK;
}

dd_status domdec_export_plan_cost(dd_ctx* c, double* Qm) {
  if (!c || !Qm) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  std::vector<double> mom((size_t)c->I * 6);
  DD_CUDA(cudaMemcpyAsync(mom.data(), c->d_mom, mom.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  // <c, pi_i> = sum_y nu_i^pre(y) E[|x - y|^2 | y] = G0 - 2 G1 + M2 (centred moments)
  for (int i = 0; i < c->I; ++i) Qm[i] = mom[6 * i + 3] - 2.0 * mom[6 * i + 4] + mom[6 * i + 5];
  return DD_OK;
}

}  // extern "C"

namespace {
__global__ void k_scale_f(float* __restrict__ a, long long n, float f) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) a[i] *= f;
}

// One cycle's record: the sweep-entry errors of A and B, 1 if the cycle's
// flow update moved mass (solver info[1] = stationary flag), and a failure
// flag (box overflow in a sweep, min-cost flow round cap, pool exhausted in
// the flow apply).  info / fcnt are null when the cycle has no flow update.
__global__ void k_record_cycle(const SweepTotals* __restrict__ ta, const SweepTotals* __restrict__ tb,
                               const long long* __restrict__ info, const unsigned long long* __restrict__ fcnt,
                               double* __restrict__ dst) {
  dst[0] = ta->e0;
  dst[1] = tb->e0;
  dst[2] = info && !info[1] ? 1.0 : 0.0;
  dst[3] = (ta->overflow || tb->overflow || (info && info[6]) || (fcnt && fcnt[1])) ? 1.0 : 0.0;
}

// One unit of G hybrid cycles on the ctx stream (recording the entry errors);
// host bookkeeping is done by the caller.
dd_status enqueue_cycles(dd_ctx* c, int G, int flow_every, int* flows) {
  *flows = 0;
  for (int k = 0; k < G; ++k) {
    for (int b = 0; b < 2; ++b) {
      dd_status s = domdec_sweep(c, (dd_partition)b, nullptr);
      if (s) return s;
    }
    const bool doflow = flow_every > 0 && k % flow_every == flow_every - 1;
    if (doflow) {
      dd_status s = flow_update_impl(c, nullptr);
      if (s) return s;
      ++*flows;
    }
    k_record_cycle<<<1, 1, 0, c->stream>>>(c->d_totals[0], c->d_totals[1],
                                           doflow ? mcf_info_ptr(c->d_mcf, c->I) : nullptr,
                                           doflow ? (const unsigned long long*)c->d_flow_info : nullptr,
                                           c->d_hist + 4 * k);
    DD_CUDA(cudaGetLastError());
  }
  return DD_OK;
}
}  // namespace

extern "C" {

dd_status domdec_run_cycles(dd_ctx* c, int32_t max_cycles, int32_t flow_every, double conv, int32_t* cycles,
                            double* entry_error, int32_t* moved_flows) {
  if (!c || max_cycles < 1 || flow_every < 0) return DD_ERR_ARG;
  NvtxRange nv("dd:run_cycles");
  if (c->stripe) {
    c->err = "stripe mode: use the cycle program of stripes.py";
    return DD_ERR_ARG;
  }
  DD_CUDA(cudaSetDevice(c->device));
  // graph unit: G cycles with an even number of pool flips (each sweep and
  // each flow update flips the double-buffered pool), so every replay starts
  // from the same buffers: 2G sweeps + G / flow_every updates
  const int G = flow_every == 0 ? 2 : 2 * flow_every;
  if (!c->d_hist || G > c->cyc_G) {
    if (c->d_hist) cudaFreeAsync(c->d_hist, c->stream);
    c->d_hist = nullptr;
    DD_CUDA(cudaMallocAsync(&c->d_hist, (size_t)4 * G * sizeof(double), c->stream));
  }
  double smu = 0.0;
  {
    std::vector<double> hm(c->I);
    DD_CUDA(cudaMemcpyAsync(hm.data(), c->d_m, (size_t)c->I * 8, cudaMemcpyDeviceToHost, c->stream));
    DD_CUDA(cudaStreamSynchronize(c->stream));
    for (double v : hm) smu += v;
  }
  int done = 0, moved = 0;
  double emax = INFINITY;
  std::vector<double> hist(4 * (size_t)G);
  // read the unit's history back (one D2H per unit) and scan it: converged
  // once a cycle meets conv (emax = that cycle's error; the rest of its unit
  // has run as well)
  bool converged = false;
  auto fetch = [&]() -> dd_status {
    unsigned long long invalid = 0;
    DD_CUDA(cudaMemcpyAsync(hist.data(), c->d_hist, hist.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    DD_CUDA(cudaMemcpyAsync(&invalid, &c->d_cum->invalid, 8, cudaMemcpyDeviceToHost, c->stream));
    DD_CUDA(cudaStreamSynchronize(c->stream));
    if (invalid) {
      c->err = "marginal pool exhausted in a sweep: the state is invalid";
      return DD_ERR_NUMERIC;
    }
    for (int k = 0; k < G; ++k) {
      if (hist[4 * k + 3] != 0.0) {
        c->err = "box capacity exceeded, min-cost flow round cap or flow-apply pool exhausted";
        return DD_ERR_NUMERIC;
      }
    }
    for (int k = 0; k < G; ++k) {
      const double a = hist[4 * k], b = hist[4 * k + 1];
      moved += hist[4 * k + 2] > 0.5 ? 1 : 0;
      ++done;
      if (converged) continue;   // keep the error of the first converged cycle
      emax = (std::isfinite(a) && std::isfinite(b)) ? std::max(a, b) / smu : INFINITY;
      converged = emax <= conv;
    }
    return DD_OK;
  };
  auto finish = [&]() {
    if (cycles) *cycles = done;
    if (entry_error) *entry_error = emax;
    if (moved_flows) *moved_flows = moved;
    return DD_OK;
  };
  // warm-up unit, uncaptured: both partitions swept, the flow workspace
  // allocated (nothing may allocate inside a capture)
  const bool need_warm = c->swept != 3 || (flow_every > 0 && !c->d_mcf) || c->cyc_flow_every != flow_every ||
                         c->cyc_G != G || !c->cyc_exec;
  if (need_warm) {
    int fl = 0;
    dd_status s = enqueue_cycles(c, G, flow_every, &fl);
    if (s) return s;
    if ((s = fetch())) return s;
    if (converged || done >= max_cycles) return finish();
    // capture one unit; host state is saved and restored around the capture
    if (c->cyc_exec) cudaGraphExecDestroy(c->cyc_exec);
    c->cyc_exec = nullptr;
    const int cur0 = c->cur, last0 = c->last_part, swept0 = c->swept;
    const long long ns0 = c->n_sweeps, nf0 = c->n_flows;
    const bool pv0 = c->primal_valid;
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      dd_status es = enqueue_cycles(c, G, flow_every, &fl);
      ok = cudaStreamEndCapture(c->stream, &g) == cudaSuccess && es == DD_OK;
      if (ok) ok = cudaGraphInstantiate(&c->cyc_exec, g, 0) == cudaSuccess;
      if (g) cudaGraphDestroy(g);
    }
    cudaGetLastError();   // a failed capture leaves a sticky-free error state
    c->cur = cur0; c->last_part = last0; c->swept = swept0;
    c->n_sweeps = ns0; c->n_flows = nf0; c->primal_valid = pv0;
    c->cyc_G = G;
    c->cyc_flow_every = flow_every;
    c->cyc_flows = fl;
    if (!ok) {
      if (c->cyc_exec) cudaGraphExecDestroy(c->cyc_exec);
      c->cyc_exec = nullptr;
    }
  }
  while (done < max_cycles) {
    int fl = c->cyc_flows;
    if (c->cyc_exec) {
      DD_CUDA(cudaGraphLaunch(c->cyc_exec, c->stream));
      c->n_sweeps += 2 * G;
      c->n_flows += fl;
      c->last_part = 1;
    } else {   // capture unsupported here: the same unit, launched eagerly
      dd_status s = enqueue_cycles(c, G, flow_every, &fl);
      if (s) return s;
    }
    dd_status s = fetch();
    if (s) return s;
    if (converged) break;
  }
  return finish();
}

dd_status domdec_set_eps(dd_ctx* c, double eps) {
  if (!c) return DD_ERR_ARG;
  const double eps_p = eps / (c->h * c->h);
  if (!(eps > 0) || !(eps_p <= c->eps_p_init * (1 + 1e-12))) {
    c->err = "domdec_set_eps: eps must be > 0 and <= the construction eps (pool capacities)";
    return DD_ERR_ARG;
  }
  DD_CUDA(cudaSetDevice(c->device));
  const float f = (float)(c->eps_p / eps_p);
  const long long NN = (long long)c->N1 * c->N2;
  for (int b = 0; b < 2; ++b)
    if (c->alpha_valid[b]) {
      k_scale_f<<<(unsigned)((NN + 255) / 256), 256, 0, c->stream>>>(c->d_alpha[b], NN, f);
      DD_CUDA(cudaGetLastError());
    }
  c->eps = eps;
  c->eps_p = eps_p;
  // the captured cycles bake eps into their kernel parameters
  if (c->cyc_exec) cudaGraphExecDestroy(c->cyc_exec);
  c->cyc_exec = nullptr;
  c->cyc_G = 0;
  return DD_OK;
}

dd_status flow_update(dd_ctx* c, dd_flow_stats* stats) {
  if (!c) return DD_ERR_ARG;
  NvtxRange nv("dd:flow_update");
  if (c->last_part < 0) {
    c->err = "flow_update needs a previous sweep (plan costs, reading R13)";
    return DD_ERR_PRECOND;
  }
  if (c->stripe) {
    c->err = "stripe mode: run the flow update through flow_edge_costs / dd_mincost_flow / flow_apply";
    return DD_ERR_ARG;
  }
  DD_CUDA(cudaSetDevice(c->device));
  return flow_update_impl(c, stats);
}

dd_status primal_dual_gap(dd_ctx* c, double* primal, double* dual, double* rel_gap, double* transport_cost) {
  if (!c) return DD_ERR_ARG;
  if (c->stripe) {
    c->err = "primal_dual_gap is not available in stripe mode";
    return DD_ERR_ARG;
  }
  if (c->swept != 3) {
    c->err = "primal_dual_gap needs at least one A and one B sweep";
    return DD_ERR_PRECOND;
  }
  if (!c->primal_valid) {
    c->err = "primal_dual_gap needs the last sweep run with options.track_primal = 1";
    return DD_ERR_PRECOND;
  }
  DD_CUDA(cudaSetDevice(c->device));
  return pd_gap_impl(c, primal, dual, rel_gap, transport_cost);
}

dd_status domdec_export_cell_stats(dd_ctx* c, dd_partition part, int32_t* iters, double* e0, double* e,
                                   int32_t* ncells) {
  if (!c || (part != DD_PART_A && part != DD_PART_B)) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  const int b = (int)part;
  if (ncells) *ncells = c->ncells[b];
  if (!(c->swept & (1 << b))) {
    c->err = "partition never swept";
    return DD_ERR_PRECOND;
  }
  std::vector<CellStats> h(c->ncells[b]);
  DD_CUDA(cudaMemcpyAsync(h.data(), c->d_stats[b], h.size() * sizeof(CellStats), cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  for (int k = 0; k < c->ncells[b]; ++k) {
    if (iters) iters[k] = h[k].iters;
    if (e0) e0[k] = (double)h[k].e0;
    if (e) e[k] = (double)h[k].e;
  }
  return DD_OK;
}

dd_status domdec_counters(dd_ctx* c, dd_counters* out) {
  if (!c || !out) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  SweepTotals t{};
  DD_CUDA(cudaMemcpyAsync(&t, c->d_cum, sizeof(t), cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  if (t.invalid) {
    c->err = "marginal pool exhausted in an earlier sweep: the state is invalid";
    return DD_ERR_NUMERIC;
  }
  out->sweeps = c->n_sweeps;
  out->flow_updates = c->n_flows;
  out->cells = (int64_t)t.cells;
  out->iters = (int64_t)t.iters;
  out->mufu_ops = (double)t.mufu;
  out->bytes = (double)t.bytes;
  return DD_OK;
}

dd_status domdec_reset_counters(dd_ctx* c) {
  if (!c) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  // the invalid-state flag is sticky (not a counter)
  DD_CUDA(cudaMemsetAsync(c->d_cum, 0, offsetof(SweepTotals, invalid), c->stream));
  c->n_sweeps = 0;
  c->n_flows = 0;
  return DD_OK;
}

static __global__ void k_mufu_probe(float* out, int iters) {
  // 8 independent ex2 chains per thread (latency hidden by ILP + occupancy)
  float x[8];
  for (int k = 0; k < 8; ++k) x[k] = -0.001f * (threadIdx.x + k);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[k]));
      x[k] = y - 1.0f;
    }
  }
  float s = 0.f;
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.f) out[0] = s;
}

dd_status dd_mufu_peak(int32_t device, double* ops_per_s) {
  if (!ops_per_s) return DD_ERR_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return DD_ERR_CUDA;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  float* d = nullptr;
  if (cudaMalloc(&d, 16) != cudaSuccess) return DD_ERR_OOM;
  const int blocks = nsm * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_mufu_probe<<<blocks, threads>>>(d, 64);   // warm-up
  cudaEventRecord(e0);
  k_mufu_probe<<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (cudaGetLastError() != cudaSuccess || ms <= 0) return DD_ERR_CUDA;
  *ops_per_s = (double)blocks * threads * iters * 8.0 / (ms * 1e-3);
  return DD_OK;
}

dd_status domdec_halo_pack(dd_ctx* c, int32_t row, void* buf, int64_t cap, int64_t* bytes) {
  if (!c || row < 0 || row >= c->n1) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  const int n2 = c->n2, i0 = row * n2;
  const long long head = 8 + 16LL * n2;
  if (!buf) {   // size query (synchronises)
    std::vector<int> he(2 * n2);
    DD_CUDA(cudaMemcpyAsync(he.data(), c->d_ext[c->cur] + 2 * i0, n2 * 8, cudaMemcpyDeviceToHost, c->stream));
    DD_CUDA(cudaStreamSynchronize(c->stream));
    long long at = 0;
    for (int k = 0; k < n2; ++k) at += (long long)he[2 * k] * he[2 * k + 1];
    if (bytes) *bytes = head + 8 * at;
    return DD_OK;
  }
  if (cap < head) {
    c->err = "halo buffer smaller than its header";
    return DD_ERR_ARG;
  }
  if (!c->d_halo) TRY(dalloc(c, &c->d_halo, 3 * (size_t)n2));
  k_halo_meta_pack<<<1, 32, 0, c->stream>>>(c->d_pos[c->cur], c->d_off[c->cur], c->d_ext[c->cur], i0, n2, cap,
                                            (char*)buf, c->d_halo);
  DD_CUDA(cudaGetLastError());
  k_copy_boxes<<<n2, 128, 0, c->stream>>>(c->d_pool[c->cur], (double*)buf, c->d_halo);
  DD_CUDA(cudaGetLastError());
  if (bytes) *bytes = cap;
  return DD_OK;
}

dd_status domdec_halo_capacity(dd_ctx* c, int64_t* bytes) {
  if (!c || !bytes) return DD_ERR_ARG;
  const long long side = c->cls.ccap[kClasses - 2];
  *bytes = 8 + 16LL * c->n2 + 8LL * c->n2 * side * side;
  return DD_OK;
}

dd_status domdec_halo_unpack(dd_ctx* c, int32_t row, const void* buf, int64_t bytes) {
  if (!c || !buf || row < 0 || row >= c->n1) return DD_ERR_ARG;
  DD_CUDA(cudaSetDevice(c->device));
  const int n2 = c->n2, i0 = row * n2;
  if (bytes < 8 + 16LL * n2) {
    c->err = "halo buffer smaller than its header";
    return DD_ERR_ARG;
  }
  if (!c->d_halo) TRY(dalloc(c, &c->d_halo, 3 * (size_t)n2));
  k_halo_meta_unpack<<<1, 32, 0, c->stream>>>((const char*)buf, bytes, i0, n2, c->N1, c->N2, c->d_poolctr + c->cur,
                                              c->pool_cap, c->d_pos[c->cur], c->d_off[c->cur], c->d_ext[c->cur],
                                              c->d_halo, &c->d_cum->invalid);
  DD_CUDA(cudaGetLastError());
  k_copy_boxes<<<n2, 128, 0, c->stream>>>((const double*)buf, c->d_pool[c->cur], c->d_halo);
  DD_CUDA(cudaGetLastError());
  return DD_OK;
}

dd_status domdec_destroy(dd_ctx* c) {
  free_ctx(c);
  return DD_OK;
}

const char* dd_last_error(const dd_ctx* c) {
  if (c) return c->err.c_str();
  return g_last_error.c_str();
}

const char* dd_version(void) { return "libdomdec 0.1 sm_100a (arXiv 2405.09400 hot path)"; }

}  // extern "C"
