// sinkhorn_global.cu — global separable log-domain Sinkhorn on the whole
// N1 x N2 grid (the SinkhornGPU comparator of the paper's benchmark,
// PAPER.md:1249-1250, Table).
//
// Potentials in units of eps (a = alpha/eps, b = beta/eps), pixel units for
// the cost, eps' = eps/h^2 (SURVEY 8 symbols):
//   b(l) = -LSE_k [ a(k) + log mu(k) - |k - l|^2 / eps' ]      (Y-update)
//   a(k) = -LSE_l [ b(l) + log nu(l) - |k - l|^2 / eps' ]      (X-update)
// each half split into two 1-D LSE stages along the axes (separable kernel,
// PAPER.md:1145).  Stop when the L1 X-marginal error after the Y-update,
// sum_k mu(k) |1 - exp(a(k) - a'(k))| (a' = the next X-update), is
// <= ||mu|| Err.
//
// Precision: the global gauge has exponents of magnitude O(N^2/eps'), which
// the paper reports as the fp32 stall, so potentials and
// terms are fp64 here; only exp2 of (term - row max) <= 0 and its sum are
// fp32.  One CTA per output row of a stage; the input row is staged in shared
// memory and every thread computes whole output entries.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <string>
#include <vector>

#include "ctx.cuh"

namespace dd {
namespace {

constexpr double kLog2eG = 1.4426950408889634;

// in[i] = w[i] > 0 ? p[i] + log w[i] : -inf
__global__ void k_sg_prep(const double* __restrict__ p, const double* __restrict__ w, double* __restrict__ in,
                          long long NN) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < NN; i += (long long)gridDim.x * blockDim.x)
    in[i] = w[i] > 0.0 ? p[i] + log(w[i]) : -INFINITY;
}

// float(v) without F2F (which runs on the XU pipe next to MUFU.EX2): the
// fp64 word's low 9 exponent bits and top 23 mantissa bits are funnel-shifted
// into place and the exponent rebased (E_f = E_d - 896 == low9 + 128 mod 512);
// mantissa truncated (<= 1 float ulp); sign copied.  |v| < 2^-126 gives 0
// (2^v = 1 to fp32 precision); |v| >= 256 gives -256 for v < 0 (2^v = 0) and
// +256 for v > 0 (2^256 overflows to +inf, so the shifted sum leaves
// [2^-60, 2^60] and that output falls back to the max pass: a stale shift
// never silently drops a dominant term).  Integer ops only.
__device__ __forceinline__ float sg_d2f(double v) {
  const unsigned hi = (unsigned)__double2hiint(v), lo = (unsigned)__double2loint(v);
  const unsigned e = hi & 0x7ff00000u;
  const unsigned bits = (__funnelshift_l(lo, hi, 3) + (128u << 23)) | (hi & 0x80000000u);
  const float f = e < (897u << 20) ? 0.f : __uint_as_float(bits);
  return e >= (1031u << 20) ? ((hi & 0x80000000u) ? -256.f : 256.f) : f;
}

__device__ __forceinline__ float sg_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// sum_z 2^(t(z) - m2) with t(z) = srow2[z] - ie2 (z - y)^2
//   = s2[z] + z (2 ie2 y) - ie2 y^2,   s2[z] = srow2[z] - ie2 z^2 (shared).
__device__ __forceinline__ float sg_sum(const double* s2, int M, int y, double ie2, double m2) {
  const double g = 2.0 * ie2 * (double)y, c = fma(ie2 * (double)y, (double)y, m2);
  float sum = 0.f;
  double zd = 0.0;
  for (int z = 0; z < M; ++z, zd += 1.0) sum += sg_ex2(sg_d2f(fma(zd, g, s2[z]) - c));
  return sum;
}

// out[y * R + x] = LSE_z [ in[x * M + z] - (z - y)^2 * inv_eps ], x < R, y, z < M
// (transposed so the next stage reads rows), computed in log2 units.  The
// shift m of each output is the previous iteration's value of the same output
// when `shift` is given (one pass; the fixed point makes it the
// LSE itself), else the true maximum (a max pass).  A shifted sum outside
// [2^-60, 2^60] (or a non-finite shift) falls back to the true maximum for
// that output.
__global__ void k_sg_stage(const double* __restrict__ in, double* __restrict__ out, int R, int M, double inv_eps,
                           const double* __restrict__ shift) {
  extern __shared__ double srow2[];
  const int x = blockIdx.x;
  const double ie2 = inv_eps * kLog2eG;
  for (int z = threadIdx.x; z < M; z += blockDim.x)
    srow2[z] = fma(-ie2 * (double)z, (double)z, in[(long long)x * M + z] * kLog2eG);   // s2[z]
  __syncthreads();
  constexpr double kLn2 = 0.6931471805599453;
  for (int y = threadIdx.x; y < M; y += blockDim.x) {
    double res = -INFINITY;
    bool done = false;
    if (shift) {
      const double m = shift[(long long)y * R + x];
      if (m > -INFINITY && m < INFINITY) {
        const double m2 = m * kLog2eG;
        const float sum = sg_sum(srow2, M, y, ie2, m2);
        if (sum > 8.67361738e-19f && sum < 1.15292150e18f) {   // 2^-60 .. 2^60
          res = (m2 + log2((double)sum)) * kLn2;
          done = true;
        }
      }
    }
    if (!done) {
      double m2 = -INFINITY;
      const double g = 2.0 * ie2 * (double)y, c = ie2 * (double)y * (double)y;
      double zd = 0.0;
      for (int z = 0; z < M; ++z, zd += 1.0) m2 = fmax(m2, fma(zd, g, srow2[z]) - c);
      if (m2 > -INFINITY) res = (m2 + log2((double)sg_sum(srow2, M, y, ie2, m2))) * kLn2;
    }
    out[(long long)y * R + x] = res;
  }
}

// dst[i] = w[i] > 0 ? -lse[i] : 0   (potential defined on the support only)
__global__ void k_sg_neg(const double* __restrict__ lse, const double* __restrict__ w, double* __restrict__ dst,
                         long long NN) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < NN; i += (long long)gridDim.x * blockDim.x)
    dst[i] = w[i] > 0.0 ? -lse[i] : 0.0;
}

// per-block partial sums of mu |expm1(a_old - a_new)| (fixed grid, fixed order)
__global__ void k_sg_err(const double* __restrict__ a_old, const double* __restrict__ a_new,
                         const double* __restrict__ mu, long long NN, double* __restrict__ part) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < NN; i += (long long)gridDim.x * blockDim.x)
    if (mu[i] > 0.0) s += mu[i] * fabs(expm1(a_old[i] - a_new[i]));
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
}

__global__ void k_sg_err_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += part[i];
    *out = t;
  }
}

constexpr int kSgThreads = 256;
constexpr int kSgErrBlocks = 296;   // 2 x 148 SMs

struct SgBuffers {
  double *mu = nullptr, *nu = nullptr, *a = nullptr, *a2 = nullptr, *b = nullptr, *in = nullptr, *part = nullptr,
         *err = nullptr;
  double *t[2] = {nullptr, nullptr}, *out[2] = {nullptr, nullptr};   // per half: stage outputs (next shifts)
  ~SgBuffers() {
    for (double* p : {mu, nu, a, a2, b, in, t[0], t[1], out[0], out[1], part, err})
      if (p) cudaFree(p);
  }
};

// One half-iteration h (0 = Y-update, 1 = X-update): dst = -LSE over the
// source grid of (src + log w_src - c/eps'), masked by w_dst.  warm: the
// half's stage outputs from the previous iteration serve as shifts.
void sg_half(const SgBuffers& B, int h, bool warm, const double* src, const double* wsrc, const double* wdst,
             double* dst, int N1, int N2, double inv_eps, int grid_ew, cudaStream_t st) {
  const long long NN = (long long)N1 * N2;
  k_sg_prep<<<grid_ew, kSgThreads, 0, st>>>(src, wsrc, B.in, NN);
  k_sg_stage<<<N1, kSgThreads, N2 * sizeof(double), st>>>(B.in, B.t[h], N1, N2, inv_eps, warm ? B.t[h] : nullptr);
  k_sg_stage<<<N2, kSgThreads, N1 * sizeof(double), st>>>(B.t[h], B.out[h], N2, N1, inv_eps,
                                                           warm ? B.out[h] : nullptr);
  k_sg_neg<<<grid_ew, kSgThreads, 0, st>>>(B.out[h], wdst, dst, NN);
}

}  // namespace
}  // namespace dd

using namespace dd;

extern "C" {

dd_status dd_sinkhorn_global(int32_t N1, int32_t N2, const double* mu, const double* nu, double eps_p, double err,
                             int32_t max_iter, int32_t check_every, int32_t device, void* stream, double* alpha,
                             double* beta, int32_t* iters, double* l1_x, double* solve_ms) {
  if (N1 <= 0 || N2 <= 0 || N1 > 8192 || N2 > 8192 || !mu || !nu || !alpha || !beta || !(eps_p > 0.0) ||
      max_iter <= 0 || check_every <= 0) {
    set_global_error("dd_sinkhorn_global: bad argument");
    return DD_ERR_ARG;
  }
  const long long NN = (long long)N1 * N2;
  double mass_mu = 0.0, mass_nu = 0.0;
  for (long long i = 0; i < NN; ++i) {
    if (!(mu[i] >= 0.0) || !(nu[i] >= 0.0)) {
      set_global_error("dd_sinkhorn_global: negative or NaN mass");
      return DD_ERR_ARG;
    }
    mass_mu += mu[i];
    mass_nu += nu[i];
  }
  if (!(mass_mu > 0.0) || std::fabs(mass_mu - mass_nu) > 1e-9 * mass_mu) {
    set_global_error("dd_sinkhorn_global: marginals must have equal positive mass");
    return DD_ERR_PRECOND;
  }
  if (cudaSetDevice(device) != cudaSuccess) return DD_ERR_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  SgBuffers B;
  const size_t bytes = NN * sizeof(double);
  if (cudaMalloc(&B.mu, bytes) || cudaMalloc(&B.nu, bytes) || cudaMalloc(&B.a, bytes) || cudaMalloc(&B.a2, bytes) ||
      cudaMalloc(&B.b, bytes) || cudaMalloc(&B.in, bytes) || cudaMalloc(&B.t[0], bytes) || cudaMalloc(&B.t[1], bytes) ||
      cudaMalloc(&B.out[0], bytes) || cudaMalloc(&B.out[1], bytes) ||
      cudaMalloc(&B.part, kSgErrBlocks * sizeof(double)) || cudaMalloc(&B.err, sizeof(double))) {
    set_global_error("dd_sinkhorn_global: cudaMalloc failed");
    return DD_ERR_OOM;
  }
  const int smem = (N1 > N2 ? N1 : N2) * (int)sizeof(double);
  if (smem > 48 * 1024 && cudaFuncSetAttribute(k_sg_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))
    return DD_ERR_CUDA;
  cudaMemcpyAsync(B.mu, mu, bytes, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(B.nu, nu, bytes, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(B.a, alpha, bytes, cudaMemcpyHostToDevice, st);
  const double inv_eps = 1.0 / eps_p;
  const int grid_ew = (int)std::min<long long>((NN + kSgThreads - 1) / kSgThreads, 148 * 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  int it = 0;
  double e = INFINITY;
  double *a = B.a, *a2 = B.a2;
  // Launch-bound at small N (8 launches per iteration): after the first
  // check_every iterations (cold first iteration), whole chunks of
  // check_every iterations + the error reduction run as one CUDA graph.  An
  // even chunk returns a/a2 to their roles, so one graph serves every chunk;
  // same kernels in the same order as the eager loop (bit-identical).
  const bool use_graph = check_every >= 2 && check_every % 2 == 0 && !getenv("DD_SG_NO_GRAPH");
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cs = nullptr;
  dd_status gs = DD_OK;
  while (it < max_iter) {
    if (use_graph && it > 0 && it % check_every == 0 && max_iter - it > check_every) {
      if (!gexec) {
        cudaGraph_t g = nullptr;
        if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
          gs = DD_ERR_CUDA;
          break;
        }
        double *ga = a, *ga2 = a2;
        for (int j = 0; j < check_every; ++j) {
          sg_half(B, 0, true, ga, B.mu, B.nu, B.b, N1, N2, inv_eps, grid_ew, cs);
          sg_half(B, 1, true, B.b, B.nu, B.mu, ga2, N1, N2, inv_eps, grid_ew, cs);
          if (j == check_every - 1) {
            k_sg_err<<<kSgErrBlocks, kSgThreads, 0, cs>>>(ga, ga2, B.mu, NN, B.part);
            k_sg_err_final<<<1, 32, 0, cs>>>(B.part, kSgErrBlocks, B.err);
          }
          std::swap(ga, ga2);
        }
        if (cudaStreamEndCapture(cs, &g) != cudaSuccess || cudaGraphInstantiate(&gexec, g, 0) != cudaSuccess) {
          if (g) cudaGraphDestroy(g);
          gs = DD_ERR_CUDA;
          break;
        }
        cudaGraphDestroy(g);
      }
      cudaGraphLaunch(gexec, st);
      it += check_every;
      cudaMemcpyAsync(&e, B.err, sizeof(double), cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) break;
      if (e <= err * mass_mu) break;
      continue;
    }
    sg_half(B, 0, it > 0, a, B.mu, B.nu, B.b, N1, N2, inv_eps, grid_ew, st);    // Y-update
    sg_half(B, 1, it > 0, B.b, B.nu, B.mu, a2, N1, N2, inv_eps, grid_ew, st);   // X-update
    ++it;
    const bool check = (it % check_every == 0) || it == max_iter;
    if (check) {
      k_sg_err<<<kSgErrBlocks, kSgThreads, 0, st>>>(a, a2, B.mu, NN, B.part);
      k_sg_err_final<<<1, 32, 0, st>>>(B.part, kSgErrBlocks, B.err);
      cudaMemcpyAsync(&e, B.err, sizeof(double), cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) break;
    }
    std::swap(a, a2);
    if (check && e <= err * mass_mu) break;
  }
  if (gexec) cudaGraphExecDestroy(gexec);
  if (cs) cudaStreamDestroy(cs);
  if (gs != DD_OK) {
    set_global_error(std::string("dd_sinkhorn_global: graph capture: ") + cudaGetErrorString(cudaGetLastError()));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return gs;
  }
  sg_half(B, 0, it > 0, a, B.mu, B.nu, B.b, N1, N2, inv_eps, grid_ew, st);   // final Y-update: beta matches alpha
  cudaEventRecord(e1, st);
  cudaMemcpyAsync(alpha, a, bytes, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(beta, B.b, bytes, cudaMemcpyDeviceToHost, st);
  const cudaError_t ce = cudaStreamSynchronize(st);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (ce != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    set_global_error(std::string("dd_sinkhorn_global: CUDA: ") + cudaGetErrorString(ce));
    return DD_ERR_CUDA;
  }
  if (iters) *iters = it;
  if (l1_x) *l1_x = e;
  if (solve_ms) *solve_ms = ms;
  if (!std::isfinite(e)) {
    set_global_error("dd_sinkhorn_global: non-finite marginal error");
    return DD_ERR_NUMERIC;
  }
  return DD_OK;
}

}  // extern "C"
