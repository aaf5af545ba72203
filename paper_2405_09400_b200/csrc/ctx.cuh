// ctx.cuh — the dd_ctx object (internal).
#pragma once
#include <string>
#include <vector>

#include "../../include/domdec.h"
#include "internal.cuh"

struct dd_ctx {
  // problem
  int N1 = 0, N2 = 0, s = 0, n1 = 0, n2 = 0, I = 0;
  double h = 0, eps = 0, eps_p = 0;
  double eps_p_init = 0;       // eps' at construction (sizes the pools; domdec_set_eps may only lower it)
  int E = 0;
  dd_options opt{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int device = 0;
  std::string err;
  // device data
  float* d_mu = nullptr;
  float* d_log2mu = nullptr;
  double* d_nu = nullptr;
  double* d_mu64 = nullptr;    // mu in fp64 (static tables of the gluing candidates)
  double* d_m = nullptr;
  int64_t* d_q = nullptr;
  double* d_pool[2] = {nullptr, nullptr};
  long long* d_pos[2] = {nullptr, nullptr};          // [I] start of box i
  unsigned long long* d_poolctr = nullptr;           // [2] elements used per pool
  long long pool_cap = 0;                            // elements per pool
  dd::SweepClasses cls{};                            // size classes (sweep.cu)
  unsigned char* d_scratch_huge = nullptr;           // global scratch of the huge class
  size_t scratch_stride = 0;
  cudaStream_t aux = nullptr;                        // large size classes run here (fork/join)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int* d_off[2] = {nullptr, nullptr};
  int* d_ext[2] = {nullptr, nullptr};
  int cur = 0;
  int* d_cls = nullptr; // [16 (counts, fetch counters) + kClasses * max ncells] size-class lists
  dd::CompCell* d_cells[2] = {nullptr, nullptr};
  int ncells[2] = {0, 0};
  std::vector<dd::CompCell> h_cells[2];
  float* d_alpha[2] = {nullptr, nullptr};
  int* d_gauge[2] = {nullptr, nullptr};
  int alpha_valid[2] = {0, 0};
  dd::CellStats* d_stats[2] = {nullptr, nullptr};
  dd::SweepTotals* d_totals[2] = {nullptr, nullptr};
  dd::SweepTotals* d_cum = nullptr;
  long long n_sweeps = 0, n_flows = 0;
  int last_part = -1;
  int swept = 0;
  int rb = 0, re = 0;          // owned basic-cell rows [rb, re) (stripe mode if not the whole grid)
  bool stripe = false;
  long long* d_halo = nullptr; // [3 * n2] halo pack/unpack metadata
  bool primal_valid = false;   // the last sweep recorded d_ecell
  // domdec_run_cycles: a CUDA graph of G hybrid cycles and the per-sweep
  // entry errors it records on the device
  cudaGraphExec_t cyc_exec = nullptr;
  int cyc_G = 0, cyc_flow_every = -1, cyc_flows = 0;
  double* d_hist = nullptr;    // [2 G] sweep-entry errors of the last graph replay
  double* d_mom = nullptr;   // [I][6] plan moments of the last sweep (R13)
  // gluing edge candidates (flow_set_candidate)
  int candidate = 0;           // 0 = product (R12), 1 = glued with entropic gamma_ij
  double eps_gamma_p = 0.25;   // eps_gamma / h^2
  double* d_pxm = nullptr;     // [N1*N2][3] PX(x), E[y - x | x] of the last sweep
  double* d_gam = nullptr;     // [I][4][s^2][3] (b, delta) of gamma~_ij per pixel (static)
  double* d_ecell = nullptr; // [max ncells] primal score per composite cell of the last sweep / h^2
  double* d_pd = nullptr;    // [4 N1 N2 + ...] primal-dual gap scratch (allocated on first use)
  // flow update
  double* d_xbar = nullptr;   // [I][2] mu-mean of X_i (pixel units)
  double* d_var = nullptr;    // [I] trace of the covariance of mu_i / m_i
  double* d_cbar = nullptr;   // [I][5]
  int64_t* d_C = nullptr;     // [I][5]
  int64_t* d_w = nullptr;     // [I][5]
  void* d_mcf = nullptr;      // solver workspace
  size_t mcf_bytes = 0;
  int* d_flow_info = nullptr; // [16] device flags of the last flow update
  // diagnostics scratch
  double* d_scratch = nullptr; // [N1*N2]
  double* d_red = nullptr;     // [64]
};

namespace dd {
// Initial coupling already on the device (multiscale.cu): compact boxes with
// their positions, plus host copies of off/ext for the capacity checks.
struct DevInit {
  const double* d_pool;
  const long long* d_pos;
  const int* d_off;
  const int* d_ext;
  long long total;        // pool entries used
  const int* h_off;       // [I][2]
  const int* h_ext;       // [I][2]
};
dd_status init_with_device_coupling(const dd_problem* P, const dd_options* O, const DevInit& dev, dd_ctx** out);
dd_status flow_update_impl(dd_ctx* c, dd_flow_stats* stats);
dd_status flow_costs_impl(dd_ctx* c);
dd_status flow_apply_impl(dd_ctx* c);
dd_status mcf_solve_device(int n1, int n2, const int64_t* d_q, const int64_t* d_C, int64_t* d_w,
                           void** d_ws, size_t* ws_bytes, int warm, cudaStream_t st, std::string& err);
dd_status flow_init_static(dd_ctx* c);
long long* mcf_info_ptr(void* ws, int I);
void keep_device_pool(int dev);   // api.cu: stream-ordered pool, pre-grown once
dd_status pd_gap_impl(dd_ctx* c, double* primal, double* dual, double* rel_gap, double* transport);
void set_global_error(const std::string& m);   // dd_last_error(NULL)
}  // namespace dd

#define DD_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      c->err = std::string(#call) + ": " + cudaGetErrorString(e_);           \
      return (e_ == cudaErrorMemoryAllocation) ? DD_ERR_OOM : DD_ERR_CUDA;   \
    }                                                                        \
  } while (0)
