// The opaque handle behind ietidp_t and the device-buffer helper.
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "impl.h"

namespace ieti {

struct Error : std::runtime_error {
  ietidp_status st;
  Error(ietidp_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

#define IETI_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      throw ::ieti::Error(e_ == cudaErrorMemoryAllocation ? IETIDP_E_NOMEM : IETIDP_E_CUDA, \
                          std::string(#call) + ": " + cudaGetErrorString(e_));       \
  } while (0)

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) IETI_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void zero(cudaStream_t s) {
    if (n) IETI_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void upload(const std::vector<T>& v, cudaStream_t s) {
    alloc(v.size());
    if (n) IETI_CUDA(cudaMemcpyAsync(p, v.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

}  // namespace ieti

// Launch tracer (IETIDP_TRACE=<file>): events recorded after each launch.
struct LaunchTrace {
  bool on = false;
  std::string path;
  std::vector<cudaEvent_t> ev;
  std::vector<std::pair<const char*, int>> tag;
  size_t used = 0;
  void start(cudaStream_t s) {
    if (!on) return;
    used = 0;
    mark(s, "start", 0);
  }
  void mark(cudaStream_t s, const char* file, int line) {
    if (used == ev.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return;
      ev.push_back(e);
      tag.push_back({file, line});
    }
    tag[used] = {file, line};
    cudaEventRecord(ev[used++], s);
  }
  void dump(const char* phase) {
    if (!on || used < 2) return;
    cudaEventSynchronize(ev[used - 1]);
    FILE* f = fopen(path.c_str(), "a");
    if (!f) return;
    for (size_t i = 1; i < used; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      const char* b = strrchr(tag[i].first, '/');
      fprintf(f, "%s %s:%d %.2f\n", phase, b ? b + 1 : tag[i].first, tag[i].second, ms * 1e3);
    }
    fclose(f);
    used = 0;
  }
  ~LaunchTrace() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

struct ietidp_s {
  ietidp_options opt{};
  int n_sub = 0, n_lambda = 0, n_primal = 0, nrhs = 1;
  std::vector<ieti::SubIn> in;
  std::string err;
  bool analyzed = false, factored = false, solved = false, factor_failed = false;
  int failed_sub = -1;
  ieti::Plan plan;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t hp = nullptr;     // highest-priority stream of the factorisation's critical path
  cudaEvent_t hp_ev = nullptr;
  cudaGraphExec_t fgraph = nullptr;  // captured factorisation + coarse set-up
  long long fgraph_launches = 0;
  cudaGraphExec_t rgraph = nullptr;  // captured recovery
  long long rgraph_launches = 0;
  cudaEvent_t fg_ev[3] = {nullptr, nullptr, nullptr};
  // side stream of the factorisation (partitioned inverse, W_k) and its events
  cudaStream_t side = nullptr;
  std::vector<cudaStream_t> gst, gside;  // per subdomain group: main and side streams
  std::vector<cudaEvent_t> gev;          // per group: events (see run_factor)
  cudaStream_t cstream = nullptr;        // host-to-device copies of ietidp_set_values
  std::vector<cudaEvent_t> kev;          // per subdomain: its last set_values copy done
  cudaEvent_t hp_ev_set = nullptr;
  std::vector<cudaEvent_t> fev;  // [0..levels): level's panels done; [levels]: side done
  std::vector<cudaEvent_t> pev;  // per panel: POTRF done (progressive inverse)
  bool fwd_in_factor = false;    // the forward sweep of the loads ran on the side stream
  long long launches = 0;
  ieti::DevBuf<unsigned long long> pcg_prof;  // IETIDP_PCG_PROF barrier timestamps
  ieti::DevBuf<unsigned long long> dbg_tl;    // IETIDP_DBG_TL chunk-pass timeline (diagnostics)
  LaunchTrace trace;
  ietidp_report rep{};

  // ---- raw values (uploaded once, refreshed by ietidp_set_values) ----
  ieti::DevBuf<double> kval, fval;
  std::vector<long long> kval_off, fval_off;
  // ---- scatter lists: dst offset <- src index ----
  ieti::DevBuf<long long> sc_front_dst;   // K lower (r and P positions) -> fronts pool, by level
  ieti::DevBuf<int> sc_front_src;
  ieti::DevBuf<long long> sc_fx_dst;      // f -> X (every non-tree DOF)
  ieti::DevBuf<int> sc_fx_src;
  ieti::DevBuf<int> kdiag_src;            // K value index of the diagonal at each r_I slot
  // ---- symbolic structures ----
  ieti::DevBuf<ieti::SnDev> d_sn;
  ieti::DevBuf<ieti::SubDev> d_sub;
  std::vector<ieti::SubDev> h_sub;
  ieti::DevBuf<int> d_rows, d_rel, d_children, d_work, d_level_sn;
  ieti::DevBuf<ieti::GemmWork> d_gwork;
  ieti::DevBuf<int> d_perm;               // position -> local DOF (per subdomain, ne entries)
  ieti::DevBuf<int> d_prim_gid;           // per primal row (prim_off + q): global primal id
  ieti::DevBuf<long long> d_uoff;
  std::vector<long long> u_off;
  // ---- numeric ----
  ieti::DevBuf<double> pool, dinv, ipool, tpool, vecw;  // fronts, Dinv blocks, L11^-1, temp, sweep workspace
  ieti::DevBuf<double> skws;                             // split-K partial products
  ieti::DevBuf<double> bpart;                            // backward-sweep partial products
  ieti::DevBuf<int> skcnt;                               // split-K arrival counters (zero between uses)
  ieti::DevBuf<double> Xf, Xr;            // forward-swept loads (kept) / recovery sweep (ne rows x nrhs)
  ieti::DevBuf<double> S, Sinv, ftil, zc0;  // coarse: S_PP, S_PP^-1, ftilde, S^-1 ftilde
  ieti::DevBuf<long long> scoef_src;      // S_PP entry <- P-front pool offsets
  ieti::DevBuf<int> scoef_ptr;
  ieti::DevBuf<int> pcon_ptr, pcon_sub, pcon_q;  // global primal <- (subdomain, local primal)
  ieti::DevBuf<int> gsrc_ptr, gsrc;              // global primal <- coarse partial rows of the loop items
  ieti::DevBuf<int> err_flag;             // [0] min failing subdomain (INT_MAX: none), [1] coarse ok
  // ---- loop ----
  ieti::DevBuf<double> tiles, itiles, lpi;  // packed L_II, L_II^-1 tiles; L_PI
  ieti::DevBuf<double> wtiles, stiles, G;   // explicit loop: W = S_II^-1 and S_II tiles, G_k
  ieti::DevBuf<double> spart;               // symmetric-pass partial blocks
  ieti::DevBuf<int2> d_blk;                 // (subdomain, block) items of the partial reduction
  int n_blk = 0;
  ieti::DevBuf<int> d_rootlist;             // subdomains by level of their r_I root (for the S_II copy)
  std::vector<std::vector<std::pair<int, int>>> rootlist_range;  // [group][level]: (offset, count) into d_rootlist
  ieti::DevBuf<long long> slot_goff;        // per r_I slot: its row of G_k
  ieti::DevBuf<int> slot_np, slot_poff;     // per r_I slot: n_P of its subdomain, primal-row offset
  ieti::DevBuf<ieti::SlotRed> slot_red;     // per r_I slot: its symmetric-pass partials
  ieti::DevBuf<ieti::LoopWork> d_loopwork;
  std::vector<ieti::LoopWork> h_loopwork;
  int n_loopwork = 0;
  ieti::DevBuf<ieti::SymWork> d_symwork;     // explicit loop: symmetric-pass items
  std::vector<ieti::SymWork> h_symwork;
  int n_symwork = 0, sym_maxseg = 1;
  ieti::DevBuf<long long> d_pboff;           // symmetric pass: first partial block of each (subdomain, block)
  long long n_pblocks = 0;
  ieti::DevBuf<int> sub_blk0, sub_nt;        // (subdomain, block) rows of each subdomain
  ieti::DevBuf<int> cta_ptr, cta_items;     // persistent PCG: work items per CTA
  int lpt_grid = 0;
  ieti::DevBuf<int> cta_ptr2, cta_items2;   // the same plan for the standalone streamed pass (k_sym_stream)
  int lpt2_grid = 0;
  // several-RHS chunk pass of the persistent PCG (pcg.cu sym_chunks), planned for a grid
  int chunk_grid = 0;
  int n_pattern_classes = 0;  // distinct subdomain patterns found by the analysis
  std::vector<int> class_rep;  // per subdomain: the representative of its pattern class
  // ietidp_set_values_lower: per pattern class, full CSR entry -> index of its value in the
  // lower-triangle list (the entry itself if j <= i, else its mirror (j, i)); built and
  // uploaded at the first call
  bool lower_ready = false;
  std::vector<long long> low_off, low_map_off;  // per subdomain: lower values offset; per class rep: map offset
  std::vector<long long> low_n;                 // per subdomain: number of lower entries
  ieti::DevBuf<int> low_map;
  ieti::DevBuf<double> klow;
  ieti::DevBuf<int> chunk_ptr, chunk_cfirst;
  ieti::DevBuf<ieti::SymChunk> chunk_list;
  ieti::DevBuf<long long> chunk_cpb;
  ieti::DevBuf<ieti::SlotRed> chunk_slot_red;
  ieti::DevBuf<double> chunk_spart;
  ieti::DevBuf<ieti::GatherRec> chunk_grec;
  ieti::DevBuf<double> chunk_wrec;
  ieti::DevBuf<double> chunk_gzv;  // G_k z_k per slot (chunk-mode gather of q)
  ieti::DevBuf<double> bsw_A, bsw_T, bsw_D;  // blocked sweep operator of large coarse problems (coarse.cu)
  std::vector<ieti::LamDev> h_lam;  // host copy of the multiplier rows (slots, signs)
  ieti::DevBuf<int> sub_cta0, sub_ncta;   // loop CTAs of each subdomain
  ieti::DevBuf<ieti::LamDev> lam;
  ieti::DevBuf<int> slot_lam;             // per r_I slot: multiplier
  ieti::DevBuf<float> slot_sign;
  ieti::DevBuf<double> delta, kdiag;      // scaling weights per slot, K diagonal per slot
  ieti::DevBuf<double> d_vec, lam_vec, r_vec, p_vec, q_vec, z_vec;
  ieti::DevBuf<double> yI, xI, sI, zI;    // per-slot vectors (sum n_I x ncols)
  ieti::DevBuf<double> pslot, rslot;      // persistent PCG: B^T p and B_D^T r in slot order
  ieti::DevBuf<double> gpart, zc, gc;     // coarse partials per loop CTA; coarse solution; coarse rhs
  ieti::DevBuf<double> partial;           // per-block dot partials
  ieti::DevBuf<double> state;             // PCG scalars (see pcg.cu)
  ieti::DevBuf<double> cgcoef;            // PCG alpha_j / beta_j per column (Lanczos condition estimate)
  int coef_ld = 0;                        // its leading dimension (max iterations)
  ieti::DevBuf<double> cond_out;          // per column: omega_min, omega_max, cond
  ieti::DevBuf<double> tmp_in, tmp_out;   // col-major <-> interleaved staging
  ieti::DevBuf<double> U;                 // subdomain solutions u^(k), n_k x nrhs col-major
  int n_slots = 0, sum_nP = 0;
  // CUDA graph of the PCG loop (while-conditional), built lazily
  void* graph_exec = nullptr;
  void* graph = nullptr;
  unsigned long long cond_handle = 0;
  bool pcg_persistent = false;          // last solve ran the persistent cooperative PCG kernel
  // ietidp_apply_F with all 16 columns through the chunk pass (pcg.cu apply_F_chunk): the
  // persistent kernel's arguments and launch shape, prepared once
  std::vector<char> fa_args;
  bool fa_tried = false;
  int fa_grid = 0, fa_smem = 0, fa_stages = 0;
  ieti::DevBuf<double> fa_state;
  // ---- sharded mode (ietidp_shard.h): this handle holds one rank's subdomains ----
  bool shard = false;
  int sh_rank = 0, sh_n = 1;
  int (*sh_allreduce)(void*, double*, int64_t, void*) = nullptr;
  void* sh_ctx = nullptr;
  void* sh_nccl_comm = nullptr;         // native NCCL transport (ietidp_shard_enable_nccl)
  void* sh_nccl_fn = nullptr;
  ieti::DevBuf<double> sh_kd2;          // K diagonal on the (+, -) sides of every multiplier
  long long sh_reduced_doubles = 0;     // doubles summed over the ranks so far (report)
  ieti::DevBuf<unsigned> gbar;          // its grid barrier
};

// Device-side entry points implemented in the .cu files (host launchers).
namespace ieti {
// Device expansion of the scatter lists (factor.cu): segment i writes n entries at
// dst_off: dst = front_off(sn_base + sl[q]) + off[q], src = kval_off + src[q] (K), or
// for the loads dst = (x_off + r[q]) nrhs + c, src = f_off + s[q] + c n_k.
struct ExpandSeg {
  long long dst_off, rel_off, base;  // base: kval_off (K) / x_off (loads)
  long long base2;                   // loads: f_off
  int n, sn_base, nk, kind;          // kind 0: K entries, 1: loads
};
// per-class relative scatter entries (analyze.cpp), uploaded at their offset
struct ClassRel {
  long long base;
  const std::vector<int>*off, *sl, *src;
};
void launch_expand_lower(ietidp_s* h, int k, cudaStream_t st);  // factor.cu (ietidp_set_values_lower)
void expand_scatter(ietidp_s* h, const std::vector<ExpandSeg>& segs, const std::vector<ClassRel>& cls, long long nrel,
                    long long nK, long long nF);
void run_factor(ietidp_s* h);                  // factor.cu
void run_coarse(ietidp_s* h);                  // coarse.cu
void run_solve(ietidp_s* h);                   // pcg.cu
void run_apply_F(ietidp_s* h, int ncols, const double* x, double* y);
void run_apply_M(ietidp_s* h, int ncols, const double* x, double* y);
void run_recover(ietidp_s* h);                 // coarse.cu
void sh_sum(ietidp_s* h, double* buf, long long n);  // sharded mode: all-reduce of a device buffer (coarse.cu)
void run_estimate_condition(ietidp_s* h, double* omega_min, double* omega_max, double* cond);  // pcg.cu
void transpose_in(ietidp_s* h, int rows, int ncols, const double* colmajor, double* inter);
void transpose_out(ietidp_s* h, int rows, int ncols, const double* inter, double* colmajor);
}  // namespace ieti
