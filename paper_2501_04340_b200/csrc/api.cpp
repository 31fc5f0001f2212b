#include <algorithm>
// C-ABI entry points of libietidp.so (include/ietidp.h). Argument checking,
// call-order state machine, error translation; the work is in analyze.cpp and
// the CUDA translation units.
#include <chrono>
#include <climits>
#include <cstring>
#include <new>

#include <nvtx3/nvToolsExt.h>

#include "handle.h"
#include "../../include/ietidp_shard.h"

namespace ieti {
void analyze_all(ietidp_s* h);
void finish_solve(ietidp_s* h, ietidp_report* rep);
void destroy_graph(ietidp_s* h);
}  // namespace ieti

using ieti::Error;

namespace {

template <class F>
ietidp_status guard(ietidp_t h, F&& f) {
  if (!h) return IETIDP_E_ARG;
  try {
    f();
    h->err.clear();
    return IETIDP_OK;
  } catch (const Error& e) {
    h->err = e.what();
    return e.st;
  } catch (const std::bad_alloc&) {
    h->err = "host allocation failed";
    return IETIDP_E_NOMEM;
  } catch (const std::exception& e) {
    h->err = e.what();
    return IETIDP_E_CUDA;
  }
}

// NVTX range of one API phase (visible in Nsight Systems / ncu --nvtx; no cost without a tool
// attached: the header-only NVTX v3 resolves to no-ops until an injection library is loaded)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

void require(bool c, ietidp_status st, const char* msg) {
  if (!c) throw Error(st, msg);
}

struct EvPair {
  cudaEvent_t a = nullptr, b = nullptr;
  EvPair() {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
  ~EvPair() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  float ms() {
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    return t;
  }
};

void set_device(ietidp_t h) {
  if (h->opt.device < 0) throw Error(IETIDP_E_STATE, "handle created in host-only analysis mode (device < 0)");
  IETI_CUDA(cudaSetDevice(h->opt.device));
}

}  // namespace

extern "C" {

void ietidp_options_default(ietidp_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->tol = 1e-10;
  o->max_iter = 500;
  o->scaling = IETIDP_SCALE_MULTIPLICITY;
  o->fixed_iters = 0;
  o->ordering = IETIDP_ORDER_NESTED_DISSECTION;
  o->leaf_size = 96;
  o->loop = IETIDP_LOOP_EXPLICIT;
  o->device = 0;
  o->stream = nullptr;
}

const char* ietidp_status_string(ietidp_status s) {
  switch (s) {
    case IETIDP_OK: return "IETIDP_OK";
    case IETIDP_E_ARG: return "IETIDP_E_ARG";
    case IETIDP_E_STATE: return "IETIDP_E_STATE";
    case IETIDP_E_B_STRUCTURE: return "IETIDP_E_B_STRUCTURE";
    case IETIDP_E_NOT_SPD: return "IETIDP_E_NOT_SPD";
    case IETIDP_E_NO_CONVERGENCE: return "IETIDP_E_NO_CONVERGENCE";
    case IETIDP_E_CUDA: return "IETIDP_E_CUDA";
    case IETIDP_E_NOMEM: return "IETIDP_E_NOMEM";
  }
  return "unknown";
}

ietidp_status ietidp_create(const ietidp_options* opt, int n_sub, int n_lambda, int n_primal, int nrhs, ietidp_t* out) {
  if (!out) return IETIDP_E_ARG;
  *out = nullptr;
  if (n_sub < 1 || n_lambda < 0 || n_primal < 0 || nrhs < 1 || nrhs > IETIDP_MAX_RHS) return IETIDP_E_ARG;
  ietidp_s* h = new (std::nothrow) ietidp_s();
  if (!h) return IETIDP_E_NOMEM;
  if (opt) h->opt = *opt;
  else ietidp_options_default(&h->opt);
  if (h->opt.leaf_size <= 0) h->opt.leaf_size = 96;
  h->n_sub = n_sub;
  h->n_lambda = n_lambda;
  h->n_primal = n_primal;
  h->nrhs = nrhs;
  h->in.resize(n_sub);
  h->rep.failed_subdomain = -1;
  *out = h;
  return guard(h, [&]() {
    require(h->opt.tol >= 0.0 && h->opt.max_iter >= 0 && h->opt.fixed_iters >= 0, IETIDP_E_ARG, "bad options");
    require(h->opt.scaling == IETIDP_SCALE_MULTIPLICITY || h->opt.scaling == IETIDP_SCALE_STIFFNESS, IETIDP_E_ARG,
            "bad scaling");
    require(h->opt.loop == IETIDP_LOOP_EXPLICIT || h->opt.loop == IETIDP_LOOP_TRIANGULAR, IETIDP_E_ARG,
            "bad loop operators");
    if (h->opt.device < 0) return;  // host-only analysis mode (tests without a GPU)
    set_device(h);
    if (h->opt.stream) {
      h->stream = (cudaStream_t)h->opt.stream;
    } else {
      IETI_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
      h->own_stream = true;
    }
    if (const char* tp = getenv("IETIDP_TRACE")) {
      h->trace.on = true;
      h->trace.path = tp;
    }
  });
}

ietidp_status ietidp_set_subdomain(ietidp_t h, int k, int n_k, const int64_t* K_rowptr, const int32_t* K_col,
                                   const double* K_val, const double* f, int nB, const int32_t* B_lambda,
                                   const int32_t* B_dof, const int8_t* B_sign, int n_tree, const int32_t* tree_dofs,
                                   int n_prim, const int32_t* prim_dofs, const int32_t* prim_global) {
  return guard(h, [&]() {
    require(!h->analyzed, IETIDP_E_STATE, "set_subdomain after analysis");
    require(k >= 0 && k < h->n_sub, IETIDP_E_ARG, "subdomain index out of range");
    require(!h->in[k].set, IETIDP_E_STATE, "subdomain set twice");
    require(n_k >= 0 && nB >= 0 && n_tree >= 0 && n_prim >= 0, IETIDP_E_ARG, "negative size");
    require(K_rowptr && (n_k == 0 || (K_col && K_val && f)), IETIDP_E_ARG, "null pointer");
    require(nB == 0 || (B_lambda && B_dof && B_sign), IETIDP_E_ARG, "null B pointer");
    require(n_tree == 0 || tree_dofs, IETIDP_E_ARG, "null tree pointer");
    require(n_prim == 0 || (prim_dofs && prim_global), IETIDP_E_ARG, "null primal pointer");
    ieti::SubIn& in = h->in[k];
    in.n = n_k;
    require(K_rowptr[0] == 0, IETIDP_E_ARG, "rowptr[0] != 0");
    const int64_t nnz = K_rowptr[n_k];
    require(nnz >= 0 && nnz < (int64_t)INT_MAX, IETIDP_E_ARG, "bad nnz");
    in.rowptr.assign(K_rowptr, K_rowptr + n_k + 1);
    in.col.assign(K_col, K_col + nnz);
    in.val.assign(K_val, K_val + nnz);
    in.f.assign(f, f + (size_t)n_k * h->nrhs);
    for (int i = 0; i < n_k; ++i) {
      require(in.rowptr[i + 1] >= in.rowptr[i], IETIDP_E_ARG, "rowptr not monotone");
      for (int64_t e = in.rowptr[i]; e < in.rowptr[i + 1]; ++e) {
        require(in.col[e] >= 0 && in.col[e] < n_k, IETIDP_E_ARG, "column index out of range");
        require(e == in.rowptr[i] || in.col[e] > in.col[e - 1], IETIDP_E_ARG, "CSR columns not sorted/unique");
      }
    }
    // pattern symmetry in one sweep: rows i in increasing order; each upper entry (i, j)
    // must be the next unvisited lower entry of row j (cursor nx[j]); afterwards every
    // row's lower entries must all have been visited
    {
      std::vector<int64_t> nx(in.rowptr.begin(), in.rowptr.end() - 1);
      for (int i = 0; i < n_k; ++i)
        for (int64_t e = in.rowptr[i]; e < in.rowptr[i + 1]; ++e) {
          const int j = in.col[e];
          if (j <= i) continue;
          const int64_t q = nx[j];
          require(q < in.rowptr[j + 1] && in.col[q] == i, IETIDP_E_ARG, "CSR pattern not symmetric");
          nx[j] = q + 1;
        }
      for (int j = 0; j < n_k; ++j)
        require(nx[j] == in.rowptr[j + 1] || in.col[nx[j]] >= j, IETIDP_E_ARG, "CSR pattern not symmetric");
    }
    in.B_lambda.assign(B_lambda, B_lambda + nB);
    in.B_dof.assign(B_dof, B_dof + nB);
    in.B_sign.assign(B_sign, B_sign + nB);
    for (int e = 0; e < nB; ++e) {
      require(in.B_lambda[e] >= 0 && in.B_lambda[e] < h->n_lambda, IETIDP_E_ARG, "B multiplier out of range");
      require(in.B_dof[e] >= 0 && in.B_dof[e] < n_k, IETIDP_E_ARG, "B DOF out of range");
      if (in.B_sign[e] != 1 && in.B_sign[e] != -1) throw Error(IETIDP_E_B_STRUCTURE, "B sign not +1/-1");
    }
    in.tree.assign(tree_dofs, tree_dofs + n_tree);
    for (int t : in.tree) require(t >= 0 && t < n_k, IETIDP_E_ARG, "tree DOF out of range");
    in.prim.assign(prim_dofs, prim_dofs + n_prim);
    in.prim_gid.assign(prim_global, prim_global + n_prim);
    for (int q = 0; q < n_prim; ++q) {
      require(in.prim[q] >= 0 && in.prim[q] < n_k, IETIDP_E_ARG, "primal DOF out of range");
      require(in.prim_gid[q] >= 0 && in.prim_gid[q] < h->n_primal, IETIDP_E_ARG, "primal id out of range");
    }
    // pattern fingerprint (the analysis groups subdomains with identical patterns and
    // compares the members of a group in full)
    in.B_dof_sorted = in.B_dof;
    std::sort(in.B_dof_sorted.begin(), in.B_dof_sorted.end());
    uint64_t x = 1469598103934665603ull;
    auto mix = [&](const void* p, size_t nb) {  // 64-bit words (tail bytes), multiply-xorshift
      const unsigned char* b = static_cast<const unsigned char*>(p);
      size_t i = 0;
      for (; i + 8 <= nb; i += 8) {
        uint64_t w;
        memcpy(&w, b + i, 8);
        x = (x ^ w) * 0x9E3779B97F4A7C15ull;
        x ^= x >> 29;
      }
      for (; i < nb; ++i) x = (x ^ b[i]) * 1099511628211ull;
    };
    auto mixv = [&](const auto& v) {
      const uint64_t nv = v.size();
      mix(&nv, sizeof(nv));
      if (nv) mix(v.data(), nv * sizeof(v[0]));
    };
    mix(&in.n, sizeof(in.n));
    mixv(in.rowptr);
    mixv(in.col);
    mixv(in.tree);
    mixv(in.prim);
    mixv(in.B_dof_sorted);
    in.fp = x;
    in.set = true;
  });
}

// ---- sharded mode (include/ietidp_shard.h) ----
ietidp_status ietidp_shard_enable(ietidp_t h, int rank, int nranks, ietidp_allreduce_fn fn, void* ctx) {
  return guard(h, [&]() {
    require(!h->analyzed, IETIDP_E_STATE, "shard_enable after analysis");
    require(fn != nullptr && nranks >= 1 && rank >= 0 && rank < nranks, IETIDP_E_ARG, "bad rank or null all-reduce");
    require(h->opt.loop == IETIDP_LOOP_EXPLICIT, IETIDP_E_ARG, "the sharded solve runs the explicit loop");
    require(h->opt.stop == IETIDP_STOP_RESIDUAL, IETIDP_E_ARG, "the sharded solve uses the residual stopping criterion");
    h->shard = true;
    h->sh_rank = rank;
    h->sh_n = nranks;
    h->sh_allreduce = fn;
    h->sh_ctx = ctx;
  });
}

namespace {
// ncclAllReduce(sendbuff, recvbuff, count, datatype, op, comm, stream); ncclFloat64 = 8, ncclSum = 0
typedef int (*nccl_allreduce_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
int nccl_trampoline(void* ctx, double* buf, int64_t n, void* stream) {
  ietidp_s* h = static_cast<ietidp_s*>(ctx);
  return reinterpret_cast<nccl_allreduce_t>(h->sh_nccl_fn)(buf, buf, (size_t)n, 8, 0, h->sh_nccl_comm,
                                                           static_cast<cudaStream_t>(stream));
}
}  // namespace

ietidp_status ietidp_shard_enable_nccl(ietidp_t h, int rank, int nranks, void* nccl_comm, void* nccl_allreduce) {
  if (h && (!nccl_comm || !nccl_allreduce)) {
    h->err = "null NCCL communicator or ncclAllReduce address";
    return IETIDP_E_ARG;
  }
  ietidp_status st = ietidp_shard_enable(h, rank, nranks, nccl_trampoline, h);
  if (st == IETIDP_OK) {
    h->sh_nccl_comm = nccl_comm;
    h->sh_nccl_fn = nccl_allreduce;
  }
  return st;
}

ietidp_status ietidp_shard_partition(int n_sub, const double* weight, int nranks, int32_t* owner) {
  if (n_sub < 1 || nranks < 1 || !weight || !owner) return IETIDP_E_ARG;
  double total = 0.0;
  for (int k = 0; k < n_sub; ++k) {
    if (!(weight[k] > 0.0)) return IETIDP_E_ARG;
    total += weight[k];
  }
  // contiguous ranges: rank r ends where the running weight passes (r + 1) / nranks of the
  // total (the subdomain straddling a cut goes to the side holding more of it), leaving at
  // least one subdomain for every later rank
  double run = 0.0;
  int r = 0;
  for (int k = 0; k < n_sub; ++k) {
    const double cut = total * (r + 1) / nranks;
    const int left_after = n_sub - k;        // subdomains k .. n_sub-1 still to place
    const int ranks_after = nranks - r - 1;  // ranks after r
    const bool must_advance = left_after <= ranks_after;  // keep one per later rank
    const bool want_advance = run + 0.5 * weight[k] > cut;
    bool started = k > 0 && owner[k - 1] == r;
    if (r < nranks - 1 && started && (must_advance || want_advance)) ++r;
    owner[k] = r;
    run += weight[k];
  }
  return IETIDP_OK;
}

ietidp_status ietidp_analyze(ietidp_t h) {
  return guard(h, [&]() {
    require(!h->analyzed, IETIDP_E_STATE, "already analyzed");
    if (h->opt.device >= 0) set_device(h);
    NvtxRange nv("ietidp_analyze");
    ieti::analyze_all(h);
    if (h->opt.device >= 0) {
      // The copy stream and the per-subdomain copy events exist before the first
      // factorisation is captured into a graph, so the graph always carries the
      // external waits on them (a later ietidp_set_values is then ordered before
      // the replayed factorisation). Each event is recorded once here (complete).
      IETI_CUDA(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
      h->kev.resize(h->n_sub);
      for (auto& e : h->kev) {
        IETI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        IETI_CUDA(cudaEventRecord(e, h->cstream));
      }
      IETI_CUDA(cudaEventCreateWithFlags(&h->hp_ev_set, cudaEventDisableTiming));
    }
    h->analyzed = true;
  });
}

ietidp_status ietidp_set_values(ietidp_t h, int k, const double* K_val, const double* f) {
  return guard(h, [&]() {
    require(h->analyzed, IETIDP_E_STATE, "set_values before analysis");
    require(k >= 0 && k < h->n_sub, IETIDP_E_ARG, "subdomain index out of range");
    const ieti::SubIn& in = h->in[k];
    // copies on a dedicated stream, one event per subdomain: the next factorisation
    // starts a subdomain group as soon as that group's values have arrived
    require(h->cstream != nullptr, IETIDP_E_STATE, "set_values on a host-only handle");
    IETI_CUDA(cudaEventRecord(h->hp_ev_set, h->stream));  // after the caller's prior work
    IETI_CUDA(cudaStreamWaitEvent(h->cstream, h->hp_ev_set, 0));
    if (K_val)
      IETI_CUDA(cudaMemcpyAsync(h->kval.p + h->kval_off[k], K_val, in.val.size() * sizeof(double),
                                cudaMemcpyHostToDevice, h->cstream));
    if (f)
      IETI_CUDA(cudaMemcpyAsync(h->fval.p + h->fval_off[k], f, (size_t)in.n * h->nrhs * sizeof(double),
                                cudaMemcpyHostToDevice, h->cstream));
    IETI_CUDA(cudaEventRecord(h->kev[k], h->cstream));
    h->factored = false;
    h->solved = false;
  });
}

ietidp_status ietidp_set_values_device(ietidp_t h, int k, const double* d_K_val, const double* d_f) {
  return guard(h, [&]() {
    require(h->analyzed, IETIDP_E_STATE, "set_values before analysis");
    require(k >= 0 && k < h->n_sub, IETIDP_E_ARG, "subdomain index out of range");
    const ieti::SubIn& in = h->in[k];
    require(h->cstream != nullptr, IETIDP_E_STATE, "set_values on a host-only handle");
    // device-to-device on the handle's stream (the producer's work on that stream, e.g. the
    // assembly kernels' results made visible by the caller, is ordered before it); the copy
    // stream's event of the subdomain is re-recorded behind it so that the captured
    // factorisation graph's external wait still covers the latest values
    if (d_K_val)
      IETI_CUDA(cudaMemcpyAsync(h->kval.p + h->kval_off[k], d_K_val, in.val.size() * sizeof(double),
                                cudaMemcpyDeviceToDevice, h->stream));
    if (d_f)
      IETI_CUDA(cudaMemcpyAsync(h->fval.p + h->fval_off[k], d_f, (size_t)in.n * h->nrhs * sizeof(double),
                                cudaMemcpyDeviceToDevice, h->stream));
    IETI_CUDA(cudaEventRecord(h->hp_ev_set, h->stream));
    IETI_CUDA(cudaStreamWaitEvent(h->cstream, h->hp_ev_set, 0));
    IETI_CUDA(cudaEventRecord(h->kev[k], h->cstream));
    h->factored = false;
    h->solved = false;
  });
}

// the lower-triangle maps of every pattern class (host integer work, once)
static void prepare_lower(ietidp_t h) {
  const int ns = h->n_sub;
  h->low_off.assign(ns + 1, 0);
  h->low_n.assign(ns, 0);
  h->low_map_off.assign(ns, -1);
  std::vector<int> map;
  for (int k = 0; k < ns; ++k) {
    const ieti::SubIn& in = h->in[k];
    long long nl = 0;
    for (int i = 0; i < in.n; ++i)
      for (int64_t e = in.rowptr[i]; e < in.rowptr[i + 1]; ++e) nl += in.col[e] <= i;
    h->low_n[k] = nl;
    h->low_off[k + 1] = h->low_off[k] + nl;
    const int r = h->class_rep[k];
    if (h->low_map_off[r] >= 0) continue;
    h->low_map_off[r] = (long long)map.size();
    const ieti::SubIn& rin = h->in[r];
    const size_t base = map.size();
    map.resize(base + rin.col.size());
    // lower index of the entries of row i: lowstart[i] + (e - rowptr[i]) for col <= i;
    // an upper entry (i, j) is the next unvisited lower entry of row j (cursor nx[j])
    std::vector<long long> lowstart(rin.n + 1, 0);
    for (int i = 0; i < rin.n; ++i) {
      long long c = 0;
      for (int64_t e = rin.rowptr[i]; e < rin.rowptr[i + 1]; ++e) c += rin.col[e] <= i;
      lowstart[i + 1] = lowstart[i] + c;
    }
    std::vector<int64_t> nx(rin.rowptr.begin(), rin.rowptr.end() - 1);
    for (int i = 0; i < rin.n; ++i)
      for (int64_t e = rin.rowptr[i]; e < rin.rowptr[i + 1]; ++e) {
        const int j = rin.col[e];
        if (j <= i) {
          map[base + e] = (int)(lowstart[i] + (e - rin.rowptr[i]));
        } else {
          const int64_t q = nx[j]++;  // (j, i): the pattern is symmetric (checked at set_subdomain)
          map[base + e] = (int)(lowstart[j] + (q - rin.rowptr[j]));
        }
      }
  }
  set_device(h);
  h->low_map.upload(map, h->stream);
  h->klow.alloc(std::max<long long>(1, h->low_off[ns]));
  IETI_CUDA(cudaStreamSynchronize(h->stream));
  h->lower_ready = true;
}

ietidp_status ietidp_set_values_lower(ietidp_t h, int k, const double* K_lower_val, const double* f) {
  return guard(h, [&]() {
    require(h->analyzed, IETIDP_E_STATE, "set_values_lower before analysis");
    require(k >= 0 && k < h->n_sub, IETIDP_E_ARG, "subdomain index out of range");
    require(h->cstream != nullptr, IETIDP_E_STATE, "set_values_lower on a host-only handle");
    if (!h->lower_ready) prepare_lower(h);
    const ieti::SubIn& in = h->in[k];
    IETI_CUDA(cudaEventRecord(h->hp_ev_set, h->stream));  // after the caller's prior work
    IETI_CUDA(cudaStreamWaitEvent(h->cstream, h->hp_ev_set, 0));
    if (K_lower_val) {
      IETI_CUDA(cudaMemcpyAsync(h->klow.p + h->low_off[k], K_lower_val, h->low_n[k] * sizeof(double),
                                cudaMemcpyHostToDevice, h->cstream));
      ieti::launch_expand_lower(h, k, h->cstream);
    }
    if (f)
      IETI_CUDA(cudaMemcpyAsync(h->fval.p + h->fval_off[k], f, (size_t)in.n * h->nrhs * sizeof(double),
                                cudaMemcpyHostToDevice, h->cstream));
    IETI_CUDA(cudaEventRecord(h->kev[k], h->cstream));
    h->factored = false;
    h->solved = false;
  });
}

ietidp_status ietidp_factor(ietidp_t h) {
  if (h && !h->analyzed) {
    ietidp_status st = ietidp_analyze(h);
    if (st != IETIDP_OK) return st;
  }
  return guard(h, [&]() {
    NvtxRange nv("ietidp_factor");
    set_device(h);
    h->factored = false;
    h->solved = false;
    h->factor_failed = true;
    // The factorisation's critical path runs on an internal highest-priority stream
    // (ordered after the caller's stream and joined back into it), so that its
    // latency-bound panel kernels are scheduled ahead of the side stream's work.
    if (!h->hp) {
      int lo = 0, hi = 0;
      IETI_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      IETI_CUDA(cudaStreamCreateWithPriority(&h->hp, cudaStreamNonBlocking, hi));
      IETI_CUDA(cudaEventCreateWithFlags(&h->hp_ev, cudaEventDisableTiming));
      for (auto& e : h->fg_ev) IETI_CUDA(cudaEventCreate(&e));
    }
    cudaStream_t user = h->stream;
    IETI_CUDA(cudaEventRecord(h->hp_ev, user));
    IETI_CUDA(cudaStreamWaitEvent(h->hp, h->hp_ev, 0));
    h->stream = h->hp;
    EvPair e1, e2;
    // The ~200 launches of the factorisation and coarse set-up (two streams, events)
    // are captured once into a CUDA graph and replayed: the plan and buffers are fixed
    // after analyze, so every factor call launches the same work. Not with the launch
    // tracer; IETIDP_GRAPH=0 launches directly.
    const bool use_graph = !h->trace.on && !(getenv("IETIDP_GRAPH") && atoi(getenv("IETIDP_GRAPH")) == 0);
    // sharded mode: the coarse set-up calls the all-reduce (host side), so only the
    // factorisation is captured and the coarse set-up is launched directly after it
    const bool coarse_in_graph = !h->shard;
    try {
      if (use_graph && !h->fgraph) {
        const long long l0 = h->launches;
        cudaGraph_t g = nullptr;
        IETI_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed));
        IETI_CUDA(cudaEventRecordWithFlags(h->fg_ev[0], h->stream, cudaEventRecordExternal));
        ieti::run_factor(h);
        IETI_CUDA(cudaEventRecordWithFlags(h->fg_ev[1], h->stream, cudaEventRecordExternal));
        if (coarse_in_graph) {
          ieti::run_coarse(h);
          IETI_CUDA(cudaEventRecordWithFlags(h->fg_ev[2], h->stream, cudaEventRecordExternal));
        }
        IETI_CUDA(cudaStreamEndCapture(h->stream, &g));
        IETI_CUDA(cudaGraphInstantiate(&h->fgraph, g, 0));
        cudaGraphDestroy(g);
        h->fgraph_launches = h->launches - l0;
        h->launches = l0;
      }
      if (use_graph) {
        IETI_CUDA(cudaGraphLaunch(h->fgraph, h->stream));
        h->launches += h->fgraph_launches;
        if (!coarse_in_graph) {
          ieti::run_coarse(h);
          IETI_CUDA(cudaEventRecord(h->fg_ev[2], h->stream));
        }
      } else {
        IETI_CUDA(cudaEventRecord(h->fg_ev[0], h->stream));
        h->trace.start(h->stream);
        ieti::run_factor(h);
        IETI_CUDA(cudaEventRecord(h->fg_ev[1], h->stream));
        ieti::run_coarse(h);
        IETI_CUDA(cudaEventRecord(h->fg_ev[2], h->stream));
      }
    } catch (...) {
      if (h->fgraph == nullptr) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(h->stream, &g);  // abandon a failed capture
        if (g) cudaGraphDestroy(g);
      }
      h->stream = user;
      throw;
    }
    h->stream = user;
    IETI_CUDA(cudaEventRecord(h->hp_ev, h->hp));
    IETI_CUDA(cudaStreamWaitEvent(user, h->hp_ev, 0));
    int flags[2];
    IETI_CUDA(cudaMemcpyAsync(flags, h->err_flag.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    IETI_CUDA(cudaStreamSynchronize(h->stream));
    h->trace.dump("factor");
    {
      float t1 = 0.f, t2 = 0.f;
      cudaEventElapsedTime(&t1, h->fg_ev[0], h->fg_ev[1]);
      cudaEventElapsedTime(&t2, h->fg_ev[1], h->fg_ev[2]);
      h->rep.ms_factor = t1;
      h->rep.ms_coarse = t2;
    }
    (void)e1;
    (void)e2;
    if (flags[0] != INT_MAX) {
      h->failed_sub = flags[0];
      h->rep.failed_subdomain = flags[0];
      throw Error(IETIDP_E_NOT_SPD, "K_rr of subdomain " + std::to_string(flags[0]) + " is not SPD");
    }
    if (flags[1] == 0) {
      h->failed_sub = -1;
      h->rep.failed_subdomain = -1;
      throw Error(IETIDP_E_NOT_SPD, "coarse matrix S_PP is not SPD");
    }
    h->rep.failed_subdomain = -1;
    h->factor_failed = false;
    h->factored = true;
  });
}

ietidp_status ietidp_solve(ietidp_t h, double* lambda, ietidp_report* report) {
  bool noconv = false;
  ietidp_status st = guard(h, [&]() {
    require(h->factored, IETIDP_E_STATE, "solve before a successful factor");
    set_device(h);
    EvPair e1, e2;
    IETI_CUDA(cudaEventRecord(e1.a, h->stream));
    h->trace.start(h->stream);
    {
      NvtxRange nv("ietidp_solve: PCG");
      ieti::run_solve(h);
    }
    NvtxRange nvr("ietidp_solve: recovery");
    IETI_CUDA(cudaEventRecord(e1.b, h->stream));
    IETI_CUDA(cudaEventRecord(e2.a, h->stream));
    // the recovery's ~40 launches (backward sweep level by level) as a captured graph
    const bool use_graph =
        !h->shard && !h->trace.on && !(getenv("IETIDP_GRAPH") && atoi(getenv("IETIDP_GRAPH")) == 0);
    if (use_graph) {
      if (!h->rgraph) {
        const long long l0 = h->launches;
        cudaGraph_t g = nullptr;
        IETI_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed));
        try {
          ieti::run_recover(h);
        } catch (...) {
          cudaStreamEndCapture(h->stream, &g);
          if (g) cudaGraphDestroy(g);
          throw;
        }
        IETI_CUDA(cudaStreamEndCapture(h->stream, &g));
        IETI_CUDA(cudaGraphInstantiate(&h->rgraph, g, 0));
        cudaGraphDestroy(g);
        h->rgraph_launches = h->launches - l0;
        h->launches = l0;
      }
      IETI_CUDA(cudaGraphLaunch(h->rgraph, h->stream));
      h->launches += h->rgraph_launches;
    } else {
      ieti::run_recover(h);
    }
    IETI_CUDA(cudaEventRecord(e2.b, h->stream));
    ieti::finish_solve(h, &h->rep);
    h->trace.dump("solve");
    h->rep.ms_pcg = e1.ms();
    h->rep.ms_recover = e2.ms();
    if (lambda && h->n_lambda) {
      ieti::transpose_out(h, h->n_lambda, h->nrhs, h->lam_vec.p, h->tmp_out.p);
      IETI_CUDA(cudaMemcpyAsync(lambda, h->tmp_out.p, (size_t)h->n_lambda * h->nrhs * sizeof(double),
                                cudaMemcpyDeviceToHost, h->stream));
      IETI_CUDA(cudaStreamSynchronize(h->stream));
    }
    h->solved = true;
    if (!h->opt.fixed_iters)
      for (int c = 0; c < h->nrhs; ++c)
        if (!h->rep.converged[c]) noconv = true;
  });
  if (h) {
    h->rep.n_sub = h->n_sub;
    h->rep.n_lambda = h->n_lambda;
    h->rep.n_primal = h->n_primal;
    h->rep.nrhs = h->nrhs;
    if (report) *report = h->rep;
  }
  if (st == IETIDP_OK && noconv) {
    h->err = "PCG reached max_iter without convergence";
    return IETIDP_E_NO_CONVERGENCE;
  }
  return st;
}

ietidp_status ietidp_get_u(ietidp_t h, int k, double* u) {
  return guard(h, [&]() {
    require(h->solved, IETIDP_E_STATE, "no solution yet");
    require(k >= 0 && k < h->n_sub && u, IETIDP_E_ARG, "bad argument");
    IETI_CUDA(cudaMemcpyAsync(u, h->U.p + h->u_off[k], (size_t)h->in[k].n * h->nrhs * sizeof(double),
                              cudaMemcpyDeviceToHost, h->stream));
    IETI_CUDA(cudaStreamSynchronize(h->stream));
  });
}

ietidp_status ietidp_get_u_device(ietidp_t h, int k, double* d_u) {
  return guard(h, [&]() {
    require(h->solved, IETIDP_E_STATE, "no solution yet");
    require(k >= 0 && k < h->n_sub && d_u, IETIDP_E_ARG, "bad argument");
    IETI_CUDA(cudaMemcpyAsync(d_u, h->U.p + h->u_off[k], (size_t)h->in[k].n * h->nrhs * sizeof(double),
                              cudaMemcpyDeviceToDevice, h->stream));
  });
}

ietidp_status ietidp_get_lambda_device(ietidp_t h, double* d_lambda) {
  return guard(h, [&]() {
    require(h->solved, IETIDP_E_STATE, "no solution yet");
    require(d_lambda || h->n_lambda == 0, IETIDP_E_ARG, "null pointer");
    if (h->n_lambda) ieti::transpose_out(h, h->n_lambda, h->nrhs, h->lam_vec.p, d_lambda);
  });
}

static ietidp_status apply_op(ietidp_t h, int ncols, const double* d_x, double* d_y, bool F) {
  return guard(h, [&]() {
    require(h->factored, IETIDP_E_STATE, "operator before a successful factor");
    require(ncols >= 1 && ncols <= h->nrhs, IETIDP_E_ARG, "ncols out of range");
    require(h->n_lambda == 0 || (d_x && d_y), IETIDP_E_ARG, "null pointer");
    if (h->n_lambda == 0) return;
    set_device(h);
    const double* xin = d_x;
    double* yout = d_y;
    if (ncols > 1) {
      ieti::transpose_in(h, h->n_lambda, ncols, d_x, h->tmp_in.p);
      xin = h->tmp_in.p;
      yout = h->tmp_out.p;
    }
    if (F) ieti::run_apply_F(h, ncols, xin, yout);
    else ieti::run_apply_M(h, ncols, xin, yout);
    if (ncols > 1) ieti::transpose_out(h, h->n_lambda, ncols, h->tmp_out.p, d_y);
  });
}

ietidp_status ietidp_apply_F(ietidp_t h, int ncols, const double* d_x, double* d_y) {
  return apply_op(h, ncols, d_x, d_y, true);
}
ietidp_status ietidp_apply_precond(ietidp_t h, int ncols, const double* d_x, double* d_y) {
  return apply_op(h, ncols, d_x, d_y, false);
}

ietidp_status ietidp_get_coarse(ietidp_t h, double* S) {
  return guard(h, [&]() {
    require(h->factored, IETIDP_E_STATE, "coarse matrix before factor");
    require(S || h->n_primal == 0, IETIDP_E_ARG, "null pointer");
    if (!h->n_primal) return;
    IETI_CUDA(cudaMemcpyAsync(S, h->S.p, (size_t)h->n_primal * h->n_primal * sizeof(double), cudaMemcpyDeviceToHost,
                              h->stream));
    IETI_CUDA(cudaStreamSynchronize(h->stream));
  });
}

ietidp_status ietidp_estimate_condition(ietidp_t h, double* omega_min, double* omega_max, double* cond) {
  return guard(h, [&]() {
    require(h->solved, IETIDP_E_STATE, "condition estimate before a solve");
    set_device(h);
    ieti::run_estimate_condition(h, omega_min, omega_max, cond);
  });
}

ietidp_status ietidp_get_pcg_coefficients(ietidp_t h, int ld, double* alpha, double* beta) {
  return guard(h, [&]() {
    require(h->solved, IETIDP_E_STATE, "PCG coefficients before a solve");
    const int nc = h->nrhs, cl = h->coef_ld;
    int kmax = 0;
    for (int c = 0; c < nc; ++c) kmax = std::max(kmax, h->rep.iters[c]);
    require(ld >= kmax && ld >= 0, IETIDP_E_ARG, "ld smaller than the iteration count");
    std::vector<double> co(2 * (size_t)nc * cl);
    IETI_CUDA(cudaMemcpyAsync(co.data(), h->cgcoef.p, co.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    IETI_CUDA(cudaStreamSynchronize(h->stream));
    for (int c = 0; c < nc; ++c) {
      const int k = std::min(h->rep.iters[c], cl);
      for (int j = 0; j < ld; ++j) {
        if (alpha) alpha[(size_t)c * ld + j] = j < k ? co[(size_t)c * cl + j] : 0.0;
        if (beta) beta[(size_t)c * ld + j] = j < k - 1 ? co[(size_t)(nc + c) * cl + j] : 0.0;
      }
    }
  });
}

ietidp_status ietidp_get_rhs(ietidp_t h, double* d) {
  return guard(h, [&]() {
    require(h->factored, IETIDP_E_STATE, "rhs before factor");
    require(d || h->n_lambda == 0, IETIDP_E_ARG, "null pointer");
    if (!h->n_lambda) return;
    ieti::transpose_out(h, h->n_lambda, h->nrhs, h->d_vec.p, h->tmp_out.p);
    IETI_CUDA(cudaMemcpyAsync(d, h->tmp_out.p, (size_t)h->n_lambda * h->nrhs * sizeof(double),
                              cudaMemcpyDeviceToHost, h->stream));
    IETI_CUDA(cudaStreamSynchronize(h->stream));
  });
}

ietidp_status ietidp_get_report(ietidp_t h, ietidp_report* r) {
  if (!h || !r) return IETIDP_E_ARG;
  h->rep.n_sub = h->n_sub;
  h->rep.n_lambda = h->n_lambda;
  h->rep.n_primal = h->n_primal;
  h->rep.nrhs = h->nrhs;
  *r = h->rep;
  return IETIDP_OK;
}

long long ietidp_kernel_launches(ietidp_t h) { return h ? h->launches : 0; }

const char* ietidp_last_error(ietidp_t h) { return h ? h->err.c_str() : "null handle"; }

void ietidp_destroy(ietidp_t h) {
  if (!h) return;
  if (h->opt.device >= 0) cudaSetDevice(h->opt.device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  ieti::destroy_graph(h);
  for (auto e : h->fev) cudaEventDestroy(e);
  for (auto e : h->pev) cudaEventDestroy(e);
  if (h->hp_ev) cudaEventDestroy(h->hp_ev);
  for (auto e : h->fg_ev)
    if (e) cudaEventDestroy(e);
  if (h->fgraph) cudaGraphExecDestroy(h->fgraph);
  if (h->rgraph) cudaGraphExecDestroy(h->rgraph);
  if (h->hp) cudaStreamDestroy(h->hp);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->cstream) cudaStreamDestroy(h->cstream);
  for (auto e : h->kev) cudaEventDestroy(e);
  if (h->hp_ev_set) cudaEventDestroy(h->hp_ev_set);
  for (auto x : h->gst)
    if (x) cudaStreamDestroy(x);
  for (auto x : h->gside)
    if (x) cudaStreamDestroy(x);
  for (auto e : h->gev) cudaEventDestroy(e);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

}  // extern "C"
