// Host-side set-up of the IETI-DP solve phase: validation of the C-ABI inputs,
// DOF classification (tree / primal / r_V / r_I),
// nested-dissection ordering of r_V with r_I last,
// symbolic supernodal factorisation and the batched level schedule.
//
// This is integer work only (the documented host exception, like a
// sparse direct solver's reordering); every floating-point operation of the
// method runs in the CUDA kernels. Values are never touched here except for
// being copied to the device.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <set>
#include <thread>
#include <unordered_map>

#include "handle.h"

namespace ieti {

namespace {

struct LocalResult {
  SubPlan sp;
  std::vector<SnHost> sn;  // local ids, parent local
  ietidp_status st = IETIDP_OK;
  std::string err;
};

// ---------------------------------------------------------------------------
// Nested dissection on the graph of K_VV (level-structure vertex separators)
// ---------------------------------------------------------------------------
// Minimum-degree ordering of r_V on the quotient graph (variables and elements, the
// approximate external degree bound of Amestoy-Davis-Duff AMD; no supervariables, no
// aggressive absorption), deterministic ties by (degree, index). Returns order[k] =
// variable eliminated k-th.
static std::vector<int> min_degree_order(const std::vector<int>& xadj, const std::vector<int>& adj, int n) {
  std::vector<std::vector<int>> av(n), ae(n), ev(n);
  std::vector<int> deg(n), state(n, 0);  // 0 live variable, 1 element, 2 absorbed element / eliminated
  std::vector<int> wstamp(n, -1), w(n, 0), mark(n, -1);
  std::set<std::pair<int, int>> pq;
  for (int i = 0; i < n; ++i) {
    av[i].assign(adj.begin() + xadj[i], adj.begin() + xadj[i + 1]);
    deg[i] = (int)av[i].size();
    pq.insert({deg[i], i});
  }
  std::vector<int> order;
  order.reserve(n);
  std::vector<int> Lp;
  for (int k = 0; k < n; ++k) {
    const int p = pq.begin()->second;
    pq.erase(pq.begin());
    order.push_back(p);
    // new element Lp = (A_p u union of the elements of p) \ {p}
    Lp.clear();
    mark[p] = k;
    for (int v : av[p])
      if (state[v] == 0 && mark[v] != k) {
        mark[v] = k;
        Lp.push_back(v);
      }
    for (int e : ae[p]) {
      if (state[e] != 1) continue;
      for (int v : ev[e])
        if (state[v] == 0 && mark[v] != k) {
          mark[v] = k;
          Lp.push_back(v);
        }
      state[e] = 2;  // absorbed into p
      std::vector<int>().swap(ev[e]);
    }
    state[p] = 1;
    ev[p] = Lp;
    std::vector<int>().swap(av[p]);
    std::vector<int>().swap(ae[p]);
    // w(e) = |L_e \ Lp| for the live elements adjacent to Lp
    for (int i : Lp)
      for (int e : ae[i]) {
        if (state[e] != 1 || e == p) continue;
        if (wstamp[e] != k) {
          wstamp[e] = k;
          w[e] = (int)ev[e].size();
        }
        --w[e];
      }
    const int nlive = n - k - 1;
    for (int i : Lp) {
      // prune: dead elements out, p in; variables of Lp (now reached through p) out
      std::vector<int>& E = ae[i];
      size_t q = 0;
      int ext = 0;
      for (int e : E)
        if (state[e] == 1 && e != p) {
          E[q++] = e;
          ext += (wstamp[e] == k) ? w[e] : (int)ev[e].size();
        }
      E.resize(q);
      E.push_back(p);
      std::vector<int>& A = av[i];
      q = 0;
      for (int v : A)
        if (state[v] == 0 && mark[v] != k) A[q++] = v;
      A.resize(q);
      int d = (int)A.size() + (int)Lp.size() - 1 + ext;
      d = std::min(d, nlive);
      d = std::min(d, deg[i] + (int)Lp.size() - 1);
      d = std::max(d, 0);
      if (d != deg[i]) {
        pq.erase({deg[i], i});
        deg[i] = d;
        pq.insert({deg[i], i});
      }
    }
  }
  return order;
}

// Fundamental supernodes of the r_V block under the elimination order `order`:
// column structures by the multifrontal merge (struct(j) = adj(j) u children's structs,
// entries > j), etree parent = min row; j joins j+1 when parent(j) = j+1, j is j+1's only
// child and |struct(j)| = |struct(j+1)| + 1. Supernodes in elimination order.
static std::vector<std::vector<int>> md_supernodes(const std::vector<int>& xadj, const std::vector<int>& adj, int n,
                                                   std::vector<int> order, bool postordered = false) {
  std::vector<int> pos(n);
  for (int k = 0; k < n; ++k) pos[order[k]] = k;
  std::vector<std::vector<int>> st(n);
  std::vector<int> parent(n, -1), nchild(n, 0), cnt(n, 0), mark(n, -1);
  std::vector<std::vector<int>> kids(n);
  for (int j = 0; j < n; ++j) {
    std::vector<int>& S = st[j];
    const int v = order[j];
    for (int e = xadj[v]; e < xadj[v + 1]; ++e) {
      const int r = pos[adj[e]];
      if (r > j && mark[r] != j) {
        mark[r] = j;
        S.push_back(r);
      }
    }
    for (int c : kids[j]) {
      for (int r : st[c])
        if (r > j && mark[r] != j) {
          mark[r] = j;
          S.push_back(r);
        }
      std::vector<int>().swap(st[c]);
    }
    std::sort(S.begin(), S.end());
    cnt[j] = (int)S.size();
    if (!S.empty()) {
      parent[j] = S[0];
      kids[S[0]].push_back(j);
      ++nchild[S[0]];
    }
  }
  if (!postordered) {
    // reorder to a postorder of the elimination tree (same fill; makes every subtree,
    // and each node with its last child, contiguous), then redo the symbolic pass
    std::vector<int> post;
    post.reserve(n);
    std::vector<std::pair<int, size_t>> stk;
    for (int r = 0; r < n; ++r) {
      if (parent[r] != -1) continue;
      stk.push_back({r, 0});
      while (!stk.empty()) {
        auto& t = stk.back();
        if (t.second < kids[t.first].size()) {
          const int c = kids[t.first][t.second++];
          stk.push_back({c, 0});
        } else {
          post.push_back(t.first);
          stk.pop_back();
        }
      }
    }
    std::vector<int> order2(n);
    for (int k = 0; k < n; ++k) order2[k] = order[post[k]];
    return md_supernodes(xadj, adj, n, std::move(order2), true);
  }
  // fundamental supernodes: [first, last] column ranges
  struct FS {
    int first, last;
    long long f;      // front size (cnt[first] + 1)
    long long nz;     // stored entries of the front's pivot columns (incl. padding)
    int parent_col;   // etree parent of the last column (-1: root)
  };
  std::vector<FS> fs;
  int first = 0;
  for (int j = 1; j <= n; ++j) {
    if (j < n && parent[j - 1] == j && nchild[j] == 1 && cnt[j - 1] == cnt[j] + 1) continue;
    FS x{first, j - 1, cnt[first] + 1LL, 0, parent[j - 1]};
    const long long np = j - first;
    x.nz = np * x.f - np * (np - 1) / 2;
    fs.push_back(x);
    first = j;
  }
  // relaxed amalgamation: a supernode merges into the next one when that is its parent
  // (contiguous in the order) and the merged front is small or adds few explicit zeros
  std::vector<FS> st2;
  for (const FS& x : fs) {
    st2.push_back(x);
    while (st2.size() >= 2) {
      FS& c = st2[st2.size() - 2];
      FS& q = st2.back();
      if (c.parent_col < q.first || c.parent_col > q.last) break;  // not the parent
      const long long npc = c.last - c.first + 1, npq = q.last - q.first + 1, np = npc + npq;
      const long long fm = npc + q.f;  // child's update rows lie in the parent's front
      const long long nzm = np * fm - np * (np - 1) / 2;
      const long long zeros = nzm - c.nz - q.nz;
      if (!(np <= 16 || (np <= 128 && zeros * 10 <= nzm))) break;
      FS m{c.first, q.last, fm, nzm, q.parent_col};
      st2.pop_back();
      st2.back() = m;
    }
  }
  std::vector<std::vector<int>> sn;
  for (const FS& x : st2) sn.emplace_back(order.begin() + x.first, order.begin() + x.last + 1);
  return sn;
}

struct NestedDissection {
  const std::vector<int>& xadj;
  const std::vector<int>& adj;
  int leaf;
  std::vector<int> reg, stamp, lev, key1, key2;
  int next_reg = 1, cur_stamp = 0;
  struct Node {
    std::vector<int> vars;
    std::vector<int> children;
  };
  std::vector<Node> nodes;

  NestedDissection(const std::vector<int>& xa, const std::vector<int>& ad, int nv, int leaf_)
      : xadj(xa), adj(ad), leaf(leaf_), reg(nv, 0), stamp(nv, 0), lev(nv, 0), key1(nv, 0), key2(nv, 0) {}

  // BFS inside region rid; returns visit order and level starts.
  void bfs(int src, int rid, std::vector<int>& order, std::vector<int>& lstart) {
    ++cur_stamp;
    order.clear();
    lstart.clear();
    order.push_back(src);
    stamp[src] = cur_stamp;
    lev[src] = 0;
    lstart.push_back(0);
    size_t head = 0;
    int curlev = 0;
    while (head < order.size()) {
      int v = order[head];
      if (lev[v] != curlev) {
        curlev = lev[v];
        lstart.push_back((int)head);
      }
      ++head;
      for (int e = xadj[v]; e < xadj[v + 1]; ++e) {
        int u = adj[e];
        if (reg[u] != rid || stamp[u] == cur_stamp) continue;
        stamp[u] = cur_stamp;
        lev[u] = lev[v] + 1;
        order.push_back(u);
      }
    }
    lstart.push_back((int)order.size());
  }

  int degree_in(int v, int rid) const {
    int d = 0;
    for (int e = xadj[v]; e < xadj[v + 1]; ++e) d += (reg[adj[e]] == rid);
    return d;
  }

  // Split the vertices of region `rid` (listed in C) into connected components,
  // each getting a fresh region id.
  std::vector<std::pair<std::vector<int>, int>> components(const std::vector<int>& C, int rid) {
    std::vector<std::pair<std::vector<int>, int>> out;
    for (int v : C) {
      if (reg[v] != rid) continue;
      int nr = next_reg++;
      std::vector<int> comp{v};
      reg[v] = nr;
      for (size_t h = 0; h < comp.size(); ++h) {
        int w = comp[h];
        for (int e = xadj[w]; e < xadj[w + 1]; ++e) {
          int u = adj[e];
          if (reg[u] == rid) {
            reg[u] = nr;
            comp.push_back(u);
          }
        }
      }
      out.emplace_back(std::move(comp), nr);
    }
    return out;
  }

  int make_node(std::vector<int> vars, std::vector<int> children) {
    std::sort(vars.begin(), vars.end());
    nodes.push_back({std::move(vars), std::move(children)});
    return (int)nodes.size() - 1;
  }

  int build(const std::vector<int>& C, int rid) {
    if ((int)C.size() <= leaf) return make_node(C, {});
    std::vector<int> order, lstart;
    // pseudo-peripheral start vertex (George-Liu style)
    int v = C[0];
    int ecc = -1;
    for (int it = 0; it < 5; ++it) {
      bfs(v, rid, order, lstart);
      int nlev = (int)lstart.size() - 1;
      if (nlev - 1 <= ecc) break;
      ecc = nlev - 1;
      int best = order[lstart[nlev - 1]], bd = INT_MAX;
      for (int i = lstart[nlev - 1]; i < lstart[nlev]; ++i) {
        int d = degree_in(order[i], rid);
        if (d < bd) bd = d, best = order[i];
      }
      v = best;
    }
    bfs(v, rid, order, lstart);
    int nlev = (int)lstart.size() - 1;
    if (nlev < 3) return make_node(C, {});
    const int n = (int)C.size();
    // Candidate separators from two keys, each a function whose value changes by at most
    // `lip` along an edge, so that `lip` consecutive values separate the smaller keys
    // from the larger ones:
    //   (1) the BFS level from the pseudo-peripheral corner v (lip 1): corner shells;
    //   (2) d_v - d_w with w the far corner of v (lip 2): on an elongated box its level
    //       sets are planes across the long axis (the shells' area is up to ~2x larger).
    // Each candidate is thinned by moving the vertices with no neighbour on the far side
    // to the near side; the smallest balanced one wins (both sides >= 30% of the rest).
    for (int i = 0; i < n; ++i) key1[order[i]] = lev[order[i]];
    int w = order[lstart[nlev - 1]], bdw = INT_MAX;
    for (int i = lstart[nlev - 1]; i < lstart[nlev]; ++i) {
      int d = degree_in(order[i], rid);
      if (d < bdw) bdw = d, w = order[i];
    }
    std::vector<int> order_w, lstart_w;
    bfs(w, rid, order_w, lstart_w);
    const bool all_reached = (int)order_w.size() == n;
    std::vector<int> best_sep;
    int best_score = INT_MAX;
    std::vector<int> half_sep;
    int hdist = INT_MAX;
    static const double nd_bal = getenv("IETIDP_ND_BAL") ? atof(getenv("IETIDP_ND_BAL")) : 0.30;  // experiments
    auto candidates = [&](const std::vector<int>& key, int kmin, int kmax, int lip) {
      // vertices bucketed by key
      const int nk = kmax - kmin + 1;
      std::vector<int> cnt(nk + 1, 0), byk(n);
      for (int u : C) ++cnt[key[u] - kmin + 1];
      for (int i = 0; i < nk; ++i) cnt[i + 1] += cnt[i];
      {
        std::vector<int> pos(cnt.begin(), cnt.end() - 1);
        for (int u : C) byk[pos[key[u] - kmin]++] = u;
      }
      for (int t = kmin + 1; t + lip - 1 < kmax; ++t) {
        const int hi = t + lip - 1;  // separator keys [t, hi]
        std::vector<int> sep;
        int nA = cnt[t - kmin], nB = n - cnt[hi - kmin + 1];
        for (int i = cnt[t - kmin]; i < cnt[hi - kmin + 1]; ++i) {
          const int x = byk[i];
          bool farB = false;
          for (int e = xadj[x]; e < xadj[x + 1] && !farB; ++e) {
            const int u = adj[e];
            if (reg[u] == rid && key[u] > hi) farB = true;
          }
          if (farB) sep.push_back(x);
          else ++nA;
        }
        const int sz = (int)sep.size(), rest = n - sz;
        const int dist = std::abs(nA - nB);
        if (dist < hdist) hdist = dist, half_sep = sep;
        if (std::min(nA, nB) >= nd_bal * rest && sz < best_score) best_score = sz, best_sep = std::move(sep);
      }
    };
    static const int nd_keys = getenv("IETIDP_ND_KEYS") ? atoi(getenv("IETIDP_ND_KEYS")) : 3;  // experiments
    if (nd_keys & 1) candidates(key1, 0, nlev - 1, 1);
    if (all_reached && (nd_keys & 2)) {
      int kmin = INT_MAX, kmax = INT_MIN;
      for (int u : C) {
        key2[u] = key1[u] - lev[u];  // lev[] now holds d_w
        kmin = std::min(kmin, key2[u]);
        kmax = std::max(kmax, key2[u]);
      }
      if (kmax - kmin >= 3) candidates(key2, kmin, kmax, 2);
    }
    std::vector<int> sep = best_sep.empty() ? half_sep : best_sep;
    if (sep.empty()) return make_node(C, {});
    for (int s : sep) reg[s] = 0;
    std::vector<int> rest;
    rest.reserve(n - sep.size());
    for (int u : C)
      if (reg[u] == rid) rest.push_back(u);
    auto comps = components(rest, rid);
    std::vector<int> ch;
    for (auto& c : comps) ch.push_back(build(c.first, c.second));
    return make_node(std::move(sep), std::move(ch));
  }
};

// Orderings of r_V shared between subdomains whose K_VV graphs are identical (a box
// tiling's subdomains differ only in their interface rows: C5's 27 pattern classes share
// one r_V graph): computed once per distinct graph (fingerprint, then a full comparison).
struct OrderCache {
  struct Entry {
    std::once_flag once;
    std::vector<int> xadj, adj;
    std::vector<std::vector<int>> sn_vars;
  };
  std::mutex mu;
  std::unordered_map<uint64_t, std::shared_ptr<Entry>> map;
};

static uint64_t graph_fingerprint(const std::vector<int>& xadj, const std::vector<int>& adj) {
  uint64_t x = 1469598103934665603ull;
  auto mix = [&](const std::vector<int>& v) {
    x = (x ^ (uint64_t)v.size()) * 0x9E3779B97F4A7C15ull;
    for (size_t i = 0; i + 1 < v.size(); i += 2) {
      const uint64_t w = (uint64_t)(uint32_t)v[i] | ((uint64_t)(uint32_t)v[i + 1] << 32);
      x = (x ^ w) * 0x9E3779B97F4A7C15ull;
      x ^= x >> 29;
    }
    if (v.size() & 1) x = (x ^ (uint64_t)(uint32_t)v.back()) * 1099511628211ull;
  };
  mix(xadj);
  mix(adj);
  return x;
}

LocalResult analyze_sub(const SubIn& in, int k, int ordering, int leaf, OrderCache* cache = nullptr) {
  LocalResult R;
  SubPlan& sp = R.sp;
  const int n = in.n;
  auto fail = [&](ietidp_status st, const std::string& m) {
    R.st = st;
    R.err = "subdomain " + std::to_string(k) + ": " + m;
    return R;
  };
  // ---- classification (tree / primal / remaining; r_I = supp B) ----
  std::vector<int8_t> cls(n, 0);
  for (int t : in.tree) {
    if (cls[t]) return fail(IETIDP_E_ARG, "tree DOF listed twice");
    cls[t] = 1;
  }
  for (int t : in.prim) {
    if (cls[t]) return fail(IETIDP_E_ARG, "primal DOF overlaps the tree or repeats");
    cls[t] = 2;
  }
  std::vector<char> isB(n, 0);
  for (int d : in.B_dof) {
    if (cls[d]) return fail(IETIDP_E_B_STRUCTURE, "B touches a tree or primal DOF");
    if (isB[d]) return fail(IETIDP_E_B_STRUCTURE, "a DOF carries two multipliers");
    isB[d] = 1;
  }
  std::vector<int> rV, rI, vidx(n, -1);
  for (int i = 0; i < n; ++i) {
    if (cls[i]) continue;
    if (isB[i]) rI.push_back(i);
    else {
      vidx[i] = (int)rV.size();
      rV.push_back(i);
    }
  }
  sp.nV = (int)rV.size();
  sp.nI = (int)rI.size();
  sp.nr = sp.nV + sp.nI;
  sp.nP = (int)in.prim.size();
  const int ne = sp.nr + sp.nP;

  // ---- graph of K_VV ----
  std::vector<int> xadj(sp.nV + 1, 0), adj;
  for (int a = 0; a < sp.nV; ++a) {
    int i = rV[a];
    for (int64_t e = in.rowptr[i]; e < in.rowptr[i + 1]; ++e) {
      int j = in.col[e];
      if (j != i && vidx[j] >= 0) adj.push_back(vidx[j]);
    }
    xadj[a + 1] = (int)adj.size();
  }

  const auto ta0 = std::chrono::steady_clock::now();
  // ---- ordering of r_V: supernode tree in postorder ----
  std::vector<std::vector<int>> sn_vars;
  auto compute_order = [&](std::vector<std::vector<int>>& sn_vars) {
  if (sp.nV > 0) {
    std::vector<int> all(sp.nV);
    std::iota(all.begin(), all.end(), 0);
    if (ordering == IETIDP_ORDER_DENSE) {
      sn_vars.push_back(all);
    } else if (ordering == IETIDP_ORDER_MIN_DEGREE) {
      sn_vars = md_supernodes(xadj, adj, sp.nV, min_degree_order(xadj, adj, sp.nV));
    } else {
      NestedDissection nd(xadj, adj, sp.nV, std::max(leaf, 8));
      for (int a = 0; a < sp.nV; ++a) nd.reg[a] = -1;
      auto comps = nd.components(all, -1);
      std::vector<int> roots;
      for (auto& c : comps) roots.push_back(nd.build(c.first, c.second));
      std::vector<std::pair<int, size_t>> st;
      for (int r : roots) {
        st.push_back({r, 0});
        while (!st.empty()) {
          auto& top = st.back();
          auto& node = nd.nodes[top.first];
          if (top.second < node.children.size()) {
            int c = node.children[top.second++];
            st.push_back({c, 0});
          } else {
            sn_vars.push_back(node.vars);
            st.pop_back();
          }
        }
      }
    }
  }
  };
  if (cache && sp.nV > 0) {
    const uint64_t fp = graph_fingerprint(xadj, adj) ^ ((uint64_t)ordering << 56) ^ ((uint64_t)leaf << 40);
    std::shared_ptr<OrderCache::Entry> ent;
    {
      std::lock_guard<std::mutex> lk(cache->mu);
      auto& slot = cache->map[fp];
      if (!slot) slot = std::make_shared<OrderCache::Entry>();
      ent = slot;
    }
    std::call_once(ent->once, [&]() {
      ent->xadj = xadj;
      ent->adj = adj;
      compute_order(ent->sn_vars);
    });
    if (ent->xadj == xadj && ent->adj == adj) sn_vars = ent->sn_vars;
    else compute_order(sn_vars);  // fingerprint collision: not shared
  } else {
    compute_order(sn_vars);
  }
  // ---- positions: r_V (ND), r_I, P ----
  sp.perm.resize(ne);
  sp.pos.assign(n, -1);
  std::vector<int> owner(ne, -1);
  int p = 0;
  auto add_sn = [&](const std::vector<int>& dofs, int coarse) {
    SnHost h;
    h.sub = k;
    h.c0 = p;
    h.npiv = (int)dofs.size();
    h.parent = -1;
    h.level = 0;
    h.coarse = coarse;
    for (int dof : dofs) {
      sp.perm[p] = dof;
      sp.pos[dof] = p;
      owner[p] = (int)R.sn.size();
      ++p;
    }
    R.sn.push_back(std::move(h));
    return (int)R.sn.size() - 1;
  };
  for (auto& vars : sn_vars) {
    std::vector<int> dofs;
    dofs.reserve(vars.size());
    for (int v : vars) dofs.push_back(rV[v]);
    add_sn(dofs, 0);
  }
  if (sp.nI > 0) sp.root = add_sn(rI, 0);
  if (sp.nP > 0) sp.pnode = add_sn(std::vector<int>(in.prim.begin(), in.prim.end()), 1);

  const auto ta1 = std::chrono::steady_clock::now();
  // ---- symbolic factorisation: row structure of every supernode ----
  std::vector<int> mark(ne, -1);
  for (size_t s = 0; s < R.sn.size(); ++s) {
    SnHost& h = R.sn[s];
    int last = h.c0 + h.npiv - 1;
    std::vector<int> rows;
    for (int q = h.c0; q <= last; ++q) {
      int dof = sp.perm[q];
      for (int64_t e = in.rowptr[dof]; e < in.rowptr[dof + 1]; ++e) {
        int pj = sp.pos[in.col[e]];
        if (pj > last && mark[pj] != (int)s) {
          mark[pj] = (int)s;
          rows.push_back(pj);
        }
      }
    }
    for (int c : h.children)
      for (int x : R.sn[c].rows)
        if (x > last && mark[x] != (int)s) {
          mark[x] = (int)s;
          rows.push_back(x);
        }
    std::sort(rows.begin(), rows.end());
    h.rows = std::move(rows);
    h.f = h.npiv + (int)h.rows.size();
    if (!h.rows.empty()) {
      h.parent = owner[h.rows[0]];
      R.sn[h.parent].children.push_back((int)s);
    }
    int lv = 0;
    for (int c : h.children) lv = std::max(lv, R.sn[c].level + 1);
    h.level = lv;
  }
  if (getenv("IETIDP_ANALYZE_PROF")) {
    const auto ta2 = std::chrono::steady_clock::now();
    fprintf(stderr, "analyze_sub %d: n %d nV %d nI %d nnz %lld: ordering %.2f ms, symbolic %.2f ms\n", k, n, sp.nV,
            sp.nI, (long long)in.rowptr[n], std::chrono::duration<double, std::milli>(ta1 - ta0).count(),
            std::chrono::duration<double, std::milli>(ta2 - ta1).count());
  }
  return R;
}

int find_in_front(const SnHost& s, int x) {
  if (x >= s.c0 && x < s.c0 + s.npiv) return x - s.c0;
  auto it = std::lower_bound(s.rows.begin(), s.rows.end(), x);
  if (it == s.rows.end() || *it != x) return -1;
  return s.npiv + (int)(it - s.rows.begin());
}

template <class F>
void parallel_for(int n, F&& fn) {
  int nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  std::atomic<int> next{0};
  for (int t = 0; t < nth; ++t)
    th.emplace_back([&]() {
      for (int k; (k = next++) < n;) fn(k);
    });
  for (auto& x : th) x.join();
}

}  // namespace

static void fill_report(ietidp_s* h) {
  const Plan& P = h->plan;
  h->rep.n_supernodes = (int)P.sn.size();
  h->rep.n_levels = P.max_level + 1;
  h->rep.max_front = P.max_front;
  h->rep.max_nI = P.max_nI;
  long long snr = 0, snI = 0, tri = 0, sIP = 0;
  for (int k = 0; k < h->n_sub; ++k) {
    const SubPlan& sp = P.subs[k];
    snr += sp.nr;
    snI += sp.nI;
    tri += (long long)sp.nI * (sp.nI + 1) / 2;
    sIP += (long long)sp.nI * sp.nP;
  }
  h->rep.sum_nr = snr;
  h->rep.sum_nI = snI;
  h->rep.nnz_L = P.nnz_L;
  h->rep.factor_flops = P.flops;
  // algorithmic bytes: one F-apply reads the lower
  // triangle of every L_II^-1 twice (forward, backward) and L_PI twice; the
  // preconditioner reads the lower triangle of every L_II twice (L^T, L).
  if (h->opt.loop == IETIDP_LOOP_EXPLICIT) {
    // explicit: one pass over the lower triangle of W_k = S_II^-1 and G_k
    // twice per F-apply, one pass over S_II per preconditioner application
    h->rep.f_apply_bytes = 8 * tri + 2 * 8 * sIP;
    h->rep.pcg_bytes_per_iter = 2 * 8 * tri + 2 * 8 * sIP;
  } else {
    h->rep.f_apply_bytes = 2 * 8 * tri + 2 * 8 * sIP;
    h->rep.pcg_bytes_per_iter = 4 * 8 * tri + 2 * 8 * sIP;
  }
}

// Build the complete plan and upload every structure and the raw values.
void analyze_all(ietidp_s* h) {
  auto t0 = std::chrono::steady_clock::now();
  // IETIDP_ANALYZE_PROF=1: host time of every stage of the analysis (stderr)
  const bool aprof = getenv("IETIDP_ANALYZE_PROF") != nullptr;
  auto tl = t0;
  auto stage = [&](const char* name) {
    if (!aprof) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "analyze %-22s %8.2f ms\n", name, std::chrono::duration<double, std::milli>(t - tl).count());
    tl = t;
  };
  const int ns = h->n_sub, nrhs = h->nrhs;
  for (int k = 0; k < ns; ++k)
    if (!h->in[k].set) throw Error(IETIDP_E_STATE, "subdomain " + std::to_string(k) + " not set");

  // ---- global B validation (R6) ----
  std::vector<int> cnt(h->n_lambda, 0), ssum(h->n_lambda, 0), firstsub(h->n_lambda, -1);
  for (int k = 0; k < ns; ++k) {
    const SubIn& in = h->in[k];
    for (size_t e = 0; e < in.B_lambda.size(); ++e) {
      int l = in.B_lambda[e];
      if (cnt[l] >= 1 && firstsub[l] == k)
        throw Error(IETIDP_E_B_STRUCTURE,
                    "multiplier " + std::to_string(l) + " twice in subdomain " + std::to_string(k));
      cnt[l]++;
      ssum[l] += in.B_sign[e];
      firstsub[l] = k;
    }
  }
  // sharded mode (ietidp_shard.h): a row may have one side, or none, on this rank
  for (int l = 0; l < h->n_lambda; ++l)
    if (h->shard ? (cnt[l] > 2 || (cnt[l] == 2 && ssum[l] != 0)) : (cnt[l] != 2 || ssum[l] != 0))
      throw Error(IETIDP_E_B_STRUCTURE,
                  "multiplier row " + std::to_string(l) + " is not {+1,-1} in two subdomains");

  stage("B validation");
  // ---- pattern classes: subdomains whose K pattern, tree, primal DOFs and r_I set
  // (supp B) coincide have identical symbolic analyses (the box tilings repeat a few
  // face/edge/corner patterns: C5 has 27 classes of 128) ----
  std::vector<int> rep(ns);
  {
    // fingerprints from ietidp_set_subdomain; members of a fingerprint group are compared
    // with the group's first subdomain in full (in parallel); a mismatch (a fingerprint
    // collision) makes the subdomain its own class
    std::unordered_map<uint64_t, int> first;
    std::vector<int> cand(ns);
    for (int k = 0; k < ns; ++k) cand[k] = first.emplace(h->in[k].fp, k).first->second;
    parallel_for(ns, [&](int k) {
      const int r = cand[k];
      const SubIn &a = h->in[k], &b = h->in[r];
      rep[k] = (r == k || (a.n == b.n && a.rowptr == b.rowptr && a.col == b.col && a.tree == b.tree &&
                           a.prim == b.prim && a.B_dof_sorted == b.B_dof_sorted))
                   ? r
                   : k;
    });
  }
  std::vector<int> reps;
  for (int k = 0; k < ns; ++k)
    if (rep[k] == k) reps.push_back(k);
  h->n_pattern_classes = (int)reps.size();
  h->class_rep = rep;
  stage("pattern classes");

  // ---- per-subdomain analysis (one per pattern class), in parallel ----
  std::vector<LocalResult> loc(ns);
  OrderCache ocache;
  parallel_for((int)reps.size(), [&](int i) {
    const int k = reps[i];
    loc[k] = analyze_sub(h->in[k], k, h->opt.ordering, h->opt.leaf_size, &ocache);
  });
  for (int k : reps)
    if (loc[k].st != IETIDP_OK) throw Error(loc[k].st, loc[k].err);
  parallel_for(ns, [&](int k) {
    if (rep[k] == k) return;
    loc[k] = loc[rep[k]];
    for (auto& x : loc[k].sn) x.sub = k;
  });

  stage("per-subdomain analysis");
  Plan& P = h->plan;
  P = Plan();
  P.subs.resize(ns);
  h->h_sub.assign(ns, SubDev{});
  // ---- global supernode numbering ----
  std::vector<int> sn_base(ns + 1, 0);
  for (int k = 0; k < ns; ++k) sn_base[k + 1] = sn_base[k] + (int)loc[k].sn.size();
  P.sn.reserve(sn_base[ns]);
  for (int k = 0; k < ns; ++k) {
    P.subs[k] = std::move(loc[k].sp);
    for (auto& s : loc[k].sn) {
      SnHost g = std::move(s);
      if (g.parent >= 0) g.parent += sn_base[k];
      for (int& c : g.children) c += sn_base[k];
      P.sn.push_back(std::move(g));
    }
    P.subs[k].sn_begin = {sn_base[k], sn_base[k + 1]};
    if (P.subs[k].root >= 0) P.subs[k].root += sn_base[k];
    if (P.subs[k].pnode >= 0) P.subs[k].pnode += sn_base[k];
  }
  const int nsn = (int)P.sn.size();
  for (auto& s : P.sn) P.max_level = std::max(P.max_level, s.level);
  std::vector<std::vector<int>> bylev(P.max_level + 1);
  for (int i = 0; i < nsn; ++i) bylev[P.sn[i].level].push_back(i);
  for (auto& v : bylev)
    std::stable_sort(v.begin(), v.end(), [&](int a, int b) { return P.sn[a].npiv > P.sn[b].npiv; });
  // subdomain groups (subdomain k in group k % G): each group's factorisation runs as an
  // independent chain of launches on its own stream, so that one group's latency-bound
  // panels overlap the other's GEMMs
  int G = ns >= 8 ? 8 : (ns >= 4 ? 2 : 1);  // measured: C2 7.87 ms with 8 groups vs 8.32 with 1
  if (const char* e = getenv("IETIDP_GROUPS")) G = std::max(1, std::min(ns, atoi(e)));
  P.ngroups = G;
  // groups are contiguous blocks of subdomains (so that a group's inputs arrive together)
  P.sub_group.resize(ns);
  for (int k = 0; k < ns; ++k) P.sub_group[k] = (int)((long long)k * G / ns);
  std::vector<std::vector<std::vector<int>>> bylev_g(G, std::vector<std::vector<int>>(P.max_level + 1));
  for (int L = 0; L <= P.max_level; ++L)
    for (int i : bylev[L]) bylev_g[P.sub_group[P.sn[i].sub]][L].push_back(i);
  P.glevels.assign(G, std::vector<LevelPlan>(P.max_level + 1));

  stage("numbering/groups");
  // ---- memory layout of the supernodes ----
  std::vector<SnDev> sd(nsn);
  std::vector<int> rows_all, rel_all, children_all, work;
  std::vector<GemmWork> gwork;
  long long pool = 0, dinv = 0, inv = 0, vec = 0;
  P.levels.resize(P.max_level + 1);
  for (int L = 0; L <= P.max_level; ++L) {
    LevelPlan& lp = P.levels[L];
    lp.sn_off = (int)P.level_sn.size();
    lp.sn_n = (int)bylev[L].size();
    for (int i : bylev[L]) {
      SnHost& s = P.sn[i];
      SnDev& d = sd[i];
      d.f = s.f;
      d.ld = (s.f + 3) & ~3;
      d.npiv = s.npiv;
      d.c0 = s.c0;
      d.sub = s.sub;
      d.parent = s.parent;
      d.coarse = s.coarse;
      d.front_off = pool;
      pool += (long long)d.ld * d.f;
      d.vec_off = vec;
      vec += s.f;
      d.bp_off = P.bpart_doubles;  // step-1 chunks, then step-2 chunks of the backward sweep
      if (!s.coarse)
        P.bpart_doubles += (long long)((s.f - s.npiv + BS_RB - 1) / BS_RB + (s.npiv + BS_RB - 1) / BS_RB) *
                           s.npiv * 16;
      d.ldi = (s.npiv + 3) & ~3;
      if (!s.coarse) {
        d.dinv_off = dinv;
        dinv += (long long)((s.npiv + TB - 1) / TB) * TILE_ELEMS;
        d.inv_off = inv;
        inv += (long long)d.ldi * s.npiv;
        for (int j = 0; j < s.npiv; ++j) {
          long long c = s.f - j;
          P.nnz_L += c;
          P.flops += c * c;
        }
        P.inv_flops += (long long)s.npiv * s.npiv * s.npiv / 3;
      }
      P.level_sn.push_back(i);
      P.max_front = std::max(P.max_front, s.f);
    }
  }
  for (int g = 0; g < G; ++g)
    for (int L = 0; L <= P.max_level; ++L) {
      P.glevels[g][L].sn_off = (int)P.level_sn.size();
      P.glevels[g][L].sn_n = (int)bylev_g[g][L].size();
      P.level_sn.insert(P.level_sn.end(), bylev_g[g][L].begin(), bylev_g[g][L].end());
    }
  P.pool_doubles = pool;
  P.dinv_doubles = dinv;
  P.inv_doubles = inv;
  P.vec_rows = vec;
  stage(" layout: fronts");
  // relative positions of every supernode's update rows in its parent's front, once
  // per pattern class (the members' supernodes are the representative's, shifted)
  std::vector<std::vector<int>> relv(nsn);
  std::vector<int> relfail(ns, 0);
  parallel_for((int)reps.size(), [&](int ri) {
    const int k = reps[ri];
    for (int i = P.subs[k].sn_begin[0]; i < P.subs[k].sn_begin[1]; ++i) {
      const SnHost& sx = P.sn[i];
      if (sx.parent < 0) continue;
      const SnHost& par = P.sn[sx.parent];
      relv[i].reserve(sx.rows.size());
      size_t q = 0;  // both row lists are sorted: one merge
      for (int x : sx.rows) {
        int r;
        if (x >= par.c0 && x < par.c0 + par.npiv) {
          r = x - par.c0;
        } else {
          while (q < par.rows.size() && par.rows[q] < x) ++q;
          r = (q < par.rows.size() && par.rows[q] == x) ? par.npiv + (int)q : -1;
        }
        if (r < 0) relfail[k] = 1;
        relv[i].push_back(r);
      }
    }
  });
  for (int k : reps)
    if (relfail[k]) throw Error(IETIDP_E_ARG, "internal: symbolic structure not nested");
  parallel_for(ns, [&](int k) {
    if (rep[k] == k) return;
    const int d0 = P.subs[rep[k]].sn_begin[0] - P.subs[k].sn_begin[0];
    for (int i = P.subs[k].sn_begin[0]; i < P.subs[k].sn_begin[1]; ++i) relv[i] = relv[i + d0];
  });
  stage(" layout: relative rows");
  {  // offsets first, then the copies in parallel (per subdomain)
    long long nr = 0, nc = 0;
    for (int i = 0; i < nsn; ++i) {
      SnDev& d = sd[i];
      d.rows_off = d.rel_off = (int)nr;
      nr += (long long)P.sn[i].rows.size();
      d.child_off = (int)nc;
      d.nchild = (int)P.sn[i].children.size();
      nc += d.nchild;
    }
    rows_all.resize(nr);
    rel_all.resize(nr);
    children_all.resize(nc);
    parallel_for(ns, [&](int k) {
      for (int i = P.subs[k].sn_begin[0]; i < P.subs[k].sn_begin[1]; ++i) {
        const SnHost& s = P.sn[i];
        const SnDev& d = sd[i];
        std::copy(s.rows.begin(), s.rows.end(), rows_all.begin() + d.rows_off);
        std::copy(relv[i].begin(), relv[i].end(), rel_all.begin() + d.rel_off);
        std::copy(s.children.begin(), s.children.end(), children_all.begin() + d.child_off);
      }
    });
  }
  stage(" layout: concatenation");

  auto push = [&](int a, int b, int c) { work.insert(work.end(), {a, b, c}); };
  // L11^-1 of the levels holding r_I roots is formed block row by block row as their
  // panels complete (it sits on the path to the loop); the other levels use recursive
  // doubling once the level is factored
  std::vector<char> prog_level(P.max_level + 1, 0);
  for (auto& sp : P.subs)
    if (sp.root >= 0) prog_level[P.sn[sp.root].level] = 1;
  auto tiles_of = [](int n) { return (n + TB - 1) / TB; };
  std::vector<std::pair<int, int>> split_group;  // split-K GemmWork entries and their group
  stage("memory layout");
  // ---- work lists: factorisation and sweeps, per level ----
  {  // capacity bounds (one allocation each; untouched capacity costs no page faults)
    long long gb = 0, wb = 0;
    for (const SnHost& x : P.sn) {
      const long long np = tiles_of(x.npiv), ft = tiles_of(x.f), ut = tiles_of(x.f - x.npiv);
      gb += np * ft * (SPLITK_MAX + 1) + 2 * np * np + ut * (ut + 1) / 2;
      wb += 6 * (np + ft + ut) + 2 * np * (x.f / BS_RB + 2);
    }
    gwork.reserve((size_t)gb);
    work.reserve((size_t)(3 * wb));
  }
  for (int L = 0; L <= P.max_level; ++L) {
    for (int grp = 0; grp < G; ++grp) {
      LevelPlan& lp = P.glevels[grp][L];
      const std::vector<int>& nodes = bylev_g[grp][L];
    int maxp = 0;
    for (int i : nodes)
      if (!P.sn[i].coarse) maxp = std::max(maxp, tiles_of(P.sn[i].npiv));
    for (int kp = 0; kp < maxp; ++kp) {
      LevelPlan::Panel pn{};
      // (a) panel columns [p0, p0+b) -= L[rows >= p0, 0:p0] L[p0:p0+b, 0:p0]^T
      pn.upd_off = (int)gwork.size();
      {
        // tiles of this panel update; long K on few tiles is split over CTAs (split-K)
        int ntile = 0;
        long long kmax = 0;
        for (int i : nodes) {
          const SnHost& s = P.sn[i];
          if (s.coarse || s.npiv <= kp * TB || kp == 0) continue;
          ntile += tiles_of(s.f - kp * TB);
          kmax = std::max<long long>(kmax, (long long)kp * TB);
        }
        int nks = 1;
        if (ntile > 0) {
          const int want = SPLITK_TARGET_CTAS / ntile;  // parts that still fit in one wave
          nks = std::max(1, std::min({SPLITK_MAX, want, (int)(kmax / SPLITK_MIN_K)}));
        }
        int tile = 0;
        long long ws = 0;
        for (int i : nodes) {
          const SnHost& s = P.sn[i];
          if (s.coarse || s.npiv <= kp * TB || kp == 0) continue;
          const SnDev& d = sd[i];
          const int p0 = kp * TB, b = std::min(TB, s.npiv - p0);
          // K range [0, p0) in nks chunks of a multiple of 32 columns
          const int chunk = ((p0 + nks - 1) / nks + 31) / 32 * 32;
          const int parts = (p0 + chunk - 1) / chunk;
          for (int r0 = p0; r0 < s.f; r0 += TB, ++tile) {
            for (int q = 0; q < parts; ++q, ++pn.upd_n) {
              const int k0 = q * chunk;
              GemmWork g{};
              g.c_off = d.front_off + (long long)p0 * d.ld + r0;
              g.a_off = d.front_off + (long long)k0 * d.ld + r0;
              g.b_off = d.front_off + (long long)k0 * d.ld + p0;  // B[k][n] = L[p0 + n][k]
              g.lda = g.ldb = g.ldc = d.ld;
              g.m = std::min(TB, s.f - r0);
              g.n = b;
              g.kdim = std::min(chunk, p0 - k0);
              g.mode = 3;  // C -= A B
              if (parts > 1) {
                split_group.push_back({(int)gwork.size(), grp});
                g.mode |= 8;
                g.ks = q;
                g.nks = parts;
                g.cnt = tile;
                g.ws_off = ws;
              }
              gwork.push_back(g);
            }
            if (parts > 1) ws += (long long)parts * TILE_ELEMS;
          }
        }
        P.splitk_doubles = std::max(P.splitk_doubles, ws);
        P.splitk_tiles = std::max(P.splitk_tiles, tile);
      }
      pn.potrf_off = (int)work.size() / 3;
      for (int i : nodes)
        if (!P.sn[i].coarse && P.sn[i].npiv > kp * TB) {
          push(i, kp, 0);
          pn.potrf_n++;
        }
      // (c) rows below the diagonal block: L = A Dinv^T (in place)
      pn.trsm_off = (int)gwork.size();
      for (int i : nodes) {
        const SnHost& s = P.sn[i];
        if (s.coarse || s.npiv <= kp * TB) continue;
        const SnDev& d = sd[i];
        const int p0 = kp * TB, b = std::min(TB, s.npiv - p0);
        for (int r0 = p0 + b; r0 < s.f; r0 += TB, ++pn.trsm_n) {
          GemmWork g{};
          g.c_off = d.front_off + (long long)p0 * d.ld + r0;
          g.a_off = g.c_off;
          g.b_off = d.dinv_off + (long long)kp * TILE_ELEMS;  // B[n][k] = Dinv[n][k], col-major
          g.lda = g.ldc = d.ld;
          g.ldb = TB;
          g.m = std::min(TB, s.f - r0);
          g.n = b;
          g.kdim = b;
          g.mode = 0;  // C = A B
          gwork.push_back(g);
        }
      }
      // (e) progressive inverse of block row kp of L11^-1 (side stream)
      pn.icopy_off = (int)work.size() / 3;
      for (int i : nodes)
        if (prog_level[L] && !P.sn[i].coarse && P.sn[i].npiv > kp * TB) {
          push(i, kp, 0);
          pn.icopy_n++;
        }
      pn.ia_off = (int)gwork.size();
      for (int i : nodes) {
        const SnHost& s = P.sn[i];
        if (!prog_level[L] || s.coarse || s.npiv <= kp * TB || kp == 0) continue;
        const SnDev& d = sd[i];
        const int p0 = kp * TB, b = std::min(TB, s.npiv - p0);
        for (int k = 0; k < kp; ++k, ++pn.ia_n) {
          // T[kp][k] = L[kp][k:kp] L11^-1[k:kp][k]  (into tpool at L11^-1[kp][k])
          GemmWork g{};
          g.c_off = d.inv_off + (long long)k * TB * d.ldi + p0;
          g.a_off = d.front_off + (long long)k * TB * d.ld + p0;  // A[r][m] = L[p0 + r][kTB + m]
          g.b_off = d.inv_off + (long long)k * TB * d.ldi + k * TB;  // B[m][n] = Linv[kTB + m][kTB + n]
          g.lda = d.ld;
          g.ldb = d.ldi;
          g.ldc = d.ldi;
          g.m = b;
          g.n = TB;
          g.kdim = p0 - k * TB;
          g.mode = 0;
          gwork.push_back(g);
        }
      }
      pn.ib_off = (int)gwork.size();
      for (int i : nodes) {
        const SnHost& s = P.sn[i];
        if (!prog_level[L] || s.coarse || s.npiv <= kp * TB || kp == 0) continue;
        const SnDev& d = sd[i];
        const int p0 = kp * TB, b = std::min(TB, s.npiv - p0);
        for (int k = 0; k < kp; ++k, ++pn.ib_n) {
          // L11^-1[kp][k] = -Dinv_kp T[kp][k]
          GemmWork g{};
          g.c_off = d.inv_off + (long long)k * TB * d.ldi + p0;
          g.a_off = d.dinv_off + (long long)kp * TILE_ELEMS;  // A = Dinv_kp (column-major TB x TB)
          g.b_off = d.inv_off + (long long)k * TB * d.ldi + p0;  // B[m][n] = T[p0 + m][kTB + n] (tpool)
          g.lda = TB;
          g.ldb = d.ldi;
          g.ldc = d.ldi;
          g.m = b;
          g.n = TB;
          g.kdim = b;
          g.mode = 1;  // negate
          gwork.push_back(g);
        }
      }
      pn.wacc_off = (int)gwork.size();  // filled below, once the loop tile offsets are known
      pn.wacc_n = 0;
      lp.panels.push_back(pn);
    }
    // (d) update block: parent[rel] += F22 - L21 L21^T (lower tiles, K = npiv), fused
    //     extend-add; one launch per child slot so that no two CTAs of a launch add
    //     into the same parent entries (deterministic, no atomics)
    {
      std::vector<int> slot(nsn, 0);
      int maxslot = 0;
      for (int i : nodes) {
        const SnHost& s = P.sn[i];
        if (s.parent < 0) continue;
        const auto& ch = P.sn[s.parent].children;
        slot[i] = (int)(std::find(ch.begin(), ch.end(), i) - ch.begin());
        maxslot = std::max(maxslot, slot[i] + 1);
      }
      for (int q = 0; q < maxslot; ++q) {
        int off = (int)gwork.size();
        for (int i : nodes) {
          const SnHost& s = P.sn[i];
          if (s.coarse || s.f == s.npiv || s.parent < 0 || slot[i] != q) continue;
          const SnDev& d = sd[i];
          const SnDev& pd = sd[s.parent];
          for (int r0 = s.npiv; r0 < s.f; r0 += TB)
            for (int c0 = s.npiv; c0 <= r0; c0 += TB) {
              GemmWork g{};
              g.c_off = d.front_off + (long long)c0 * d.ld + r0;
              g.a_off = d.front_off + r0;
              g.b_off = d.front_off + c0;
              g.lda = g.ldb = g.ldc = d.ld;
              g.m = std::min(TB, s.f - r0);
              g.n = std::min(TB, s.f - c0);
              g.kdim = s.npiv;
              g.mode = 4 | 1;  // extend-add of C - A B
              // no children: the update block F22 received nothing (K entries go to the
              // front owning their first position), so C is zero and not read
              if (s.children.empty()) g.mode |= 32;
              g.diag = (r0 == c0);
              g.p_off = pd.front_off;
              g.p_ld = pd.ld;
              g.rel_r = d.rel_off + (r0 - s.npiv);
              g.rel_c = d.rel_off + (c0 - s.npiv);
              gwork.push_back(g);
            }
        }
        if ((int)gwork.size() > off) lp.syrk.push_back({off, (int)gwork.size() - off});
      }
    }
      // the group's assembly (zero the lower trapezoids; see the global lists below)
      lp.zr_off = (int)work.size() / 3;
      for (int i : nodes) {
        const bool leaf = P.sn[i].children.empty() && !P.sn[i].coarse;
        const int ncol = leaf ? P.sn[i].npiv : P.sn[i].f;
        for (int t = 0; t < tiles_of(ncol); ++t, ++lp.zr_n) push(i, t, leaf ? 1 : 0);
      }
      // the group's forward-sweep lists (the factorisation's side stream)
      lp.fs_off = (int)work.size() / 3;
      for (int i : nodes)
        if (!P.sn[i].coarse)
          for (int t = 0; t < tiles_of(P.sn[i].npiv); ++t, ++lp.fs_n) push(i, t, 0);
      lp.fu_off = (int)work.size() / 3;
      for (int i : nodes)
        if (!P.sn[i].coarse)
          for (int t = 0; t < tiles_of(P.sn[i].f - P.sn[i].npiv); ++t, ++lp.fu_n) push(i, t, 0);
    }
    LevelPlan& lp = P.levels[L];
    // assembly: zero the lower trapezoid of every front of this level (coarse node too)
    lp.zr_off = (int)work.size() / 3;
    for (int i : bylev[L]) {
      // a childless front's update block is never read (its SYRK treats it as zero):
      // zero only its pivot columns
      const bool leaf = P.sn[i].children.empty() && !P.sn[i].coarse;
      const int ncol = leaf ? P.sn[i].npiv : P.sn[i].f;
      for (int t = 0; t < tiles_of(ncol); ++t, ++lp.zr_n) push(i, t, leaf ? 1 : 0);
    }
    // sweeps
    lp.fs_off = (int)work.size() / 3;
    for (int i : bylev[L])
      if (!P.sn[i].coarse)
        for (int t = 0; t < tiles_of(P.sn[i].npiv); ++t, ++lp.fs_n) push(i, t, 0);
    lp.fu_off = (int)work.size() / 3;
    for (int i : bylev[L])
      if (!P.sn[i].coarse)
        for (int t = 0; t < tiles_of(P.sn[i].f - P.sn[i].npiv); ++t, ++lp.fu_n) push(i, t, 0);
    lp.bt_off = (int)work.size() / 3;
    for (int i : bylev[L])
      if (!P.sn[i].coarse && P.sn[i].f > P.sn[i].npiv) {
        const int nch = (P.sn[i].f - P.sn[i].npiv + BS_RB - 1) / BS_RB;
        for (int t = 0; t < tiles_of(P.sn[i].npiv); ++t)
          for (int rc = 0; rc < nch; ++rc, ++lp.bt_n) push(i, t, rc);
      }
    lp.bx_off = (int)work.size() / 3;  // (sn, pivot col tile, row chunk >= the tile's)
    for (int i : bylev[L])
      if (!P.sn[i].coarse) {
        const int nch = (P.sn[i].npiv + BS_RB - 1) / BS_RB;
        for (int t = 0; t < tiles_of(P.sn[i].npiv); ++t)
          for (int rc = t * TB / BS_RB; rc < nch; ++rc, ++lp.bx_n) push(i, t, rc);
      }
    lp.bxr_off = (int)work.size() / 3;
    for (int i : bylev[L])
      if (!P.sn[i].coarse)
        for (int t = 0; t < tiles_of(P.sn[i].npiv); ++t, ++lp.bxr_n) push(i, t, 0);
  }
  stage("work lists");
  if (aprof) fprintf(stderr, "analyze: %d supernodes, %zu GemmWork, %zu Work, %zu rows\n", nsn, gwork.size(), work.size() / 3, rows_all.size());
  // ---- partitioned inverse L11^-1 by recursive doubling over TB-blocks, per level ----
  // each group's split-K launches use their own slice of the workspace and counters
  for (auto& sg : split_group) {
    gwork[sg.first].ws_off += (long long)sg.second * P.splitk_doubles;
    gwork[sg.first].cnt += sg.second * P.splitk_tiles;
  }
  for (int grp = 0; grp < G; ++grp)
  for (int L = 0; L <= P.max_level; ++L) {
    LevelPlan& lp = P.glevels[grp][L];
    const std::vector<int>& nodes = bylev_g[grp][L];
    if (prog_level[L]) continue;  // progressive, per panel (above)
    lp.inv_copy_off = (int)work.size() / 3;
    int maxnb = 0;
    for (int i : nodes)
      if (!P.sn[i].coarse) {
        for (int kp = 0; kp < tiles_of(P.sn[i].npiv); ++kp, ++lp.inv_copy_n) push(i, kp, 0);
        maxnb = std::max(maxnb, tiles_of(P.sn[i].npiv));
      }
    for (int half = 1; half < maxnb; half *= 2) {
      // step 1: T(second, first) = L11(second, first-half) * Linv(first, first)
      int off1 = (int)gwork.size();
      for (int i : nodes) {
        const SnHost& s = P.sn[i];
        if (s.coarse) continue;
        const SnDev& d = sd[i];
        const int nb = tiles_of(s.npiv);
        for (int fs = 0; fs < nb; fs += 2 * half) {
          int ss = fs + half, se = std::min(fs + 2 * half, nb);
          if (ss >= nb) continue;
          for (int ti = ss; ti < se; ++ti)
            for (int tj = fs; tj < ss; ++tj) {
              GemmWork g{};
              int k0 = tj * TB, k1 = std::min(ss * TB, s.npiv);
              g.c_off = d.inv_off + (long long)tj * TB * d.ldi + ti * TB;  // T stored in tpool, same layout
              g.a_off = d.front_off + (long long)k0 * d.ld + ti * TB;
              g.b_off = d.inv_off + (long long)tj * TB * d.ldi + k0;
              g.lda = d.ld;
              g.ldb = d.ldi;
              g.ldc = d.ldi;
              g.m = std::min(TB, s.npiv - ti * TB);
              g.n = std::min(TB, s.npiv - tj * TB);
              g.kdim = k1 - k0;
              g.mode = 0;
              gwork.push_back(g);
            }
        }
      }
      lp.inv_rounds.push_back({off1, (int)gwork.size() - off1});
      // step 2: Linv(second, first) = -Linv(second, second) * T(second, first)
      int off2 = (int)gwork.size();
      for (int i : nodes) {
        const SnHost& s = P.sn[i];
        if (s.coarse) continue;
        const SnDev& d = sd[i];
        const int nb = tiles_of(s.npiv);
        for (int fs = 0; fs < nb; fs += 2 * half) {
          int ss = fs + half, se = std::min(fs + 2 * half, nb);
          if (ss >= nb) continue;
          for (int ti = ss; ti < se; ++ti)
            for (int tj = fs; tj < ss; ++tj) {
              GemmWork g{};
              int k0 = ss * TB, k1 = std::min((ti + 1) * TB, s.npiv);
              g.c_off = d.inv_off + (long long)tj * TB * d.ldi + ti * TB;
              g.a_off = d.inv_off + (long long)k0 * d.ldi + ti * TB;
              g.b_off = d.inv_off + (long long)tj * TB * d.ldi + k0;  // T in tpool
              g.lda = d.ldi;
              g.ldb = d.ldi;
              g.ldc = d.ldi;
              g.m = std::min(TB, s.npiv - ti * TB);
              g.n = std::min(TB, s.npiv - tj * TB);
              g.kdim = k1 - k0;
              g.mode = 1;  // negate
              gwork.push_back(g);
            }
        }
      }
      lp.inv_rounds.push_back({off2, (int)gwork.size() - off2});
    }
  }

  stage("inverse plan");
  // ---- per-subdomain offsets ----
  long long kv = 0, fv = 0, xo = 0, rio = 0, lpio = 0, to = 0, uo = 0, spo = 0;
  int po = 0, permo = 0, cta = 0;
  P.nPmax = 0;
  h->kval_off.resize(ns);
  h->fval_off.resize(ns);
  h->u_off.resize(ns);
  std::vector<LoopWork> loopwork;
  std::vector<SymWork> symwork;
  std::vector<int> sub_cta0(ns), sub_ncta(ns), sub_blk0(ns), sub_nt(ns);
  int maxnt_all = 0;
  for (int k = 0; k < ns; ++k) maxnt_all = std::max(maxnt_all, tiles_of(P.subs[k].nI));
  const int maxseg = std::max(1, (maxnt_all + SYM_SEG - 1) / SYM_SEG);
  long long npo = 0;
  int blk = 0;
  for (int k = 0; k < ns; ++k) {
    SubPlan& sp = P.subs[k];
    SubDev& d = h->h_sub[k];
    const SubIn& in = h->in[k];
    P.nPmax = std::max(P.nPmax, sp.nP);
    d.nk = in.n;
    d.nr = sp.nr;
    d.nI = sp.nI;
    d.nV = sp.nV;
    d.nP = sp.nP;
    d.ne = sp.nr + sp.nP;
    d.root = sp.root;
    d.pnode = sp.pnode;
    d.x_off = xo;
    xo += d.ne;
    d.rI_off = rio;
    rio += sp.nI;
    d.kval_off = kv;
    h->kval_off[k] = kv;
    kv += (long long)in.val.size();
    d.f_off = fv;
    h->fval_off[k] = fv;
    fv += (long long)in.n * nrhs;
    d.lpi_off = lpio;
    d.g_off = lpio;  // G_k has the same size as L_PI (nI x nP)
    lpio += (long long)sp.nP * sp.nI;
    d.nt = tiles_of(sp.nI);
    d.spart_off = spo;
    spo += (long long)d.nt * (d.nt - 1) / 2;
    d.tile_off = to;
    d.itile_off = to;  // same offsets in the two tile arrays
    to += (long long)d.nt * (d.nt + 1) / 2 * TILE_ELEMS;
    d.prim_off = po;
    po += sp.nP;
    d.perm_off = permo;
    permo += d.ne;
    h->u_off[k] = uo;
    uo += (long long)in.n * nrhs;
    P.max_nI = std::max(P.max_nI, sp.nI);
    // loop CTAs: block pairs (i, nt-1-i)
    d.cta0 = cta;
    sub_cta0[k] = cta;
    for (int i = 0; i < (d.nt + 1) / 2; ++i) {
      int j = d.nt - 1 - i;
      loopwork.push_back({k, i == j ? 1 : 2, i, j, i == j ? i + 1 : d.nt + 1});
      ++cta;
    }
    sub_ncta[k] = cta - d.cta0;
    // symmetric-pass items (explicit loop): segments of SYM_SEG tiles of each block row
    d.blk0 = blk;
    sub_blk0[k] = blk;
    sub_nt[k] = d.nt;
    blk += d.nt;
    d.npart_off = npo;
    npo += (long long)d.nt * maxseg;
    for (int o = 0; o < d.nt; ++o)
      for (int seg = 0; seg * SYM_SEG <= o; ++seg) {
        const int j0 = seg * SYM_SEG, j1 = std::min(o, j0 + SYM_SEG - 1);
        symwork.push_back({k, o, j0, j1, seg, j1 - j0 + 2});
      }
  }
  h->sym_maxseg = maxseg;
  if (P.max_nI > 32 * TB) throw Error(IETIDP_E_ARG, "interface block larger than 2048 DOFs is not supported");
  // the loop kernels' coarse partials: two (primal, column) outputs per thread of 256,
  // the G_k rows of one block (TB x nP) staged in shared memory
  if (P.nPmax > 32) throw Error(IETIDP_E_ARG, "more than 32 primal DOFs in one subdomain is not supported");
  h->n_slots = (int)rio;
  h->sum_nP = po;
  h->n_loopwork = (int)loopwork.size();
  h->n_symwork = (int)symwork.size();
  // the r_I roots by level (S_II is copied before the root is factored)
  P.roots_by_level.assign(P.max_level + 1, {});
  for (int k = 0; k < ns; ++k)
    if (h->h_sub[k].root >= 0) P.roots_by_level[P.sn[h->h_sub[k].root].level].push_back(k);
  // W_k = L_II^-T L_II^-1 accumulated from groups of W_GROUP block rows of L_II^-1 as
  // the r_I root's panels complete: after the group [k0, kp], W[i][j] += sum over
  // the group's rows k >= i of L11^-1[k][i]^T L11^-1[k][j], j <= i <= kp, written into
  // the loop's row-major lower tiles (zeroed before the factorisation). Groups keep
  // the read-modify-write traffic of the tiles W_GROUP times below per-row updates.
  constexpr int W_GROUP = 4;
  for (int grp = 0; grp < G; ++grp)
  for (int L = 0; L <= P.max_level; ++L)
    for (int kp = 0; kp < (int)P.glevels[grp][L].panels.size(); ++kp) {
      LevelPlan::Panel& pn = P.glevels[grp][L].panels[kp];
      pn.wacc_off = (int)gwork.size();
      if (h->opt.loop != IETIDP_LOOP_EXPLICIT) continue;
      for (int k : P.roots_by_level[L]) {
        if (P.sub_group[k] != grp) continue;
        const SubDev& d = h->h_sub[k];
        if (kp >= d.nt) continue;
        if ((kp + 1) % W_GROUP != 0 && kp != d.nt - 1) continue;  // not the end of a group
        const int k0 = kp / W_GROUP * W_GROUP;
        const SnDev& r = sd[d.root];
        for (int i = 0; i <= kp; ++i)
          for (int j = 0; j <= i; ++j, ++pn.wacc_n) {
            const int ks = std::max(i, k0);  // L11^-1[k][i] = 0 for k < i
            GemmWork g{};
            g.c_off = d.tile_off + (long long)(i * (i + 1) / 2 + j) * TILE_ELEMS;
            g.a_off = r.inv_off + (long long)(i * TB) * r.ldi + ks * TB;  // A[rr][m] = Linv[ksTB + m][iTB + rr]
            g.b_off = r.inv_off + (long long)(j * TB) * r.ldi + ks * TB;  // B[m][c] = Linv[ksTB + m][jTB + c]
            g.lda = g.ldb = r.ldi;
            g.ldc = TB;
            g.m = std::min(TB, d.nI - i * TB);
            g.n = std::min(TB, d.nI - j * TB);
            g.kdim = std::min(d.nI, (kp + 1) * TB) - ks * TB;
            g.mode = 16 | 2;  // accumulate into the row-major tile
            g.diag = (i == j);
            gwork.push_back(g);
          }
      }
    }
  // G_k^T = L_PI L_II^-1 (n_P x n_I, column-major = G_k row-major), per 64-column tile
  // of a: K = [a0, n_I) since L_II^-1[m][a] = 0 for m < a
  P.g_off = (int)gwork.size();
  for (int k = 0; k < ns; ++k) {
    const SubDev& d = h->h_sub[k];
    if (d.root < 0 || d.nP == 0 || d.nI == 0) continue;
    const SnDev& r = sd[d.root];
    for (int i = 0; i < d.nt; ++i) {
      GemmWork g{};
      const int a0 = i * TB;
      g.c_off = d.g_off + (long long)a0 * d.nP;
      g.a_off = d.lpi_off + a0;                          // A[q][k] = L_PI[q][a0 + k]
      g.b_off = r.inv_off + (long long)a0 * r.ldi + a0;  // B[k][n] = Linv[a0 + k][a0 + n]
      g.lda = d.nI;
      g.ldb = r.ldi;
      g.ldc = d.nP;
      g.m = d.nP;
      g.n = std::min(TB, d.nI - a0);
      g.kdim = d.nI - a0;
      g.mode = 0;
      gwork.push_back(g);
    }
  }
  P.g_n = (int)gwork.size() - P.g_off;

  stage("offsets/items");
  // ---- scatter lists: relative entries once per pattern class (in parallel), then
  // every subdomain's absolute lists written in parallel into the merged arrays ----
  struct Rel {
    std::vector<std::vector<int>> off, sl, src;  // per level: in-front offset, local supernode, CSR index
    std::vector<int> fxr, fxs;                   // loads: position, local DOF
    std::vector<int> kdiag;                      // r_I diagonal entries: CSR index
    std::vector<int> foff, fsl, fsrc;            // the levels, then the loads, one after another
    std::vector<long long> lev;                  // start of level L (L = NL: the loads) in f*
    std::string err;
  };
  std::vector<Rel> rel(ns);
  parallel_for((int)reps.size(), [&](int ri) {
    const int k = reps[ri];
    Rel& S = rel[k];
    const SubIn& in = h->in[k];
    const SubPlan& sp = P.subs[k];
    const SubDev& d = h->h_sub[k];
    const int ne = d.ne;
    const int sb = sp.sn_begin[0];
    S.off.resize(P.max_level + 1);
    S.sl.resize(P.max_level + 1);
    S.src.resize(P.max_level + 1);
    std::vector<int> own(ne);
    for (int sn = sp.sn_begin[0]; sn < sp.sn_begin[1]; ++sn)
      for (int q = 0; q < P.sn[sn].npiv; ++q) own[P.sn[sn].c0 + q] = sn;
    S.kdiag.assign(sp.nI, -1);
    // K lower triangle in position order, column by column (pi >= pj); the owning
    // front's row positions in a position map while its columns are visited
    std::vector<int> pmap(ne, -1);
    int cur = -1;
    for (int pj = 0; pj < ne; ++pj) {
      const int j = sp.perm[pj];
      const int sn = own[pj];
      const SnHost& hs = P.sn[sn];
      const SnDev& ds = sd[sn];
      if (sn != cur) {
        if (cur >= 0)
          for (int x : P.sn[cur].rows) pmap[x] = -1;
        for (size_t q = 0; q < hs.rows.size(); ++q) pmap[hs.rows[q]] = hs.npiv + (int)q;
        cur = sn;
      }
      const int lcol = pj - hs.c0;
      for (int64_t e = in.rowptr[j]; e < in.rowptr[j + 1]; ++e) {
        const int pi = sp.pos[in.col[e]];
        if (pi < pj) continue;  // tree DOF (-1) or upper triangle
        const int lrow = pi < hs.c0 + hs.npiv ? pi - hs.c0 : pmap[pi];
        if (lrow < 0) {
          S.err = "internal: entry outside the symbolic structure";
          return;
        }
        S.off[hs.level].push_back(lcol * ds.ld + lrow);
        S.sl[hs.level].push_back(sn - sb);
        S.src[hs.level].push_back((int)e);
        if (pi == pj && pj >= sp.nV && pj < sp.nr) S.kdiag[pj - sp.nV] = (int)e;
      }
      S.fxr.push_back(pj);
      S.fxs.push_back(j);
    }
    for (int a = 0; a < sp.nI; ++a)
      if (S.kdiag[a] < 0) S.err = "subdomain " + std::to_string(k) + ": missing diagonal entry";
    // one contiguous array per class (uploaded as it is)
    const int nl = P.max_level + 1;
    S.lev.assign(nl + 2, 0);
    for (int L = 0; L < nl; ++L) S.lev[L + 1] = S.lev[L] + (long long)S.off[L].size();
    S.lev[nl + 1] = S.lev[nl] + (long long)S.fxr.size();
    S.foff.reserve(S.lev[nl + 1]);
    S.fsl.reserve(S.lev[nl + 1]);
    S.fsrc.reserve(S.lev[nl + 1]);
    for (int L = 0; L < nl; ++L) {
      S.foff.insert(S.foff.end(), S.off[L].begin(), S.off[L].end());
      S.fsl.insert(S.fsl.end(), S.sl[L].begin(), S.sl[L].end());
      S.fsrc.insert(S.fsrc.end(), S.src[L].begin(), S.src[L].end());
      std::vector<int>().swap(S.sl[L]);
      std::vector<int>().swap(S.src[L]);
    }
    S.foff.insert(S.foff.end(), S.fxr.begin(), S.fxr.end());
    S.fsl.insert(S.fsl.end(), S.fxr.size(), 0);
    S.fsrc.insert(S.fsrc.end(), S.fxs.begin(), S.fxs.end());
  });
  for (int k : reps)
    if (!rel[k].err.empty()) throw Error(IETIDP_E_ARG, rel[k].err);
  stage(" scatter: relative entries");
  // segment offsets in the merged arrays: by level, then subdomain (groups contiguous)
  const int NL = P.max_level + 1;
  std::vector<long long> segoff((size_t)NL * ns + 1, 0);
  {
    long long o = 0;
    for (int L = 0; L < NL; ++L) {
      P.levels[L].sc_off = o;
      for (int k = 0; k < ns; ++k) {
        LevelPlan& gl = P.glevels[P.sub_group[k]][L];
        if (k == 0 || P.sub_group[k] != P.sub_group[k - 1]) gl.sc_off = o;
        segoff[(size_t)L * ns + k] = o;
        o += (long long)rel[rep[k]].off[L].size();
        gl.sc_n = o - gl.sc_off;
      }
      P.levels[L].sc_n = o - P.levels[L].sc_off;
    }
    segoff[(size_t)NL * ns] = o;
  }
  std::vector<long long> fxoff(ns + 1, 0), kdoff(ns + 1, 0);
  for (int k = 0; k < ns; ++k) {
    fxoff[k + 1] = fxoff[k] + (long long)rel[rep[k]].fxr.size() * nrhs;
    kdoff[k + 1] = kdoff[k] + (long long)rel[rep[k]].kdiag.size();
  }
  P.gfx.assign(P.ngroups, {0, 0});
  for (int k = 0; k < ns; ++k) {
    auto& gx = P.gfx[P.sub_group[k]];
    if (k == 0 || P.sub_group[k] != P.sub_group[k - 1]) gx.first = fxoff[k];
    gx.second = fxoff[k + 1] - gx.first;
  }
  stage(" scatter: offsets");
  // relative entries of the pattern classes, concatenated; one expansion segment per
  // (level, subdomain) and per subdomain's loads (expanded on the device at upload)
  std::vector<long long> relbase((size_t)ns * (NL + 1), -1);  // per class rep: start of level L / loads
  std::vector<long long> class_base(ns, -1);
  long long nrel = 0;
  for (int k : reps) {
    const Rel& S = rel[k];
    class_base[k] = nrel;
    for (int L = 0; L <= NL; ++L) relbase[(size_t)k * (NL + 1) + L] = nrel + S.lev[L];
    nrel += S.lev[NL + 1];
  }
  stage(" scatter: concatenation");
  std::vector<ExpandSeg> segs;
  for (int L = 0; L < NL; ++L)
    for (int k = 0; k < ns; ++k) {
      const int n = (int)rel[rep[k]].off[L].size();
      if (n == 0) continue;
      segs.push_back({segoff[(size_t)L * ns + k], relbase[(size_t)rep[k] * (NL + 1) + L], h->h_sub[k].kval_off, 0, n,
                      P.subs[k].sn_begin[0], h->h_sub[k].nk, 0});
    }
  for (int k = 0; k < ns; ++k) {
    const int n = (int)rel[rep[k]].fxr.size();
    if (n == 0) continue;
    segs.push_back({fxoff[k], relbase[(size_t)rep[k] * (NL + 1) + NL], h->h_sub[k].x_off, h->h_sub[k].f_off, n, 0,
                    h->h_sub[k].nk, 1});
  }
  std::vector<int> kdiag(kdoff[ns]);
  for (int k = 0; k < ns; ++k) {
    const Rel& S = rel[rep[k]];
    for (size_t a = 0; a < S.kdiag.size(); ++a) kdiag[kdoff[k] + a] = (int)(h->h_sub[k].kval_off + S.kdiag[a]);
  }
  for (int k : reps) std::vector<std::vector<int>>().swap(rel[k].off);  // (only the flattened lists are kept)
  stage("scatter lists");

  // ---- multipliers, slots, primal bookkeeping ----
  std::vector<int> slot_lam(h->n_slots);
  std::vector<float> slot_sign(h->n_slots);
  std::vector<LamDev> lam(h->n_lambda);
  std::vector<int> lamfill(h->n_lambda, 0);
  std::vector<int> prim_gid(po);
  std::vector<int> perm_all(permo);
  std::vector<char> gid_seen(h->n_primal, 0);
  for (int k = 0; k < ns; ++k) {
    const SubIn& in = h->in[k];
    const SubPlan& sp = P.subs[k];
    const SubDev& d = h->h_sub[k];
    for (size_t e = 0; e < in.B_dof.size(); ++e) {
      int slot = (int)d.rI_off + sp.pos[in.B_dof[e]] - sp.nV;
      int l = in.B_lambda[e];
      slot_lam[slot] = l;
      slot_sign[slot] = (float)in.B_sign[e];
      lam[l].slot[lamfill[l]] = slot;
      lam[l].sign[lamfill[l]] = (float)in.B_sign[e];
      lamfill[l]++;
    }
    for (int q = 0; q < sp.nP; ++q) {
      prim_gid[d.prim_off + q] = in.prim_gid[q];
      gid_seen[in.prim_gid[q]] = 1;
    }
    std::copy(sp.perm.begin(), sp.perm.end(), perm_all.begin() + d.perm_off);
  }
  for (int g = 0; g < h->n_primal; ++g)
    if (!gid_seen[g] && !h->shard) throw Error(IETIDP_E_ARG, "global primal " + std::to_string(g) + " has no local DOF");
  // S_PP entry (g1, g2) <- lower entries of the P fronts; global primal g <- (k, q)
  const int ng = h->n_primal;
  std::vector<std::vector<long long>> sl((size_t)ng * ng);
  std::vector<std::vector<std::pair<int, int>>> pc(ng);
  for (int k = 0; k < ns; ++k) {
    const SubDev& d = h->h_sub[k];
    if (d.pnode < 0) continue;
    const SnDev& pn = sd[d.pnode];
    for (int a = 0; a < d.nP; ++a) {
      int ga = prim_gid[d.prim_off + a];
      pc[ga].push_back({k, a});
      for (int b = 0; b < d.nP; ++b) {
        int gb = prim_gid[d.prim_off + b];
        int r = std::max(a, b), c = std::min(a, b);
        sl[(size_t)ga * ng + gb].push_back(pn.front_off + (long long)c * pn.ld + r);
      }
    }
  }
  std::vector<int> scoef_ptr((size_t)ng * ng + 1, 0), pcon_ptr(ng + 1, 0), pcon_sub, pcon_q;
  std::vector<long long> scoef_src;
  for (size_t e = 0; e < sl.size(); ++e) {
    scoef_src.insert(scoef_src.end(), sl[e].begin(), sl[e].end());
    scoef_ptr[e + 1] = (int)scoef_src.size();
  }
  for (int g = 0; g < ng; ++g) {
    for (auto& x : pc[g]) {
      pcon_sub.push_back(x.first);
      pcon_q.push_back(x.second);
    }
    pcon_ptr[g + 1] = (int)pcon_sub.size();
  }
  // the same, flattened to the loop work items' coarse partial rows: g_gi = sum over
  // gsrc[gsrc_ptr[gi] ..) of gpart[row][.]  (row = item * nPmax + local primal)
  std::vector<int> gsrc_ptr(ng + 1, 0), gsrc;
  {
    const int npm = std::max(P.nPmax, 1);
    for (int g = 0; g < ng; ++g) {
      for (auto& x : pc[g]) {
        const SubDev& d = h->h_sub[x.first];
        if (h->opt.loop == IETIDP_LOOP_EXPLICIT)  // symmetric pass: one row per (subdomain, block)
          for (int it = d.blk0; it < d.blk0 + d.nt; ++it) gsrc.push_back(it * npm + x.second);
        else  // triangular loop: one row per block-pair item
          for (int it = d.cta0; it < d.cta0 + sub_ncta[x.first]; ++it) gsrc.push_back(it * npm + x.second);
      }
      gsrc_ptr[g + 1] = (int)gsrc.size();
    }
  }
  auto t1 = std::chrono::steady_clock::now();
  h->rep.ms_analyze = std::chrono::duration<double, std::milli>(t1 - t0).count();  // host symbolic part
  h->rep.n_pattern_classes = h->n_pattern_classes;
  fill_report(h);
  if (getenv("IETIDP_DEBUG")) {
    int crit = 0;
    for (int L = 0; L <= P.max_level; ++L) {
      int mx = 0, mf = 0, n = 0;
      long long fl = 0;
      for (int i : bylev[L]) {
        const SnHost& sh = P.sn[i];
        if (sh.coarse) continue;
        ++n;
        mx = std::max(mx, sh.npiv);
        mf = std::max(mf, sh.f);
        for (int j = 0; j < sh.npiv; ++j) fl += (long long)(sh.f - j) * (sh.f - j);
      }
      crit += (mx + TB - 1) / TB;
      fprintf(stderr, "level %d: %d fronts, max npiv %d, max f %d, panels %d, GF %.2f\n", L, n, mx, mf,
              (mx + TB - 1) / TB, fl / 1e9);
    }
    fprintf(stderr, "critical-path panels %d, pool %.1f MB, inv %.1f MB\n", crit, P.pool_doubles * 8e-6, P.inv_doubles * 8e-6);
    auto gflops = [&](int off, int n) {
      long long f = 0;
      for (int q = off; q < off + n; ++q) f += 2LL * gwork[q].m * gwork[q].n * gwork[q].kdim;
      return f / 1e9;
    };
    for (int L = 0; L <= P.max_level; ++L) {
      double up = 0, tr = 0;
      std::vector<std::pair<int, int>> syrks;
      for (auto& gl : P.glevels) {
        for (auto& pn : gl[L].panels) {
          up += gflops(pn.upd_off, pn.upd_n);
          tr += gflops(pn.trsm_off, pn.trsm_n);
        }
        syrks.insert(syrks.end(), gl[L].syrk.begin(), gl[L].syrk.end());
      }
      fprintf(stderr, "level %d: upd %.2f GF, trsm %.2f GF, syrk:", L, up, tr);
      for (auto& sy : syrks) {
        int kmin = 1 << 30, kmax = 0;
        for (int q = sy.first; q < sy.first + sy.second; ++q) {
          kmin = std::min(kmin, gwork[q].kdim);
          kmax = std::max(kmax, gwork[q].kdim);
        }
        fprintf(stderr, " [%d tiles, K %d-%d, %.2f GF]", sy.second, kmin, kmax, gflops(sy.first, sy.second));
      }
      fprintf(stderr, "\n");
    }
  }
  if (h->opt.device < 0) {  // host-only analysis mode: no device work
    stage("rest (host only)");
    return;
  }

  stage("slots/primal");
  // ---- upload ----
  cudaStream_t s = h->stream;
  h->d_sn.upload(sd, s);
  h->d_sub.upload(h->h_sub, s);
  h->d_rows.upload(rows_all, s);
  h->d_rel.upload(rel_all, s);
  h->d_children.upload(children_all, s);
  h->d_work.upload(work, s);
  h->d_gwork.upload(gwork, s);
  h->d_level_sn.upload(P.level_sn, s);
  h->d_perm.upload(perm_all, s);
  h->d_uoff.upload(h->u_off, s);
  h->d_prim_gid.upload(prim_gid, s);
  {
    std::vector<ClassRel> cls;
    for (int k : reps) cls.push_back({class_base[k], &rel[k].foff, &rel[k].fsl, &rel[k].fsrc});
    expand_scatter(h, segs, cls, nrel, segoff[(size_t)NL * ns], fxoff[ns]);
  }
  h->kdiag_src.upload(kdiag, s);
  h->slot_lam.upload(slot_lam, s);
  h->slot_sign.upload(slot_sign, s);
  h->lam.upload(lam, s);
  h->h_lam = lam;
  h->scoef_ptr.upload(scoef_ptr, s);
  h->scoef_src.upload(scoef_src, s);
  h->pcon_ptr.upload(pcon_ptr, s);
  h->gsrc_ptr.upload(gsrc_ptr, s);
  h->gsrc.upload(gsrc, s);
  h->pcon_sub.upload(pcon_sub, s);
  h->pcon_q.upload(pcon_q, s);
  h->d_loopwork.upload(loopwork, s);
  h->d_symwork.upload(symwork, s);
  h->h_symwork = symwork;
  h->h_loopwork = loopwork;
  h->lpt_grid = 0;
  {
    std::vector<int> rl;
    h->rootlist_range.assign(P.ngroups, std::vector<std::pair<int, int>>(P.max_level + 1, {0, 0}));
    for (int g = 0; g < P.ngroups; ++g)
      for (int L = 0; L <= P.max_level; ++L) {
        const int off = (int)rl.size();
        for (int k : P.roots_by_level[L])
          if (P.sub_group[k] == g) rl.push_back(k);
        h->rootlist_range[g][L] = {off, (int)rl.size() - off};
      }
    h->d_rootlist.upload(rl, s);
    std::vector<long long> goff(h->n_slots);
    std::vector<int> np(h->n_slots), poff(h->n_slots);
    for (int k = 0; k < ns; ++k) {
      const SubDev& d = h->h_sub[k];
      for (int a = 0; a < d.nI; ++a) {
        goff[d.rI_off + a] = d.g_off + (long long)a * d.nP;
        np[d.rI_off + a] = d.nP;
        poff[d.rI_off + a] = d.prim_off;
      }
    }
    h->slot_goff.upload(goff, s);
    // symmetric-pass partial blocks per (subdomain, block)
    std::vector<long long> pboff;
    long long pbo = 0;
    for (int k = 0; k < ns; ++k) {
      const SubDev& d = h->h_sub[k];
      for (int j = 0; j < d.nt; ++j) {
        pboff.push_back(pbo);
        pbo += (j / SYM_SEG + 1) + (d.nt - 1 - j);
      }
    }
    h->d_pboff.upload(pboff, s);
    h->n_pblocks = pbo;
    std::vector<SlotRed> sred(h->n_slots);
    for (int k = 0; k < ns; ++k) {
      const SubDev& d = h->h_sub[k];
      for (int a = 0; a < d.nI; ++a) {
        const int j = a / TB, r = a % TB;
        sred[d.rI_off + a] = {pboff[d.blk0 + j] * TB + r, (j / SYM_SEG + 1) + (d.nt - 1 - j), 0};
      }
    }
    h->slot_red.upload(sred, s);
    std::vector<int2> blk;
    for (int k = 0; k < ns; ++k)
      for (int j = 0; j < h->h_sub[k].nt; ++j) blk.push_back(make_int2(k, j));
    h->n_blk = (int)blk.size();
    h->d_blk.upload(blk, s);
    h->slot_np.upload(np, s);
    h->slot_poff.upload(poff, s);
  }
  h->sub_cta0.upload(sub_cta0, s);
  h->sub_ncta.upload(sub_ncta, s);
  h->sub_blk0.upload(sub_blk0, s);
  h->sub_nt.upload(sub_nt, s);
  std::vector<double> kvals(kv), fvals(fv);
  for (int k = 0; k < ns; ++k) {
    std::copy(h->in[k].val.begin(), h->in[k].val.end(), kvals.begin() + h->kval_off[k]);
    std::copy(h->in[k].f.begin(), h->in[k].f.end(), fvals.begin() + h->fval_off[k]);
  }
  h->kval.upload(kvals, s);
  h->fval.upload(fvals, s);
  const int nc = nrhs;
  h->pool.alloc(P.pool_doubles);
  h->dinv.alloc(P.dinv_doubles);
  h->ipool.alloc(P.inv_doubles);
  h->tpool.alloc(P.inv_doubles);
  h->skws.alloc(std::max<long long>(1, P.splitk_doubles * P.ngroups));
  h->bpart.alloc(std::max<long long>(1, P.bpart_doubles));
  h->skcnt.alloc(std::max(1, P.splitk_tiles * P.ngroups));
  IETI_CUDA(cudaMemset(h->skcnt.p, 0, h->skcnt.n * sizeof(int)));
  h->vecw.alloc((size_t)P.vec_rows * 16);  // sweeps use up to 16 interleaved columns
  h->Xf.alloc((size_t)xo * nc);
  h->Xr.alloc((size_t)xo * nc);
  h->S.alloc((size_t)ng * ng);
  h->Sinv.alloc((size_t)ng * ng);
  h->ftil.alloc((size_t)ng * nc);
  h->zc0.alloc((size_t)ng * nc);
  h->err_flag.alloc(4);
  h->tiles.alloc(to);
  h->itiles.alloc(to);
  h->lpi.alloc(lpio);
  h->G.alloc(lpio);
  if (h->opt.loop == IETIDP_LOOP_EXPLICIT) {
    h->wtiles.alloc(to);
    h->stiles.alloc(to);
  }
  h->spart.alloc((size_t)std::max(h->n_pblocks, 1LL) * TB * nc);
  (void)spo;
  (void)npo;
  h->delta.alloc(h->n_slots);
  h->kdiag.alloc(h->n_slots);
  const size_t m = (size_t)h->n_lambda * nc;
  h->d_vec.alloc(m);
  h->lam_vec.alloc(m);
  h->r_vec.alloc(m);
  h->p_vec.alloc(m);
  h->q_vec.alloc(m);
  h->z_vec.alloc(m);
  h->yI.alloc((size_t)h->n_slots * nc);
  h->xI.alloc((size_t)h->n_slots * nc);
  h->sI.alloc((size_t)h->n_slots * nc);
  h->zI.alloc((size_t)h->n_slots * nc);
  h->gpart.alloc((size_t)std::max({cta, blk, 1}) * std::max(P.nPmax, 1) * nc);
  h->zc.alloc((size_t)std::max(ng, 1) * nc);
  h->gc.alloc((size_t)std::max(ng, 1) * nc);
  h->partial.alloc(4 * 1024 * (size_t)nc);
  h->state.alloc(16 * IETIDP_MAX_RHS + 64);
  h->coef_ld = std::max(1, std::max(h->opt.max_iter, h->opt.fixed_iters));
  h->cgcoef.alloc(2 * (size_t)nc * h->coef_ld);
  h->cgcoef.zero(h->stream);
  h->cond_out.alloc(3 * (size_t)nc);
  h->tmp_in.alloc(m);
  h->tmp_out.alloc(m);
  h->U.alloc(uo);
  IETI_CUDA(cudaStreamSynchronize(s));
  stage("upload/alloc");
  auto t2 = std::chrono::steady_clock::now();
  h->rep.ms_upload = std::chrono::duration<double, std::milli>(t2 - t1).count();
}

}  // namespace ieti
