// Host-side symbolic analysis for the multifrontal factorization
// (multifrontal.py): nested dissection of a block graph into a post-ordered
// elimination forest, and each front's boundary set.  Native because the
// setup runs inside the solve timer (the reference's lazy SuperLU
// factorizations count there too, solvers.py:300-305 / SURVEY 8(d)).
//
// Nested dissection: per connected component (in order of their lowest
// vertex), recursively: BFS from the first vertex, BFS again from the last
// vertex reached (pseudo-peripheral); the level set k minimising
// 2 max(|levels < k|, |levels > k|) + |level k| is chosen and thinned to the
// smaller one-sided vertex cut between levels k and k+1 (level-k vertices
// adjacent to level k+1, or level-(k+1) vertices adjacent to level k: 8 %
// fewer factor bytes on the cfg2 low-order system); the parts before and
// after it are dissected first (children), the separator is their parent.  Subsets of at most `leaf` vertices, or BFS depth < 3, are
// leaves.  Level sets are sorted, so the result equals the reference
// Python restatement kept in multifrontal.nested_dissection_py.
#include <stdint.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "xdg_common.cuh"

namespace {

struct ND {
  const int64_t* ptr;
  const int64_t* col;
  int64_t leaf;
  // per-vertex scratch shared by the workers of xdg_nd_order: a worker only
  // touches the vertices of its own connected components
  char* active;
  int64_t* dist;
  std::vector<int64_t> node_ptr{0};
  std::vector<int64_t> node_verts;
  std::vector<int64_t> parent;

  // BFS over active vertices; levels returned flattened (order) with
  // offsets; each level sorted ascending.
  void bfs(int64_t start, std::vector<int64_t>& order, std::vector<int64_t>& off) {
    order.clear();
    off.assign(1, 0);
    order.push_back(start);
    dist[start] = 0;
    off.push_back(1);
    int64_t b = 0, e = 1, d = 0;
    while (true) {
      ++d;
      for (int64_t i = b; i < e; ++i) {
        const int64_t v = order[i];
        for (int64_t k = ptr[v]; k < ptr[v + 1]; ++k) {
          const int64_t w = col[k];
          if (active[w] && dist[w] < 0) {
            dist[w] = d;
            order.push_back(w);
          }
        }
      }
      if ((int64_t)order.size() == e) break;
      std::sort(order.begin() + e, order.end());
      b = e;
      e = (int64_t)order.size();
      off.push_back(e);
    }
    for (int64_t v : order) dist[v] = -1;
  }

  int64_t make_node(std::vector<int64_t>& P, const std::vector<int64_t>& kids) {
    std::sort(P.begin(), P.end());
    const int64_t id = (int64_t)node_ptr.size() - 1;
    node_verts.insert(node_verts.end(), P.begin(), P.end());
    node_ptr.push_back((int64_t)node_verts.size());
    parent.push_back(-1);
    for (int64_t c : kids) parent[c] = id;
    return id;
  }

  // V sorted; returns the roots created for V (in creation order)
  std::vector<int64_t> run(std::vector<int64_t> V) {
    std::vector<int64_t> roots;
    if (V.empty()) return roots;
    for (int64_t v : V) active[v] = 1;
    std::vector<int64_t> order, off;
    bfs(V[0], order, off);
    if (order.size() < V.size()) {
      for (int64_t v : V) active[v] = 0;
      std::vector<int64_t> reached(order), rest;
      std::sort(reached.begin(), reached.end());
      std::set_difference(V.begin(), V.end(), reached.begin(), reached.end(),
                          std::back_inserter(rest));
      roots = run(reached);
      std::vector<int64_t> r2 = run(rest);
      roots.insert(roots.end(), r2.begin(), r2.end());
      return roots;
    }
    const int64_t nlev = (int64_t)off.size() - 1;
    if ((int64_t)V.size() <= leaf || nlev < 3) {
      for (int64_t v : V) active[v] = 0;
      roots.push_back(make_node(V, {}));
      return roots;
    }
    bfs(order[off[nlev - 1]], order, off);  // first vertex of the last level
    for (int64_t v : V) active[v] = 0;
    const int64_t L = (int64_t)off.size() - 1;
    if (L < 3) {
      roots.push_back(make_node(V, {}));
      return roots;
    }
    const int64_t n = (int64_t)V.size();
    int64_t best = -1, bestk = 1;
    for (int64_t k = 1; k <= L - 2; ++k) {
      const int64_t left = off[k], right = n - off[k + 1], size = off[k + 1] - off[k];
      const int64_t score = 2 * std::max(left, right) + size;
      if (best < 0 || score < best) {
        best = score;
        bestk = k;
      }
    }
    // thin the level-set separator to a minimal one-sided cut between
    // levels k and k+1: S1 = level-k vertices with a neighbour in level k+1
    // (the rest of level k joins the left part) or S2 = level-(k+1)
    // vertices with a neighbour in level k (the rest of level k+1 joins the
    // right part), the smaller of the two (S1 on ties)
    const int64_t k = bestk;
    for (int64_t i = off[k + 1]; i < off[k + 2]; ++i) dist[order[i]] = 1;  // level k+1
    std::vector<int64_t> S1, R1;
    for (int64_t i = off[k]; i < off[k + 1]; ++i) {
      const int64_t v = order[i];
      bool adj = false;
      for (int64_t e = ptr[v]; e < ptr[v + 1] && !adj; ++e) adj = dist[col[e]] == 1;
      (adj ? S1 : R1).push_back(v);
    }
    for (int64_t i = off[k + 1]; i < off[k + 2]; ++i) dist[order[i]] = -1;
    for (int64_t i = off[k]; i < off[k + 1]; ++i) dist[order[i]] = 1;  // level k
    std::vector<int64_t> S2, R2;
    for (int64_t i = off[k + 1]; i < off[k + 2]; ++i) {
      const int64_t v = order[i];
      bool adj = false;
      for (int64_t e = ptr[v]; e < ptr[v + 1] && !adj; ++e) adj = dist[col[e]] == 1;
      (adj ? S2 : R2).push_back(v);
    }
    for (int64_t i = off[k]; i < off[k + 1]; ++i) dist[order[i]] = -1;
    std::vector<int64_t> Lp(order.begin(), order.begin() + off[k]);
    std::vector<int64_t> Rp(order.begin() + off[k + 2], order.end());
    std::vector<int64_t> S;
    if (S2.size() < S1.size()) {
      Lp.insert(Lp.end(), order.begin() + off[k], order.begin() + off[k + 1]);
      Rp.insert(Rp.end(), R2.begin(), R2.end());
      S = std::move(S2);
    } else {
      Lp.insert(Lp.end(), R1.begin(), R1.end());
      Rp.insert(Rp.end(), order.begin() + off[k + 1], order.begin() + off[k + 2]);
      S = std::move(S1);
    }
    std::sort(Lp.begin(), Lp.end());
    std::sort(Rp.begin(), Rp.end());
    std::vector<int64_t> kids = run(std::move(Lp));
    std::vector<int64_t> k2 = run(std::move(Rp));
    kids.insert(kids.end(), k2.begin(), k2.end());
    roots.push_back(make_node(S, kids));
    return roots;
  }
};

std::vector<int64_t> g_bptr, g_bverts;  // last boundaries result (copied out)

}  // namespace

// Nested dissection of the graph (ptr, col) with nv vertices.  Writes the
// fronts in post-order: node_ptr[nnodes+1], node_verts[nv], parent[nnodes]
// (capacities nv+1, nv, nv).  Returns nnodes.
extern "C" int64_t xdg_nd_order(int64_t nv, const int64_t* ptr, const int64_t* col,
                                int64_t leaf, int64_t* node_ptr, int64_t* node_verts,
                                int64_t* parent) {
  if (nv <= 0) {
    node_ptr[0] = 0;
    return 0;
  }
  std::vector<char> active(nv, 0);
  std::vector<int64_t> dist(nv, -1);
  // connected components in order of their lowest vertex
  std::vector<int64_t> comp(nv, -1), cverts, cptr{0};
  cverts.reserve(nv);
  for (int64_t s = 0; s < nv; ++s) {
    if (comp[s] >= 0) continue;
    const size_t q0 = cverts.size();
    cverts.push_back(s);
    comp[s] = s;
    for (size_t i = q0; i < cverts.size(); ++i) {
      const int64_t v = cverts[i];
      for (int64_t k = ptr[v]; k < ptr[v + 1]; ++k)
        if (comp[col[k]] < 0) {
          comp[col[k]] = s;
          cverts.push_back(col[k]);
        }
    }
    std::sort(cverts.begin() + q0, cverts.end());
    cptr.push_back((int64_t)cverts.size());
  }
  // the components are independent (the Schwarz blocks' systems: thousands
  // of them): contiguous chunks of components per worker thread, results
  // appended in component order -- the same forest as one thread builds
  const int64_t nc = (int64_t)cptr.size() - 1;
  int64_t nthreads = (int64_t)std::thread::hardware_concurrency();
  nthreads = std::max<int64_t>(1, std::min<int64_t>({nthreads, 32, nc / 8}));
  std::vector<ND> nds(nthreads);
  std::vector<int64_t> cut(nthreads + 1, nc);
  cut[0] = 0;
  for (int64_t t = 1; t < nthreads; ++t) {  // chunks of about equal vertex counts
    const int64_t want = nv * t / nthreads;
    cut[t] = std::lower_bound(cptr.begin(), cptr.end(), want) - cptr.begin();
    cut[t] = std::min(std::max(cut[t], cut[t - 1]), nc);
  }
  auto work = [&](int64_t t) {
    ND& nd = nds[t];
    nd.ptr = ptr;
    nd.col = col;
    nd.leaf = leaf < 1 ? 1 : leaf;
    nd.active = active.data();
    nd.dist = dist.data();
    for (int64_t c = cut[t]; c < cut[t + 1]; ++c)
      nd.run(std::vector<int64_t>(cverts.begin() + cptr[c], cverts.begin() + cptr[c + 1]));
  };
  if (nthreads == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int64_t t = 0; t < nthreads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  int64_t nn = 0, nvert = 0;
  node_ptr[0] = 0;
  for (int64_t t = 0; t < nthreads; ++t) {
    const ND& nd = nds[t];
    const int64_t k = (int64_t)nd.parent.size();
    for (int64_t i = 0; i < k; ++i) {
      node_ptr[nn + i + 1] = nvert + nd.node_ptr[i + 1];
      parent[nn + i] = nd.parent[i] < 0 ? -1 : nd.parent[i] + nn;
    }
    std::copy(nd.node_verts.begin(), nd.node_verts.end(), node_verts + nvert);
    nn += k;
    nvert += (int64_t)nd.node_verts.size();
  }
  return nn;
}

// Boundary set of every front: B_t = (neighbours of P_t  U  B of t's
// children) minus the fronts of t's subtree (owner <= t in post-order),
// sorted by (owner, vertex).  Returns the total size; the sets are copied
// out by xdg_nd_boundaries_copy.
extern "C" int64_t xdg_nd_boundaries(int64_t nv, const int64_t* ptr, const int64_t* col,
                                     int64_t nnodes, const int64_t* node_ptr,
                                     const int64_t* node_verts, const int64_t* parent) {
  std::vector<int64_t> owner(nv, -1), stamp(nv, -1);
  for (int64_t t = 0; t < nnodes; ++t)
    for (int64_t i = node_ptr[t]; i < node_ptr[t + 1]; ++i) owner[node_verts[i]] = t;
  std::vector<std::vector<int64_t>> kids(nnodes);
  for (int64_t t = 0; t < nnodes; ++t)
    if (parent[t] >= 0) kids[parent[t]].push_back(t);
  g_bptr.assign(nnodes + 1, 0);
  g_bverts.clear();
  std::vector<int64_t> cand;
  for (int64_t t = 0; t < nnodes; ++t) {
    cand.clear();
    auto add = [&](int64_t w) {
      if (owner[w] > t && stamp[w] != t) {
        stamp[w] = t;
        cand.push_back(w);
      }
    };
    for (int64_t i = node_ptr[t]; i < node_ptr[t + 1]; ++i) {
      const int64_t v = node_verts[i];
      for (int64_t k = ptr[v]; k < ptr[v + 1]; ++k) add(col[k]);
    }
    for (int64_t c : kids[t])
      for (int64_t i = g_bptr[c]; i < g_bptr[c + 1]; ++i) add(g_bverts[i]);
    std::sort(cand.begin(), cand.end(), [&](int64_t a, int64_t b) {
      return owner[a] != owner[b] ? owner[a] < owner[b] : a < b;
    });
    g_bverts.insert(g_bverts.end(), cand.begin(), cand.end());
    g_bptr[t + 1] = (int64_t)g_bverts.size();
  }
  return (int64_t)g_bverts.size();
}

extern "C" int xdg_nd_boundaries_copy(int64_t* b_ptr, int64_t* b_verts) {
  std::copy(g_bptr.begin(), g_bptr.end(), b_ptr);
  std::copy(g_bverts.begin(), g_bverts.end(), b_verts);
  return XDG_OK;
}

// ---------------------------------------------------------------------------
// Overlapping Schwarz partition (cutdg schwarz_partition, solvers.py:384-457;
// host setup, must match the reference exactly): greedy breadth-first cores
// seeded at the lowest unassigned node, neighbours (sorted adjacency) queued
// in order if neither taken nor already queued for this core; a core closes
// once it holds >= target DOFs; then every core grows by one neighbour layer
// (sorted, deduplicated).  Returns the number of cores; the cores and the
// extended blocks are copied out by xdg_schwarz_copy.
namespace {
std::vector<int64_t> g_cptr, g_cnodes, g_eptr, g_enodes;
}

extern "C" int64_t xdg_schwarz_partition(int64_t n, const int64_t* adj_ptr,
                                         const int64_t* adj, const int64_t* dofs,
                                         int64_t target) {
  std::vector<char> taken(n, 0);
  std::vector<int64_t> seen(n, -1), queue, core;
  g_cptr.assign(1, 0);
  g_cnodes.clear();
  int64_t next_free = 0, ncore = 0;
  while (true) {
    while (next_free < n && taken[next_free]) ++next_free;
    if (next_free == n) break;
    core.clear();
    queue.assign(1, next_free);
    seen[next_free] = ncore;
    int64_t acc = 0;
    for (size_t qi = 0; qi < queue.size() && acc < target; ++qi) {
      const int64_t c = queue[qi];
      if (taken[c]) continue;
      taken[c] = 1;
      core.push_back(c);
      acc += dofs[c];
      for (int64_t k = adj_ptr[c]; k < adj_ptr[c + 1]; ++k) {
        const int64_t nb = adj[k];
        if (!taken[nb] && seen[nb] != ncore) {
          seen[nb] = ncore;
          queue.push_back(nb);
        }
      }
    }
    std::sort(core.begin(), core.end());
    g_cnodes.insert(g_cnodes.end(), core.begin(), core.end());
    g_cptr.push_back((int64_t)g_cnodes.size());
    ++ncore;
  }
  // one neighbour layer
  g_eptr.assign(1, 0);
  g_enodes.clear();
  std::vector<int64_t> stamp(n, -1), grown;
  for (int64_t q = 0; q < ncore; ++q) {
    grown.clear();
    for (int64_t i = g_cptr[q]; i < g_cptr[q + 1]; ++i) {
      const int64_t c = g_cnodes[i];
      if (stamp[c] != q) {
        stamp[c] = q;
        grown.push_back(c);
      }
      for (int64_t k = adj_ptr[c]; k < adj_ptr[c + 1]; ++k)
        if (stamp[adj[k]] != q) {
          stamp[adj[k]] = q;
          grown.push_back(adj[k]);
        }
    }
    std::sort(grown.begin(), grown.end());
    g_enodes.insert(g_enodes.end(), grown.begin(), grown.end());
    g_eptr.push_back((int64_t)g_enodes.size());
  }
  return ncore;
}

// sizes: out[0] = #core nodes, out[1] = #extended nodes
extern "C" int xdg_schwarz_sizes(int64_t* out) {
  out[0] = (int64_t)g_cnodes.size();
  out[1] = (int64_t)g_enodes.size();
  return XDG_OK;
}

extern "C" int xdg_schwarz_copy(int64_t* core_ptr, int64_t* core_nodes, int64_t* ext_ptr,
                                int64_t* ext_nodes) {
  std::copy(g_cptr.begin(), g_cptr.end(), core_ptr);
  std::copy(g_cnodes.begin(), g_cnodes.end(), core_nodes);
  std::copy(g_eptr.begin(), g_eptr.end(), ext_ptr);
  std::copy(g_enodes.begin(), g_enodes.end(), ext_nodes);
  return XDG_OK;
}
