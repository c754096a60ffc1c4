// Host-side symbolic analysis, native.
//
// Restates the reference's ordering/symbolic algorithms with identical
// outputs (the reference's rules are deterministic: ties by lowest index):
//   * nested dissection        reference ordering.py:225-266 (+ helpers :94-222)
//   * elimination tree (Liu)   reference ordering.py:269-291
//   * postorder                reference ordering.py:294-311
//   * column structures + fundamental supernodes
//                              reference symbolic.py:36-53 and :88-104
// The column structures are streamed (a child's structure is freed once its
// parent consumed it) so 120^3 analysis does not hold nnz(L) row indices.
// Exposed through a C ABI (ctypes in ordering.py / symbolic.py).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <set>
#include <vector>

typedef int64_t i64;

namespace {

struct Graph {
  i64 n;
  const i64* ptr;
  const i64* idx;
};

struct SepNode {
  i64 nverts;
  std::vector<int> kids;
};

class Dissector {
 public:
  Dissector(const Graph& g, i64 leaf) : G(g), leaf_(leaf), tag_(g.n, -1), seen_(g.n, -1), side_(g.n, 0) {}

  int run() {
    std::vector<i64> all(G.n);
    for (i64 i = 0; i < G.n; ++i) all[i] = i;
    return visit(all);
  }

  std::vector<i64> order;
  std::vector<SepNode> nodes;

 private:
  const Graph G;
  i64 leaf_;
  std::vector<int> tag_;   // stamp of the current vertex set
  std::vector<int> seen_;  // stamp for traversals
  std::vector<signed char> side_;
  int stamp_ = 0;
  int seen_stamp_ = 0;

  int mark(const std::vector<i64>& vs) {
    ++stamp_;
    for (i64 v : vs) tag_[v] = stamp_;
    return stamp_;
  }

  // connected components of the induced subgraph, each sorted, ordered by min vertex
  std::vector<std::vector<i64>> components(const std::vector<i64>& verts) {
    int cur = mark(verts);
    int s = ++seen_stamp_;
    std::vector<std::vector<i64>> comps;
    std::vector<i64> stack;
    for (i64 start : verts) {  // verts sorted ascending
      if (seen_[start] == s) continue;
      std::vector<i64> comp;
      stack.clear();
      stack.push_back(start);
      seen_[start] = s;
      while (!stack.empty()) {
        i64 v = stack.back();
        stack.pop_back();
        comp.push_back(v);
        for (i64 e = G.ptr[v]; e < G.ptr[v + 1]; ++e) {
          i64 w = G.idx[e];
          if (tag_[w] == cur && seen_[w] != s) {
            seen_[w] = s;
            stack.push_back(w);
          }
        }
      }
      std::sort(comp.begin(), comp.end());
      comps.push_back(std::move(comp));
    }
    return comps;
  }

  // BFS level sets inside the set stamped `cur`, each level sorted
  std::vector<std::vector<i64>> bfs_levels(i64 start, int cur) {
    int s = ++seen_stamp_;
    std::vector<std::vector<i64>> levels;
    levels.push_back({start});
    seen_[start] = s;
    while (true) {
      std::vector<i64> nxt;
      for (i64 v : levels.back()) {
        for (i64 e = G.ptr[v]; e < G.ptr[v + 1]; ++e) {
          i64 w = G.idx[e];
          if (tag_[w] == cur && seen_[w] != s) {
            seen_[w] = s;
            nxt.push_back(w);
          }
        }
      }
      if (nxt.empty()) break;
      std::sort(nxt.begin(), nxt.end());
      levels.push_back(std::move(nxt));
    }
    return levels;
  }

  // reference _pseudo_peripheral: up to 4 eccentricity-increasing sweeps
  std::vector<std::vector<i64>> pseudo_peripheral(const std::vector<i64>& verts, int cur) {
    i64 v = verts.front();
    i64 last_depth = -1;
    std::vector<std::vector<i64>> levels;
    bool have = false;
    for (int it = 0; it < 4; ++it) {
      levels = bfs_levels(v, cur);
      if ((i64)levels.size() - 1 <= last_depth) {
        have = true;  // v unchanged; levels == bfs(v)
        break;
      }
      last_depth = (i64)levels.size() - 1;
      v = levels.back().front();
    }
    if (!have) levels = bfs_levels(v, cur);
    return levels;
  }

  // reference _split_once; returns false for "None"
  bool split_once(const std::vector<i64>& verts, std::vector<i64>& A, std::vector<i64>& B,
                  std::vector<i64>& S) {
    int cur = mark(verts);
    auto levels = pseudo_peripheral(verts, cur);
    if (levels.size() < 2) return false;
    i64 total = 0;
    for (auto& l : levels) total += (i64)l.size();
    size_t best_l = 0;
    i64 best_gap = -1, left = 0;
    for (size_t l = 0; l < levels.size(); ++l) {
      i64 right = total - left - (i64)levels[l].size();
      i64 gap = left > right ? left - right : right - left;
      if (best_gap < 0 || gap < best_gap) {
        best_gap = gap;
        best_l = l;
      }
      left += (i64)levels[l].size();
    }
    i64 na = 0, nb = 0;
    for (size_t l = 0; l < levels.size(); ++l) {
      signed char sd = l < best_l ? 0 : (l == best_l ? 2 : 1);
      for (i64 v : levels[l]) side_[v] = sd;
      if (sd == 0) na += (i64)levels[l].size();
      if (sd == 1) nb += (i64)levels[l].size();
    }
    const std::vector<i64>& sep = levels[best_l];  // sorted
    if (na > 0 && nb > 0) {
      // one refinement pass in ascending separator order; sides mutate as we go
      for (i64 s : sep) {
        bool in_a = false, in_b = false;
        for (i64 e = G.ptr[s]; e < G.ptr[s + 1]; ++e) {
          i64 w = G.idx[e];
          if (tag_[w] != cur) continue;
          if (side_[w] == 0) in_a = true;
          else if (side_[w] == 1) in_b = true;
        }
        if (in_a && !in_b) {
          side_[s] = 0; ++na;
        } else if (in_b && !in_a) {
          side_[s] = 1; ++nb;
        } else if (!in_a && !in_b) {
          if (na <= nb) { side_[s] = 0; ++na; }
          else { side_[s] = 1; ++nb; }
        }
      }
    }
    A.clear(); B.clear(); S.clear();
    for (i64 v : verts) {  // sorted
      if (side_[v] == 0) A.push_back(v);
      else if (side_[v] == 1) B.push_back(v);
      else S.push_back(v);
    }
    return true;
  }

  // reference _min_degree_order (naive, quotient-graph clique fill)
  void min_degree(const std::vector<i64>& verts) {
    const size_t k = verts.size();
    if (k == 0) return;
    int cur = mark(verts);
    // local index of each vertex: position in sorted verts
    std::vector<std::vector<int>> nb(k);
    for (size_t a = 0; a < k; ++a) {
      i64 v = verts[a];
      for (i64 e = G.ptr[v]; e < G.ptr[v + 1]; ++e) {
        i64 w = G.idx[e];
        if (tag_[w] != cur) continue;
        int b = (int)(std::lower_bound(verts.begin(), verts.end(), w) - verts.begin());
        nb[a].push_back(b);
      }
    }
    if (k <= 4096) {
      std::vector<unsigned char> adj(k * k, 0);
      std::vector<int> deg(k, 0);
      for (size_t a = 0; a < k; ++a)
        for (int b : nb[a])
          if (!adj[a * k + b]) { adj[a * k + b] = 1; ++deg[a]; }
      std::vector<unsigned char> alive(k, 1);
      std::vector<int> nbrs;
      for (size_t step = 0; step < k; ++step) {
        int best = -1;
        for (size_t a = 0; a < k; ++a)
          if (alive[a] && (best < 0 || deg[a] < deg[best])) best = (int)a;
        order.push_back(verts[best]);
        alive[best] = 0;
        nbrs.clear();
        for (size_t a = 0; a < k; ++a)
          if (adj[(size_t)best * k + a]) nbrs.push_back((int)a);
        for (int u : nbrs) {
          if (adj[(size_t)u * k + best]) { adj[(size_t)u * k + best] = 0; --deg[u]; }
        }
        for (int a = 0; a < (int)k; ++a) adj[(size_t)best * k + a] = 0;
        deg[best] = 0;
        for (int u : nbrs)
          for (int w : nbrs)
            if (w != u && !adj[(size_t)u * k + w]) { adj[(size_t)u * k + w] = 1; ++deg[u]; }
      }
    } else {
      std::vector<std::set<int>> adj(k);
      for (size_t a = 0; a < k; ++a) adj[a].insert(nb[a].begin(), nb[a].end());
      std::set<std::pair<size_t, int>> pq;
      for (size_t a = 0; a < k; ++a) pq.insert({adj[a].size(), (int)a});
      while (!pq.empty()) {
        int v = pq.begin()->second;
        pq.erase(pq.begin());
        order.push_back(verts[v]);
        std::vector<int> nbrs(adj[v].begin(), adj[v].end());
        adj[v].clear();
        for (int u : nbrs) {
          pq.erase({adj[u].size(), u});
          adj[u].erase(v);
        }
        for (int u : nbrs)
          for (int w : nbrs)
            if (w != u) adj[u].insert(w);
        for (int u : nbrs) pq.insert({adj[u].size(), u});
      }
    }
  }

  int new_node(i64 nverts) {
    nodes.push_back(SepNode{nverts, {}});
    return (int)nodes.size() - 1;
  }

  int visit(const std::vector<i64>& vertices) {
    auto comps = components(vertices);
    if (comps.size() > 1) {
      int node = new_node(0);
      for (auto& c : comps) {
        int kid = visit(c);
        nodes[node].kids.push_back(kid);
      }
      return node;
    }
    std::vector<i64> verts;
    if (!comps.empty()) verts = std::move(comps[0]);
    if ((i64)verts.size() <= leaf_) {
      min_degree(verts);
      return new_node((i64)verts.size());
    }
    std::vector<i64> A, B, S;
    if (!split_once(verts, A, B, S)) {
      min_degree(verts);
      return new_node((i64)verts.size());
    }
    verts.clear();
    verts.shrink_to_fit();
    int node = new_node((i64)S.size());
    if (!A.empty()) {
      int kid = visit(A);
      nodes[node].kids.push_back(kid);
    }
    if (!B.empty()) {
      int kid = visit(B);
      nodes[node].kids.push_back(kid);
    }
    order.insert(order.end(), S.begin(), S.end());
    return node;
  }
};

struct Symbolic {
  i64 nnz_l = 0;
  std::vector<i64> starts;   // fundamental supernode starts (+ n)
  std::vector<i64> rowptr;   // per supernode, rows >= lc
  std::vector<i64> rows;
};

}  // namespace

extern "C" {

// Nested dissection (reference ordering.py:225-266).
// iperm_out[n]: new -> old.  sep_sizes_out: sizes of non-leaf separator-tree
// nodes in the reference's all_nodes() order; capacity `cap`, count returned
// in *nsep.  Returns 0, or -1 if cap is too small.
int psh_nested_dissection(i64 n, const i64* indptr, const i64* indices, i64 leaf,
                          i64* iperm_out, i64* sep_sizes_out, i64 cap, i64* nsep) {
  Graph g{n, indptr, indices};
  Dissector d(g, leaf);
  int root = d.run();
  if ((i64)d.order.size() != n) return -2;
  std::memcpy(iperm_out, d.order.data(), sizeof(i64) * n);
  // all_nodes(): stack = [root]; pop; append; extend(children)
  std::vector<int> stack{root};
  i64 cnt = 0;
  while (!stack.empty()) {
    int v = stack.back();
    stack.pop_back();
    const SepNode& nd = d.nodes[v];
    if (!nd.kids.empty()) {
      if (cnt >= cap) return -1;
      sep_sizes_out[cnt++] = nd.nverts;
    }
    for (int c : nd.kids) stack.push_back(c);
  }
  *nsep = cnt;
  return 0;
}

// Elimination tree of a symmetric-lower CSC pattern (reference ordering.py:269-291).
void psh_etree(i64 n, const i64* colptr, const i64* rowidx, i64* parent) {
  // row lists of the strict lower triangle: row i -> columns k < i (ascending)
  std::vector<i64> cnt(n + 1, 0);
  for (i64 k = 0; k < n; ++k)
    for (i64 e = colptr[k]; e < colptr[k + 1]; ++e)
      if (rowidx[e] > k) ++cnt[rowidx[e] + 1];
  for (i64 i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  std::vector<i64> rl(cnt[n]), pos(cnt.begin(), cnt.end() - 1);
  for (i64 k = 0; k < n; ++k)
    for (i64 e = colptr[k]; e < colptr[k + 1]; ++e)
      if (rowidx[e] > k) rl[pos[rowidx[e]]++] = k;
  std::vector<i64> anc(n, -1);
  for (i64 j = 0; j < n; ++j) parent[j] = -1;
  for (i64 j = 0; j < n; ++j) {
    for (i64 t = cnt[j]; t < cnt[j + 1]; ++t) {
      i64 r = rl[t];
      while (anc[r] != -1 && anc[r] != j) {
        i64 nx = anc[r];
        anc[r] = j;
        r = nx;
      }
      if (anc[r] == -1) {
        anc[r] = j;
        parent[r] = j;
      }
    }
  }
}

// Post-order (roots ascending, children ascending); po[new] = old
// (reference ordering.py:294-311).
void psh_postorder(i64 n, const i64* parent, i64* po) {
  std::vector<i64> head(n, -1), next(n, -1);
  // children lists ascending: insert in descending order at the head
  for (i64 v = n - 1; v >= 0; --v) {
    i64 p = parent[v];
    if (p >= 0) {
      next[v] = head[p];
      head[p] = v;
    }
  }
  i64 pos = 0;
  std::vector<std::pair<i64, i64>> stack;  // (vertex, next child cursor)
  for (i64 r = 0; r < n; ++r) {
    if (parent[r] >= 0) continue;
    stack.push_back({r, head[r]});
    while (!stack.empty()) {
      auto& top = stack.back();
      if (top.second >= 0) {
        i64 c = top.second;
        top.second = next[c];
        stack.push_back({c, head[c]});
      } else {
        po[pos++] = top.first;
        stack.pop_back();
      }
    }
  }
}

// Column structures of L and the fundamental supernode partition
// (reference symbolic.py:36-53 + find_supernodes :88-104).  Requires a
// postordered tree (parent[v] > v).  Returns a handle or nullptr.
void* psh_symbolic(i64 n, const i64* colptr, const i64* rowidx, const i64* parent) {
  auto* out = new Symbolic();
  std::vector<std::vector<i64>> kids(n);
  for (i64 v = 0; v < n; ++v)
    if (parent[v] >= 0) kids[parent[v]].push_back(v);
  std::vector<std::vector<i64>> st(n);
  std::vector<i64> mark(n, -1);
  std::vector<i64> cnt(n, 0);
  std::vector<i64> start_struct_of;  // unused
  std::vector<i64> cur_struct;
  out->starts.push_back(0);
  std::vector<i64> panel_first_struct;  // struct of the current panel's first column
  std::vector<std::vector<i64>> pstruct;
  for (i64 j = 0; j < n; ++j) {
    std::vector<i64> s;
    mark[j] = j;
    s.push_back(j);
    for (i64 e = colptr[j]; e < colptr[j + 1]; ++e) {
      i64 r = rowidx[e];
      if (r >= j && mark[r] != j) { mark[r] = j; s.push_back(r); }
    }
    for (i64 c : kids[j]) {
      for (i64 r : st[c]) {
        if (r > c && mark[r] != j) { mark[r] = j; s.push_back(r); }
      }
      std::vector<i64>().swap(st[c]);  // consumed
    }
    std::sort(s.begin(), s.end());
    cnt[j] = (i64)s.size();
    out->nnz_l += cnt[j];
    bool merge = j > 0 && parent[j - 1] == j && cnt[j - 1] == cnt[j] + 1;
    if (!merge && j > 0) out->starts.push_back(j);
    if (!merge) pstruct.push_back(s);
    if (parent[j] >= 0) st[j] = std::move(s);
  }
  out->starts.push_back(n);
  if (n == 0) out->starts.assign(1, 0);
  const i64 np = (i64)out->starts.size() - 1;
  out->rowptr.assign(np + 1, 0);
  for (i64 p = 0; p < np; ++p) {
    i64 lc = out->starts[p + 1];
    const auto& s = pstruct[p];
    auto it = std::lower_bound(s.begin(), s.end(), lc);
    out->rows.insert(out->rows.end(), it, s.end());
    out->rowptr[p + 1] = (i64)out->rows.size();
  }
  return out;
}

void psh_symbolic_sizes(void* h, i64* npanels, i64* nrows, i64* nnz_l) {
  auto* s = (Symbolic*)h;
  *npanels = (i64)s->starts.size() - 1;
  *nrows = (i64)s->rows.size();
  *nnz_l = s->nnz_l;
}

void psh_symbolic_fetch(void* h, i64* starts, i64* rowptr, i64* rows) {
  auto* s = (Symbolic*)h;
  std::memcpy(starts, s->starts.data(), sizeof(i64) * s->starts.size());
  std::memcpy(rowptr, s->rowptr.data(), sizeof(i64) * s->rowptr.size());
  if (!s->rows.empty()) std::memcpy(rows, s->rows.data(), sizeof(i64) * s->rows.size());
}

void psh_symbolic_free(void* h) { delete (Symbolic*)h; }

}  // extern "C"
