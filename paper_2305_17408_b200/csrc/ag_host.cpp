// Host-side preprocessing of the AdaptGear path.
//
// ag_cluster_bfs restates reorder.py:92-153 (+ _undirected_adjacency :44-53,
// _refine_swaps :56-89) bit-exactly.  The algorithm is inherently sequential
// (greedy heap BFS, then Gauss-Seidel swap refinement whose tie-breaks depend
// on the visiting order), so it runs on the host; what changes vs. the
// reference is the data structure, not the decisions:
//   * neighbour histograms are sparse (only touched communities) instead of a
//     dense bincount(minlength=ncomm) per vertex;
//   * community member lists are kept sorted incrementally instead of an
//     O(n) flatnonzero(assigned == cstar) scan per vertex.
// ag_partition_from_ids restates load_partition's core (reorder.py:177-203).
#include <stdint.h>

#include <algorithm>
#include <numeric>
#include <queue>
#include <string>
#include <vector>

#include "adaptgear_b200.h"

namespace ag {
std::string &last_error();
}

namespace {

int host_fail(int code, const std::string &msg) {
  ag::last_error() = msg;
  return code;
}

struct Adjacency {
  std::vector<int64_t> start;  // n+1
  std::vector<int32_t> nbr;    // sorted unique per vertex
};

// reorder.py:44-53: sorted unique neighbours ignoring direction (a vertex is
// its own neighbour iff it has a self loop).
Adjacency undirected_adjacency(int64_t n, int64_t m, const int32_t *dst, const int32_t *src) {
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t i = 0; i < m; ++i) {
    ++cnt[dst[i] + 1];
    ++cnt[src[i] + 1];
  }
  for (int64_t v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
  std::vector<int32_t> raw(cnt[n]);
  std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (int64_t i = 0; i < m; ++i) {
    raw[fill[dst[i]]++] = src[i];
    raw[fill[src[i]]++] = dst[i];
  }
  Adjacency a;
  a.start.assign(n + 1, 0);
  a.nbr.reserve(raw.size());
  for (int64_t v = 0; v < n; ++v) {
    auto b = raw.begin() + cnt[v], e = raw.begin() + cnt[v + 1];
    std::sort(b, e);
    auto last = std::unique(b, e);
    a.nbr.insert(a.nbr.end(), b, last);
    a.start[v + 1] = static_cast<int64_t>(a.nbr.size());
  }
  return a;
}

// reorder.py:56-89
void refine_swaps(const Adjacency &adj, std::vector<int64_t> &assigned, int sweeps) {
  const int64_t n = static_cast<int64_t>(assigned.size());
  if (n == 0) return;
  const int64_t ncomm = *std::max_element(assigned.begin(), assigned.end()) + 1;
  std::vector<std::vector<int32_t>> members(ncomm);
  for (int64_t v = 0; v < n; ++v) members[assigned[v]].push_back(static_cast<int32_t>(v));
  std::vector<int64_t> hist(ncomm, 0);
  std::vector<int64_t> touched;
  touched.reserve(64);
  auto erase_sorted = [](std::vector<int32_t> &vec, int32_t x) {
    vec.erase(std::lower_bound(vec.begin(), vec.end(), x));
  };
  auto insert_sorted = [](std::vector<int32_t> &vec, int32_t x) {
    vec.insert(std::upper_bound(vec.begin(), vec.end(), x), x);
  };
  for (int s = 0; s < sweeps; ++s) {
    int64_t moved = 0;
    for (int64_t v = 0; v < n; ++v) {
      const int64_t c0 = assigned[v];
      const int64_t b = adj.start[v], e = adj.start[v + 1];
      if (b == e) continue;  // argmax of an all-zero histogram is 0: never moves
      touched.clear();
      for (int64_t k = b; k < e; ++k) {
        const int64_t c = assigned[adj.nbr[k]];
        if (hist[c]++ == 0) touched.push_back(c);
      }
      int64_t cstar = -1, best = -1;
      for (int64_t c : touched) {
        if (hist[c] > best || (hist[c] == best && c < cstar)) {
          best = hist[c];
          cstar = c;
        }
      }
      const int64_t cnt_star = hist[cstar];
      const int64_t cnt_c0 = hist[c0];
      for (int64_t c : touched) hist[c] = 0;
      if (cstar == c0 || cnt_star <= cnt_c0) continue;
      int64_t best_delta = 0, best_u = -1;
      const int32_t *vb = adj.nbr.data() + b;
      const int32_t *ve = adj.nbr.data() + e;
      for (int32_t u : members[cstar]) {
        int64_t cu_c0 = 0, cu_star = 0;
        for (int64_t k = adj.start[u]; k < adj.start[u + 1]; ++k) {
          const int64_t c = assigned[adj.nbr[k]];
          cu_c0 += (c == c0);
          cu_star += (c == cstar);
        }
        const int64_t vu = std::binary_search(vb, ve, u) ? 2 : 0;
        const int64_t delta = cnt_star + cu_c0 - cnt_c0 - cu_star - vu;
        if (delta > best_delta) {
          best_delta = delta;
          best_u = u;
        }
      }
      if (best_u >= 0) {
        assigned[v] = cstar;
        assigned[best_u] = c0;
        erase_sorted(members[c0], static_cast<int32_t>(v));
        insert_sorted(members[cstar], static_cast<int32_t>(v));
        erase_sorted(members[cstar], static_cast<int32_t>(best_u));
        insert_sorted(members[c0], static_cast<int32_t>(best_u));
        ++moved;
      }
    }
    if (!moved) break;
  }
}

}  // namespace

extern "C" int ag_cluster_bfs(int64_t n, int64_t m, const int32_t *dst, const int32_t *src,
                              int64_t comm_size, int64_t *community_out,
                              int64_t *permutation_out) {
  if (comm_size < 1) return host_fail(AG_ERR_VALUE, "comm_size must be >= 1");
  try {
    Adjacency adj = undirected_adjacency(n, m, dst, src);
    std::vector<int64_t> degree(n);
    for (int64_t v = 0; v < n; ++v) degree[v] = adj.start[v + 1] - adj.start[v];
    // lexsort((arange(n), -degree)): degree descending, id ascending
    std::vector<int32_t> seed_order(n);
    std::iota(seed_order.begin(), seed_order.end(), 0);
    std::stable_sort(seed_order.begin(), seed_order.end(),
                     [&](int32_t a, int32_t b) { return degree[a] > degree[b]; });
    std::vector<int64_t> assigned(n, -1);
    std::vector<int64_t> attach(n, 0);
    std::vector<int32_t> attach_touched;
    typedef std::pair<int64_t, int32_t> Entry;  // (-attachment, vertex): heapq order
    std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> heap;
    int64_t placed = 0, seed_pos = 0, comm = 0;
    while (placed < n) {
      while (assigned[seed_order[seed_pos]] >= 0) ++seed_pos;
      const int32_t start = seed_order[seed_pos];
      assigned[start] = comm;
      ++placed;
      int64_t size = 1;
      for (int64_t k = adj.start[start]; k < adj.start[start + 1]; ++k) {
        const int32_t u = adj.nbr[k];
        if (assigned[u] < 0) {
          if (attach[u] == 0) attach_touched.push_back(u);
          attach[u] = 1;
          heap.push(Entry(-1, u));
        }
      }
      while (size < comm_size && !heap.empty()) {
        const Entry top = heap.top();
        heap.pop();
        const int32_t v = top.second;
        if (assigned[v] >= 0 || attach[v] != -top.first) continue;  // stale entry
        assigned[v] = comm;
        ++placed;
        ++size;
        attach[v] = 0;  // del attach[v]
        for (int64_t k = adj.start[v]; k < adj.start[v + 1]; ++k) {
          const int32_t u = adj.nbr[k];
          if (assigned[u] < 0) {
            if (attach[u] == 0) attach_touched.push_back(u);
            attach[u] += 1;
            heap.push(Entry(-attach[u], u));
          }
        }
      }
      // a fresh frontier per community
      while (!heap.empty()) heap.pop();
      for (int32_t u : attach_touched) attach[u] = 0;
      attach_touched.clear();
      ++comm;
    }
    refine_swaps(adj, assigned, 3);
    // order = lexsort((arange(n), assigned)); permutation[order] = arange(n)
    std::vector<int32_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return assigned[a] < assigned[b]; });
    for (int64_t i = 0; i < n; ++i) {
      permutation_out[order[i]] = i;
      community_out[i] = assigned[i];
    }
  } catch (const std::exception &ex) {
    return host_fail(AG_ERR_CUDA, std::string("cluster_bfs: ") + ex.what());
  }
  return AG_OK;
}

extern "C" int ag_partition_from_ids(int64_t n, const int64_t *ids, int64_t comm_size,
                                     int64_t *community_out, int64_t *permutation_out) {
  if (comm_size < 1) return host_fail(AG_ERR_VALUE, "comm_size must be >= 1");
  for (int64_t i = 0; i < n; ++i)
    if (ids[i] < 0) return host_fail(AG_ERR_VALUE, "negative community id");
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t a, int64_t b) { return ids[a] < ids[b]; });
  int64_t chunk = -1, within = 0;
  for (int64_t i = 0; i < n; ++i) {
    const bool run_start = (i == 0) || ids[order[i]] != ids[order[i - 1]];
    within = run_start ? 0 : within + 1;
    if (within % comm_size == 0) ++chunk;
    community_out[order[i]] = chunk;
    permutation_out[order[i]] = i;
  }
  return AG_OK;
}
