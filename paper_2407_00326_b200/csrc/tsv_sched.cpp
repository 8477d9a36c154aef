// tsv_sched.cpp - native engine queue for the topology-aware batch scheduler.
//
// The reference forms every batch of an engine with form_batch_topo
// (pkg/src/teola_sim/runtime.py:189-268): per-query buckets of the queued node tasks in order of
// earliest arrival; each pass takes the requests of every bucket's deepest pending nodes (node
// id order) while slots remain; passes repeat until the cap is reached or nothing fits. The
// Python mirror (paper_2407_00326_b200/runtime.py, form_batch_topo) rebuilds that state from
// every queued task object on every call: with thousands of queued stage tasks (the
// embedding / LLM engines of a workflow) batch formation dominated the host time of the
// real-time runtime. Here the queue lives in native memory: a task is pushed once (its static
// fields and request loads), batches are formed over flat arrays, and a dispatched batch is
// committed (requests consumed, drained tasks dropped). Decisions are the mirror's, bit for
// bit: the same pass structure, the same comparisons and the same left-to-right double sums
// (tests/test_mirror_reference.py runs the 300 reference snapshots through both).
//
// Host-only code: no CUDA calls, usable without a GPU.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "tsv.h"

namespace {

struct Task {
  int64_t handle = 0;
  int query = 0;             // index into Queue::queries
  std::string node_id;
  int depth = 0;
  int phase = 0;
  double arrival = 0.0;
  std::vector<double> loads;
  int64_t next = 0;          // first unconsumed request
  int64_t scratch_next = 0;  // form()'s private copy of next
  bool pending() const { return static_cast<int64_t>(loads.size()) > next; }
};

struct Query {
  std::string id;
  std::vector<int> tasks;  // slots in Queue::tasks
};

struct Bucket {
  int query;
  double min_arrival;
};

}  // namespace

struct tsv_topo_queue {
  double eps = 1e-9;
  std::vector<Task> tasks;  // slot storage; free slots are recycled
  std::vector<int> free_slots;
  std::unordered_map<int64_t, int> slot_of;  // handle -> slot
  std::vector<Query> queries;
  std::unordered_map<std::string, int> query_of;
  std::vector<int> free_queries;
  // form() scratch
  std::vector<Bucket> buckets;
  std::vector<int> cands;
  std::vector<std::pair<int, int64_t>> entries;  // (slot, n) in pass order
};

namespace {

// _fill_at: requests of `loads` from `begin` that fit next to `used` under `cap`; a request
// that alone exceeds the cap is admitted when nothing else is in the batch.
inline int64_t fill_at(const std::vector<double>& loads, int64_t begin, double used, double cap,
                       bool nonempty, double eps, double* acc_out) {
  int64_t n = 0;
  double acc = 0.0;
  const int64_t len = static_cast<int64_t>(loads.size());
  for (int64_t i = begin; i < len; ++i) {
    const double r = loads[i];
    if (used + acc + r > cap + eps && (nonempty || n)) break;
    ++n;
    acc += r;
  }
  *acc_out = acc;
  return n;
}

inline bool bucket_before(const tsv_topo_queue* q, const Bucket& a, const Bucket& b) {
  if (a.min_arrival != b.min_arrival) return a.min_arrival < b.min_arrival;
  return q->queries[a.query].id < q->queries[b.query].id;
}

void drop_task(tsv_topo_queue* q, int slot) {
  Task& t = q->tasks[slot];
  Query& qu = q->queries[t.query];
  auto it = std::find(qu.tasks.begin(), qu.tasks.end(), slot);
  if (it != qu.tasks.end()) qu.tasks.erase(it);
  if (qu.tasks.empty()) {
    q->query_of.erase(qu.id);
    qu.id.clear();
    q->free_queries.push_back(t.query);
  }
  q->slot_of.erase(t.handle);
  t.loads.clear();
  t.loads.shrink_to_fit();
  t.node_id.clear();
  t.handle = 0;
  q->free_slots.push_back(slot);
}

}  // namespace

extern "C" {

TSV_API int tsv_topo_create(double eps, tsv_topo_queue** out) {
  if (out == nullptr) return TSV_ERR_ARGUMENT;
  auto* q = new tsv_topo_queue();
  q->eps = eps;
  *out = q;
  return TSV_OK;
}

TSV_API int tsv_topo_destroy(tsv_topo_queue* q) {
  delete q;
  return TSV_OK;
}

TSV_API int64_t tsv_topo_size(const tsv_topo_queue* q) {
  return q ? static_cast<int64_t>(q->slot_of.size()) : -1;
}

TSV_API int tsv_topo_push(tsv_topo_queue* q, int64_t handle, const char* query_id,
                          const char* node_id, int depth, int phase, double arrival_ms,
                          const double* loads, int64_t n_loads, int64_t next) {
  if (q == nullptr || query_id == nullptr || node_id == nullptr || n_loads < 0 ||
      (n_loads > 0 && loads == nullptr) || next < 0)
    return TSV_ERR_ARGUMENT;
  if (q->slot_of.count(handle)) return TSV_ERR_ARGUMENT;
  int slot;
  if (!q->free_slots.empty()) {
    slot = q->free_slots.back();
    q->free_slots.pop_back();
  } else {
    slot = static_cast<int>(q->tasks.size());
    q->tasks.emplace_back();
  }
  int qi;
  auto it = q->query_of.find(query_id);
  if (it != q->query_of.end()) {
    qi = it->second;
  } else {
    if (!q->free_queries.empty()) {
      qi = q->free_queries.back();
      q->free_queries.pop_back();
    } else {
      qi = static_cast<int>(q->queries.size());
      q->queries.emplace_back();
    }
    q->queries[qi].id = query_id;
    q->queries[qi].tasks.clear();
    q->query_of.emplace(query_id, qi);
  }
  Task& t = q->tasks[slot];
  t.handle = handle;
  t.query = qi;
  t.node_id = node_id;
  t.depth = depth;
  t.phase = phase;
  t.arrival = arrival_ms;
  t.loads.assign(loads, loads + n_loads);
  t.next = next;
  q->queries[qi].tasks.push_back(slot);
  q->slot_of.emplace(handle, slot);
  return TSV_OK;
}

// Form one batch under `max_slots`. Writes up to `cap_entries` (task handle, request count)
// pairs, merged per task in order of first appearance; *n_entries = the number of entries
// (when it exceeds cap_entries nothing is written and the call returns TSV_ERR_CAPACITY: grow
// the buffers and call again). *phase = the anchor task's phase (unchanged when empty).
TSV_API int tsv_topo_form(tsv_topo_queue* q, double max_slots, int64_t cap_entries,
                          int64_t* handles, int64_t* counts, int64_t* n_entries, double* load,
                          int* phase) {
  if (q == nullptr || n_entries == nullptr || load == nullptr || phase == nullptr)
    return TSV_ERR_ARGUMENT;
  *n_entries = 0;
  *load = 0.0;
  const double eps = q->eps;
  // anchor: the bucket of earliest arrival over all pending tasks (any phase), then its
  // deepest task (node id breaks ties)
  int anchor_q = -1;
  double anchor_arr = 0.0;
  for (int qi = 0; qi < static_cast<int>(q->queries.size()); ++qi) {
    const Query& qu = q->queries[qi];
    bool any = false;
    double m = 0.0;
    for (int s : qu.tasks) {
      const Task& t = q->tasks[s];
      if (!t.pending()) continue;
      if (!any || t.arrival < m) m = t.arrival;
      any = true;
    }
    if (!any) continue;
    if (anchor_q < 0 || m < anchor_arr ||
        (m == anchor_arr && qu.id < q->queries[anchor_q].id)) {
      anchor_q = qi;
      anchor_arr = m;
    }
  }
  if (anchor_q < 0) return TSV_OK;
  int anchor = -1;
  for (int s : q->queries[anchor_q].tasks) {
    const Task& t = q->tasks[s];
    if (!t.pending()) continue;
    if (anchor < 0) {
      anchor = s;
      continue;
    }
    const Task& a = q->tasks[anchor];
    if (t.depth > a.depth || (t.depth == a.depth && t.node_id < a.node_id)) anchor = s;
  }
  const int ph = q->tasks[anchor].phase;
  *phase = ph;
  for (const Query& qu : q->queries)
    for (int s : qu.tasks) q->tasks[s].scratch_next = q->tasks[s].next;
  auto& entries = q->entries;
  entries.clear();
  double used = 0.0;
  while (used < max_slots - eps) {
    auto& buckets = q->buckets;
    buckets.clear();
    for (int qi = 0; qi < static_cast<int>(q->queries.size()); ++qi) {
      bool any = false;
      double m = 0.0;
      for (int s : q->queries[qi].tasks) {
        const Task& t = q->tasks[s];
        if (t.phase != ph || static_cast<int64_t>(t.loads.size()) <= t.scratch_next) continue;
        if (!any || t.arrival < m) m = t.arrival;
        any = true;
      }
      if (any) buckets.push_back({qi, m});
    }
    if (buckets.empty()) break;
    std::sort(buckets.begin(), buckets.end(),
              [q](const Bucket& a, const Bucket& b) { return bucket_before(q, a, b); });
    bool progressed = false;
    for (const Bucket& b : buckets) {
      if (max_slots - used <= eps) break;
      // the bucket's rows: this phase, pending at the start of the pass (bucket membership is
      // fixed per pass, as in the mirror)
      auto& cands = q->cands;
      cands.clear();
      int deepest = 0;
      bool first = true;
      for (int s : q->queries[b.query].tasks) {
        const Task& t = q->tasks[s];
        if (t.phase != ph || static_cast<int64_t>(t.loads.size()) <= t.scratch_next) continue;
        if (first || t.depth > deepest) deepest = t.depth;
        first = false;
      }
      for (int s : q->queries[b.query].tasks) {
        const Task& t = q->tasks[s];
        if (t.phase != ph || static_cast<int64_t>(t.loads.size()) <= t.scratch_next) continue;
        if (t.depth == deepest) cands.push_back(s);
      }
      std::sort(cands.begin(), cands.end(),
                [q](int x, int y) { return q->tasks[x].node_id < q->tasks[y].node_id; });
      for (int s : cands) {
        if (max_slots - used <= eps) break;
        Task& t = q->tasks[s];
        double acc = 0.0;
        const int64_t n = fill_at(t.loads, t.scratch_next, used, max_slots, !entries.empty(),
                                  eps, &acc);
        if (n) {
          entries.emplace_back(s, n);
          used += acc;
          t.scratch_next += n;
          progressed = true;
        }
      }
    }
    if (!progressed) break;
  }
  *load = used;
  // merge per task, first appearance order (_merge_plan_entries)
  int64_t m = 0;
  for (size_t i = 0; i < entries.size(); ++i) {
    bool seen = false;
    for (size_t j = 0; j < i; ++j)
      if (entries[j].first == entries[i].first) {
        seen = true;
        break;
      }
    if (!seen) ++m;
  }
  *n_entries = m;
  if (m > cap_entries) return TSV_ERR_CAPACITY;
  int64_t w = 0;
  for (size_t i = 0; i < entries.size(); ++i) {
    int64_t j = 0;
    for (; j < w; ++j)
      if (handles[j] == q->tasks[entries[i].first].handle) break;
    if (j < w) {
      counts[j] += entries[i].second;
    } else {
      handles[w] = q->tasks[entries[i].first].handle;
      counts[w] = entries[i].second;
      ++w;
    }
  }
  return TSV_OK;
}

// A dispatched batch: the tasks' next unconsumed requests advance by the counts; tasks left
// with nothing pending leave the queue.
TSV_API int tsv_topo_commit(tsv_topo_queue* q, const int64_t* handles, const int64_t* counts,
                            int64_t n) {
  if (q == nullptr || n < 0 || (n > 0 && (handles == nullptr || counts == nullptr)))
    return TSV_ERR_ARGUMENT;
  for (int64_t i = 0; i < n; ++i) {
    auto it = q->slot_of.find(handles[i]);
    if (it == q->slot_of.end()) return TSV_ERR_ARGUMENT;
    Task& t = q->tasks[it->second];
    t.next += counts[i];
    if (!t.pending()) drop_task(q, it->second);
  }
  return TSV_OK;
}

}  // extern "C"
