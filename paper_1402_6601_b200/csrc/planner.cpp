// Bit-exact native planner: the reference's discrete-event engine
// (/root/reference/pkg/src/hetsim/sim.py:97-385) driving its HEFT and DADA
// strategies (sched.py:90-412), replayed in virtual time with noise = 0.
//
// Everything that feeds a decision is reproduced with CPython 3.12 float
// semantics: IEEE double, no FMA contraction (-ffp-contract=off), builtin
// sum() emulated as Neumaier compensated summation (Appendix A.17 of
// SURVEY.md), Python min/max/sort tie-breaking (first of equal keys, stable
// sorts on the same key tuples), the (time, seq) event-heap order and the
// exact order of dict/list appends.  Residency sets are node bitmasks
// (k <= 62 GPUs).
//
// On top of the reference semantics the planner records the executable plan
// (dispatch order, transfer jobs with the version they move and where that
// version came from) exactly as paper_1402_6601_b200/sim.py does.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <limits>
#include <queue>
#include <string>
#include <vector>

#include "../../include/hetgpu.h"

namespace hg {
void set_error(const char* fmt, ...);
}

namespace {

using hg::set_error;
typedef uint64_t NodeSet;
constexpr int HOST = 0;

inline bool has(NodeSet s, int n) { return (s >> n) & 1ull; }
inline int lowest(NodeSet s) { return __builtin_ctzll(s); }

// CPython 3.12 builtin sum() over floats (Neumaier), starting from int 0.
struct PySum {
  double f = 0.0, c = 0.0;
  bool any = false;
  void add(double x) {
    if (!any) {  // 0 + x1 -> x1 exactly (int + float)
      f = 0 + x;
      any = true;
      return;
    }
    double t = f + x;
    if (std::fabs(f) >= std::fabs(x)) c += (f - t) + x;
    else c += (x - t) + f;
    f = t;
  }
  double value() const {
    if (!any) return 0.0;
    double r = f;
    if (c != 0.0 && std::isfinite(c)) r += c;
    return r;
  }
};

struct Hop {
  int src, dst;
  double bw, lat;
  int sw[2], nsw;
  int ep[2], nep;
};

struct Route {
  Hop h[2];
  int n = 0;
};

struct Platform {
  int m, k, n_workers, n_cpu, n_switches, slots;  // slots < 0: unlimited
  double bw, lat;
  bool p2p;
  int link_switch(int node) const { return (node - 1) % n_switches; }
  Hop host_leg(int src, int dst) const {
    Hop h{};
    h.src = src;
    h.dst = dst;
    h.bw = bw;
    h.lat = lat;
    int dev = src == HOST ? dst : src;
    h.sw[0] = link_switch(dev);
    h.nsw = 1;
    h.ep[0] = dev;
    h.nep = 1;
    return h;
  }
  Route route(int src, int dst) const {
    Route r;
    if (src == dst) return r;
    if (src == HOST || dst == HOST) {
      r.h[0] = host_leg(src, dst);
      r.n = 1;
      return r;
    }
    if (p2p) {
      Hop h{};
      h.src = src;
      h.dst = dst;
      h.bw = std::min(bw, bw);
      h.lat = lat + lat;
      int a = link_switch(src), b = link_switch(dst);
      if (a == b) {
        h.sw[0] = a;
        h.nsw = 1;
      } else {
        h.sw[0] = std::min(a, b);
        h.sw[1] = std::max(a, b);
        h.nsw = 2;
      }
      h.ep[0] = src;
      h.ep[1] = dst;
      h.nep = 2;
      r.h[0] = h;
      r.n = 1;
      return r;
    }
    r.h[0] = host_leg(src, HOST);
    r.h[1] = host_leg(HOST, dst);
    r.n = 2;
    return r;
  }
  // platform.py:119-123
  double raw(int64_t nbytes, int src, int dst) const {
    Route r = route(src, dst);
    PySum s;
    for (int i = 0; i < r.n; ++i) s.add(r.h[i].lat + double(nbytes) / r.h[i].bw);
    return s.value();
  }
  bool is_cpu(int w) const { return w < n_cpu; }
  int mem(int w) const { return w < n_cpu ? HOST : (w - n_cpu) + 1; }
};

struct Model {
  int n_kinds;
  std::vector<double> fb[2];
  std::vector<int64_t> cnt[2];
  std::vector<double> mean[2];
  int64_t threshold;
  bool predict(int kind, int cls, double* out) const {
    if (cnt[cls][kind] >= 0 && cnt[cls][kind] >= threshold) {
      *out = mean[cls][kind];
      return true;
    }
    double v = fb[cls][kind];
    if (std::isnan(v)) return false;
    *out = v;
    return true;
  }
  void record(int kind, int cls, double d) {
    if (cnt[cls][kind] < 0) {
      cnt[cls][kind] = 0;
      mean[cls][kind] = 0.0;
    }
    cnt[cls][kind] += 1;
    mean[cls][kind] += (d - mean[cls][kind]) / double(cnt[cls][kind]);
  }
};

struct Graph {
  int n, nb;
  const int32_t* kind;
  const double* flops;
  const int64_t* ap;
  const int32_t* ab;
  const int8_t* am;
  const int64_t* sp;
  const int32_t* su;
  const int64_t* bytes;
  bool reads(int64_t a) const { return am[a] != HG_ACCESS_W; }
  bool writes(int64_t a) const { return am[a] != HG_ACCESS_R; }
};

struct View {
  int id;
  double p_cpu, p_gpu, speedup;
  bool has_tr = false;
  std::vector<double> tr;   // per node
  std::vector<double> aff;  // per node
};

struct Job {
  int block;
  int64_t nbytes;
  Route route;
  int leg = 0;
  int dest;
  std::vector<int> waiters;
  int requester;
  std::vector<int> riders;
  int src, version, src_job = -1, stage_job = -1, req_task;
};

struct Event {
  double t;
  int64_t seq;
  int kind;  // 0 task end (payload worker), 1 transfer end (payload job)
  int payload;
  bool operator>(const Event& o) const { return t > o.t || (t == o.t && seq > o.seq); }
};

struct Failure {
  int code;
};

class Planner {
 public:
  Planner(const Graph& g, const Platform& p, const Model& m, const hg_sched_desc& s)
      : G(g), P(p), M(m), S(s) {}

  void run(hg_plan_out* out);

 private:
  const Graph& G;
  const Platform& P;
  Model M;
  hg_sched_desc S;
  // engine state
  std::vector<std::deque<int>> queues;
  std::vector<int> run_task;
  std::vector<double> run_start, run_dur;
  std::vector<int> wait_task, wait_pending;
  std::vector<double> busy, ready_at, last_completion;
  std::vector<NodeSet> res;
  std::vector<int> preds_left;
  std::priority_queue<Event, std::vector<Event>, std::greater<Event>> heap;
  int64_t seq = 0;
  int ndone = 0;
  std::vector<int> sched_worker;
  std::vector<double> sched_start, sched_end;
  std::vector<int> inflight;  // block*(k+1)+node -> job or -1
  std::vector<int> staging;   // block -> job or -1
  std::vector<double> link_free;
  std::vector<std::vector<double>> sw_busy;  // min-heaps
  int64_t b_h2d = 0, b_d2h = 0, b_d2d = 0;
  // plan recording
  std::vector<int> version;
  std::vector<int> arrived;  // block*(k+1)+node -> job
  std::vector<Job> jobs;
  std::vector<std::vector<int>> waits;
  std::vector<int> dispatch_seq;
  int n_act = 0, n_fallback = 0;
  // scratch for the overlay
  std::vector<NodeSet> ov_delta;
  std::vector<char> ov_set;
  std::vector<int> ov_touched;
  std::vector<char> placed_scratch;

  int nn() const { return P.k + 1; }
  double predict(int kind, int cls) {
    double v;
    if (!M.predict(kind, cls, &v)) {
      set_error("uncalibrated kind %d on %s", kind, cls ? "GPU" : "CPU");
      throw Failure{HG_EMODEL};
    }
    return v;
  }
  double true_exec(int kind, int cls) {
    double v = M.fb[cls][kind];
    if (std::isnan(v)) {
      set_error("no ground-truth timing for kind %d on %s", kind, cls ? "GPU" : "CPU");
      throw Failure{HG_EMODEL};
    }
    return v;
  }
  int cls_of(int w) const { return P.is_cpu(w) ? 0 : 1; }

  // perfmodel.py:84-103 over an arbitrary residency lookup
  template <class Res>
  double predict_transfer(int t, int node, const Res& r) {
    double total = 0.0;
    for (int64_t a = G.ap[t]; a < G.ap[t + 1]; ++a) {
      if (!G.reads(a)) continue;
      NodeSet h = r(G.ab[a]);
      if (has(h, node)) continue;
      if (!h) {
        set_error("data block %d has no valid copy anywhere", G.ab[a]);
        throw Failure{HG_EINVAL};
      }
      int src = has(h, HOST) ? HOST : lowest(h);
      total += P.raw(G.bytes[G.ab[a]], src, node);
    }
    return total;
  }

  void post(double t, int kind, int payload) { heap.push(Event{t, seq++, kind, payload}); }
  bool free_w(int w) const { return run_task[w] < 0 && wait_task[w] < 0; }

  // -- schedulers ----------------------------------------------------------
  std::vector<View> make_views(const std::vector<int>& ready, bool with_tr, bool with_aff) {
    std::vector<View> vs;
    vs.reserve(ready.size());
    auto base = [&](int b) { return res[b]; };
    for (int tid : ready) {
      View v;
      v.id = tid;
      v.p_cpu = predict(G.kind[tid], 0);
      v.p_gpu = predict(G.kind[tid], 1);
      v.speedup = v.p_cpu / v.p_gpu;
      if (with_tr) {
        v.has_tr = true;
        v.tr.resize(nn());
        for (int node = 0; node < nn(); ++node) v.tr[node] = predict_transfer(tid, node, base);
      }
      if (with_aff) {
        v.aff.assign(nn(), 0.0);
        for (int64_t a = G.ap[tid]; a < G.ap[tid + 1]; ++a) {
          if (!G.writes(a)) continue;
          NodeSet h = res[G.ab[a]];
          for (int node = 1; node < nn(); ++node)
            if (has(h, node)) v.aff[node] += double(G.bytes[G.ab[a]]);
        }
      }
      vs.push_back(std::move(v));
    }
    return vs;
  }
  static void sort_views(std::vector<View*>& v) {
    std::stable_sort(v.begin(), v.end(), [](const View* a, const View* b) {
      double ka = -a->speedup, kb = -b->speedup;
      if (ka != kb) return ka < kb;
      return a->id < b->id;
    });
  }
  double exec_of(const View& v, int w) const { return P.is_cpu(w) ? v.p_cpu : v.p_gpu; }
  double charge(const View& v, int w) const {
    double p = exec_of(v, w);
    if (v.has_tr) p += v.tr[P.mem(w)];
    return p;
  }

  struct Asg {
    std::vector<std::vector<int>> order;  // per worker
    std::vector<double> added;
  };

  void heft(const std::vector<int>& ready, Asg& out) {
    std::vector<View> vs = make_views(ready, false, false);
    std::vector<View*> order;
    for (auto& v : vs) order.push_back(&v);
    sort_views(order);
    out.order.assign(P.n_workers, {});
    ov_touched.clear();
    auto ov = [&](int b) { return ov_set[b] ? ov_delta[b] : res[b]; };
    std::vector<double> tr(nn());
    for (View* v : order) {
      for (int node = 0; node < nn(); ++node) tr[node] = predict_transfer(v->id, node, ov);
      int best_w = -1;
      double best = std::numeric_limits<double>::infinity();
      for (int w = 0; w < P.n_workers; ++w) {
        double eft = ready_at[w] + tr[P.mem(w)] + (P.is_cpu(w) ? v->p_cpu : v->p_gpu);
        if (eft < best) {
          best = eft;
          best_w = w;
        }
      }
      if (best_w < 0) {
        set_error("heft: no finite finish time");
        throw Failure{HG_EINVAL};
      }
      ready_at[best_w] = best;
      out.order[best_w].push_back(v->id);
      const int node = P.mem(best_w);
      for (int64_t a = G.ap[v->id]; a < G.ap[v->id + 1]; ++a) {
        int b = G.ab[a];
        NodeSet cur = ov(b);
        NodeSet nxt;
        if (G.writes(a)) nxt = NodeSet(1) << node;
        else if (has(cur, node)) continue;
        else nxt = cur | (NodeSet(1) << node);
        if (!ov_set[b]) {
          ov_set[b] = 1;
          ov_touched.push_back(b);
        }
        ov_delta[b] = nxt;
      }
    }
    for (int b : ov_touched) ov_set[b] = 0;
  }

  // sched.py:229-298
  bool dual_assign(const std::vector<View*>& rest, double lam, std::vector<double>& loads,
                   std::vector<double>& added, std::vector<std::vector<int>>& order) {
    std::vector<View*> fgpu, fcpu, flex;
    for (View* v : rest) {
      bool bc = v->p_cpu > lam, bg = v->p_gpu > lam;
      if (bc && bg) return false;
      if (bc) fgpu.push_back(v);
      else if (bg) fcpu.push_back(v);
      else flex.push_back(v);
    }
    const int ncpu = P.n_cpu, nw = P.n_workers;
    const bool have_gpu = nw > ncpu, have_cpu = ncpu > 0;
    if (!fgpu.empty() && !have_gpu) return false;
    if (!fcpu.empty() && !have_cpu) return false;
    auto place = [&](View* v, int w) {
      double c = charge(*v, w);
      loads[w] += c;
      added[w] += c;
      order[w].push_back(v->id);
    };
    auto place_gpu = [&](View* v, bool must) {
      int best = -1;
      double bkey = 0.0;
      for (int w = ncpu; w < nw; ++w) {
        if (loads[w] > lam) continue;
        double key = loads[w] + charge(*v, w);
        if (best < 0 || key < bkey) {
          best = w;
          bkey = key;
        }
      }
      if (best < 0) {
        if (!must) return false;
        best = ncpu;
        for (int w = ncpu + 1; w < nw; ++w)
          if (loads[w] < loads[best]) best = w;
      }
      place(v, best);
      return true;
    };
    for (View* v : fgpu) place_gpu(v, true);
    std::vector<View*> cpu_stream = fcpu;
    for (View* v : flex)
      if (!place_gpu(v, !have_cpu)) cpu_stream.push_back(v);
    sort_views(cpu_stream);
    for (View* v : cpu_stream) {
      int best = 0;
      for (int w = 1; w < ncpu; ++w)
        if (loads[w] < loads[best]) best = w;
      place(v, best);
    }
    return true;
  }

  // sched.py:301-369; returns false when no guess was accepted
  bool dada(const std::vector<int>& ready, double now, Asg& out) {
    const bool with_aff = S.alpha > 0;
    std::vector<View> vs = make_views(ready, S.with_cp != 0, with_aff);
    std::vector<View*> views;
    for (auto& v : vs) views.push_back(&v);
    sort_views(views);
    const int nw = P.n_workers;
    std::vector<double> backlog(nw);
    for (int w = 0; w < nw; ++w) backlog[w] = std::max(ready_at[w] - now, 0.0);
    struct Cand {
      double negs;
      int tid, wid;
      View* v;
    };
    std::vector<Cand> cands;
    if (with_aff) {
      for (View* v : views) {
        double best_s = 0.0;
        int best_w = -1;
        for (int w = 0; w < nw; ++w) {
          double s = v->aff[P.mem(w)];
          if (s > best_s) {
            best_s = s;
            best_w = w;
          }
        }
        if (best_w >= 0) cands.push_back(Cand{-best_s, v->id, best_w, v});
      }
      std::stable_sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
        if (a.negs != b.negs) return a.negs < b.negs;
        if (a.tid != b.tid) return a.tid < b.tid;
        return a.wid < b.wid;
      });
    }
    const double thr = S.rho + S.alpha;
    PySum up;
    for (View* v : views) up.add(v->p_gpu > v->p_cpu ? v->p_gpu : v->p_cpu);  // Python max(a, b)
    double upper = up.value(), lower = 0.0;
    bool kept = false;
    std::vector<double> loads, added;
    std::vector<std::vector<int>> order;
    std::vector<char>& placed = placed_scratch;
    std::vector<int> placed_ids;
    std::vector<View*> rest;
    while (upper - lower > S.epsilon) {
      const double lam = (lower + upper) / 2.0;
      loads = backlog;
      added.assign(nw, 0.0);
      order.assign(nw, {});
      for (int t : placed_ids) placed[t] = 0;
      placed_ids.clear();
      if (S.alpha > 0.0 && !cands.empty()) {
        const double budget = S.alpha * lam;
        for (const Cand& c : cands) {
          if (added[c.wid] <= budget && exec_of(*c.v, c.wid) <= lam) {
            double ch = charge(*c.v, c.wid);
            loads[c.wid] += ch;
            added[c.wid] += ch;
            order[c.wid].push_back(c.tid);
            placed[c.tid] = 1;
            placed_ids.push_back(c.tid);
          }
        }
      }
      rest.clear();
      for (View* v : views)
        if (!placed[v->id]) rest.push_back(v);
      bool fits = dual_assign(rest, lam, loads, added, order);
      if (fits) {
        bool anyw = false;
        double span = 0.0;
        for (int w = 0; w < nw; ++w) {
          if (added[w] > 0.0) {
            if (!anyw || loads[w] > span) span = loads[w];
            anyw = true;
          }
        }
        if (!anyw) {
          set_error("dual_search: max() of an empty sequence (no positive charge)");
          throw Failure{HG_EINVAL};
        }
        if (span <= thr * lam) {
          upper = lam;
          out.order = order;
          out.added = added;
          kept = true;
          continue;
        }
      }
      lower = lam;
    }
    for (int t : placed_ids) placed[t] = 0;
    return kept;
  }

  void activate(std::vector<int> ready, double now) {
    // sim.py:192-203
    for (int w = 0; w < P.n_workers; ++w) {
      bool idle = free_w(w) && queues[w].empty();
      if (idle || ready_at[w] < now) ready_at[w] = now;
    }
    std::sort(ready.begin(), ready.end());
    if (ready.empty()) {
      set_error("empty activation batch");
      throw Failure{HG_EINVAL};
    }
    ++n_act;
    Asg asg;
    if (S.type == 1) {
      if (dada(ready, now, asg)) {
        for (int w = 0; w < P.n_workers; ++w)
          if (asg.added[w] > 0.0) ready_at[w] += asg.added[w];
      } else {
        ++n_fallback;
        heft(ready, asg);
      }
    } else {
      heft(ready, asg);
    }
    for (int w = 0; w < P.n_workers; ++w)
      for (int t : asg.order[w]) queues[w].push_back(t);
  }

  void dispatch_round(double now) {
    bool moved = true;
    while (moved) {
      moved = false;
      for (int w = 0; w < P.n_workers; ++w) {
        if (free_w(w) && !queues[w].empty()) {
          int t = queues[w].front();
          queues[w].pop_front();
          dispatch(w, t, now);
          moved = true;
        }
      }
    }
  }

  int new_job(int block, int src, int dest, int w, int tid) {
    Job j;
    j.block = block;
    j.nbytes = G.bytes[block];
    j.route = P.route(src, dest);
    j.dest = dest;
    j.requester = w;
    j.src = src;
    j.version = version[block];
    j.src_job = arrived[size_t(block) * nn() + src];
    j.req_task = tid;
    jobs.push_back(std::move(j));
    return int(jobs.size()) - 1;
  }

  void account(const Job& j) {
    for (int i = 0; i < j.route.n; ++i) {
      const Hop& h = j.route.h[i];
      if (h.src == HOST) b_h2d += j.nbytes;
      else if (h.dst == HOST) b_d2h += j.nbytes;
      else b_d2d += j.nbytes;
    }
  }

  void dispatch(int w, int tid, double now) {
    const int node = P.mem(w);
    dispatch_seq.push_back(tid);
    int pending = 0;
    for (int64_t a = G.ap[tid]; a < G.ap[tid + 1]; ++a) {
      if (!G.reads(a)) continue;
      const int b = G.ab[a];
      NodeSet h = res[b];
      if (has(h, node)) continue;
      const size_t key = size_t(b) * nn() + node;
      int jid = inflight[key];
      if (jid < 0) {
        if (!h) {
          set_error("data block %d lost all copies", b);
          throw Failure{HG_EINVAL};
        }
        int src = has(h, HOST) ? HOST : lowest(h);
        int stage = src != HOST ? staging[b] : -1;
        if (stage >= 0) {
          jid = new_job(b, HOST, node, w, tid);
          jobs[jid].stage_job = stage;
          jobs[stage].riders.push_back(jid);
        } else {
          jid = new_job(b, src, node, w, tid);
          if (jobs[jid].route.n > 0 && jobs[jid].route.h[0].dst == HOST) staging[b] = jid;
          issue(jid, now);
        }
        inflight[key] = jid;
        account(jobs[jid]);
      }
      jobs[jid].waiters.push_back(w);
      waits[tid].push_back(jid);
      ++pending;
    }
    if (pending) {
      wait_task[w] = tid;
      wait_pending[w] = pending;
    } else {
      start(w, tid, now);
    }
  }

  double admit(int sw, double t) {
    std::vector<double>& hb = sw_busy[sw];
    auto cmp = std::greater<double>();
    while (true) {
      while (!hb.empty() && hb.front() <= t) {
        std::pop_heap(hb.begin(), hb.end(), cmp);
        hb.pop_back();
      }
      if (int(hb.size()) < P.slots) return t;
      t = hb.front();
    }
  }

  void issue(int jid, double now) {
    Job& j = jobs[jid];
    const Hop& h = j.route.h[j.leg];
    double t0 = now;
    for (int e = 0; e < h.nep; ++e)
      if (link_free[h.ep[e]] > t0) t0 = link_free[h.ep[e]];
    if (P.slots >= 0)
      for (int s = 0; s < h.nsw; ++s) t0 = admit(h.sw[s], t0);
    const double t1 = t0 + h.lat + double(j.nbytes) / h.bw;
    for (int e = 0; e < h.nep; ++e) link_free[h.ep[e]] = t1;
    if (P.slots >= 0)
      for (int s = 0; s < h.nsw; ++s) {
        sw_busy[h.sw[s]].push_back(t1);
        std::push_heap(sw_busy[h.sw[s]].begin(), sw_busy[h.sw[s]].end(), std::greater<double>());
      }
    post(t1, 1, jid);
  }

  void transfer_end(int jid, double now) {
    Job& j = jobs[jid];
    const Hop& h = j.route.h[j.leg];
    if (h.dst == HOST) {
      res[j.block] |= NodeSet(1);
      arrived[size_t(j.block) * nn() + HOST] = jid;
      if (staging[j.block] == jid) staging[j.block] = -1;
      std::vector<int> riders;
      riders.swap(jobs[jid].riders);
      for (int r : riders) {
        if (jobs[r].route.n > 0) issue(r, now);
        else finish(r, now);
      }
      Job& jj = jobs[jid];
      if (jj.leg + 1 < jj.route.n) {
        jj.leg += 1;
        issue(jid, now);
        return;
      }
    }
    finish(jid, now);
  }

  void finish(int jid, double now) {
    Job& j = jobs[jid];
    res[j.block] |= NodeSet(1) << j.dest;
    arrived[size_t(j.block) * nn() + j.dest] = jid;
    inflight[size_t(j.block) * nn() + j.dest] = -1;
    std::vector<int> ws = j.waiters;
    for (int w : ws) {
      wait_pending[w] -= 1;
      if (wait_pending[w] == 0 && wait_task[w] >= 0) {
        int t = wait_task[w];
        wait_task[w] = -1;
        start(w, t, now);
      }
    }
  }

  void start(int w, int tid, double now) {
    double dur = true_exec(G.kind[tid], cls_of(w)) * 1.0;
    run_task[w] = tid;
    run_start[w] = now;
    run_dur[w] = dur;
    busy[w] += dur;
    post(now + dur, 0, w);
  }

  void task_end(int w, double now) {
    const int tid = run_task[w];
    const double began = run_start[w], dur = run_dur[w];
    run_task[w] = -1;
    sched_worker[tid] = w;
    sched_start[tid] = began;
    sched_end[tid] = now;
    const int node = P.mem(w);
    for (int64_t a = G.ap[tid]; a < G.ap[tid + 1]; ++a) {
      if (!G.writes(a)) continue;
      const int b = G.ab[a];
      res[b] = NodeSet(1) << node;
      version[b] = tid;
      for (int nd = 0; nd < nn(); ++nd) arrived[size_t(b) * nn() + nd] = -1;
    }
    M.record(G.kind[tid], cls_of(w), dur);
    last_completion[w] = now;
    if (ready_at[w] < now) ready_at[w] = now;
    ++ndone;
    std::vector<int> ready;
    for (int64_t s = G.sp[tid]; s < G.sp[tid + 1]; ++s) {
      int sc = G.su[s];
      if (--preds_left[sc] < 0) {
        set_error("negative predecessor count for task %d", sc);
        throw Failure{HG_EINVAL};
      }
      if (preds_left[sc] == 0) ready.push_back(sc);
    }
    if (!ready.empty()) activate(ready, now);
    dispatch_round(now);
  }
};

template <class T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(std::max<size_t>(v.size(), 1) * sizeof(T)));
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

void Planner::run(hg_plan_out* out) {
  const int nw = P.n_workers;
  queues.assign(nw, {});
  run_task.assign(nw, -1);
  run_start.assign(nw, 0.0);
  run_dur.assign(nw, 0.0);
  wait_task.assign(nw, -1);
  wait_pending.assign(nw, 0);
  busy.assign(nw, 0.0);
  ready_at.assign(nw, 0.0);
  last_completion.assign(nw, 0.0);
  res.assign(G.nb, NodeSet(1));
  preds_left.assign(G.n, 0);
  for (int t = 0; t < G.n; ++t)
    for (int64_t s = G.sp[t]; s < G.sp[t + 1]; ++s) preds_left[G.su[s]]++;
  sched_worker.assign(G.n, -1);
  sched_start.assign(G.n, 0.0);
  sched_end.assign(G.n, 0.0);
  inflight.assign(size_t(G.nb) * nn(), -1);
  staging.assign(G.nb, -1);
  link_free.assign(nn(), 0.0);
  sw_busy.assign(std::max(1, P.n_switches), {});
  version.assign(G.nb, -1);
  arrived.assign(size_t(G.nb) * nn(), -1);
  waits.assign(G.n, {});
  ov_delta.assign(G.nb, 0);
  ov_set.assign(G.nb, 0);
  placed_scratch.assign(G.n, 0);

  if (G.n) {
    std::vector<int> init;
    for (int t = 0; t < G.n; ++t)
      if (preds_left[t] == 0) init.push_back(t);
    activate(init, 0.0);
    dispatch_round(0.0);
  }
  while (!heap.empty()) {
    Event e = heap.top();
    heap.pop();
    if (e.kind == 0) task_end(e.payload, e.t);
    else transfer_end(e.payload, e.t);
  }
  if (ndone != G.n) {
    set_error("simulation deadlocked: %d of %d tasks never ran", G.n - ndone, G.n);
    throw Failure{HG_EDEADLOCK};
  }
  double span = 0.0;
  for (int t = 0; t < G.n; ++t)
    if (t == 0 || sched_end[t] > span) span = sched_end[t];
  PySum fl;
  for (int t = 0; t < G.n; ++t) fl.add(G.flops[t]);
  const double work = fl.value();

  out->worker = dup(sched_worker);
  out->start = dup(sched_start);
  out->end = dup(sched_end);
  out->dispatch = dup(dispatch_seq);
  std::vector<int64_t> wp(G.n + 1, 0);
  std::vector<int32_t> wj;
  for (int t = 0; t < G.n; ++t) {
    for (int j : waits[t]) wj.push_back(j);
    wp[t + 1] = int64_t(wj.size());
  }
  out->wait_ptr = dup(wp);
  out->wait_job = dup(wj);
  const int nj = int(jobs.size());
  out->n_jobs = nj;
  std::vector<int32_t> c_block(nj), c_src(nj), c_dst(nj), c_ver(nj), c_sj(nj), c_st(nj), c_req(nj);
  std::vector<int64_t> c_bytes(nj);
  for (int j = 0; j < nj; ++j) {
    c_block[j] = jobs[j].block;
    c_src[j] = jobs[j].src;
    c_dst[j] = jobs[j].dest;
    c_ver[j] = jobs[j].version;
    c_sj[j] = jobs[j].src_job;
    c_st[j] = jobs[j].stage_job;
    c_req[j] = jobs[j].req_task;
    c_bytes[j] = jobs[j].nbytes;
  }
  out->job_block = dup(c_block);
  out->job_src = dup(c_src);
  out->job_dst = dup(c_dst);
  out->job_version = dup(c_ver);
  out->job_src_job = dup(c_sj);
  out->job_stage_job = dup(c_st);
  out->job_requester = dup(c_req);
  out->job_bytes = dup(c_bytes);
  out->bytes_h2d = b_h2d;
  out->bytes_d2h = b_d2h;
  out->bytes_d2d = b_d2d;
  out->makespan = span;
  out->gflops = span > 0 ? work / span / 1e9 : 0.0;
  out->busy = dup(busy);
  out->n_workers = nw;
  out->n_activations = n_act;
  out->n_fallbacks = n_fallback;
}

}  // namespace

extern "C" int hg_plan_build(const hg_graph_desc* g, const hg_platform_desc* p, const hg_model_desc* m,
                             const hg_sched_desc* s, hg_plan_out* out) {
  auto t0 = std::chrono::steady_clock::now();
  if (!g || !p || !m || !s || !out) {
    set_error("hg_plan_build: null argument");
    return HG_EINVAL;
  }
  std::memset(out, 0, sizeof(*out));
  if (p->k < 0 || p->k > 62 || p->m < p->k || p->m < 1) {
    set_error("hg_plan_build: unsupported platform m=%d k=%d (k <= 62)", p->m, p->k);
    return HG_EINVAL;
  }
  if (s->type != 0 && s->type != 1) {
    set_error("hg_plan_build: scheduler type %d", s->type);
    return HG_EINVAL;
  }
  Graph G{g->n_tasks, g->n_blocks, g->task_kind, g->task_flops, g->acc_ptr, g->acc_block,
          g->acc_mode, g->succ_ptr, g->succ, g->block_bytes};
  Platform P{};
  P.m = p->m;
  P.k = p->k;
  P.n_workers = p->m;
  P.n_cpu = p->m - p->k;
  P.n_switches = std::max(1, p->n_switches);
  P.slots = p->switch_slots;
  P.bw = p->link_bandwidth;
  P.lat = p->link_latency;
  P.p2p = p->p2p != 0;
  Model M;
  M.n_kinds = m->n_kinds;
  M.threshold = m->sample_threshold;
  for (int c = 0; c < 2; ++c) {
    const double* fb = c ? m->fallback_gpu : m->fallback_cpu;
    const int64_t* cn = c ? m->count_gpu : m->count_cpu;
    const double* mn = c ? m->mean_gpu : m->mean_cpu;
    M.fb[c].assign(fb, fb + m->n_kinds);
    M.cnt[c].assign(cn, cn + m->n_kinds);
    M.mean[c].assign(mn, mn + m->n_kinds);
  }
  try {
    Planner pl(G, P, M, *s);
    pl.run(out);
  } catch (const Failure& f) {
    hg_plan_free(out);
    return f.code;
  } catch (const std::bad_alloc&) {
    hg_plan_free(out);
    set_error("hg_plan_build: out of memory");
    return HG_EINVAL;
  }
  out->plan_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return HG_OK;
}

extern "C" void hg_plan_free(hg_plan_out* out) {
  if (!out) return;
  void* ptrs[] = {out->worker, out->start, out->end, out->dispatch, out->wait_ptr, out->wait_job,
                  out->job_block, out->job_src, out->job_dst, out->job_version, out->job_src_job,
                  out->job_stage_job, out->job_requester, out->job_bytes, out->busy};
  for (void* q : ptrs) std::free(q);
  std::memset(out, 0, sizeof(*out));
}

extern "C" double hg_pysum(const double* x, int64_t n) {
  PySum s;
  for (int64_t i = 0; i < n; ++i) s.add(x[i]);
  return s.value();
}
