// TEST INFRASTRUCTURE ONLY — a flat C API over the reference's own hot-path
// code (/root/reference/proj/src, compiled in place by oracle/Makefile into
// oracle/_ref/libdearsim_ref.so). It exists so Python tests and bench.py's
// reference arm can call the UNMODIFIED reference functions:
//   build_fusion_plan / per_layer_plan   (fusion.cpp:29-70)
//   preset_model                          (model.cpp:111-168)
//   chunk_ranges                          (collective.cpp:39-57)
//   ring_reduce_scatter/ring_all_gather   (collective.cpp:59-152)
//   all_reduce_sum / all_reduce_average   (collective.cpp:154-164)
//   sgd_step                              (collective.cpp:166-194)
//   build_graph + simulate                (task_graph.cpp:271, simulate.cpp:65)
// Nothing here is linked into or called by the product library.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "dearsim/analysis.hpp"
#include "dearsim/cost_model.hpp"
#include "dearsim/gp.hpp"
#include "dearsim/tuner.hpp"
#include "dearsim/collective.hpp"
#include "dearsim/fusion.hpp"
#include "dearsim/model.hpp"
#include "dearsim/simulate.hpp"
#include "dearsim/task_graph.hpp"

using namespace dearsim;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

ModelSpec model_from_counts(const int64_t* counts, int L, int bytes_per_elem,
                            const double* t_ff, const double* t_bp) {
  ModelSpec m;
  m.name = "capi";
  for (int i = 0; i < L; ++i) {
    LayerSpec l;
    l.index = i + 1;
    l.param_count = counts[i];
    l.bytes_per_element = bytes_per_elem;
    l.t_ff = t_ff ? t_ff[i] : 1.0;
    l.t_bp = t_bp ? t_bp[i] : 2.0;
    m.layers.push_back(l);
  }
  return m;
}

std::vector<Vector> unpack(int P, int64_t d, const double* in) {
  std::vector<Vector> v(static_cast<std::size_t>(P));
  for (int w = 0; w < P; ++w) {
    v[static_cast<std::size_t>(w)].resize(d);
    std::memcpy(v[static_cast<std::size_t>(w)].data(), in + static_cast<int64_t>(w) * d,
                sizeof(double) * static_cast<std::size_t>(d));
  }
  return v;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Uniform (imbalanced=0) or imbalanced preset; writes up to `cap` counts.
int ref_preset_params(const char* name, int imbalanced, int64_t* out, int cap) {
  try {
    const ModelSpec m = preset_model(
        name, 1.0, 2.0, imbalanced ? ParamProfile::Imbalanced : ParamProfile::Uniform);
    if (m.layer_count() > cap) throw std::invalid_argument("cap too small");
    for (int i = 0; i < m.layer_count(); ++i) out[i] = m.layers[static_cast<std::size_t>(i)].param_count;
    return m.layer_count();
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// buffer_bytes == 0 -> per_layer_plan. Returns the group count.
int ref_build_plan(const int64_t* counts, int L, int bytes_per_elem, int64_t buffer_bytes,
                   int32_t* low, int32_t* high) {
  try {
    const ModelSpec m = model_from_counts(counts, L, bytes_per_elem, nullptr, nullptr);
    const FusionPlan plan =
        buffer_bytes == 0 ? per_layer_plan(m) : build_fusion_plan(m, buffer_bytes);
    validate(plan, m);
    for (int g = 0; g < plan.group_count(); ++g) {
      low[g] = plan.groups[static_cast<std::size_t>(g)].low_layer;
      high[g] = plan.groups[static_cast<std::size_t>(g)].high_layer;
    }
    return plan.group_count();
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_chunk_ranges(int64_t d, int P, int64_t* begin, int64_t* end) {
  try {
    const auto r = chunk_ranges(d, P);
    for (int c = 0; c < P; ++c) {
      begin[c] = r[static_cast<std::size_t>(c)].begin;
      end[c] = r[static_cast<std::size_t>(c)].end;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The reference tests' input generator (test_collective.cpp:27-37): one
// mt19937_64(seed), U(-1,1) doubles, worker-major.
int ref_random_vectors(int P, int64_t d, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int64_t i = 0; i < static_cast<int64_t>(P) * d; ++i) out[i] = dist(rng);
  return 0;
}

// ring_reduce_scatter: chunk c written at its range [begin_c, end_c) of out
// (length d). Also returns the owner map check and round count via rounds.
int ref_ring_reduce_scatter(int P, int64_t d, const double* in, double* out, int* rounds) {
  try {
    const ReduceScatterResult rs = ring_reduce_scatter(unpack(P, d, in));
    for (int c = 0; c < P; ++c) {
      const ChunkRange& r = rs.ranges[static_cast<std::size_t>(c)];
      std::memcpy(out + r.begin, rs.chunks[static_cast<std::size_t>(c)].data(),
                  sizeof(double) * static_cast<std::size_t>(r.size()));
    }
    if (rounds) *rounds = rs.rounds;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// all_reduce_sum (average=0) or all_reduce_average (average=1); out is P x d.
int ref_all_reduce(int P, int64_t d, const double* in, double* out, int average) {
  try {
    const auto v = average ? all_reduce_average(unpack(P, d, in)) : all_reduce_sum(unpack(P, d, in));
    for (int w = 0; w < P; ++w)
      std::memcpy(out + static_cast<int64_t>(w) * d, v[static_cast<std::size_t>(w)].data(),
                  sizeof(double) * static_cast<std::size_t>(d));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// sgd_step on P replicas that all start from w_in; writes the P resulting
// weight vectors (P x d) to w_out.
int ref_sgd_step(int P, int64_t d, double lr, const double* w_in, const double* grads,
                 double* w_out) {
  try {
    Vector w(d);
    std::memcpy(w.data(), w_in, sizeof(double) * static_cast<std::size_t>(d));
    std::vector<SgdState> states(static_cast<std::size_t>(P), SgdState{w, lr});
    const auto next = sgd_step(states, unpack(P, d, grads));
    for (int k = 0; k < P; ++k)
      std::memcpy(w_out + static_cast<int64_t>(k) * d, next[static_cast<std::size_t>(k)].weights.data(),
                  sizeof(double) * static_cast<std::size_t>(d));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// sgd_step with caller-supplied (possibly divergent) replicas: P x d weights.
int ref_sgd_step_replicas(int P, int64_t d, double lr, const double* w_in, const double* grads,
                          double* w_out) {
  try {
    std::vector<SgdState> states(static_cast<std::size_t>(P));
    const auto ws = unpack(P, d, w_in);
    for (int k = 0; k < P; ++k) states[static_cast<std::size_t>(k)] = {ws[static_cast<std::size_t>(k)], lr};
    const auto next = sgd_step(states, unpack(P, d, grads));
    for (int k = 0; k < P; ++k)
      std::memcpy(w_out + static_cast<int64_t>(k) * d, next[static_cast<std::size_t>(k)].weights.data(),
                  sizeof(double) * static_cast<std::size_t>(d));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// build_graph + simulate; returns a malloc'ed JSON document (free with
// ref_free) listing tasks (id, label, kind, subject, group_subject,
// issue_order, duration, deps, resource, start, end) and the makespan.
// policy: 0 WFBP, 1 WFBP_FUSED, 2 PRIORITY_PARTITION, 3 DEAR, 4 DEAR_FUSED.
char* ref_simulate_json_ex(const int64_t* counts, int L, const double* t_ff, const double* t_bp,
                           int policy, int64_t fusion_buffer_bytes, int group_dependency,
                           int workers, double alpha, double beta, int64_t partition_bytes,
                           int negotiation_rounds, int negotiation_floating);

char* ref_simulate_json(const int64_t* counts, int L, const double* t_ff, const double* t_bp,
                        int policy, int64_t fusion_buffer_bytes, int group_dependency,
                        int workers, double alpha, double beta) {
  return ref_simulate_json_ex(counts, L, t_ff, t_bp, policy, fusion_buffer_bytes,
                              group_dependency, workers, alpha, beta, 0, 1, 0);
}

// Same, with PolicySpec's PRIORITY_PARTITION fields (policy.hpp:36-45).
char* ref_simulate_json_ex(const int64_t* counts, int L, const double* t_ff, const double* t_bp,
                           int policy, int64_t fusion_buffer_bytes, int group_dependency,
                           int workers, double alpha, double beta, int64_t partition_bytes,
                           int negotiation_rounds, int negotiation_floating) {
  try {
    const ModelSpec m = model_from_counts(counts, L, 4, t_ff, t_bp);
    PolicySpec p;
    p.kind = static_cast<PolicyKind>(policy);
    p.fusion_buffer_bytes = fusion_buffer_bytes;
    p.dear_group_dependency = group_dependency != 0;
    p.partition_bytes = partition_bytes;
    p.negotiation_rounds = negotiation_rounds;
    p.negotiation_floating = negotiation_floating != 0;
    const ClusterSpec c{"capi", workers, alpha, beta};
    const TaskGraph g = build_graph(m, p, c);
    const Timeline tl = simulate(g);
    std::vector<const TimelineEvent*> by(g.tasks.size());
    for (const auto& ev : tl.events) by[static_cast<std::size_t>(ev.task_id)] = &ev;
    std::string os;
    char num[64];
    auto put = [&](double x) {
      std::snprintf(num, sizeof num, "%.17g", x);
      os += num;
    };
    auto puti = [&](long long x) { os += std::to_string(x); };
    os += "{\"iteration_seconds\":";
    put(tl.iteration_seconds);
    os += ",\"tasks\":[";
    for (std::size_t i = 0; i < g.tasks.size(); ++i) {
      const Task& t = g.tasks[i];
      if (i) os += ",";
      os += "{\"id\":";
      puti(t.id);
      os += ",\"label\":\"" + task_label(t) + "\",\"kind\":\"" + to_string(t.kind) +
            "\",\"subject\":";
      puti(t.subject);
      os += std::string(",\"group_subject\":") + (t.group_subject ? "true" : "false");
      os += ",\"issue_order\":";
      puti(t.issue_order);
      os += ",\"duration\":";
      put(t.duration);
      os += ",\"resource\":";
      puti(static_cast<int>(resource_of(t.kind)));
      os += ",\"start\":";
      put(by[i]->start);
      os += ",\"end\":";
      put(by[i]->end);
      os += ",\"part\":";
      puti(t.part);
      os += ",\"release\":";
      put(t.release_delay);
      os += ",\"deps\":[";
      for (std::size_t k = 0; k < t.deps.size(); ++k) {
        if (k) os += ",";
        puti(t.deps[k]);
      }
      os += "]}";
    }
    os += "],\"groups\":[";
    if (g.plan) {
      for (std::size_t k = 0; k < g.plan->groups.size(); ++k) {
        if (k) os += ",";
        os += "[" + std::to_string(g.plan->groups[k].low_layer) + "," +
              std::to_string(g.plan->groups[k].high_layer) + "]";
      }
    }
    os += "]}";
    const std::string& s = os;
    char* out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(out, s.c_str(), s.size() + 1);
    return out;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_free(void* p) { std::free(p); }

// calibrate_alpha_beta (cost_model.cpp:79-133) on (bytes, seconds) pairs.
int ref_calibrate(const double* bytes, const double* seconds, int n, int workers, double* alpha,
                  double* beta, int* clamped) {
  try {
    std::vector<std::pair<double, double>> m;
    for (int i = 0; i < n; ++i) m.push_back({bytes[i], seconds[i]});
    const Calibration c = calibrate_alpha_beta(m, workers);
    *alpha = c.alpha;
    *beta = c.beta;
    *clamped = c.clamped ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// reduce_scatter_time / all_reduce_time (cost_model.cpp:34-48);
// theoretical_times (analysis.cpp:50-60); max_speedup (:34-48).
int ref_costs(double bytes, int workers, double alpha, double beta, double* rs, double* ar) {
  try {
    const ClusterSpec c{"capi", workers, alpha, beta};
    *rs = reduce_scatter_time(bytes, c);
    *ar = all_reduce_time(bytes, c);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// gp_fit + predict (gp.cpp:46-158) and expected_improvement (:172-183) on
// caller observations; defaults of GpHyperParams / TunerConfig bounds.
int ref_gp(const double* xb, const double* ty, int n, const double* q, int m, double* mean,
           double* var, double* ei) {
  try {
    std::vector<Observation> obs;
    for (int i = 0; i < n; ++i) obs.push_back({xb[i], ty[i], 1});
    const GpPosterior gp = gp_fit(obs, GpHyperParams{}, 1e6, 1e8);
    for (int j = 0; j < m; ++j) {
      const auto p = gp.predict(q[j]);
      mean[j] = p.mean;
      var[j] = p.variance;
      ei[j] = expected_improvement(gp, q[j], gp.best_throughput(), 0.1);
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// tune (tuner.cpp:176-203) on the analytic objective
// peak - ((x/1e6 - opt_mb) / width_mb)^2; writes the trial trace.
int ref_tune_quadratic(double opt_mb, double width_mb, double peak, int max_trials,
                       int measure_steps, double* buffers, double* thr, int* n) {
  try {
    TunerConfig cfg;
    cfg.max_trials = max_trials;
    cfg.measure_steps = measure_steps;
    auto obj = [&](double x) {
      const double r = (x / 1e6 - opt_mb) / width_mb;
      return peak - r * r;
    };
    const TuneResult res = tune(obj, cfg);
    *n = static_cast<int>(res.trace.size());
    for (size_t i = 0; i < res.trace.size(); ++i) {
      buffers[i] = res.trace[i].buffer_bytes;
      thr[i] = res.trace[i].throughput;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_theory(double t_ff, double t_bp, double t_rs, double t_ag, int workers, double* dear,
               double* baseline, double* smax) {
  try {
    const TheoreticalTimes t = theoretical_times(t_ff, t_bp, t_rs, t_ag);
    *dear = t.dear;
    *baseline = t.baseline;
    *smax = max_speedup(t_ff, t_bp, t_rs, t_ag, workers);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// CPU baseline: the reference's per-bucket S-SGD step (sgd_step =
// ring RS + ring AG + 1/P + w -= lr*mean, fp64) over `n_buckets` buckets of
// `bucket_elems[b]` elements each, P virtual workers, `steps` timed steps.
// Buckets are independent, so `threads` host threads split them (the
// reference is single-threaded and pure). Inputs are generated
// before timing; per-step wall seconds are written to out_seconds.
int ref_time_sgd_steps(const int64_t* bucket_elems, int n_buckets, int P, int threads,
                       int steps, uint64_t seed, double lr, double* out_seconds) {
  try {
    if (threads < 1) threads = 1;
    std::vector<std::vector<SgdState>> states(static_cast<std::size_t>(n_buckets));
    std::vector<std::vector<Vector>> grads(static_cast<std::size_t>(n_buckets));
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (int b = 0; b < n_buckets; ++b) {
      const int64_t d = bucket_elems[b];
      Vector w(d);
      for (int64_t i = 0; i < d; ++i) w(i) = dist(rng);
      states[static_cast<std::size_t>(b)].assign(static_cast<std::size_t>(P), SgdState{w, lr});
      auto& gs = grads[static_cast<std::size_t>(b)];
      gs.resize(static_cast<std::size_t>(P));
      for (auto& g : gs) {
        g.resize(d);
        for (int64_t i = 0; i < d; ++i) g(i) = dist(rng);
      }
    }
    // Balance buckets over threads by element count (greedy, largest first).
    std::vector<std::vector<int>> work(static_cast<std::size_t>(threads));
    std::vector<int64_t> load(static_cast<std::size_t>(threads), 0);
    for (int b = 0; b < n_buckets; ++b) {
      std::size_t best = 0;
      for (std::size_t t = 1; t < load.size(); ++t)
        if (load[t] < load[best]) best = t;
      work[best].push_back(b);
      load[best] += bucket_elems[b];
    }
    for (int s = 0; s < steps; ++s) {
      const auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
          for (int b : work[static_cast<std::size_t>(t)])
            states[static_cast<std::size_t>(b)] =
                sgd_step(states[static_cast<std::size_t>(b)], grads[static_cast<std::size_t>(b)]);
        });
      }
      for (auto& th : pool) th.join();
      const auto t1 = std::chrono::steady_clock::now();
      out_seconds[s] = std::chrono::duration<double>(t1 - t0).count();
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
