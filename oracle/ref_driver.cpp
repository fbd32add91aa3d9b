// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// Thin extern "C" driver over the UNMODIFIED reference sources
// (/root/reference/proj/src/*.cpp), compiled by oracle/Makefile into
// oracle/_ref/libwarpred_ref.so. It lets the Python tests and golden-vector
// generator call the reference's own hot path directly:
//   workload::generate          /root/reference/proj/src/workload.cpp:99-153
//   reducers::apply_policy      /root/reference/proj/src/reducers.cpp:222-237
//   reducers::oracle_sum        /root/reference/proj/src/reducers.cpp:208-220
//   trace_io::save/load_binary  /root/reference/proj/src/trace_io.cpp:209-276
// and time the reference's CPU path for bench.py's `cpu_baseline` /
// `--impl reference` arm. No reference source is copied into this repo; the
// driver only includes the reference headers in place.

#include <random>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "warpred/experiment.hpp"
#include "warpred/hwsim.hpp"
#include "warpred/reducers.hpp"
#include "warpred/trace_io.hpp"
#include "warpred/workload.hpp"

using namespace warpred;

namespace {
thread_local std::string g_err = "ok";

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

struct RefScene {  // identical layout to wr_scene_spec (warpred.h:42-53)
  int32_t num_primitives;
  int32_t params_per_primitive;
  int32_t image_width;
  int32_t image_height;
  double mean_fragment_span;
  double fragments_per_pixel_mean;
  double activity_prob;
  double locality;
  uint64_t seed;
  int32_t quantized_values;
};

workload::SceneSpec to_scene(const RefScene& s) {
  workload::SceneSpec o;
  o.num_primitives = s.num_primitives;
  o.params_per_primitive = s.params_per_primitive;
  o.image_width = s.image_width;
  o.image_height = s.image_height;
  o.mean_fragment_span = s.mean_fragment_span;
  o.fragments_per_pixel_mean = s.fragments_per_pixel_mean;
  o.activity_prob = s.activity_prob;
  o.locality = s.locality;
  o.seed = s.seed;
  o.quantized_values = s.quantized_values != 0;
  return o;
}

reducers::PolicyKind to_kind(int k) {
  switch (k) {
    case 0: return reducers::PolicyKind::native;
    case 1: return reducers::PolicyKind::sw_s;
    case 2: return reducers::PolicyKind::sw_b;
    case 3: return reducers::PolicyKind::cccl;
    case 4: return reducers::PolicyKind::hw_atomred;
  }
  throw std::invalid_argument("unknown policy kind");
}

// Accumulate one policy over [begin, end) records into a dense per-address
// buffer (prim * N + param), in the order the reference emits requests.
void apply_range(const workload::Trace& t, size_t begin, size_t end,
                 const reducers::Policy& pol, double* sums, int n,
                 uint64_t* nreq, uint64_t* ninstr, uint64_t* nfp) {
  uint64_t q = 0, ins = 0, fp = 0;
  for (size_t r = begin; r < end; ++r) {
    const auto out = reducers::apply_policy(t.records[r], pol);
    for (const auto& req : out.requests)
      sums[static_cast<size_t>(req.addr.primitive) * n + req.addr.param] +=
          req.value;
    q += out.requests.size();
    ins += out.core_instructions;
    fp += out.core_fp_adds;
  }
  *nreq = q;
  *ninstr = ins;
  *nfp = fp;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_generate(const RefScene* s, void** out) {
  return guarded([&] {
    auto* t = new workload::Trace(workload::generate(to_scene(*s)));
    *out = t;
  });
}

int ref_load_binary(const char* path, void** out) {
  return guarded([&] {
    *out = new workload::Trace(trace_io::load_trace_binary(std::string(path)));
  });
}

int ref_save_binary(const void* h, const char* path) {
  return guarded([&] {
    trace_io::save_trace_binary(*static_cast<const workload::Trace*>(h),
                                std::string(path));
  });
}

// Builds a trace from flat arrays (lane-major grads, f64), e.g. records tapped
// from the rasterizer backward; scene fields other than N/P are zero.
int ref_from_arrays(int64_t nrec, int32_t n, int32_t num_prims,
                    const int32_t* warp_id, const int32_t* iteration,
                    const uint32_t* active, const int32_t* prim,
                    const double* grads, void** out) {
  return guarded([&] {
    auto* t = new workload::Trace();
    t->scene.params_per_primitive = n;
    t->scene.num_primitives = num_prims;
    t->records.resize(static_cast<size_t>(nrec));
    for (int64_t r = 0; r < nrec; ++r) {
      auto& rec = t->records[static_cast<size_t>(r)];
      rec.warp_id = warp_id ? warp_id[r] : 0;
      rec.iteration = iteration ? iteration[r] : 0;
      rec.active = active[r];
      for (int l = 0; l < 32; ++l) rec.lane_primitive[l] = prim[r * 32 + l];
      rec.lane_grads.assign(grads + r * 32 * n, grads + (r + 1) * 32 * n);
    }
    *out = t;
  });
}

void ref_free(void* h) { delete static_cast<workload::Trace*>(h); }

int64_t ref_record_count(const void* h) {
  return static_cast<int64_t>(
      static_cast<const workload::Trace*>(h)->records.size());
}

int32_t ref_params(const void* h) {
  return static_cast<const workload::Trace*>(h)->scene.params_per_primitive;
}

int32_t ref_num_primitives(const void* h) {
  return static_cast<const workload::Trace*>(h)->scene.num_primitives;
}

// Copies the records out as flat arrays (lane-major grads, as WarpRecord).
void ref_export(const void* h, int32_t* warp_id, int32_t* iteration,
                uint32_t* active, int32_t* prim, double* grads) {
  const auto& t = *static_cast<const workload::Trace*>(h);
  const int n = t.scene.params_per_primitive;
  for (size_t r = 0; r < t.records.size(); ++r) {
    const auto& rec = t.records[r];
    warp_id[r] = rec.warp_id;
    iteration[r] = rec.iteration;
    active[r] = rec.active;
    std::memcpy(prim + r * 32, rec.lane_primitive.data(), 32 * sizeof(int32_t));
    std::memcpy(grads + r * 32 * n, rec.lane_grads.data(),
                32 * n * sizeof(double));
  }
}

// reducers::oracle_sum densified: sums[prim*N+param], touched[...] = 1 for
// every address present in the reference's std::map.
int ref_oracle_sum(const void* h, int32_t num_prims, double* sums,
                   uint8_t* touched) {
  return guarded([&] {
    const auto& t = *static_cast<const workload::Trace*>(h);
    const int n = t.scene.params_per_primitive;
    const auto m = reducers::oracle_sum(t);
    for (const auto& [addr, v] : m) {
      if (addr.primitive < 0 || addr.primitive >= num_prims)
        throw std::invalid_argument("primitive out of range");
      const size_t i = static_cast<size_t>(addr.primitive) * n + addr.param;
      sums[i] = v;
      if (touched) touched[i] = 1;
    }
  });
}

// apply_policy over the whole trace, per-address sums in request order (the
// reference idiom of test_reducers.cpp:304-308, densified), plus the request
// / instruction / fp-add counts of reducers::PolicyOutput.
int ref_apply_policy(const void* h, int kind, int threshold, int32_t num_prims,
                     double* sums, uint64_t* counts3) {
  return guarded([&] {
    const auto& t = *static_cast<const workload::Trace*>(h);
    const int n = t.scene.params_per_primitive;
    std::memset(sums, 0, sizeof(double) * static_cast<size_t>(num_prims) * n);
    apply_range(t, 0, t.records.size(), {to_kind(kind), threshold}, sums, n,
                &counts3[0], &counts3[1], &counts3[2]);
  });
}

// One record through one policy: request stream in emission order.
int ref_record_policy(const uint32_t active, const int32_t* prim,
                      const double* grads, int32_t n, int kind, int threshold,
                      int32_t* out_prim, int32_t* out_param, double* out_val,
                      int64_t* out_count, uint64_t* instr, uint64_t* fp_adds) {
  return guarded([&] {
    workload::WarpRecord rec;
    rec.active = active;
    for (int l = 0; l < 32; ++l) rec.lane_primitive[l] = prim[l];
    rec.lane_grads.assign(grads, grads + 32 * n);
    const auto out = reducers::apply_policy(rec, {to_kind(kind), threshold});
    for (size_t i = 0; i < out.requests.size(); ++i) {
      out_prim[i] = out.requests[i].addr.primitive;
      out_param[i] = out.requests[i].addr.param;
      out_val[i] = out.requests[i].value;
    }
    *out_count = static_cast<int64_t>(out.requests.size());
    *instr = out.core_instructions;
    *fp_adds = out.core_fp_adds;
  });
}

// CPU baseline: wall seconds for apply_policy + per-address accumulation over
// the first `max_records` records (<=0: all), sharded over `threads` host
// threads by contiguous record ranges (per-record parallelism is permitted by
// SPEC.md:262), each into its own dense buffer, merged at the end.
int ref_time_policy(const void* h, int kind, int threshold, int32_t num_prims,
                    int threads, int64_t max_records, double* seconds,
                    uint64_t* contributions, uint64_t* requests) {
  return guarded([&] {
    const auto& t = *static_cast<const workload::Trace*>(h);
    const int n = t.scene.params_per_primitive;
    size_t nrec = t.records.size();
    if (max_records > 0 && static_cast<size_t>(max_records) < nrec)
      nrec = static_cast<size_t>(max_records);
    if (threads < 1) threads = 1;
    const size_t words = static_cast<size_t>(num_prims) * n;
    std::vector<std::vector<double>> bufs(threads, std::vector<double>(words));
    std::vector<uint64_t> q(threads), ins(threads), fp(threads);
    const reducers::Policy pol{to_kind(kind), threshold};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) {
      const size_t b = nrec * i / threads, e = nrec * (i + 1) / threads;
      pool.emplace_back([&, i, b, e] {
        apply_range(t, b, e, pol, bufs[i].data(), n, &q[i], &ins[i], &fp[i]);
      });
    }
    for (auto& th : pool) th.join();
    // merge the per-thread buffers in parallel, each thread one slice of the
    // addresses (a serial merge would cost O(threads * P * N) whatever the
    // sample size)
    pool.clear();
    for (int i = 0; i < threads; ++i) {
      const size_t b = words * i / threads, e = words * (i + 1) / threads;
      pool.emplace_back([&, b, e] {
        for (int k = 1; k < threads; ++k)
          for (size_t w = b; w < e; ++w) bufs[0][w] += bufs[k][w];
      });
    }
    for (auto& th : pool) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    uint64_t c = 0, qq = 0;
    for (size_t r = 0; r < nrec; ++r)
      c += static_cast<uint64_t>(__builtin_popcount(t.records[r].active)) * n;
    for (int i = 0; i < threads; ++i) qq += q[i];
    *contributions = c;
    *requests = qq;
  });
}

// experiment::read_metrics_csv (experiment.cpp:319-336) over a metrics.csv
// file: the reference's own reader accepting a file this repo writes
// (tools/metrics_csv.py). Copies up to max_rows rows out:
// policy kind, threshold (-1 when "-"), the 7 integer RunMetrics fields, and
// energy_proxy / grad_speedup / end_to_end_speedup.
int ref_read_metrics_csv(const char* path, int32_t max_rows, int64_t* nrows, int32_t* policy,
                         int32_t* threshold, uint64_t* ints7, double* doubles3) {
  return guarded([&] {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error(std::string("cannot open ") + path);
    const auto rows = experiment::read_metrics_csv(in);
    *nrows = static_cast<int64_t>(rows.size());
    for (size_t i = 0; i < rows.size() && static_cast<int32_t>(i) < max_rows; ++i) {
      const auto& c = rows[i];
      policy[i] = static_cast<int32_t>(c.policy);
      threshold[i] = c.threshold ? *c.threshold : -1;
      const auto& m = c.metrics;
      const uint64_t v[7] = {m.total_cycles, m.stalls_lsu, m.stalls_other,
                             m.atomic_requests_to_l2, m.core_instructions, m.core_fp_adds,
                             m.interconnect_packets};
      std::memcpy(ints7 + 7 * i, v, sizeof v);
      doubles3[3 * i + 0] = m.energy_proxy;
      doubles3[3 * i + 1] = c.grad_speedup;
      doubles3[3 * i + 2] = c.end_to_end_speedup;
    }
  });
}

// The draw sequence of the reference's acceptance criterion 1
// (tests/acceptance.cpp:93-146): one mt19937_64(20240801) stream; per trace
// the nine SceneSpec draws in source order, then per preset (3) and policy
// (native, sw_s, sw_b, cccl, hw_atomred) a threshold draw for the threshold
// policies only (reducers::policy_uses_threshold). thresholds[i*6 + 2*p + k]
// is preset p's sw_s (k = 0) / sw_b (k = 1) threshold of trace i.
int ref_criterion1_draws(int32_t ntraces, RefScene* specs, int32_t* thresholds) {
  return guarded([&] {
    std::mt19937_64 mix(20240801);
    const int npresets = static_cast<int>(hwsim::preset_names().size());
    if (npresets != 3) throw std::runtime_error("expected 3 presets");
    for (int32_t i = 0; i < ntraces; ++i) {
      RefScene& s = specs[i];
      s.num_primitives = 50 + static_cast<int32_t>(mix() % 400);
      s.params_per_primitive = 1 + static_cast<int>(mix() % 4);
      s.image_width = 32 + 8 * static_cast<int>(mix() % 5);
      s.image_height = 16 + 4 * static_cast<int>(mix() % 5);
      s.mean_fragment_span = 8.0 + static_cast<double>(mix() % 48);
      s.fragments_per_pixel_mean = 1.0 + 0.25 * static_cast<double>(mix() % 5);
      s.locality = 0.5 + 0.5 * static_cast<double>(mix() % 101) / 100.0;
      s.activity_prob = 0.3 + 0.7 * static_cast<double>(mix() % 101) / 100.0;
      s.seed = mix();
      s.quantized_values = 1;
      for (int p = 0; p < npresets; ++p) {
        thresholds[i * 6 + 2 * p + 0] = static_cast<int32_t>(mix() % 33);  // sw_s
        thresholds[i * 6 + 2 * p + 1] = static_cast<int32_t>(mix() % 33);  // sw_b
      }
    }
  });
}

}  // extern "C"
