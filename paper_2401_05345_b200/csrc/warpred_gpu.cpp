// libwarpred_gpu.so: the reference's C interface (warpred.h:20-133) with its
// hot path on the B200. Every wr_* symbol keeps the reference's signature,
// struct layout, status codes and error conventions (capi.cpp:16-44: a
// thread-local message, invalid_argument -> WR_ERR_INVALID_ARGUMENT,
// ios_base::failure -> WR_ERR_IO, other exceptions -> WR_ERR_RUNTIME), so a
// program built against warpred.h relinks against this library unchanged.
// It is a thin adapter over libdistwar.so's C ABI (include/distwar.h); the
// semantics that change because the machine is real are listed in
// include/warpred_gpu.h.
#include <charconv>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../../include/distwar.h"
#include "../../include/warpred_gpu.h"

static_assert(sizeof(wr_scene_spec) == sizeof(dw_scene_spec), "scene spec layout");
static_assert(offsetof(wr_scene_spec, seed) == offsetof(dw_scene_spec, seed), "scene spec layout");
static_assert(offsetof(wr_scene_spec, quantized_values) ==
                  offsetof(dw_scene_spec, quantized_values),
              "scene spec layout");
static_assert(static_cast<int>(WR_POLICY_HW_ATOMRED) == static_cast<int>(DW_POLICY_HW_ATOMRED),
              "policy enum");

struct wr_trace {
  dw_trace* t = nullptr;
  mutable dw_device_trace* d = nullptr;  // uploaded on first wr_simulate
  ~wr_trace() {
    if (d) dw_device_trace_free(d);
    if (t) dw_trace_free(t);
  }
};

namespace {

thread_local std::string last_error = "ok";

wr_status fail(wr_status code, const std::string& m) {
  last_error = m;
  return code;
}
wr_status fail_invalid(const std::string& m) { return fail(WR_ERR_INVALID_ARGUMENT, m); }

// A failing libdistwar call: same status numbering (distwar.h mirrors warpred.h:20-25).
struct DwError : std::runtime_error {
  dw_status code;
  DwError(dw_status c, const char* m) : std::runtime_error(m), code(c) {}
};
void dw_ok(dw_status s) {
  if (s != DW_OK) throw DwError(s, dw_last_error());
}

template <typename Fn>
wr_status guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const DwError& e) {
    return fail(static_cast<wr_status>(e.code), e.what());
  } catch (const std::invalid_argument& e) {
    return fail(WR_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::ios_base::failure& e) {
    return fail(WR_ERR_IO, e.what());
  } catch (const std::exception& e) {
    return fail(WR_ERR_RUNTIME, e.what());
  }
}

// Machine presets (hwsim.hpp:27-38 defaults, hwsim.cpp:35-55 SM / ROP counts):
// kept so wr_machine_preset callers work unchanged; the B200 run ignores them.
struct Preset {
  const char* name;
  int32_t sms, rops;
};
constexpr Preset kPresets[] = {{"tiny", 1, 2}, {"rtx3060like", 28, 48}, {"rtx4090like", 144, 176}};

void preset_defaults(wr_machine_config* c) {
  c->num_sms = 1;
  c->subcores_per_sm = 4;
  c->lsu_queue_depth = 32;
  c->rop_units = 2;
  c->rop_throughput = 1.0;
  c->interconnect_latency = 20;
  c->interconnect_bandwidth = 256;
  c->red_unit_latency_per_add = 1;
  c->red_pipe_depth = 4;
  c->warp_issue_width = 4;
}

// SM clock used to express measured kernel time as cycles.
double clock_hz() {
  const int khz = dw_device_clock_khz();
  if (khz <= 0) throw std::runtime_error("no CUDA device: " + std::string(dw_last_error()));
  return 1e3 * static_cast<double>(khz);
}

// ---- text trace format (trace_io.cpp:64-157 layout) ----------------------
constexpr char kTextMagic[] = "WRTRACE v1";

std::string fmt_double(double v) {
  char buf[32];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);  // shortest round-trip
  return std::string(buf, r.ptr);
}

[[noreturn]] void bad_format(const std::string& what) {
  throw std::runtime_error("trace format error: " + what);
}

void save_text(const wr_trace* tr, const std::string& path) {
  const uint32_t* active = nullptr;
  const int32_t* prim = nullptr;
  const double* grads = nullptr;
  dw_scene_spec sc{};
  dw_ok(dw_trace_arrays(tr->t, &active, &prim, &grads, &sc));
  const int32_t* wid = nullptr;
  const int32_t* it = nullptr;
  dw_ok(dw_trace_ids(tr->t, &wid, &it));
  const int64_t R = dw_trace_record_count(tr->t);
  const int n = sc.params_per_primitive;
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  out << kTextMagic << "; N=" << n << "; seed=" << sc.seed << "\n";
  static const char hex[] = "0123456789abcdef";
  for (int64_t r = 0; r < R; ++r) {
    char mask[9];
    for (int i = 0; i < 8; ++i) mask[i] = hex[(active[r] >> (28 - 4 * i)) & 0xfu];
    mask[8] = 0;
    out << wid[r] << ',' << it[r] << ',' << mask;
    for (int l = 0; l < 32; ++l) {
      out << ',';
      if ((active[r] >> l) & 1u) out << prim[r * 32 + l];
      else out << '-';
    }
    out << ',';
    for (int l = 0; l < 32; ++l) {
      if (l) out << ';';
      for (int p = 0; p < n; ++p) {
        if (p) out << ',';
        out << fmt_double(grads[(r * 32 + l) * n + p]);
      }
    }
    out << '\n';
  }
  if (!out) throw std::runtime_error("write failed: " + path);
}

template <typename T>
T parse_int(std::string_view s) {
  T v{};
  const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  if (r.ec != std::errc{} || r.ptr != s.data() + s.size())
    throw std::invalid_argument("bad integer field: " + std::string(s));
  return v;
}

double parse_double(std::string_view s) {
  double v = 0;
  const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  if (r.ec != std::errc{} || r.ptr != s.data() + s.size())
    throw std::invalid_argument("bad floating point field: " + std::string(s));
  return v;
}

std::vector<std::string_view> split(std::string_view s, char d) {
  std::vector<std::string_view> out;
  size_t b = 0;
  for (;;) {
    const size_t e = s.find(d, b);
    out.push_back(s.substr(b, e == std::string_view::npos ? std::string_view::npos : e - b));
    if (e == std::string_view::npos) return out;
    b = e + 1;
  }
}

dw_trace* load_text(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open for reading: " + path);
  std::string line;
  if (!std::getline(in, line)) bad_format("missing header");
  const auto hdr = split(line, ';');
  if (hdr.size() != 3 || hdr[0] != kTextMagic) bad_format("bad header: " + line);
  auto field = [](std::string_view f, std::string_view key) {
    while (!f.empty() && f.front() == ' ') f.remove_prefix(1);
    if (f.substr(0, key.size()) != key) bad_format("bad header field");
    return f.substr(key.size());
  };
  const int n = parse_int<int>(field(hdr[1], "N="));
  const uint64_t seed = parse_int<uint64_t>(field(hdr[2], "seed="));
  if (n < 1) bad_format("N must be >= 1");
  std::vector<int32_t> wid, it, prim;
  std::vector<uint32_t> act;
  std::vector<double> grads;
  int32_t max_prim = 0;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    size_t pos = 0;
    auto next = [&]() -> std::string_view {
      const size_t e = line.find(',', pos);
      if (e == std::string::npos) bad_format("truncated record: " + line);
      std::string_view f(line.data() + pos, e - pos);
      pos = e + 1;
      return f;
    };
    wid.push_back(parse_int<int32_t>(next()));
    it.push_back(parse_int<int32_t>(next()));
    const auto m = next();
    if (m.size() != 8) bad_format("active mask must be 8 hex digits");
    uint32_t mask = 0;
    for (char ch : m) {
      mask <<= 4;
      if (ch >= '0' && ch <= '9') mask |= static_cast<uint32_t>(ch - '0');
      else if (ch >= 'a' && ch <= 'f') mask |= static_cast<uint32_t>(ch - 'a' + 10);
      else bad_format("bad hex digit in active mask");
    }
    act.push_back(mask);
    for (int l = 0; l < 32; ++l) {
      const auto f = next();
      const int32_t id = f == "-" ? -1 : parse_int<int32_t>(f);
      if (id > max_prim) max_prim = id;
      prim.push_back(id);
    }
    const auto lanes = split(std::string_view(line).substr(pos), ';');
    if (lanes.size() != 32) bad_format("expected 32 lane grads");
    for (int l = 0; l < 32; ++l) {
      const auto vals = split(lanes[l], ',');
      if (static_cast<int>(vals.size()) != n) bad_format("expected N grads per lane");
      for (int p = 0; p < n; ++p) grads.push_back(parse_double(vals[p]));
    }
  }
  dw_trace* t = nullptr;
  dw_ok(dw_trace_from_arrays(static_cast<int64_t>(act.size()), n, max_prim + 1, wid.data(),
                             it.data(), act.data(), prim.data(), grads.data(), &t));
  dw_scene_spec sc{};
  dw_scene_spec_init(&sc);  // the text format carries N and the seed only
  sc.params_per_primitive = n;
  sc.num_primitives = max_prim + 1;
  sc.seed = seed;
  const dw_status s = dw_trace_set_scene(t, &sc);
  if (s != DW_OK) {
    dw_trace_free(t);
    dw_ok(s);
  }
  return t;
}

void write_hist(const std::filesystem::path& p, const char* key, const uint64_t h[33]) {
  std::ofstream out(p, std::ios::binary);
  if (!out) throw std::ios_base::failure("cannot write histogram csv");
  out << key << ",frequency\n";
  for (int k = 0; k <= 32; ++k)  // std::map order: present keys ascending
    if (h[k]) out << k << ',' << h[k] << '\n';
}

}  // namespace

extern "C" {

const char* wr_version(void) { return "1.0.0+b200"; }

const char* wr_last_error(void) { return last_error.c_str(); }

void wr_scene_spec_init(wr_scene_spec* scene) {
  if (scene) dw_scene_spec_init(reinterpret_cast<dw_scene_spec*>(scene));
}

wr_status wr_scene_from_config(const char* config_path, wr_scene_spec* out) {
  if (!config_path || !out) return fail_invalid("null argument");
  return fail(WR_ERR_RUNTIME,
              "wr_scene_from_config: the JSON experiment harness is not part of the GPU backend");
}

int wr_preset_count(void) { return static_cast<int>(sizeof kPresets / sizeof kPresets[0]); }

const char* wr_preset_name(int index) {
  if (index < 0 || index >= wr_preset_count()) return nullptr;
  return kPresets[index].name;
}

wr_status wr_machine_preset(const char* name, wr_machine_config* out) {
  if (!name || !out) return fail_invalid("null argument");
  for (const auto& p : kPresets)
    if (std::strcmp(p.name, name) == 0) {
      preset_defaults(out);
      out->num_sms = p.sms;
      out->rop_units = p.rops;
      return WR_OK;
    }
  return fail_invalid(std::string("unknown machine preset: ") + name);
}

wr_status wr_trace_generate(const wr_scene_spec* scene, wr_trace** out) {
  if (!scene || !out) return fail_invalid("null argument");
  return guarded([&] {
    auto t = std::make_unique<wr_trace>();
    dw_ok(dw_trace_generate(reinterpret_cast<const dw_scene_spec*>(scene), &t->t));
    *out = t.release();
    return WR_OK;
  });
}

void wr_trace_free(wr_trace* trace) { delete trace; }

int64_t wr_trace_record_count(const wr_trace* trace) {
  return trace ? dw_trace_record_count(trace->t) : -1;
}

wr_status wr_trace_save(const wr_trace* trace, const char* path, int binary) {
  if (!trace || !path) return fail_invalid("null argument");
  return guarded([&] {
    if (binary) dw_ok(dw_trace_save(trace->t, path, 1));
    else save_text(trace, path);
    return WR_OK;
  });
}

wr_status wr_trace_load(const char* path, int binary, wr_trace** out) {
  if (!path || !out) return fail_invalid("null argument");
  return guarded([&] {
    auto t = std::make_unique<wr_trace>();
    if (binary) dw_ok(dw_trace_load(path, 1, &t->t));
    else t->t = load_text(path);
    *out = t.release();
    return WR_OK;
  });
}

wr_status wr_trace_histogram_distinct(const wr_trace* trace, uint64_t out_counts[33]) {
  if (!trace || !out_counts) return fail_invalid("null argument");
  return guarded([&] {
    dw_ok(dw_trace_histogram_distinct(trace->t, out_counts));
    return WR_OK;
  });
}

wr_status wr_trace_histogram_active(const wr_trace* trace, uint64_t out_counts[33]) {
  if (!trace || !out_counts) return fail_invalid("null argument");
  return guarded([&] {
    dw_ok(dw_trace_histogram_active(trace->t, out_counts));
    return WR_OK;
  });
}

wr_status wr_trace_write_histograms(const wr_trace* trace, const char* dir) {
  if (!trace || !dir) return fail_invalid("null argument");
  return guarded([&] {
    uint64_t d[33], a[33];
    dw_ok(dw_trace_histogram_distinct(trace->t, d));
    dw_ok(dw_trace_histogram_active(trace->t, a));
    std::filesystem::create_directories(dir);
    write_hist(std::filesystem::path(dir) / "histogram_distinct.csv", "distinct_count", d);
    write_hist(std::filesystem::path(dir) / "histogram_active.csv", "active_lanes", a);
    return WR_OK;
  });
}

wr_status wr_simulate(const wr_trace* trace, const wr_machine_config* machine,
                      wr_policy_kind policy, int threshold, wr_run_metrics* out) {
  if (!trace || !machine || !out) return fail_invalid("null argument");
  return guarded([&] {
    if (policy == WR_POLICY_HW_ATOMRED)
      throw std::invalid_argument(
          "hw_atomred: the B200 has no atomred unit (DISTWAR-HW is a simulator-only policy)");
    if ((policy == WR_POLICY_SW_S || policy == WR_POLICY_SW_B) && (threshold < 0 || threshold > 33))
      throw std::invalid_argument("policy threshold out of range");
    if (!trace->d) dw_ok(dw_trace_upload(trace->t, nullptr, &trace->d));
    const auto kind = static_cast<dw_policy_kind>(policy);
    const int thr = (policy == WR_POLICY_SW_S || policy == WR_POLICY_SW_B) ? threshold : 0;
    dw_gpu_metrics m{};
    dw_ok(dw_gpu_run(trace->d, kind, thr, nullptr, &m));
    uint64_t costs[2] = {0, 0};
    dw_ok(dw_model_costs(trace->d, kind, thr, costs));
    std::memset(out, 0, sizeof *out);
    out->total_cycles = static_cast<uint64_t>(std::llround(m.kernel_ms * 1e-3 * clock_hz()));
    if (out->total_cycles == 0 && m.records) out->total_cycles = 1;
    out->atomic_requests_to_l2 = m.atomic_requests_to_l2;
    out->core_instructions = costs[0];
    out->core_fp_adds = costs[1];
    out->interconnect_packets = m.atomic_requests_to_l2;
    out->energy_proxy = 10.0 * static_cast<double>(out->interconnect_packets) +
                        static_cast<double>(out->atomic_requests_to_l2 + out->core_fp_adds);
    return WR_OK;
  });
}

wr_status wr_tune(const wr_trace* trace, const wr_machine_config* machine,
                  wr_policy_family family, int32_t iteration, wr_tune_report* out) {
  if (!trace || !machine || !out) return fail_invalid("null argument");
  return guarded([&] {
    dw_tune_report rep{};
    dw_ok(dw_tune(trace->t, family == WR_FAMILY_SW_S ? DW_FAMILY_SW_S : DW_FAMILY_SW_B,
                  iteration, 3, &rep));
    const double hz = clock_hz();
    out->chosen = 0;
    for (int t = 0; t <= 32; ++t) {
      out->cycles_by_threshold[t] =
          static_cast<uint64_t>(std::llround(rep.us_by_threshold[t] * 1e-6 * hz));
      if (out->cycles_by_threshold[t] < out->cycles_by_threshold[out->chosen]) out->chosen = t;
    }
    out->profile_iteration = rep.profile_iteration;
    out->reprofile_period = rep.reprofile_period;
    return WR_OK;
  });
}

wr_status wr_tune_report_save_csv(const wr_tune_report* report, const char* path) {
  if (!report || !path) return fail_invalid("null argument");
  return guarded([&] {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::ios_base::failure(std::string("cannot write: ") + path);
    out << "threshold,cycles\n";  // tuner.cpp:54-62 layout
    for (int t = 0; t <= 32; ++t) out << t << ',' << report->cycles_by_threshold[t] << '\n';
    out << "# chosen=" << report->chosen << " profile_iteration=" << report->profile_iteration
        << " reprofile_period=" << report->reprofile_period << '\n';
    return WR_OK;
  });
}

wr_status wr_experiment_run(const char* config_path, const char* output_dir_override,
                            int64_t seed_override, int emit_events) {
  (void)output_dir_override;
  (void)seed_override;
  (void)emit_events;
  if (!config_path) return fail_invalid("null argument");
  return fail(WR_ERR_RUNTIME,
              "wr_experiment_run: the JSON experiment harness is not part of the GPU backend");
}

}  // extern "C"
