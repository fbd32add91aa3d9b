// Host-side input side of the path: the seeded WarpRecord generator, the
// WRTRACEB container and the Observation-1/2 histograms. Byte-compatible with
// the reference (workload.cpp:15-153, trace_io.cpp:159-276,
// workload.cpp:155-197): equal SceneSpecs give byte-identical traces, which
// tests/test_gpu_trace.py checks against the oracle and tests/golden/.
#include <cmath>
#include <cstring>
#include <fstream>
#include <random>
#include <stdexcept>
#include <string>

#include "dw_internal.h"

namespace dw {
namespace {

// std::mt19937_64 is fully specified by the standard; the variate transforms
// are hand-rolled exactly as the reference's (workload.cpp:15-52), so the
// stream does not depend on the standard library build.
double uniform01(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
bool bernoulli(std::mt19937_64& g, double p) { return uniform01(g) < p; }
int poisson(std::mt19937_64& g, double mean) {
  const double limit = std::exp(-mean);
  int k = 0;
  double p = 1.0;
  do {
    ++k;
    p *= uniform01(g);
  } while (p > limit);
  return k - 1;
}
int64_t geometric_at_least_one(std::mt19937_64& g, double mean) {
  if (mean <= 1.0) return 1;
  const double p = 1.0 / mean;
  const double u = uniform01(g);
  const double len = std::floor(std::log1p(-u) / std::log1p(-p)) + 1.0;
  return static_cast<int64_t>(std::max(1.0, len));
}
double draw_grad(std::mt19937_64& g, bool quantized) {
  if (quantized) return static_cast<double>(1 + static_cast<int>(g() % 255)) / 256.0;
  return 2.0 * uniform01(g) - 1.0;
}

void validate(const dw_scene_spec& s) {
  auto bad = [](const char* f) {
    throw std::invalid_argument(std::string("SceneSpec: invalid field ") + f);
  };
  if (s.num_primitives < 1) bad("num_primitives");
  if (s.params_per_primitive < 1) bad("params_per_primitive");
  if (s.image_width < 1) bad("image_width");
  if (s.image_height < 1) bad("image_height");
  if (!(s.mean_fragment_span >= 1.0)) bad("mean_fragment_span");
  if (!(s.fragments_per_pixel_mean > 0.0)) bad("fragments_per_pixel_mean");
  if (!(s.activity_prob >= 0.0 && s.activity_prob <= 1.0)) bad("activity_prob");
  if (!(s.locality >= 0.0 && s.locality <= 1.0)) bad("locality");
}

[[noreturn]] void bad_format(const std::string& what) {
  throw std::runtime_error("trace format error: " + what);
}

template <typename T>
void put(std::ofstream& f, const T& v) {
  f.write(reinterpret_cast<const char*>(&v), sizeof(T));  // little-endian host
}
template <typename T>
void get(std::ifstream& f, T* v, size_t n = 1) {
  f.read(reinterpret_cast<char*>(v), static_cast<std::streamsize>(sizeof(T) * n));
  if (!f) bad_format("truncated binary trace");
}

}  // namespace

void scene_defaults(dw_scene_spec* s) {  // SceneSpec, workload.hpp:16-36
  s->num_primitives = 1024;
  s->params_per_primitive = 3;
  s->image_width = 64;
  s->image_height = 32;
  s->mean_fragment_span = 64.0;
  s->fragments_per_pixel_mean = 1.0;
  s->activity_prob = 1.0;
  s->locality = 1.0;
  s->seed = 0;
  s->quantized_values = 1;
}

HostTrace generate(const dw_scene_spec& s) {
  validate(s);
  HostTrace t;
  t.scene = s;
  std::mt19937_64 g(s.seed);
  // FragmentStream (workload.cpp:56-81): geometric runs of one primitive.
  int32_t cur = static_cast<int32_t>(g() % static_cast<uint64_t>(s.num_primitives));
  int64_t remaining = geometric_at_least_one(g, s.mean_fragment_span);
  const int num_warps = ((s.image_width + 7) / 8) * ((s.image_height + 3) / 4);
  const int n = s.params_per_primitive;
  const bool q = s.quantized_values != 0;
  for (int32_t warp = 0; warp < num_warps; ++warp) {
    const int trips = std::max(1, poisson(g, s.fragments_per_pixel_mean));
    for (int32_t iter = 0; iter < trips; ++iter) {
      const size_t r = t.active.size();
      uint32_t active = 0;
      for (int lane = 0; lane < 32; ++lane)
        if (bernoulli(g, s.activity_prob)) active |= 1u << lane;
      const int32_t base = cur;
      remaining -= 32;
      if (remaining <= 0) {
        cur = static_cast<int32_t>(g() % static_cast<uint64_t>(s.num_primitives));
        remaining = geometric_at_least_one(g, s.mean_fragment_span);
      }
      t.warp_id.push_back(warp);
      t.iteration.push_back(iter);
      t.active.push_back(active);
      t.prim.resize((r + 1) * 32);
      t.grads.resize((r + 1) * 32 * static_cast<size_t>(n), 0.0);
      int32_t* prim = t.prim.data() + r * 32;
      if (bernoulli(g, s.locality)) {
        for (int lane = 0; lane < 32; ++lane) prim[lane] = base;
      } else {
        const int k = 2 + static_cast<int>(g() % 7);
        for (int lane = 0; lane < 32; ++lane)
          prim[lane] = (base + static_cast<int32_t>(g() % static_cast<uint64_t>(k))) %
                       s.num_primitives;
      }
      double* gr = t.grads.data() + r * 32 * n;
      for (int lane = 0; lane < 32; ++lane) {
        if (!(active >> lane & 1u)) continue;
        for (int p = 0; p < n; ++p) gr[lane * n + p] = draw_grad(g, q);
      }
    }
  }
  return t;
}

void save_binary(const HostTrace& t, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::ios_base::failure("cannot open for writing: " + path);
  f.write("WRTRACEB", 8);
  const auto& s = t.scene;
  put<uint32_t>(f, 1);
  put(f, s.num_primitives);
  put(f, s.params_per_primitive);
  put(f, s.image_width);
  put(f, s.image_height);
  put(f, s.mean_fragment_span);
  put(f, s.fragments_per_pixel_mean);
  put(f, s.activity_prob);
  put(f, s.locality);
  put(f, s.seed);
  put<uint32_t>(f, s.quantized_values ? 1u : 0u);
  put<uint64_t>(f, static_cast<uint64_t>(t.records()));
  const int n = s.params_per_primitive;
  for (int64_t r = 0; r < t.records(); ++r) {
    put(f, t.warp_id[r]);
    put(f, t.iteration[r]);
    put(f, t.active[r]);
    f.write(reinterpret_cast<const char*>(t.prim.data() + r * 32), 128);
    f.write(reinterpret_cast<const char*>(t.grads.data() + r * 32 * n), 256 * n);
  }
  if (!f) throw std::ios_base::failure("write failed: " + path);
}

HostTrace load_binary(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open for reading: " + path);
  char magic[8];
  f.read(magic, 8);
  if (!f || std::memcmp(magic, "WRTRACEB", 8) != 0) bad_format("bad binary magic");
  uint32_t version, q;
  get(f, &version);
  if (version != 1) bad_format("unsupported binary version");
  HostTrace t;
  auto& s = t.scene;
  get(f, &s.num_primitives);
  get(f, &s.params_per_primitive);
  get(f, &s.image_width);
  get(f, &s.image_height);
  get(f, &s.mean_fragment_span);
  get(f, &s.fragments_per_pixel_mean);
  get(f, &s.activity_prob);
  get(f, &s.locality);
  get(f, &s.seed);
  get(f, &q);
  s.quantized_values = q != 0;
  uint64_t count;
  get(f, &count);
  const int n = s.params_per_primitive;
  if (n < 1) bad_format("N must be >= 1");
  t.warp_id.resize(count);
  t.iteration.resize(count);
  t.active.resize(count);
  t.prim.resize(count * 32);
  t.grads.resize(count * 32 * static_cast<size_t>(n));
  for (uint64_t r = 0; r < count; ++r) {
    get(f, &t.warp_id[r]);
    get(f, &t.iteration[r]);
    get(f, &t.active[r]);
    get(f, t.prim.data() + r * 32, 32);
    get(f, t.grads.data() + r * 32 * n, 32 * static_cast<size_t>(n));
  }
  return t;
}

void histograms(const HostTrace& t, uint64_t distinct[33], uint64_t act[33]) {
  if (t.records() == 0) throw std::invalid_argument("histogram: empty trace");
  for (int i = 0; i < 33; ++i) distinct[i] = act[i] = 0;
  for (int64_t r = 0; r < t.records(); ++r) {
    const uint32_t a = t.active[r];
    act[__builtin_popcount(a)]++;
    if (!a) continue;
    int32_t seen[32];
    int c = 0;
    for (int l = 0; l < 32; ++l) {
      if (!(a >> l & 1u)) continue;
      const int32_t id = t.prim[r * 32 + l];
      bool found = false;
      for (int i = 0; i < c && !found; ++i) found = seen[i] == id;
      if (!found) seen[c++] = id;
    }
    distinct[c]++;
  }
}

}  // namespace dw
