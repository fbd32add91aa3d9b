// Internal host-side helpers shared by the distwar translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/distwar.h"

namespace dw {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " +
                             cudaGetErrorString(e));
}
#define DW_CUDA(x) ::dw::cuda_check((x), #x)

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int sm_count();  // cached per device

// Trace-driven reduction kernels (trace_reduce.cu).
void launch_reduce_records(const uint32_t* active, const int32_t* prim, const float* vals,
                           int64_t num_records, int n, int policy, int thr, float* grad,
                           unsigned long long* red_count, cudaStream_t stream);
// The reference's instruction / FP-add cost model of the same records (out[2], accumulated).
void launch_model_costs(const uint32_t* active, const int32_t* prim, int64_t num_records, int n,
                        int policy, int thr, unsigned long long* out, cudaStream_t stream);

// Host-side WarpRecord trace (workload.cpp): flat arrays as in
// reference workload.hpp:41-65, lane-major f64 grads.
struct HostTrace {
  dw_scene_spec scene{};
  std::vector<int32_t> warp_id, iteration;
  std::vector<uint32_t> active;
  std::vector<int32_t> prim;   // R*32
  std::vector<double> grads;   // R*32*N
  int64_t records() const { return static_cast<int64_t>(active.size()); }
};

void scene_defaults(dw_scene_spec* s);
HostTrace generate(const dw_scene_spec& s);
void save_binary(const HostTrace& t, const std::string& path);
HostTrace load_binary(const std::string& path);
void histograms(const HostTrace& t, uint64_t distinct[33], uint64_t active[33]);

// RED-throughput microbenchmarks (microbench.cu).
double microbench_red(int pattern, int64_t ops, cudaStream_t stream);

}  // namespace dw

struct dw_trace {
  dw::HostTrace t;
};

struct dw_device_trace {
  uint32_t* active = nullptr;
  int32_t* prim = nullptr;
  float* vals = nullptr;
  int64_t records = 0;
  int32_t params = 0;
  int32_t num_primitives = 0;
  uint64_t contributions = 0;
};
