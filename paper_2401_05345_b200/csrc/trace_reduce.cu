// Trace-driven DISTWAR kernels: one warp per WarpRecord, grid-stride over a
// device-resident SoA trace. This is the reference's hot loop #3
// (`for rec in trace: apply_policy(rec); sums[addr] += value`,
// test_reducers.cpp:304-308, reducers.cpp:222-237) with the requests issued
// as real RED.ADD.F32 to L2 instead of std::map inserts.
//
// Layout (dw_trace_upload): active u32[R]; prim i32[R][32]; vals f32[R][N][32].
// Per record a warp reads 4 + 128 + 128*N bytes, every load a full 128 B
// line; HBM roofline: (132 + 128N) B/record.
#include <cuda_runtime.h>

#include <atomic>

#include "distwar.cuh"
#include "dw_internal.h"

namespace dw {

template <int N, int POL, bool COUNT>
__global__ void __launch_bounds__(256) k_reduce_trace(const uint32_t* __restrict__ active,
                                                      const int32_t* __restrict__ prim,
                                                      const float* __restrict__ vals,
                                                      int64_t R, int thr,
                                                      float* __restrict__ grad,
                                                      unsigned long long* __restrict__ ctr) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  uint32_t nred = 0;
  bool issuer = false;
  const int slot = bfly_slot<N>(lane, &issuer);
  // software pipeline: the next record's N+2 loads are in flight while this
  // record is reduced (streaming, L1-bypassing loads)
  uint32_t a_n = 0;
  int idx_n = 0;
  float v_n[N];
  if (w0 < R) {
    a_n = __ldcs(active + w0);
    idx_n = __ldcs(prim + w0 * 32 + lane);
#pragma unroll
    for (int p = 0; p < N; ++p) v_n[p] = __ldcs(vals + w0 * (32 * N) + p * 32 + lane);
  }
  for (int64_t r = w0; r < R; r += nw) {
    const uint32_t a = a_n;
    const int idx = idx_n;
    float v[N];
#pragma unroll
    for (int p = 0; p < N; ++p) v[p] = v_n[p];
    const int64_t rn = r + nw;
    if (rn < R) {
      a_n = __ldcs(active + rn);
      idx_n = __ldcs(prim + rn * 32 + lane);
#pragma unroll
      for (int p = 0; p < N; ++p) v_n[p] = __ldcs(vals + rn * (32 * N) + p * 32 + lane);
    }
    const bool act = (a >> lane) & 1u;
    if (POL == kNative) {
      native_atomics<N, COUNT>(grad + static_cast<int64_t>(idx) * N, v, act, nred);
    } else if (POL == kSwB) {
      reduce_bfly<N, COUNT, false>(idx, grad, v, thr, act, lane, nred, a, slot, issuer);
    } else if (POL == kSwS) {
      reduce_serial<N, COUNT>(idx, grad, v, thr, act, lane, nred, a, slot, issuer);
    } else {
      reduce_cccl<N, COUNT>(idx, grad, v, act, lane, nred, a);
    }
  }
  if (COUNT) flush_count(ctr, nred, lane);
}

// Any N: params are streamed from memory one at a time (per-param full-warp
// butterflies for SW-B, per-param folds for SW-S). Same request semantics.
template <int POL, bool COUNT>
__global__ void __launch_bounds__(256) k_reduce_trace_any(const uint32_t* __restrict__ active,
                                                          const int32_t* __restrict__ prim,
                                                          const float* __restrict__ vals,
                                                          int64_t R, int N, int thr,
                                                          float* __restrict__ grad,
                                                          unsigned long long* __restrict__ ctr) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  uint32_t nred = 0;
  for (int64_t r = w0; r < R; r += nw) {
    const uint32_t a = __ldg(active + r);
    const int idx = __ldg(prim + r * 32 + lane);
    const float* vr = vals + r * (32 * static_cast<int64_t>(N)) + lane;
    const bool act = (a >> lane) & 1u;
    const int cnt = __popc(a);
    const int idx0 = __shfl_sync(kFull, idx, 0);
    const bool same = __all_sync(kFull, idx == idx0) && idx0 >= 0;
    if (POL == kNative || ((POL == kSwB) && !(same && cnt > 0 && cnt >= thr)) ||
        (POL == kCccl && !(same && cnt > 0))) {
      if (act) {
        for (int p = 0; p < N; ++p) red_add(grad + static_cast<int64_t>(idx) * N + p, vr[p * 32]);
        if (COUNT) nred += N;
      }
    } else if (POL == kSwB || POL == kCccl) {
      for (int p = 0; p < N; ++p) {
        float x = __ldg(vr + p * 32);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) x += __shfl_xor_sync(kFull, x, off);
        if (lane == 0) {
          red_add(grad + static_cast<int64_t>(idx0) * N + p, x);
          if (COUNT) nred += 1;
        }
      }
    } else if (act) {  // SW-S, active lanes only
      const unsigned group = __match_any_sync(a, idx);
      const bool reduce = __popc(group) >= thr;
      const int leader = __ffs(group) - 1;
      for (int p = 0; p < N; ++p) {
        const float mine = __ldg(vr + p * 32);
        float s = mine;
        unsigned fetch = reduce ? (group & ~(1u << leader)) : 0u;
        while (__any_sync(a, fetch != 0u)) {
          const int src = fetch ? __ffs(fetch) - 1 : lane;
          const float x = __shfl_sync(a, mine, src);
          if (fetch && lane == leader) s += x;
          fetch &= fetch - 1u;
        }
        if (!reduce || lane == leader) {
          red_add(grad + static_cast<int64_t>(idx) * N + p, s);
          if (COUNT) nred += 1;
        }
      }
    }
  }
  if (COUNT) flush_count(ctr, nred, lane);
}

namespace {

template <int N, int POL, bool COUNT>
void launch_n(const uint32_t* a, const int32_t* p, const float* v, int64_t R, int thr,
              float* g, unsigned long long* c, cudaStream_t s) {
  static std::atomic<int> cached{0};  // occupancy of this instantiation (thread-safe)
  int blocks_per_sm = cached.load(std::memory_order_relaxed);
  if (!blocks_per_sm) {
    DW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm,
                                                          k_reduce_trace<N, POL, COUNT>, 256, 0));
    cached.store(blocks_per_sm, std::memory_order_relaxed);
  }
  const int64_t want = (R + 7) / 8;
  const int64_t cap = static_cast<int64_t>(sm_count()) * (blocks_per_sm ? blocks_per_sm : 1);
  const int grid = static_cast<int>(want < cap ? want : cap);
  k_reduce_trace<N, POL, COUNT><<<grid, 256, 0, s>>>(a, p, v, R, thr, g, c);
}

template <int POL, bool COUNT>
void launch_any(const uint32_t* a, const int32_t* p, const float* v, int64_t R, int N, int thr,
                float* g, unsigned long long* c, cudaStream_t s) {
  const int64_t want = (R + 7) / 8;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
  const int grid = static_cast<int>(want < cap ? want : cap);
  k_reduce_trace_any<POL, COUNT><<<grid, 256, 0, s>>>(a, p, v, R, N, thr, g, c);
}

template <int POL, bool COUNT>
void dispatch_n(const uint32_t* a, const int32_t* p, const float* v, int64_t R, int N, int thr,
                float* g, unsigned long long* c, cudaStream_t s) {
  switch (N) {
    case 1: return launch_n<1, POL, COUNT>(a, p, v, R, thr, g, c, s);
    case 2: return launch_n<2, POL, COUNT>(a, p, v, R, thr, g, c, s);
    case 3: return launch_n<3, POL, COUNT>(a, p, v, R, thr, g, c, s);
    case 4: return launch_n<4, POL, COUNT>(a, p, v, R, thr, g, c, s);
    case 9: return launch_n<9, POL, COUNT>(a, p, v, R, thr, g, c, s);
    default: return launch_any<POL, COUNT>(a, p, v, R, N, thr, g, c, s);
  }
}

template <bool COUNT>
void dispatch_pol(const uint32_t* a, const int32_t* p, const float* v, int64_t R, int N,
                  int pol, int thr, float* g, unsigned long long* c, cudaStream_t s) {
  switch (pol) {
    case kNative: return dispatch_n<kNative, COUNT>(a, p, v, R, N, thr, g, c, s);
    case kSwS: return dispatch_n<kSwS, COUNT>(a, p, v, R, N, thr, g, c, s);
    case kSwB: return dispatch_n<kSwB, COUNT>(a, p, v, R, N, thr, g, c, s);
    default: return dispatch_n<kCccl, COUNT>(a, p, v, R, N, thr, g, c, s);
  }
}

}  // namespace

// The reference's per-record instruction / FP-add cost model
// (reducers.cpp:84-206, every InstructionCosts entry 1: reducers.hpp:51-61),
// evaluated on the device over the same records the policy kernels reduce, so
// wr_simulate on the B200 reports the reference's core_instructions /
// core_fp_adds beside the measured REDs and cycles. One warp per record;
// out[0] += instructions, out[1] += fp adds.
__global__ void __launch_bounds__(256) k_model_costs(const uint32_t* __restrict__ active,
                                                     const int32_t* __restrict__ prim, int64_t R,
                                                     int N, int pol, int thr,
                                                     unsigned long long* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  unsigned long long ins = 0, fp = 0;  // lane-local shares, warp-summed at the end
  const unsigned long long n = static_cast<unsigned long long>(N);
  for (int64_t r = w0; r < R; r += nw) {
    const uint32_t a = active[r];
    const int idx = prim[r * 32 + lane];
    const unsigned long long cnt = static_cast<unsigned long long>(__popc(a));
    const int idx0 = __shfl_sync(kFull, idx, 0);
    const bool same = __all_sync(kFull, idx == idx0) && idx0 >= 0;  // all_lanes_same_primitive
    if (pol == kNative) {  // reducers.cpp:84-93
      if (lane == 0) ins += cnt * n;
    } else if (pol == kSwB) {  // reducers.cpp:138-175
      if (lane == 0) {
        ins += 4;
        if (same && cnt > 0 && cnt >= static_cast<unsigned long long>(thr)) {
          ins += 6 * n;
          fp += 160 * n;
        } else {
          ins += cnt * n;
        }
      }
    } else if (pol == kCccl) {  // reducers.cpp:177-206, per param
      if (lane == 0) {
        if (same && cnt > 0) {
          ins += n * 10;
          fp += n * 160;
        } else {
          ins += n * (4 + cnt);
        }
      }
    } else if ((a >> lane) & 1u) {  // SW-S, reducers.cpp:95-136: per match_any group
      const unsigned g = __match_any_sync(a, idx);
      if (lane == __ffs(g) - 1) {  // the group's leader accounts for it
        const unsigned long long gc = static_cast<unsigned long long>(__popc(g));
        ins += 3;
        if (gc >= static_cast<unsigned long long>(thr)) {
          ins += 1 + (gc - 1) * (2 + n) + n;
          fp += n * (gc - 1);
        } else {
          ins += gc * n;
        }
      }
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    ins += __shfl_xor_sync(kFull, ins, off);
    fp += __shfl_xor_sync(kFull, fp, off);
  }
  if (lane == 0 && (ins || fp)) {
    atomicAdd(out, ins);
    atomicAdd(out + 1, fp);
  }
}

void launch_model_costs(const uint32_t* active, const int32_t* prim, int64_t R, int n, int policy,
                        int thr, unsigned long long* out, cudaStream_t stream) {
  if (R <= 0) return;
  const int64_t want = (R + 7) / 8;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
  k_model_costs<<<static_cast<int>(want < cap ? want : cap), 256, 0, stream>>>(active, prim, R, n,
                                                                              policy, thr, out);
  DW_CUDA(cudaGetLastError());
}

void launch_reduce_records(const uint32_t* active, const int32_t* prim, const float* vals,
                           int64_t R, int n, int policy, int thr, float* grad,
                           unsigned long long* red_count, cudaStream_t stream) {
  if (R <= 0) return;
  if (red_count)
    dispatch_pol<true>(active, prim, vals, R, n, policy, thr, grad, red_count, stream);
  else
    dispatch_pol<false>(active, prim, vals, R, n, policy, thr, grad, nullptr, stream);
  DW_CUDA(cudaGetLastError());
}

}  // namespace dw
