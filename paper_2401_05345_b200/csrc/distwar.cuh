// DISTWAR device-side reduction primitives for sm_100a.
//
// Each function is called by ALL 32 lanes of a warp in place of the N
// per-lane atomicAdds of the gradient step (the SW-B
// calling convention of PAPER.md:1858-1888: inactive lanes participate with
// zero values and an `active` flag). Policy semantics follow the reference
// restatement exactly -- which lanes issue, how many RED.ADD requests reach
// L2, the balancing-threshold comparison `count >= t` -- while the arithmetic
// is laid out for the B200 SM:
//
//   native   reducers.cpp:84-93   one RED per (active lane, param)
//   sw_s     reducers.cpp:95-136  __match_any_sync groups; a group of size
//                                 >= t is summed (masked reduce-scatter
//                                 butterfly), then N REDs
//   sw_b     reducers.cpp:138-175 all 32 lanes on one primitive and
//                                 popc(active) >= t: a full-warp butterfly,
//                                 then N REDs; else per-lane REDs
//   cccl     reducers.cpp:177-206 per-param eligibility + per-param
//                                 cub::WarpReduce, lane 0 issues
//
// SW-B's butterfly is a *reduce-scatter* xor butterfly: at each of the 5
// levels a lane keeps half of its live params and ships the other half to
// its partner, so N=9 needs 5+3+2+1+1 = 12 SHFL+FADD instead of 5*9 = 45, and
// the N sums end in N distinct lanes which issue ONE RED instruction (N
// active lanes, contiguous addresses) instead of N single-lane REDs. The
// per-param sum is the same balanced 32-leaf tree as the reference's
// shfl_down tree up to a relabelling of the leaves, so it is exact wherever
// the reference's is (the k/256 grid) and otherwise within fp32 rounding.
#pragma once

#include <cuda_runtime.h>
#include <cub/warp/warp_reduce.cuh>
#include <cstdint>

// Per-lane fallback of the rasterizer's SW-B as vector REDs (red_row9); 0 = one
// scalar RED per param (the A/B baseline; also selectable at run time,
// DW_VEC_RED=0 in the environment, for bench.py's speed-up decomposition).
#ifndef DW_VEC_RED
#define DW_VEC_RED 1
#endif

namespace dw {

constexpr unsigned kFull = 0xffffffffu;

enum PolicyKind : int { kNative = 0, kSwS = 1, kSwB = 2, kCccl = 3 };

// One fire-and-forget fp32 reduction at L2 (SASS RED.E.ADD.F32.FTZ.RN).
__device__ __forceinline__ void red_add(float* addr, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(addr), "f"(v) : "memory");
}

// Vector fp32 reductions (sm_90+: RED.E.ADD.F32x2 / x4): one L2 atomic request
// carries 2 or 4 consecutive floats. `addr` must be 8- / 16-byte aligned.
__device__ __forceinline__ void red_add_v2(float* addr, float a, float b) {
  asm volatile("red.relaxed.gpu.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(a), "f"(b)
               : "memory");
}
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a),
               "f"(b), "f"(c), "f"(d)
               : "memory");
}

// One primitive's nine consecutive gradient floats (Address order,
// reducers.hpp:19-23) added with the fewest aligned vector REDs the row's
// 16-byte phase allows: 3 requests (phase 0 or 3) or 4 (phase 1 or 2) instead
// of 9. Each float is still one fp32 add at L2, so the per-param semantics
// (and the reference's request count, which counts params) are unchanged.
// The phase is warp-uniform where the caller's lanes share a primitive.
__device__ __forceinline__ void red_row9(float* b, const float (&s)[9]) {
  switch ((reinterpret_cast<uintptr_t>(b) >> 2) & 3u) {
    case 0:
      red_add_v4(b, s[0], s[1], s[2], s[3]);
      red_add_v4(b + 4, s[4], s[5], s[6], s[7]);
      red_add(b + 8, s[8]);
      break;
    case 1:
      red_add(b, s[0]);
      red_add_v2(b + 1, s[1], s[2]);
      red_add_v4(b + 3, s[3], s[4], s[5], s[6]);
      red_add_v2(b + 7, s[7], s[8]);
      break;
    case 2:
      red_add_v2(b, s[0], s[1]);
      red_add_v4(b + 2, s[2], s[3], s[4], s[5]);
      red_add_v2(b + 6, s[6], s[7]);
      red_add(b + 8, s[8]);
      break;
    default:
      red_add(b, s[0]);
      red_add_v4(b + 1, s[1], s[2], s[3], s[4]);
      red_add_v4(b + 5, s[5], s[6], s[7], s[8]);
  }
}

// ---------------------------------------------------------------------------
// Reduce-scatter butterfly over compile-time N (<= 32 params).
//
// Register layout: at a level with CNT virtual slots, lanes with the level's
// bit clear keep slots [0, H) and lanes with it set keep [H, 2H) moved down
// to [0, H), H = ceil(CNT/2); slots past the parent's real range are
// garbage that only ever meets garbage. Once CNT == 1 both partners keep the
// slot (a plain butterfly step), so on exit v[0] of every lane is the full
// 32-lane sum of the param bfly_slot() names.
template <int CNT, int OFF>
struct ReduceScatter {
  template <int CAP>
  __device__ __forceinline__ static void run(float (&v)[CAP], int lane) {
    if constexpr (OFF >= 1) {
      if constexpr (CNT <= 1) {
        v[0] += __shfl_xor_sync(kFull, v[0], OFF);
        ReduceScatter<1, OFF / 2>::run(v, lane);
      } else {
        constexpr int H = (CNT + 1) / 2;
        const bool up = (lane & OFF) != 0;
#pragma unroll
        for (int k = 0; k < H; ++k) {
          if (k + H < CNT) {
            const float send = up ? v[k] : v[k + H];
            const float recv = __shfl_xor_sync(kFull, send, OFF);
            v[k] = (up ? v[k + H] : v[k]) + recv;
          } else {  // odd CNT: the upper lane has no slot k+H
            const float send = up ? v[k] : 0.0f;
            const float recv = __shfl_xor_sync(kFull, send, OFF);
            v[k] = v[k] + recv;  // garbage in upper lanes, never emitted
          }
        }
        ReduceScatter<H, OFF / 2>::run(v, lane);
      }
    }
  }
};

// N = 9 specialisation with the level sums done as packed FP32 pairs
// (sm_100 FADD2): same slot algebra as ReduceScatter<9, 16> (bfly_slot<9>
// applies unchanged), 8 adds instead of 12.
__device__ __forceinline__ void reduce_scatter9(float (&v)[9], int lane) {
  // level 16: 9 -> 5 slots
  bool up = (lane & 16) != 0;
  float sd[5], kp[5];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    sd[k] = up ? v[k] : v[k + 5];
    kp[k] = up ? v[k + 5] : v[k];
  }
  sd[4] = up ? v[4] : 0.0f;
  kp[4] = v[4];
  float rv[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) rv[k] = __shfl_xor_sync(kFull, sd[k], 16);
  const float2 s01 = __fadd2_rn(make_float2(kp[0], kp[1]), make_float2(rv[0], rv[1]));
  const float2 s23 = __fadd2_rn(make_float2(kp[2], kp[3]), make_float2(rv[2], rv[3]));
  const float s4 = kp[4] + rv[4];
  // level 8: 5 -> 3
  up = (lane & 8) != 0;
  const float a0 = up ? s01.x : s23.y, a1 = up ? s01.y : s4, a2 = up ? s23.x : 0.0f;
  const float b0 = up ? s23.y : s01.x, b1 = up ? s4 : s01.y, b2 = s23.x;
  const float r0 = __shfl_xor_sync(kFull, a0, 8), r1 = __shfl_xor_sync(kFull, a1, 8),
              r2 = __shfl_xor_sync(kFull, a2, 8);
  const float2 t01 = __fadd2_rn(make_float2(b0, b1), make_float2(r0, r1));
  const float t2 = b2 + r2;
  // level 4: 3 -> 2
  up = (lane & 4) != 0;
  const float c0 = up ? t01.x : t2, c1 = up ? t01.y : 0.0f;
  const float d0 = up ? t2 : t01.x, d1 = t01.y;
  const float2 u = __fadd2_rn(make_float2(d0, d1),
                              make_float2(__shfl_xor_sync(kFull, c0, 4), __shfl_xor_sync(kFull, c1, 4)));
  // level 2: 2 -> 1
  up = (lane & 2) != 0;
  const float e0 = up ? u.x : u.y, f0 = up ? u.y : u.x;
  float w = f0 + __shfl_xor_sync(kFull, e0, 2);
  // level 1: plain butterfly
  w += __shfl_xor_sync(kFull, w, 1);
  v[0] = w;
}

// Which param lane `lane` holds after ReduceScatter<N,16>, and whether it is
// the one designated lane that issues that param's RED.
template <int N>
__device__ __forceinline__ int bfly_slot(int lane, bool* issuer) {
  int lo = 0, real = N, cnt = N;
  bool designated = true;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    if (cnt <= 1) {
      if (lane & off) designated = false;  // both partners hold it; keep bit-0 side
    } else {
      const int h = (cnt + 1) / 2;
      if (lane & off) {
        lo += h;
        real = real - h > 0 ? real - h : 0;
      } else {
        real = real < h ? real : h;
      }
      cnt = h;
    }
  }
  *issuer = designated && real >= 1;
  return lo;
}

// ---------------------------------------------------------------------------
// Policies. `base` is this lane's &grad[idx * N]; `v` its N values (zeros
// when inactive, as the SW-B convention requires); `active` its was_active
// flag; `nred` counts the REDs this lane issues when COUNT. reduce_bfly
// takes the lane's (slot, issuer) from bfly_slot<N>(), computed once per
// kernel.

template <int N, bool COUNT>
__device__ __forceinline__ void native_atomics(float* base, const float (&v)[N], bool active,
                                               uint32_t& nred) {
  if (active) {
#pragma unroll
    for (int p = 0; p < N; ++p) red_add(base + p, v[p]);
    if (COUNT) nred += N;
  }
}

// SW-B (reduce_bfly, PAPER.md:1779-1813 with the listing's bugs fixed: the
// threshold is compared with popc(ballot), not the ballot mask). UNIFORM=true
// skips the all-lanes-same-primitive vote when the caller guarantees it (the
// rasterizer: every lane of a warp walks the same Gaussian list).
template <int N, bool COUNT, bool UNIFORM>
__device__ __forceinline__ void reduce_bfly(int idx, float* grad, float (&v)[N], int thr,
                                            bool active, int lane, uint32_t& nred,
                                            unsigned ballot, int slot, bool issuer) {
  bool same = true;
  int idx0 = idx;
  if (!UNIFORM) {
    idx0 = __shfl_sync(kFull, idx, 0);
    same = __all_sync(kFull, idx == idx0) && idx0 >= 0;
  }
  const int cnt = __popc(ballot);
  if (same && cnt > 0 && cnt >= thr) {
    ReduceScatter<N, 16>::run(v, lane);
    if (issuer) {
      red_add(grad + static_cast<int64_t>(idx0) * N + slot, v[0]);
      if (COUNT) nred += 1;
    }
  } else {
    native_atomics<N, COUNT>(grad + static_cast<int64_t>(idx) * N, v, active, nred);
  }
}

// SW-B for callers that hand in gradients with a per-param constant factor
// still to apply (grad[p] = scale[p] * v[p]): the factor is linear in the sum,
// so the reducing path multiplies once after the butterfly (`lane_scale` =
// scale[slot], precomputed per lane) and only the per-lane fallback scales all
// N values. Same request semantics as reduce_bfly<N, COUNT, true>.
// S: floats per gradient row -- N (the Address-order [P][N] buffer), or 12
// for N = 9: a padded [P][12] accumulation buffer whose 48-byte rows are
// 16-byte aligned, so the per-lane fallback is always v4 + v4 + scalar (no
// phase switch, no register shuffles) and folded into [P][9] once per batch
// (launch_fold_rows).
template <int N, bool COUNT, bool VEC = DW_VEC_RED != 0, int S = N>
__device__ __forceinline__ void reduce_bfly_scaled(int idx, float* grad, float (&v)[N], int thr,
                                                   bool active, int lane, uint32_t& nred,
                                                   unsigned ballot, int slot, bool issuer,
                                                   float lane_scale, const float (&scale)[N]) {
  const int cnt = __popc(ballot);
  if (cnt >= thr) {  // cnt > 0: callers skip empty ballots
    if constexpr (N == 9)
      reduce_scatter9(v, lane);
    else
      ReduceScatter<N, 16>::run(v, lane);
    if (issuer) {
      red_add(grad + static_cast<int64_t>(idx) * S + slot, v[0] * lane_scale);
      if (COUNT) nred += 1;
    }
  } else if (active) {
    float* base = grad + static_cast<int64_t>(idx) * S;
    if constexpr (VEC && N == 9 && S == 12) {  // 16-byte aligned padded row: phase 0 always
      red_add_v4(base, v[0] * scale[0], v[1] * scale[1], v[2] * scale[2], v[3] * scale[3]);
      red_add_v4(base + 4, v[4] * scale[4], v[5] * scale[5], v[6] * scale[6], v[7] * scale[7]);
      red_add(base + 8, v[8] * scale[8]);
    } else if constexpr (VEC && N == 9) {
      float sv[9];
#pragma unroll
      for (int p = 0; p < 9; ++p) sv[p] = v[p] * scale[p];
      red_row9(base, sv);
    } else {
#pragma unroll
      for (int p = 0; p < N; ++p) red_add(base + p, v[p] * scale[p]);
    }
    if (COUNT) nred += N;
  }
}

// SW-S (reduce_serial; request semantics
// reducers.cpp:95-136): the active lanes split into __match_any_sync groups
// (one per distinct primitive); a group of size >= thr issues its N sums once,
// from the lanes the reduce-scatter leaves them in; smaller groups issue
// per-lane REDs. The paper's leader folds its group serially (O(group) SHFLs
// per param, a warp-uniform trip count set by the largest group); here each
// reducing group is summed by the same reduce-scatter butterfly as SW-B with
// the lanes outside the group contributing zero, so a warp pays one
// butterfly per reducing group -- and one in total when the active lanes
// share a primitive, as every warp of the rasterizer and ~99 % of the C3
// trace's records do. The per-group sum is a balanced tree rather than the
// leader's ascending fold: identical on the reference's exact grid (any
// order is exact below 65,793 addends), within fp32 rounding elsewhere.
// Must be called by all 32 lanes.
template <int N, bool COUNT>
__device__ __forceinline__ void group_bfly(float (&x)[N], int lane) {
  if constexpr (N == 9)
    reduce_scatter9(x, lane);
  else
    ReduceScatter<N, 16>::run(x, lane);
}

template <int N, bool COUNT>
__device__ __forceinline__ void reduce_serial(int idx, float* grad, const float (&v)[N], int thr,
                                              bool active, int lane, uint32_t& nred,
                                              unsigned ballot, int slot, bool issuer) {
  if (ballot == 0u) return;  // no active lane: no groups, no requests
  const unsigned group = active ? __match_any_sync(ballot, idx) : 0u;
  if (__all_sync(kFull, !active || group == ballot)) {  // one group: every active lane
    const int cnt = __popc(ballot);
    if (cnt >= thr) {
      float x[N];
#pragma unroll
      for (int p = 0; p < N; ++p) x[p] = active ? v[p] : 0.0f;
      group_bfly<N, COUNT>(x, lane);
      const int leader = __ffs(ballot) - 1;
      const int idx0 = __shfl_sync(kFull, idx, leader);
      if (issuer) {
        red_add(grad + static_cast<int64_t>(idx0) * N + slot, x[0]);
        if (COUNT) nred += 1;
      }
    } else if (active) {
      float* base = grad + static_cast<int64_t>(idx) * N;
#pragma unroll
      for (int p = 0; p < N; ++p) red_add(base + p, v[p]);
      if (COUNT) nred += N;
    }
    return;
  }
  // divergent record: one pass per group, in ascending-leader order
  unsigned remaining = ballot;
  while (remaining) {
    const int leader = __ffs(remaining) - 1;
    const unsigned g = __shfl_sync(kFull, group, leader);
    remaining &= ~g;
    const bool mine = (g >> lane) & 1u;
    if (__popc(g) >= thr) {
      float x[N];
#pragma unroll
      for (int p = 0; p < N; ++p) x[p] = mine ? v[p] : 0.0f;
      group_bfly<N, COUNT>(x, lane);
      const int idx0 = __shfl_sync(kFull, idx, leader);
      if (issuer) {
        red_add(grad + static_cast<int64_t>(idx0) * N + slot, x[0]);
        if (COUNT) nred += 1;
      }
    } else if (mine) {
      float* base = grad + static_cast<int64_t>(idx) * N;
#pragma unroll
      for (int p = 0; p < N; ++p) red_add(base + p, v[p]);
      if (COUNT) nred += N;
    }
  }
}

// CCCL-style baseline (reducers.cpp:177-206): the eligibility check and a
// library warp reduction repeated for every param, lane 0 issuing each RED.
template <int N, bool COUNT>
__device__ __forceinline__ void reduce_cccl(int idx, float* grad, const float (&v)[N],
                                            bool active, int lane, uint32_t& nred,
                                            unsigned ballot) {
  using WR = cub::WarpReduce<float>;
  typename WR::TempStorage tmp;  // shuffle-based for a full warp: no smem traffic
#pragma unroll
  for (int p = 0; p < N; ++p) {
    const int idx0 = __shfl_sync(kFull, idx, 0);
    const bool same = __all_sync(kFull, idx == idx0) && idx0 >= 0;
    const int cnt = __popc(__ballot_sync(kFull, active));
    if (same && cnt > 0) {
      const float s = WR(tmp).Sum(v[p]);
      if (lane == 0) {
        red_add(grad + static_cast<int64_t>(idx0) * N + p, s);
        if (COUNT) nred += 1;
      }
    } else if (active) {
      red_add(grad + static_cast<int64_t>(idx) * N + p, v[p]);
      if (COUNT) nred += 1;
    }
  }
  (void)ballot;
}

// Warp-sum a per-lane counter and add it to a global u64 once per warp.
__device__ __forceinline__ void flush_count(unsigned long long* ctr, uint32_t n, int lane) {
  unsigned long long s = n;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
  if (lane == 0 && s) atomicAdd(ctr, s);
}

}  // namespace dw
