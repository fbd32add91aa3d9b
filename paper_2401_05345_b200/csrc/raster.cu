// Host orchestration of one view: render_forward / render_backward.
//
// Per-view device state lives in grow-only HBM buffers owned by the
// dw_rasterizer handle, so a training loop re-renders without reallocating:
//   per Gaussian: means2D f32x2, depth, radius, conic+opacity f32x4,
//                 rgb f32x4, tiles_touched u32, depth keys u32 x2 + ids u32
//                 x2 (double-buffered depth sort), inclusive offsets u64
//   per instance: tile ids u32 x2, values u32 x2 (double-buffered tile sort)
//   per tile:     ranges u32x2;  per pixel: final_T f32, n_contrib u32
// Binning uses the hand-written sort of raster_sort.cu (no library calls).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "distwar.cuh"
#include "dw_internal.h"
#include "raster.cuh"

#ifndef DW_SCATTER
// scatter binning (raster_scatter.cu) on by default? A/B on B200 (tools/forward_ab.py,
// profiles/r02/forward_binning_ab.md): C3 forward 0.594 vs 0.598 ms depth-first,
// C5 view 0 0.926 vs 0.910 ms -- a tie, so the depth-first sort stays the default
#define DW_SCATTER 0
#endif
#ifndef DW_TILE_FIRST
#define DW_TILE_FIRST 1  // sort path: duplicate by index, sort by tile, depth-sort per tile
#endif
#ifndef DW_LPT
#define DW_LPT 1  // the backward takes tiles longest-list first (0: row-major)
#endif

namespace {

template <typename T>
void grow(T*& p, size_t& cap, size_t want) {
  if (want <= cap && p) return;
  if (p) DW_CUDA(cudaFree(p));
  p = nullptr;
  const size_t n = std::max<size_t>(want, 1) + std::max<size_t>(want, 1) / 8;
  DW_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), n * sizeof(T)));
  cap = n;
}

// grow() for state that kernels expect zeroed (and leave zeroed) between
// calls; the zeroing is ordered on the stream that will use the buffer (a
// synchronous cudaMemset runs on the legacy default stream, which does not
// order with non-blocking streams)
template <typename T>
void grow_zeroed(T*& p, size_t& cap, size_t want, cudaStream_t s) {
  if (want <= cap && p) return;
  grow(p, cap, want);
  DW_CUDA(cudaMemsetAsync(p, 0, cap * sizeof(T), s));
}

}  // namespace

#ifndef DW_BLOCK_BINNING
#define DW_BLOCK_BINNING 1
#endif

struct dw_rasterizer {
  int P = 0, W = 0, H = 0;
  int64_t num_rendered = 0;
  dw::CamParams cam{};
  int tile_bits = 0;
  bool forward_done = false;

  size_t cap_p = 0, cap_p2 = 0, cap_p3 = 0, cap_p4 = 0, cap_p5 = 0, cap_p6 = 0, cap_p7 = 0;
  float2* means2D = nullptr;
  float* depths = nullptr;
  int* radii = nullptr;
  float4* conic_opacity = nullptr;
  float4* rgb = nullptr;
  uint32_t* tiles_touched = nullptr;
  uint64_t* offsets = nullptr;

  size_t cap_d[4] = {0};
  uint32_t* dkey[2] = {nullptr, nullptr};  // depth keys (double buffer)
  uint32_t* dids[2] = {nullptr, nullptr};  // Gaussian ids (double buffer)
  const uint32_t* order = nullptr;         // Gaussians in (depth, id) order

  size_t cap_i[4] = {0};
  uint32_t* itile[2] = {nullptr, nullptr};  // instance tile ids (double buffer)
  uint32_t* ivals[2] = {nullptr, nullptr};  // instance Gaussian ids
  uint32_t* tiles_sorted = nullptr;
  uint32_t* vals = nullptr;                 // sorted Gaussian ids (the lists)

  size_t cap_t = 0, cap_px = 0, cap_px2 = 0, cap_to = 0;
  uint2* ranges = nullptr;
  uint32_t* tile_order = nullptr;  // tiles, longest list first (the backward's CTA order)
  uint32_t* area_sorted = nullptr; // tiles_touched in depth order (the offsets scan's input)
  size_t cap_as = 0;
  unsigned long long* seg_scratch = nullptr;  // tile-first: long lists' merge buffers (2 x I)
  size_t cap_seg = 0;
  bool dense = false;              // last forward used dense (tile-major) binning
  bool scatter = false;            // last forward used scatter binning (raster_scatter.cu)
  uint32_t* sc_scratch = nullptr;  // scatter binning: per-(segment, tile) counts + totals
  size_t cap_sc = 0;
  float4* packed = nullptr;        // bulk-copy staging: 48-byte staged record per Gaussian
  size_t cap_pk = 0;
  bool bulk = false;               // DW_BULK_STAGING=1: the backward stages by cp.async.bulk
  bool tile_first = false;         // last forward binned tile-first (per-tile depth sort)
  double last_list_mean = -1.0;    // instances per tile of the last counted forward
  static constexpr double kTileFirstMaxMean = 384.0;
  uint2* rects = nullptr;          // dense / block binning: packed tile rectangle + id, depth order
  bool blocked = false;            // last forward built its lists by block binning
  uint2* branges = nullptr;        // block binning: coarse block ranges
  uint32_t* bb_cnt = nullptr;      // block binning: per-(warp, tile) counts + tile totals
  uint32_t* bb_rect_id = nullptr;  // block binning: packed rectangle by Gaussian id
  uint32_t* bb_hist = nullptr;     // block binning, fused level 1: per-(block, tile) counts
  size_t cap_br = 0, cap_bbc = 0, cap_bri = 0, cap_bbh = 0;
  bool bb_fused = false;           // fused level 1 (DW_BB_FUSED=1, <= 256 blocks)
  int* diff = nullptr;             // dense binning: per-segment difference grids + offsets
  size_t cap_r = 0, cap_diff = 0;
  float* final_T = nullptr;
  uint32_t* n_contrib = nullptr;

  size_t cap_tmp = 0, cap_scan = 0, cap_keys = 0;
  unsigned char* tmp = nullptr;
  unsigned char* scan_tmp = nullptr;
  uint64_t* keys_dbg = nullptr;            // u64 keys, materialised on request
  unsigned long long* counters = nullptr;  // [pairs, reds]
  uint64_t* h_total = nullptr;             // pinned

  // host-entry scratch (dw_render_host / dw_render_views_host)
  size_t cap_h[12] = {0};
  float* h_bufs[12] = {nullptr};
  cudaStream_t s_in = nullptr, s_out = nullptr;  // copy streams of the batched host path
  static constexpr int kMaxFwdStreams = 4;
  cudaStream_t s_fwd[kMaxFwdStreams] = {};  // the batched host path's forward streams
  // the batched host path's forward states: a probe state for its first frame
  // and a pool of kWave states the frames of a wave rotate through
  dw_rasterizer* probe = nullptr;
  std::vector<dw_rasterizer*> pool;
  std::vector<cudaEvent_t> pev;  // per pool slot: forward done, dL uploaded, images downloaded
  cudaEvent_t ev[6] = {};

  // Per-stage forward timing (dw_rasterizer_stage_timing): events recorded
  // between the forward's stages. Diagnostic only: an event between two
  // programmatic-dependent launches serialises them, so the stages add up
  // to a little more than the untimed forward.
  static constexpr int kStages = 6;  // preprocess, depth sort, offsets, binning, ranges, blend
  bool stage_timing = false;
  bool stage_valid = false;
  cudaEvent_t st_ev[kStages + 1] = {};
  void stage_mark(int i, cudaStream_t s) {
    if (!stage_timing) return;
    if (!st_ev[0])
      for (auto& e : st_ev) DW_CUDA(cudaEventCreate(&e));
    DW_CUDA(cudaEventRecord(st_ev[i], s));
  }

  void ensure_streams() {
    if (s_in) return;
    DW_CUDA(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
    DW_CUDA(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    for (auto& f : s_fwd) DW_CUDA(cudaStreamCreateWithFlags(&f, cudaStreamNonBlocking));
    for (auto& e : ev) DW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }

  ~dw_rasterizer() {
    void* ps[] = {means2D, depths, radii, conic_opacity, rgb, tiles_touched, offsets, dkey[0],
                  dkey[1], dids[0], dids[1], itile[0], itile[1], ivals[0], ivals[1], ranges,
                  final_T, n_contrib, tmp, scan_tmp, keys_dbg, counters, small_dev,
                  tile_order, rects, diff, area_sorted, seg_scratch, sc_scratch, packed,
                  branges, bb_cnt, bb_rect_id, bb_hist, pad_grad};
    for (void* p : ps)
      if (p) cudaFree(p);
    for (float* p : h_bufs)
      if (p) cudaFree(p);
    if (h_total) cudaFreeHost(h_total);
    if (h_small) cudaFreeHost(h_small);
    if (st_ev[0])
      for (auto& e : st_ev) cudaEventDestroy(e);
    delete probe;
    for (auto* q : pool) delete q;
    for (auto e : pev) cudaEventDestroy(e);
    if (s_in) {
      cudaStreamDestroy(s_in);
      cudaStreamDestroy(s_out);
      for (auto f : s_fwd) cudaStreamDestroy(f);
      for (auto e : ev) cudaEventDestroy(e);
    }
  }

  // no-sync forward state: live instance count + overflow flag on the device
  // one device block [live count, live entries, overflow flag] so the host
  // reads all three with a single copy (and its pinned mirror)
  unsigned long long* small_dev = nullptr;
  unsigned long long* h_small = nullptr;
  unsigned long long* live_dev = nullptr;
  unsigned long long* live_c_dev = nullptr;  // block binning: live level-1 entry count
  unsigned int* overflow_dev = nullptr;
  cudaStream_t last_stream = nullptr;        // stream of the last forward
  bool count_pending = false;  // num_rendered not read back yet (no-sync forward)

  void ensure_small(cudaStream_t s) {
    if (!counters) DW_CUDA(cudaMalloc(&counters, 2 * sizeof(unsigned long long)));
    if (!h_total) DW_CUDA(cudaMallocHost(&h_total, sizeof(uint64_t)));
    if (!small_dev) {
      DW_CUDA(cudaMalloc(&small_dev, 3 * sizeof(unsigned long long)));
      DW_CUDA(cudaMallocHost(&h_small, 3 * sizeof(unsigned long long)));
      live_dev = small_dev;
      live_c_dev = small_dev + 1;
      overflow_dev = reinterpret_cast<unsigned int*>(small_dev + 2);
      DW_CUDA(cudaMemsetAsync(small_dev, 0, 3 * sizeof(unsigned long long), s));
    }
  }

  // Dense-binning choice: DW_DENSE_BINNING=0/1 forces it, else the heuristic.
  static bool dense_env_ok(bool heuristic) {
    const char* env = std::getenv("DW_DENSE_BINNING");
    return env && *env ? *env == '1' : heuristic;
  }

  // Block binning's entry scan (depth sort done: order, area_sorted = packed
  // rectangles in depth order): entries into itile[0] / ivals[0], totals to
  // offsets[P-1]. bb_entry_cap: the entries those buffers held.
  uint64_t bb_entry_cap = 0;
  void bb_entries_scan(cudaStream_t s, bool skip_entries) {
    if (bb_fused) {  // counts only: the entries are written after the buffers are sized
      bb_entry_cap = ~uint64_t(0);
      DW_CUDA(cudaMemsetAsync(offsets + P - 1, 0, sizeof(uint64_t), s));
      dw::launch_bb_hist(area_sorted, P, cam, bb_hist, offsets + P - 1, s);
      return;
    }
    // (a frame expected to take dense binning writes no entries; should it
    // not, the synced path rescans)
    bb_entry_cap = skip_entries ? 0 : static_cast<uint64_t>(std::min(cap_i[0], cap_i[2]));
    dw::block_entries_scan(area_sorted, order, P, offsets, scan_tmp,
                           dw::block_binning_nbx(cam.tiles_x), itile[0], ivals[0], bb_entry_cap,
                           s);
  }

  // Pre-size every buffer (no allocation happens in a later forward/backward
  // that stays within these sizes -- required before CUDA-graph capture).
  // nv > 1: for frames of nv stacked views (forward_views) -- P_ scene
  // Gaussians, W_ x H_ per view, max_instances over the whole frame.
  void reserve(int32_t P_, int32_t W_, int32_t H_, int64_t max_instances, int nv = 1) {
    if (P_ < 0 || W_ < 1 || H_ < 1 || max_instances < 0 || nv < 1 ||
        static_cast<int64_t>(P_) * nv > INT32_MAX)
      throw std::invalid_argument("invalid reserve sizes");
    const size_t np = static_cast<size_t>(std::max(P_ * nv, 1));
    const size_t npx = static_cast<size_t>(W_) * H_ * nv;
    const size_t ntiles = static_cast<size_t>((W_ + dw::kTile - 1) / dw::kTile) *
                          (nv * ((H_ + dw::kTile - 1) / dw::kTile));
    grow(means2D, cap_p, np);
    grow(depths, cap_p2, np);
    grow(radii, cap_p3, np);
    grow(conic_opacity, cap_p4, np);
    grow(rgb, cap_p5, np);
    grow(tiles_touched, cap_p6, np);
    grow(offsets, cap_p7, np);
    for (int b = 0; b < 2; ++b) {
      grow(dkey[b], cap_d[b], np);
      grow(dids[b], cap_d[2 + b], np);
    }
    grow(area_sorted, cap_as, np);
    grow_zeroed(scan_tmp, cap_scan, dw::scan_temp_bytes(static_cast<int64_t>(np)), nullptr);
    grow(ranges, cap_t, ntiles);
    grow(tile_order, cap_to, ntiles);
    grow(final_T, cap_px, npx);
    grow(n_contrib, cap_px2, npx);
    const size_t ni = static_cast<size_t>(std::max<int64_t>(max_instances, 1));
    for (int b = 0; b < 2; ++b) {
      grow(itile[b], cap_i[b], ni);
      grow(ivals[b], cap_i[2 + b], ni);
    }
    grow(seg_scratch, cap_seg, 2 * ni);
    if (nv == 1 && dw::scatter_binning_fits(static_cast<int>(ntiles)))
      grow(sc_scratch, cap_sc, dw::scatter_scratch_words(P_, static_cast<int>(ntiles)));
    const int tx = (W_ + dw::kTile - 1) / dw::kTile, ty = nv * ((H_ + dw::kTile - 1) / dw::kTile);
    if (dw::dense_binning_fits(tx, ty)) {  // dense binning allocates nothing in the forward
      grow(rects, cap_r, np);
      grow(diff, cap_diff, dw::dense_scratch_words(tx, ty));
    }
    if (dw::block_binning_fits(tx, ty)) {  // nor does block binning
      grow(rects, cap_r, np);
      grow(branges, cap_br, static_cast<size_t>(dw::block_binning_blocks(tx, ty)));
      grow(bb_cnt, cap_bbc, dw::block_binning_count_words(tx, ty));
      grow(bb_rect_id, cap_bri, np);
      if (dw::block_binning_blocks(tx, ty) <= 256)
        grow(bb_hist, cap_bbh, dw::block_binning_hist_words(static_cast<int64_t>(np)));
    }
    ensure_tmp(std::max(dw::radix_sort_temp_bytes(static_cast<int64_t>(np)),
                        dw::radix_sort_temp_bytes(static_cast<int64_t>(std::min(cap_i[0], cap_i[2])))));
    ensure_small(nullptr);
    // reserve() takes no stream: the zeroing above ran on the legacy stream,
    // so complete it before any stream (blocking or not) uses the buffers
    DW_CUDA(cudaDeviceSynchronize());
  }

  // Host view of the instance count (reads the device value back after a
  // no-sync forward); overflow = the no-sync forward exceeded the reserve.
  int64_t resolve_count(bool* overflowed) {
    unsigned int ovf = 0;
    if (count_pending) {
      // one copy on the forward's stream (ordered after its kernels)
      DW_CUDA(cudaMemcpyAsync(h_small, small_dev, 3 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, last_stream));
      DW_CUDA(cudaStreamSynchronize(last_stream));
      std::memcpy(&ovf, h_small + 2, sizeof(ovf));
      num_rendered = static_cast<int64_t>(h_small[0]);
      count_pending = false;
      last_overflow = ovf != 0;
      if (blocked && !last_overflow) last_entries = static_cast<int64_t>(h_small[1]);
    }
    if (overflowed) *overflowed = last_overflow;
    return num_rendered;
  }
  bool last_overflow = false;
  int64_t last_entries = -1;  // block binning: level-1 entries of the last counted frame

  void forward(int32_t P_, const float* means3D, const float* scales, const float* rotations,
               const float* opacities, const float* colors, const dw_camera& c, float* out_color,
               int32_t* radii_out, cudaStream_t s, bool nosync = false,
               bool sticky_overflow = false) {
    forward_views(P_, means3D, scales, rotations, opacities, colors, &c, 1, out_color, radii_out,
                  s, nosync, sticky_overflow);
  }

  // Views stacked into one frame (nv > 1: the batched host path). The nv
  // views of one scene share every launch of the forward -- one preprocess per
  // view into consecutive id ranges [v P, (v + 1) P), then ONE depth sort, one
  // entry scan, one block binning and one blend over a frame whose tile rows
  // [v rows, (v + 1) rows) are view v. A tile holds only its own view's
  // Gaussians (the rectangles never leave the view's rows) in that view's
  // (depth, id) order -- the global sort interleaves views but keeps each
  // view's relative order -- so every tile's list is the single-view list with
  // ids offset by v P, bit for bit. The latency-bound binning launches then do
  // nv views' work each (a 1080p frame's block-binning kernels run one wave
  // either way). Images / final_T / n_contrib (and the backward's dL/dpixel)
  // are [nv][...] arrays; the backward adds view v's gradients at id - v P.
  // Requires block binning (its rectangle packing bounds the frame to 255 tile
  // rows) and one background colour.
  static constexpr int kMaxStack = 3;
  int nviews = 1;
  int P_scene = 0;           // scene Gaussians (P = nviews * P_scene)
  int nviews_reserved = 0;   // views per frame the last reserve() sized for
  bool stack_unfit = false;  // the last stacked frame would have preferred dense binning
  static int stack_limit(int W_, int H_) {
    const int tx = (W_ + dw::kTile - 1) / dw::kTile, ty = (H_ + dw::kTile - 1) / dw::kTile;
    if (!dw::block_binning_fits(tx, ty)) return 1;
    return std::max(1, std::min(kMaxStack, 255 / ty));
  }
  void forward_views(int32_t P_, const float* means3D, const float* scales, const float* rotations,
                     const float* opacities, const float* colors, const dw_camera* cs, int nv,
                     float* out_color, int32_t* radii_out, cudaStream_t s, bool nosync = false,
                     bool sticky_overflow = false) {
    last_overflow = false;
    last_stream = s;
    const dw_camera& c = cs[0];
    if (P_ < 0) throw std::invalid_argument("P must be >= 0");
    if (c.width < 1 || c.height < 1) throw std::invalid_argument("camera size must be >= 1");
    if (nv < 1 || nv > stack_limit(c.width, c.height))
      throw std::invalid_argument("too many stacked views for this image size");
    for (int v = 0; v < nv; ++v) {
      if (!(cs[v].tan_fovx > 0.0f) || !(cs[v].tan_fovy > 0.0f))
        throw std::invalid_argument("tan_fov must be > 0");
      if (cs[v].width != c.width || cs[v].height != c.height ||
          std::memcmp(cs[v].bg, c.bg, sizeof(c.bg)) != 0)
        throw std::invalid_argument("stacked views must share image size and background");
    }
    if (static_cast<int64_t>(P_) * nv > INT32_MAX)
      throw std::invalid_argument("stacked frame has too many Gaussians");
    nviews = nv;
    stack_unfit = false;
    P_scene = P_;
    const int Ps = P_;
    P = P_ * nv;
    W = c.width;
    H = c.height;
    std::memcpy(cam.vm, c.viewmatrix, sizeof(cam.vm));
    std::memcpy(cam.pm, c.projmatrix, sizeof(cam.pm));
    cam.tan_fovx = c.tan_fovx;
    cam.tan_fovy = c.tan_fovy;
    std::memcpy(cam.bg, c.bg, sizeof(cam.bg));
    cam.scale_modifier = c.scale_modifier;
    cam.W = W;
    cam.H = H;
    cam.tiles_x = (W + dw::kTile - 1) / dw::kTile;
    cam.rows_v = (H + dw::kTile - 1) / dw::kTile;
    cam.tiles_y = nv * cam.rows_v;
    cam.vstride = nv > 1 ? Ps : 0;
    const int ntiles = cam.tiles_x * cam.tiles_y;
    tile_bits = 0;
    while ((1 << tile_bits) < ntiles) ++tile_bits;

    const size_t np = static_cast<size_t>(std::max(P, 1));
    grow(means2D, cap_p, np);
    grow(depths, cap_p2, np);
    grow(radii, cap_p3, np);
    grow(conic_opacity, cap_p4, np);
    grow(rgb, cap_p5, np);
    grow(tiles_touched, cap_p6, np);
    grow(offsets, cap_p7, np);
    grow(ranges, cap_t, static_cast<size_t>(ntiles));
    grow(tile_order, cap_to, static_cast<size_t>(ntiles));
    grow(final_T, cap_px, static_cast<size_t>(W) * H * nv);
    grow(n_contrib, cap_px2, static_cast<size_t>(W) * H * nv);
    ensure_small(s);

    for (int b = 0; b < 2; ++b) {
      grow(dkey[b], cap_d[b], np);
      grow(dids[b], cap_d[2 + b], np);
    }
    grow(area_sorted, cap_as, np);
    grow_zeroed(scan_tmp, cap_scan, dw::scan_temp_bytes(P), s);

    // Tile-first binning (default): instances duplicated in index order, sorted
    // by tile, each tile's list then depth-sorted on chip. Depth-first: all P
    // Gaussians depth-sorted first (also what dense binning needs).
    // Tile-first pays only for short lists (the per-tile sort is a bitonic
    // network: C2, ~190 per tile: 0.240 -> 0.220 ms; C3, ~570: 0.655 -> 0.848),
    // so it is chosen from the previous frame's mean list length.
    const char* tf_env = std::getenv("DW_TILE_FIRST");  // "0" / "1" force
    // Scatter binning (DW_SCATTER=1, or the compile-time default): per-tile
    // counts, placement, on-chip depth sort per tile -- no global sort at
    // all (raster_scatter.cu). A forced tile-first path turns it off.
    const char* sc_env = std::getenv("DW_SCATTER");
    scatter = nv == 1 && (sc_env && *sc_env ? *sc_env == '1' : DW_SCATTER != 0) &&
              !(tf_env && *tf_env == '1') && dw::scatter_binning_fits(ntiles);
    tile_first = nv == 1 && !scatter &&
                 (tf_env && *tf_env ? *tf_env == '1'
                                    : DW_TILE_FIRST != 0 && last_list_mean >= 0.0 &&
                                          last_list_mean < kTileFirstMaxMean);
    // Block binning (default on the depth-first path): the lists through
    // coarse 8x4-tile blocks (raster_blockbin.cu); DW_BLOCK_BINNING=0 selects
    // the duplicate + tile-sort construction (same output). Block totals must
    // stay < 2^30 for its packed scan: not used once a frame came near that.
    const char* bb_env = std::getenv("DW_BLOCK_BINNING");
    const bool block_mode = !tile_first && !scatter &&
                            (nv > 1 || (bb_env && *bb_env ? *bb_env == '1' : DW_BLOCK_BINNING != 0)) &&
                            dw::block_binning_fits(cam.tiles_x, cam.tiles_y) &&
                            last_list_mean * ntiles < static_cast<double>(1 << 29) &&
                            static_cast<int64_t>(P) < (int64_t(1) << 29);
    if (nv > 1 && !block_mode)
      throw std::invalid_argument("stacked views need block binning (list too long for it)");
    // the depth-first paths' sort keys come straight out of the preprocess
    const bool keys_ready = !tile_first && !scatter;
    stage_valid = stage_timing;
    stage_mark(0, s);
    const char* bulk_env = std::getenv("DW_BULK_STAGING");
    bulk = nv == 1 && bulk_env && *bulk_env == '1';
    if (bulk) grow(packed, cap_pk, 3 * np);
    if (block_mode) {
      const char* fe = std::getenv("DW_BB_FUSED");
      // (not kept by default: the per-entry shared-memory atomics of its two
      // counting sweeps cost what the radix pass saved -- profiles/r02/ab/bb_fused.md)
      bb_fused = fe && *fe == '1' && dw::block_binning_blocks(cam.tiles_x, cam.tiles_y) <= 256;
      grow(bb_rect_id, cap_bri, np);
      if (bb_fused) grow(bb_hist, cap_bbh, dw::block_binning_hist_words(P));
    }
    for (int v = 0; v < nv; ++v) {  // view v: ids [v Ps, (v + 1) Ps), tile rows from v rows_v
      dw::CamParams cv = cam;
      std::memcpy(cv.vm, cs[v].viewmatrix, sizeof(cv.vm));
      std::memcpy(cv.pm, cs[v].projmatrix, sizeof(cv.pm));
      cv.tan_fovx = cs[v].tan_fovx;
      cv.tan_fovy = cs[v].tan_fovy;
      cv.scale_modifier = cs[v].scale_modifier;
      cv.tiles_y = cam.rows_v;
      const size_t o = static_cast<size_t>(v) * Ps;
      dw::launch_preprocess(Ps, means3D, scales, rotations, opacities, colors, cv, means2D + o,
                            depths + o, radii + o, conic_opacity + o, rgb + o, tiles_touched + o,
                            keys_ready ? dkey[0] + o : nullptr, keys_ready ? dids[0] + o : nullptr,
                            s, bulk ? packed : nullptr, block_mode ? bb_rect_id + o : nullptr,
                            v * cam.rows_v, static_cast<uint32_t>(o));
    }
    stage_mark(1, s);
    // Instance count: read back (one host sync) to size the buffers, or --
    // nosync -- kept on the device against the reserved capacity
    // (dw_rasterizer_reserve), so the whole forward is graph-capturable.
    int64_t n_grid = 0;                        // element count the grids are sized for
    const unsigned long long* n_dev = nullptr;  // live count on the device (nosync)
    int64_t n_entries = 0;                      // block binning: level-1 entries (or capacity)
    const unsigned long long* nc_dev = nullptr;  // block binning: live entries (nosync)
    num_rendered = 0;
    count_pending = false;
    bool depth_sorted = false;
    auto depth_sort = [&](bool with_area) {
      if (!keys_ready) dw::launch_depth_keys(P, depths, radii, dkey[0], dids[0], s);
      ensure_tmp(dw::radix_sort_temp_bytes(P));
      // (its last pass can also lay tiles_touched -- block binning: the packed
      // rectangles -- out in that order: area_sorted)
      const uint32_t* payload = block_mode ? bb_rect_id : tiles_touched;
      order = dids[dw::radix_sort_pairs(dkey, dids, P, 32, tmp, s, nullptr,
                                        with_area ? payload : nullptr, area_sorted)];
      depth_sorted = true;
    };
    if (P > 0) {
      if (tile_first || scatter) {
        stage_mark(2, s);  // no depth sort on these paths
        // instance offsets in index order
        dw::inclusive_scan_gather(tiles_touched, nullptr, P, offsets, scan_tmp, s);
      } else if (block_mode) {
        // 1. Gaussians in (depth, id) order; one scan over their packed
        // rectangles in that order gives both the tile and the block offsets
        depth_sort(true);
        stage_mark(2, s);
        bb_entries_scan(s, dense && !nosync);  // dense: the previous frame's choice
      } else {
        // 1. Gaussians in (depth, id) order: stable 32-bit LSD sort
        depth_sort(true);
        stage_mark(2, s);
        // instance offsets in that order (a sequential scan, no gather)
        dw::inclusive_scan_gather(area_sorted, nullptr, P, offsets, scan_tmp, s);
      }
      if (nosync) {
        if (cap_i[0] == 0 || cap_i[2] == 0)
          throw std::invalid_argument("no-sync forward needs dw_rasterizer_reserve first");
        n_grid = static_cast<int64_t>(std::min(cap_i[0], cap_i[2]));
        if (block_mode) {
          // entries <= instances; the level-1 sort's grid is sized from the
          // last counted frame's entries (+25 %) when known (fused: no sort,
          // the entries need only fit the buffers)
          n_entries = last_entries > 0 && !bb_fused
                          ? std::min<int64_t>(n_grid, last_entries + last_entries / 4 + 4096)
                          : n_grid;
          dw::launch_bb_clamp(offsets, P, static_cast<uint64_t>(n_grid),
                              static_cast<uint64_t>(n_entries), live_dev, live_c_dev,
                              overflow_dev, sticky_overflow, s);
          nc_dev = live_c_dev;
        } else {
          dw::launch_clamp_total(offsets, P, static_cast<uint64_t>(n_grid), live_dev,
                                 overflow_dev, sticky_overflow, s);
        }
        n_dev = live_dev;
        count_pending = true;
      } else {
        DW_CUDA(cudaMemcpyAsync(h_total, offsets + P - 1, sizeof(uint64_t),
                                cudaMemcpyDeviceToHost, s));
        DW_CUDA(cudaStreamSynchronize(s));
        num_rendered = static_cast<int64_t>(*h_total);
        if (block_mode) {  // (blocks << 34 | tiles)
          n_entries = static_cast<int64_t>(*h_total >> dw::kBBTileBits);
          num_rendered = static_cast<int64_t>(*h_total & dw::kBBTileMask);
          last_entries = n_entries;
          // the scan wrote the entries into buffers that must hold every
          // instance (the later grows keep them): else grow and rescan
          const bool will_dense =
              nv == 1 && num_rendered > 0 && dw::dense_binning_fits(cam.tiles_x, cam.tiles_y) &&
              dense_env_ok(static_cast<double>(P) * ntiles <= 4.0 * static_cast<double>(num_rendered));
          // a stacked frame of a scene whose single views take dense binning
          // (large rectangles): the caller goes back to one view per frame
          if (nv > 1)
            stack_unfit = num_rendered > 0 && dw::dense_binning_fits(cam.tiles_x, cam.rows_v) &&
                          dense_env_ok(static_cast<double>(Ps) * cam.tiles_x * cam.rows_v <=
                                       4.0 * static_cast<double>(num_rendered) / nv);
          if (!will_dense && static_cast<uint64_t>(num_rendered) > bb_entry_cap) {
            const size_t ni = static_cast<size_t>(num_rendered);
            for (int b = 0; b < 2; ++b) {
              grow(itile[b], cap_i[b], ni);
              grow(ivals[b], cap_i[2 + b], ni);
            }
            bb_entries_scan(s, false);
          }
        }
        n_grid = num_rendered;
        last_list_mean = static_cast<double>(num_rendered) / ntiles;
      }
    }
    if (P == 0) {
      stage_mark(2, s);
    }
    stage_mark(3, s);
    if (n_grid >= (int64_t(1) << 32)) throw std::runtime_error("more than 2^32 tile instances");
    const size_t ni = static_cast<size_t>(std::max<int64_t>(n_grid, 1));
    for (int b = 0; b < 2; ++b) {
      grow(itile[b], cap_i[b], ni);
      grow(ivals[b], cap_i[2 + b], ni);
    }
    tiles_sorted = itile[0];
    vals = ivals[0];
    blocked = false;
    // Dense scenes (large tile rectangles: P x tiles <= 4 x instances) build the
    // per-tile lists directly; the rest duplicate + radix-sort (same output).
    dense = nv == 1 && n_grid > 0 && dw::dense_binning_fits(cam.tiles_x, cam.tiles_y) &&
            dense_env_ok(static_cast<double>(P) * ntiles <= 4.0 * static_cast<double>(n_grid));
    if (dense) {
      grow(rects, cap_r, static_cast<size_t>(P));
      grow(diff, cap_diff, dw::dense_scratch_words(cam.tiles_x, cam.tiles_y));
      if (!depth_sorted) depth_sort(false);
      dw::launch_dense_binning(P, order, means2D, radii, cam, rects, diff, ranges, ivals[0],
                               n_dev, static_cast<uint64_t>(n_grid), s);
    } else if (scatter && n_grid > 0) {
      grow(sc_scratch, cap_sc, dw::scatter_scratch_words(P, ntiles));
      grow(seg_scratch, cap_seg, 2 * static_cast<size_t>(n_grid));
      dw::launch_scatter_binning(P, means2D, radii, depths, cam, sc_scratch, ranges, ivals[0],
                                 seg_scratch, n_grid, n_dev, s);
    } else if (block_mode && n_grid > 0) {
      // 2. entries per coarse block, sorted by block; 3. per-tile lists
      const int nb = dw::block_binning_blocks(cam.tiles_x, cam.tiles_y);
      grow(branges, cap_br, static_cast<size_t>(nb));
      grow(bb_cnt, cap_bbc, dw::block_binning_count_words(cam.tiles_x, cam.tiles_y));
      grow(seg_scratch, cap_seg, 2 * static_cast<size_t>(std::max<int64_t>(n_grid, 1)));
      // the sorted entries' rectangles land in seg_scratch (>= n_grid >= entries words)
      if (bb_fused) {
        dw::launch_block_binning_fused(area_sorted, order, P, cam, bb_hist, ivals,
                                       static_cast<uint64_t>(n_grid),
                                       reinterpret_cast<uint32_t*>(seg_scratch), branges, bb_cnt,
                                       ranges, &vals, n_dev, nc_dev, s);
      } else {
        ensure_tmp(dw::radix_sort_temp_bytes(std::max<int64_t>(n_entries, 1)));
        dw::launch_block_binning(bb_rect_id, cam, itile, ivals, n_entries, tmp,
                                 reinterpret_cast<uint32_t*>(seg_scratch), branges, bb_cnt,
                                 ranges, &vals, n_dev, nc_dev, s);
      }
      tiles_sorted = nullptr;
      blocked = true;
    } else if (n_grid > 0) {
      // 2. duplicate (index order, or depth order), 3. stable sort by tile id
      dw::launch_duplicate_sorted(P, tile_first ? nullptr : order, means2D, radii, offsets, cam,
                                  itile[0], ivals[0], static_cast<uint64_t>(n_grid), s);
      ensure_tmp(dw::radix_sort_temp_bytes(n_grid));
      const int cur = dw::radix_sort_pairs(itile, ivals, n_grid, tile_bits, tmp, s, n_dev);
      tiles_sorted = itile[cur];
      vals = ivals[cur];
    }
    stage_mark(4, s);
    const bool scattered = scatter && !dense && n_grid > 0;  // ranges already written
    if (!scattered) scatter = false;
    if (!dense && !scattered && !blocked)
      dw::launch_ranges_u32(n_grid, tiles_sorted, ranges, ntiles, s, n_dev);
    if (!dense && !scattered && tile_first && n_grid > 0) {
      // 4. every tile's list (index order) -> (depth, index) order
      grow(seg_scratch, cap_seg, 2 * static_cast<size_t>(n_grid));
      dw::launch_segsort_depth(ranges, depths, vals, seg_scratch, n_grid, ntiles, s);
    }
    order_stale = true;  // the backward derives its tile order from these ranges
    stage_mark(5, s);
    dw::launch_forward_impl(cam, ranges, vals, means2D, conic_opacity, rgb, nullptr, final_T,
                            n_contrib, out_color, s);
    stage_mark(6, s);
    if (radii_out && P > 0)  // (a stacked frame: [nv][P] radii)
      DW_CUDA(cudaMemcpyAsync(radii_out, radii, sizeof(int) * P, cudaMemcpyDeviceToDevice, s));
    forward_done = true;
  }

  // grad_stride 12: grad is a padded [P_scene][12] accumulation buffer (the
  // batch path, raster_backward_views), SW-B / SW-S only.
  void backward(const float* dL_dpixels, int policy, int thr, float* grad, uint64_t* pairs_out,
                cudaStream_t s, bool chained = false, int grad_stride = dw::kNParam) {
    if (!forward_done) throw std::invalid_argument("render_backward before render_forward");
    if (policy == DW_POLICY_HW_ATOMRED || policy < 0 || policy > 4)
      throw std::invalid_argument("policy has no B200 kernel (hw_atomred is simulated hardware)");
    if (thr < 0 || thr > 33) throw std::invalid_argument("balance threshold out of range 0..33");
    if (P == 0) {
      if (pairs_out) *pairs_out = 0;
      return;
    }
    unsigned long long* ctr = nullptr;
    if (pairs_out) {
      DW_CUDA(cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned long long), s));
      ctr = counters;
    }
    // A chained launch skips the wait for the previous kernel, so it launches
    // nothing before itself, and takes the tiles in their natural (row-major)
    // order: longest-list-first only shortens a lone launch's last wave, which
    // a chain overlaps anyway (C5: 0.7496 vs 0.7493 ms per view), while
    // neighbouring tiles running together re-read far less -- DRAM reads of
    // the C5 view 0 backward 439 MB in LPT order vs 339 MB (= the algorithmic
    // bytes) in row order (profiles/r02/ab/chained_backward.md).
    if (!chained) ensure_order(s);
    dw::launch_backward_impl(cam, ranges, vals, means2D, conic_opacity, rgb,
                             chained ? nullptr : order_or_null(),
                             final_T, n_contrib, dL_dpixels, policy, thr, grad, ctr, s,
                             bulk ? packed : nullptr, chained && !ctr, grad_stride);
    if (pairs_out) {
      unsigned long long h[2];
      DW_CUDA(cudaMemcpyAsync(h, counters, sizeof(h), cudaMemcpyDeviceToHost, s));
      DW_CUDA(cudaStreamSynchronize(s));
      *pairs_out = h[0];
      last_reds = h[1];
    }
  }

  uint64_t last_reds = 0;

  void ensure_tmp(size_t bytes) { grow(tmp, cap_tmp, bytes); }
  const uint32_t* order_or_null() const { return DW_LPT ? tile_order : nullptr; }
  // Longest-list-first tile order of the last forward's ranges, computed once
  // by the first backward after it (any permutation is correct; this one
  // shortens the backward's last wave: C2 0.156 -> 0.148 ms, C3 -1 %).
  bool order_stale = true;
  void ensure_order(cudaStream_t s) {
    if (!DW_LPT || !order_stale) return;
    dw::launch_tile_order(ranges, cam.tiles_x * cam.tiles_y, tile_order, s);
    order_stale = false;
  }

  // padded [P][12] gradient accumulation of the batch paths, kept zeroed
  // between batches by launch_fold_rows; pad_dirty: a batch started adding
  // into it and did not fold (an error between the two) -- zero it again
  float* pad_grad = nullptr;
  size_t cap_pad = 0;
  bool pad_dirty = false;
  float* padded_grad(int64_t P_, cudaStream_t s) {
    grow_zeroed(pad_grad, cap_pad, static_cast<size_t>(std::max<int64_t>(P_, 1)) * 12, s);
    if (pad_dirty) DW_CUDA(cudaMemsetAsync(pad_grad, 0, cap_pad * sizeof(float), s));
    pad_dirty = true;
    return pad_grad;
  }
  void fold_padded(int64_t P_, float* grad, cudaStream_t s) {
    dw::launch_fold_rows(P_, pad_grad, grad, s);
    pad_dirty = false;
  }

  float* host_scratch(int slot, size_t n) {
    grow(h_bufs[slot], cap_h[slot], n);
    return h_bufs[slot];
  }
};

namespace dw {

// SM count of the current device, cached per device (thread-safe: a racing
// first query just stores the same value twice).
int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  DW_CUDA(cudaGetDevice(&dev));
  int n = (dev >= 0 && dev < 64) ? cache[dev].load(std::memory_order_relaxed) : 0;
  if (!n) {
    DW_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    if (dev >= 0 && dev < 64) cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

}  // namespace dw

// Entry points used by capi.cpp.
namespace dw {

void raster_forward(dw_rasterizer* r, int32_t P, const float* m, const float* sc, const float* rot,
                    const float* op, const float* col, const dw_camera* cam, float* out,
                    int32_t* radii, int64_t* nr, cudaStream_t s, bool nosync) {
  r->forward(P, m, sc, rot, op, col, *cam, out, radii, s, nosync);
  if (nr) *nr = nosync ? -1 : r->num_rendered;
}

void raster_forward_views(dw_rasterizer* r, int32_t P, const float* m, const float* sc,
                          const float* rot, const float* op, const float* col,
                          const dw_camera* cams, int32_t nv, float* out, int64_t* nr,
                          cudaStream_t s) {
  r->forward_views(P, m, sc, rot, op, col, cams, nv, out, nullptr, s);
  if (nr) *nr = r->num_rendered;
}

int raster_max_stacked_views(int32_t W, int32_t H) { return dw_rasterizer::stack_limit(W, H); }

// The backwards of n rendered views of one scene (one rasterizer each) added
// into grad[P][9] as one chain: the first launch waits for the stream, the
// rest are chained (no wait for the previous grid). SW-B / SW-S accumulate
// into a padded [P][12] buffer (16-byte aligned rows: the per-lane fallback
// is v4 + v4 + scalar with no phase switch; C5 chained 0.745 -> 0.714 ms per
// view, profiles/r02/ab/chained_backward.md) folded into grad at the end.
bool padded_rows_ok(int policy, dw_rasterizer* const* rs, int n) {
  if (policy != kSwB && policy != kSwS) return false;
  for (int k = 0; k < n; ++k)
    if (rs[k]->bulk) return false;  // bulk-copy staging keeps the [P][9] layout
  return true;
}

void raster_backward_views(dw_rasterizer* const* rs, const float* const* dLs, int32_t n,
                           int policy, int thr, float* grad, cudaStream_t s) {
  if (n < 1) throw std::invalid_argument("need at least one view");
  for (int k = 0; k < n; ++k) {
    if (!rs[k] || !dLs[k]) throw std::invalid_argument("null argument");
    if (!rs[k]->forward_done) throw std::invalid_argument("render_backward before render_forward");
    if (rs[k]->P_scene != rs[0]->P_scene)
      throw std::invalid_argument("the views of a batch must render one scene");
  }
  const int Ps = rs[0]->P_scene;
  if (Ps == 0) return;
  const bool pad = padded_rows_ok(policy, rs, n);
  float* acc = pad ? rs[0]->padded_grad(Ps, s) : grad;
  for (int k = 0; k < n; ++k)
    rs[k]->backward(dLs[k], policy, thr, acc, nullptr, s, /*chained=*/k > 0, pad ? 12 : kNParam);
  if (pad) rs[0]->fold_padded(Ps, grad, s);
}

void raster_backward(dw_rasterizer* r, const float* dL, int policy, int thr, float* grad,
                     uint64_t* pairs, cudaStream_t s, bool chained) {
  r->backward(dL, policy, thr, grad, pairs, s, chained);
}

uint64_t raster_last_reds(const dw_rasterizer* r) { return r->last_reds; }

void raster_stage_timing(dw_rasterizer* r, bool on) { r->stage_timing = on; }

int raster_stage_ms(dw_rasterizer* r, double* out, int cap) {
  if (!r->stage_valid || !r->st_ev[0]) throw std::invalid_argument("no stage-timed forward");
  DW_CUDA(cudaEventSynchronize(r->st_ev[dw_rasterizer::kStages]));
  const int n = std::min(cap, dw_rasterizer::kStages);
  for (int i = 0; i < n; ++i) {
    float ms = 0;
    DW_CUDA(cudaEventElapsedTime(&ms, r->st_ev[i], r->st_ev[i + 1]));
    out[i] = ms;
  }
  return n;
}

void raster_reserve(dw_rasterizer* r, int32_t P, int32_t W, int32_t H, int64_t max_instances) {
  r->reserve(P, W, H, max_instances);
}

int64_t raster_resolve(dw_rasterizer* r, bool* overflowed) { return r->resolve_count(overflowed); }

// SW-B backward that also taps its WarpRecords into a host
// trace: records sorted by (warp, descending list position) -- the order
// each warp executed them; prim = the warp-uniform Gaussian id in all 32
// lanes; grads lane-major f64 with zeros in inactive lanes (workload.hpp:41-65).
dw::HostTrace raster_backward_tap(dw_rasterizer* r, const float* dL, int thr, float* grad,
                                  int64_t max_records, int64_t* total, cudaStream_t s) {
  if (!r->forward_done) throw std::invalid_argument("render_backward before render_forward");
  if (r->nviews != 1) throw std::invalid_argument("the tap takes a single-view forward");
  if (max_records < 0) throw std::invalid_argument("max_records must be >= 0");
  const size_t cap = static_cast<size_t>(std::max<int64_t>(max_records, 1));
  TapBuf tb;
  tb.cap = static_cast<unsigned long long>(max_records);
  DW_CUDA(cudaMalloc(&tb.count, sizeof(unsigned long long)));
  DW_CUDA(cudaMalloc(&tb.warp_id, cap * sizeof(int32_t)));
  DW_CUDA(cudaMalloc(&tb.iteration, cap * sizeof(int32_t)));
  DW_CUDA(cudaMalloc(&tb.active, cap * sizeof(uint32_t)));
  DW_CUDA(cudaMalloc(&tb.prim, cap * 32 * sizeof(int32_t)));
  DW_CUDA(cudaMalloc(&tb.vals, cap * 32 * kNParam * sizeof(float)));
  struct Free {
    TapBuf& t;
    ~Free() {
      cudaFree(t.count); cudaFree(t.warp_id); cudaFree(t.iteration); cudaFree(t.active);
      cudaFree(t.prim); cudaFree(t.vals);
    }
  } guard{tb};
  DW_CUDA(cudaMemsetAsync(tb.count, 0, sizeof(unsigned long long), s));
  if (r->P > 0) {  // an empty scene has no lists (and no tile order) to walk
    r->ensure_order(s);
    launch_backward_tap(r->cam, r->ranges, r->vals, r->means2D, r->conic_opacity, r->rgb,
                        r->order_or_null(), r->final_T, r->n_contrib, dL, thr, grad, tb, s);
  }
  unsigned long long count = 0;
  DW_CUDA(cudaMemcpyAsync(&count, tb.count, sizeof(count), cudaMemcpyDeviceToHost, s));
  DW_CUDA(cudaStreamSynchronize(s));
  *total = static_cast<int64_t>(count);
  const size_t R = std::min<size_t>(count, static_cast<size_t>(max_records));
  std::vector<int32_t> wid(R), it(R), prim(R * 32);
  std::vector<uint32_t> act(R);
  std::vector<float> vals(R * 32 * kNParam);
  if (R) {
    DW_CUDA(cudaMemcpy(wid.data(), tb.warp_id, R * 4, cudaMemcpyDeviceToHost));
    DW_CUDA(cudaMemcpy(it.data(), tb.iteration, R * 4, cudaMemcpyDeviceToHost));
    DW_CUDA(cudaMemcpy(act.data(), tb.active, R * 4, cudaMemcpyDeviceToHost));
    DW_CUDA(cudaMemcpy(prim.data(), tb.prim, R * 128, cudaMemcpyDeviceToHost));
    DW_CUDA(cudaMemcpy(vals.data(), tb.vals, vals.size() * 4, cudaMemcpyDeviceToHost));
  }
  std::vector<size_t> order(R);
  for (size_t i = 0; i < R; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    return wid[a] != wid[b] ? wid[a] < wid[b] : it[a] > it[b];
  });
  dw::HostTrace t;
  dw::scene_defaults(&t.scene);
  t.scene.num_primitives = std::max(r->P, 1);
  t.scene.params_per_primitive = kNParam;
  t.scene.image_width = r->W;
  t.scene.image_height = r->H;
  t.scene.quantized_values = 0;
  t.warp_id.resize(R);
  t.iteration.resize(R);
  t.active.resize(R);
  t.prim.resize(R * 32);
  t.grads.resize(R * 32 * kNParam);
  for (size_t k = 0; k < R; ++k) {
    const size_t i = order[k];
    t.warp_id[k] = wid[i];
    t.iteration[k] = it[i];
    t.active[k] = act[i];
    for (int l = 0; l < 32; ++l) {
      t.prim[k * 32 + l] = prim[i * 32 + l];
      for (int p = 0; p < kNParam; ++p)
        t.grads[(k * 32 + l) * kNParam + p] = vals[(i * kNParam + p) * 32 + l];
    }
  }
  return t;
}

void raster_preprocess_backward(dw_rasterizer* r, const float* means3D, const float* scales,
                                const float* rotations, const float* grad2d, float* grad3d,
                                cudaStream_t s) {
  if (!r->forward_done) throw std::invalid_argument("preprocess_backward before render_forward");
  if (r->nviews != 1) throw std::invalid_argument("preprocess_backward after a stacked forward");
  launch_preprocess_backward(r->P, means3D, scales, rotations, r->radii, r->cam, grad2d, grad3d, s);
}

void raster_buffer(const dw_rasterizer* r, int which, const void** p, int64_t* count) {
  const int64_t P = r->P, npx = int64_t(r->W) * r->H * r->nviews;
  const int64_t I = const_cast<dw_rasterizer*>(r)->resolve_count(nullptr);
  const int64_t nt = int64_t(r->cam.tiles_x) * r->cam.tiles_y;
  switch (which) {
    case 0: *p = r->means2D; *count = 2 * P; break;
    case 1: *p = r->depths; *count = P; break;
    case 2: *p = r->radii; *count = P; break;
    case 3: *p = r->conic_opacity; *count = 4 * P; break;
    case 4: *p = r->tiles_touched; *count = P; break;
    case 5: {  // (tile << 32 | depth bits) of the sorted instances, built on request
      auto* m = const_cast<dw_rasterizer*>(r);
      grow(m->keys_dbg, m->cap_keys, static_cast<size_t>(std::max<int64_t>(I, 1)));
      const bool no_tiles = r->dense || r->scatter || r->blocked;  // no tile-id array: from the ranges
      if (no_tiles)
        launch_tiles_from_ranges(r->ranges, r->cam.tiles_x * r->cam.tiles_y, r->itile[0],
                                 nullptr);
      launch_make_keys(I, no_tiles ? r->itile[0] : r->tiles_sorted, r->vals, r->depths,
                       m->keys_dbg, nullptr);
      DW_CUDA(cudaDeviceSynchronize());
      *p = r->keys_dbg;
      *count = I;
      break;
    }
    case 6: *p = r->vals; *count = I; break;
    case 7: *p = r->ranges; *count = 2 * nt; break;
    case 8: *p = r->final_T; *count = npx; break;
    case 9: *p = r->n_contrib; *count = npx; break;
    default: throw std::invalid_argument("unknown rasterizer buffer");
  }
}

void raster_host(dw_rasterizer* r, int32_t P, const float* m, const float* sc, const float* rot,
                 const float* op, const float* col, const dw_camera* cam, const float* dL,
                 int policy, int thr, float* out_color, float* grad, cudaStream_t s) {
  const size_t np = static_cast<size_t>(std::max(P, 1));
  const size_t npx = static_cast<size_t>(cam->width) * cam->height;
  float* d_m = r->host_scratch(0, 3 * np);
  float* d_sc = r->host_scratch(1, 3 * np);
  float* d_rot = r->host_scratch(2, 4 * np);
  float* d_op = r->host_scratch(3, np);
  float* d_col = r->host_scratch(4, 3 * np);
  float* d_dl = r->host_scratch(5, 3 * npx);
  float* d_img = r->host_scratch(6, 3 * npx);
  float* d_g = r->host_scratch(7, kNParam * np);
  auto h2d = [&](float* d, const float* h, size_t n) {
    if (n) DW_CUDA(cudaMemcpyAsync(d, h, n * sizeof(float), cudaMemcpyHostToDevice, s));
  };
  h2d(d_m, m, 3 * size_t(P));
  h2d(d_sc, sc, 3 * size_t(P));
  h2d(d_rot, rot, 4 * size_t(P));
  h2d(d_op, op, size_t(P));
  h2d(d_col, col, 3 * size_t(P));
  h2d(d_dl, dL, 3 * npx);
  r->forward(P, d_m, d_sc, d_rot, d_op, d_col, *cam, d_img, nullptr, s);
  DW_CUDA(cudaMemsetAsync(d_g, 0, kNParam * np * sizeof(float), s));
  r->backward(d_dl, policy, thr, d_g, nullptr, s);
  DW_CUDA(cudaMemcpyAsync(out_color, d_img, 3 * npx * sizeof(float), cudaMemcpyDeviceToHost, s));
  if (P > 0)
    DW_CUDA(cudaMemcpyAsync(grad, d_g, kNParam * size_t(P) * sizeof(float),
                            cudaMemcpyDeviceToHost, s));
  DW_CUDA(cudaStreamSynchronize(s));
}

// One training step's rasterization from host buffers: the scene is uploaded
// once, then V views are rendered and back-propagated into one gradient
// buffer. dL/dpixel uploads (copy stream s_in) and image downloads (copy
// stream s_out) are double-buffered against the compute stream, so with
// pinned host memory the PCIe traffic of view k+1 / k-1 overlaps view k.
// grad_on_device: `grad` is a device buffer of P*9 floats that receives the
// batch's gradient (overwritten) and stays in HBM -- for a caller that reduces
// it across GPUs before the one device-to-host copy; otherwise `grad` is host
// memory and the gradient is copied there.
// device gradient scratch of the host-buffer paths (host_scratch slot 7)
float* raster_scratch_grad(dw_rasterizer* r, int32_t P) {
  return r->host_scratch(7, kNParam * static_cast<size_t>(std::max(P, 1)));
}

void raster_views_host(dw_rasterizer* r, int32_t P, const float* m, const float* sc,
                       const float* rot, const float* op, const float* col, const dw_camera* cams,
                       int32_t V, const float* dL, int policy, int thr, float* out_images,
                       float* grad, cudaStream_t s, bool grad_on_device) {
  if (V < 1) throw std::invalid_argument("need at least one view");
  bool same_bg = true;
  for (int k = 1; k < V; ++k) {
    if (cams[k].width != cams[0].width || cams[k].height != cams[0].height)
      throw std::invalid_argument("all views must share one image size");
    same_bg = same_bg && std::memcmp(cams[k].bg, cams[0].bg, sizeof(cams[0].bg)) == 0;
  }
  r->ensure_streams();
  // Views per frame (dw_rasterizer::forward_views): G consecutive views share
  // every forward launch and one backward launch. DW_VIEWS_STACK=n overrides
  // the default (profiles/r02/ab/stacked_views.md); one view per frame when
  // the views differ in background, the image is too tall for the packed
  // rectangles, the scene takes dense binning (decided on the first frame) or
  // another list construction is forced.
  int G = 1;  // stacked frames: a tie or a loss once backwards chain (stacked_views.md)
  if (const char* e = std::getenv("DW_VIEWS_STACK"); e && *e) G = std::atoi(e);
  G = std::max(1, std::min({G, dw_rasterizer::stack_limit(cams[0].width, cams[0].height),
                            static_cast<int>(V)}));
  if (!same_bg || P == 0) G = 1;
  auto forced = [](const char* name, char v) {
    const char* e = std::getenv(name);
    return e && *e == v;
  };
  if (forced("DW_BLOCK_BINNING", '0') || forced("DW_TILE_FIRST", '1') ||
      forced("DW_SCATTER", '1') || forced("DW_DENSE_BINNING", '1'))
    G = 1;
  const size_t np = static_cast<size_t>(std::max(P, 1));
  const size_t npx = static_cast<size_t>(cams[0].width) * cams[0].height;
  float* d_m = r->host_scratch(0, 3 * np);
  float* d_sc = r->host_scratch(1, 3 * np);
  float* d_rot = r->host_scratch(2, 4 * np);
  float* d_op = r->host_scratch(3, np);
  float* d_col = r->host_scratch(4, 3 * np);
  float* d_g = grad_on_device ? grad : r->host_scratch(7, kNParam * np);
  // SW-B / SW-S add into a padded [P][12] buffer folded into d_g at the end
  const bool pad = P > 0 && (policy == kSwB || policy == kSwS) &&
                   !forced("DW_BULK_STAGING", '1');
  float* d_acc = pad ? r->padded_grad(P, s) : d_g;
  cudaEvent_t e_scene = r->ev[0], e_start = r->ev[1], e_chain = r->ev[2];
  int NF = 4;  // forward streams the frames of a wave rotate over (1 / 2 / 3 / 4: C5 101.1 / 98.4 / 98.3 / 97.6 ms)
  if (const char* e = std::getenv("DW_VIEWS_FSTREAMS"); e && *e)
    NF = std::max(1, std::min(dw_rasterizer::kMaxFwdStreams, std::atoi(e)));
  const cudaStream_t* F = r->s_fwd;
  // Waves of up to kWave frames: the wave's forwards (NF streams, each frame
  // into its own state) and uploads first, then its backwards as ONE chain on
  // `s` (dw_render_backward_chained after the first: every frame is rendered
  // and independent, so a launch starts on the SMs the previous one's last
  // wave leaves idle). Forwards of different views overlap each other well;
  // a forward interleaved with another view's backward (the previous
  // two-state pipeline) only competes for the SMs the backward fills.
  // 64 views, C5: 103.5 -> 97.6 ms per step; C3: 80.7 -> 76.4 ms
  // (profiles/r02/ab/chained_backward.md). The next wave reuses the states
  // once this wave's chain is done.
  int kWave = 16;
  if (const char* e = std::getenv("DW_VIEWS_WAVE"); e && *e) kWave = std::max(1, std::atoi(e));
  const int NG0 = (V + G - 1) / G;
  const int K = std::min(kWave, NG0);
  if (!r->probe) r->probe = new dw_rasterizer();
  while (static_cast<int>(r->pool.size()) < K) r->pool.push_back(new dw_rasterizer());
  while (static_cast<int>(r->pev.size()) < 3 * K) {
    cudaEvent_t e;
    DW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    r->pev.push_back(e);
  }
  auto h2d = [&](float* d, const float* h, size_t n, cudaStream_t st) {
    if (n) DW_CUDA(cudaMemcpyAsync(d, h, n * sizeof(float), cudaMemcpyHostToDevice, st));
  };
  // nothing may run ahead of work already queued on `s`
  DW_CUDA(cudaEventRecord(e_start, s));
  for (auto st : {r->s_in, r->s_out}) DW_CUDA(cudaStreamWaitEvent(st, e_start, 0));
  for (int f = 0; f < NF; ++f) DW_CUDA(cudaStreamWaitEvent(F[f], e_start, 0));
  h2d(d_m, m, 3 * size_t(P), r->s_in);
  h2d(d_sc, sc, 3 * size_t(P), r->s_in);
  h2d(d_rot, rot, 4 * size_t(P), r->s_in);
  h2d(d_op, op, size_t(P), r->s_in);
  h2d(d_col, col, 3 * size_t(P), r->s_in);
  DW_CUDA(cudaEventRecord(e_scene, r->s_in));
  DW_CUDA(cudaStreamWaitEvent(s, e_scene, 0));
  for (int f = 0; f < NF; ++f) DW_CUDA(cudaStreamWaitEvent(F[f], e_scene, 0));
  // Frame 0 reads its instance count back (a host sync on its stream) into
  // the probe state; the pool states get a 1.5x reserve from it and every
  // later frame keeps its count on the device (no host sync: the host runs
  // ahead and every copy overlaps). A frame that outgrows its reserve raises
  // its state's sticky overflow flag and the batch is redone with host-read
  // counts; a stacked first frame that would have preferred dense binning
  // restarts the batch with one view per frame.
  bool nosync_ok = true;
  for (int pass = 0; pass < 3; ++pass) {
    const int NG = (V + G - 1) / G;  // frames
    nosync_ok = nosync_ok && NG > 1;
    auto first = [&](int g) { return g * G; };
    auto count = [&](int g) { return std::min(G, static_cast<int>(V) - g * G); };
    auto state = [&](int g) { return g == 0 ? r->probe : r->pool[g % K]; };
    DW_CUDA(cudaMemsetAsync(d_g, 0, kNParam * np * sizeof(float), s));  // (the chain's stream)
    if (pad) DW_CUDA(cudaMemsetAsync(d_acc, 0, 12 * np * sizeof(float), s));
    bool restack = false;
    for (int w0 = 0; w0 < NG && !restack; w0 += K) {
      const int w1 = std::min(NG, w0 + K);
      for (int g = w0; g < w1; ++g) {
        const int j = g - w0;
        dw_rasterizer* Rg = state(g);
        cudaStream_t Fg = F[j % NF];
        cudaEvent_t e_fwd = r->pev[3 * j], e_in = r->pev[3 * j + 1], e_img = r->pev[3 * j + 2];
        float* d_dl = Rg->host_scratch(5, 3 * npx * G);
        float* d_img = Rg->host_scratch(6, 3 * npx * G);
        if (w0 > 0) {  // the previous wave's chain is done with the states and dL buffers
          DW_CUDA(cudaStreamWaitEvent(Fg, e_chain, 0));
          DW_CUDA(cudaStreamWaitEvent(Fg, e_img, 0));  // its images downloaded
          DW_CUDA(cudaStreamWaitEvent(r->s_in, e_chain, 0));
        }
        h2d(d_dl, dL + static_cast<size_t>(first(g)) * 3 * npx, 3 * npx * count(g), r->s_in);
        DW_CUDA(cudaEventRecord(e_in, r->s_in));
        const bool nosync = nosync_ok && g > 0;
        Rg->forward_views(P, d_m, d_sc, d_rot, d_op, d_col, cams + first(g), count(g), d_img,
                          nullptr, Fg, nosync, /*sticky_overflow=*/true);
        if (g == 0 && count(0) > 1 && Rg->stack_unfit) {  // counted: known on the host now
          restack = true;
          break;
        }
        Rg->ensure_order(Fg);  // the backward's tile order, so the chain launches nothing else
        DW_CUDA(cudaEventRecord(e_fwd, Fg));
        if (out_images) {
          DW_CUDA(cudaStreamWaitEvent(r->s_out, e_fwd, 0));
          DW_CUDA(cudaMemcpyAsync(out_images + static_cast<size_t>(first(g)) * 3 * npx, d_img,
                                  3 * npx * count(g) * sizeof(float), cudaMemcpyDeviceToHost,
                                  r->s_out));
          DW_CUDA(cudaEventRecord(e_img, r->s_out));
        } else {
          DW_CUDA(cudaEventRecord(e_img, Fg));
        }
        if (g == 0 && nosync_ok) {  // size the pool's reserves from frame 0's count
          const int64_t want = Rg->num_rendered + Rg->num_rendered / 2 + 4096;
          for (int q = 0; q < K; ++q) {
            dw_rasterizer* Rq = r->pool[q];
            if (static_cast<int64_t>(std::min(Rq->cap_i[0], Rq->cap_i[2])) < want ||
                Rq->nviews_reserved < G)
              Rq->reserve(P, cams[0].width, cams[0].height, want, G);
            Rq->nviews_reserved = G;
            Rq->last_entries = Rg->last_entries;
            // the pass's sticky overflow flag, cleared before the state's
            // first frame (frame q, or frame K for pool[0], on F[q % NF])
            DW_CUDA(cudaMemsetAsync(Rq->overflow_dev, 0, sizeof(unsigned int), F[q % NF]));
          }
        }
      }
      if (restack) break;
      for (int g = w0; g < w1; ++g) {  // the chain waits for the whole wave up front
        DW_CUDA(cudaStreamWaitEvent(s, r->pev[3 * (g - w0)], 0));
        DW_CUDA(cudaStreamWaitEvent(s, r->pev[3 * (g - w0) + 1], 0));
      }
      for (int g = w0; g < w1; ++g)
        state(g)->backward(state(g)->host_scratch(5, 3 * npx * G), policy, thr, d_acc, nullptr,
                           s, /*chained=*/g > w0, pad ? 12 : kNParam);
      DW_CUDA(cudaEventRecord(e_chain, s));
    }
    for (int f = 0; f <= NF; ++f) {  // join every stream into `s`
      DW_CUDA(cudaEventRecord(e_start, f < NF ? F[f] : r->s_in));
      DW_CUDA(cudaStreamWaitEvent(s, e_start, 0));
    }
    if (restack) {
      DW_CUDA(cudaStreamSynchronize(s));
      DW_CUDA(cudaStreamSynchronize(r->s_out));
      G = 1;
      continue;
    }
    if (!nosync_ok) break;
    DW_CUDA(cudaStreamSynchronize(s));
    bool ovf = false;
    for (int q = 0; q < K; ++q) {
      bool o = false;
      r->pool[q]->resolve_count(&o);  // the batch's sticky flags
      ovf = ovf || o;
    }
    if (!ovf) break;
    nosync_ok = false;  // redo every view with host-read instance counts
  }
  if (pad) r->fold_padded(P, d_g, s);
  if (P > 0 && !grad_on_device)
    DW_CUDA(cudaMemcpyAsync(grad, d_g, kNParam * size_t(P) * sizeof(float),
                            cudaMemcpyDeviceToHost, s));
  DW_CUDA(cudaStreamSynchronize(s));
  DW_CUDA(cudaStreamSynchronize(r->s_out));
  DW_CUDA(cudaStreamSynchronize(r->s_in));
}

}  // namespace dw

namespace dw {
dw_rasterizer* raster_new() { return new dw_rasterizer(); }
void raster_delete(dw_rasterizer* r) { delete r; }
}  // namespace dw
