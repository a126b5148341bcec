// scan_mamba1.cu -- fused Mamba-1 selective scan for sm_100a (fp32).
//
// Semantics (mamba_ssm selective_scan_fn, the paper's kernel),
// recurrence core identical to chunklab::scan_window (scan.hpp:77-100) under the
// mapping a = exp(delta'*A), x = delta'*u, b/c = B/C (SURVEY.md finding 1):
//   delta' = softplus(delta + bias)            (identity above 20, mamba_ssm)
//   h_s    = exp(delta'*A[c,s]) * h_s + B[b,s,t] * (delta'*u)     s = 0..N-1
//   y      = (sum_s C[b,s,t]*h_s + D[c]*u) * z*sigmoid(z)
//
// Kernels:
//   * rowpair_ws_kernel (the hot path, N = 16): warp-specialised.  Consumer warps own
//     16-row tiles (two lanes per (b, c) row, 8 states each in FFMA2 register pairs);
//     producer warps feed each consumer a 2-stage TMA ring of 16-timestep boxes
//     (u / delta / z with 64B swizzle, one interleaved [B^T | C^T] box).  y is stored
//     from registers.  Work items are (row tile, L-segment) pairs with segment length
//     = the chunk chosen by the device rule (read from device memory, rounded up to
//     whole boxes), dispatched segment-major through an atomic ticket; the state carry
//     between consecutive segments of a tile is a chained scan (flag + release /
//     acquire), so chunking never changes a single floating-point operation: outputs
//     are bit-identical for every chunk size.
//   * rowseq_tma_kernel: one lane per row (32-row tiles), each warp feeding its own
//     TMA ring and TMA-storing y; kept as a selectable variant (CL_SCAN_CFG=1..3).
//   * generic_kernel: any N <= 64, any alignment; one thread per row, direct loads.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "cl_internal.h"
#include "scan_common.cuh"

namespace cl {
namespace {



template <int BOX, int STAGES>
constexpr int warp_bytes() {
  return STAGES * Geo<BOX>::kStageBytes + 2 * Geo<BOX>::kTileBytes;  // + 2 y staging buffers
}

template <int BOX, int WARPS, int STAGES, bool SP, bool HZ>
__global__ void __launch_bounds__(WARPS * 32, 1)
    rowseq_tma_kernel(const __grid_constant__ CUtensorMap map_u,
                      const __grid_constant__ CUtensorMap map_dt,
                      const __grid_constant__ CUtensorMap map_z,
                      const __grid_constant__ CUtensorMap map_out,
                      const __grid_constant__ CUtensorMap map_Bt,
                      const __grid_constant__ CUtensorMap map_Ct, TmaArgs a) {
  using G = Geo<BOX>;
  int status;
  const int chunk = read_chunk(a.decision, a.fixed_chunk, &status);
  if (status != 0) return;
  int seg_len = chunk < BOX ? BOX : chunk;
  seg_len = (seg_len + BOX - 1) / BOX * BOX;
  const int L = static_cast<int>(a.L);
  const int n_seg = (L + seg_len - 1) / seg_len;
  const int n_items = n_seg * a.n_tiles;

  extern __shared__ unsigned char smem_raw[];
  // align to 1024 B (128B swizzle atom) with pointer arithmetic on the __shared__
  // base, so every access below stays in the shared window (LDS/STS, not generic LD)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int kWB = warp_bytes<BOX, STAGES>();
  unsigned char* wbase = smem + size_t(warp) * kWB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(WARPS) * kWB) + warp * 4;
  int meta_item[STAGES], meta_box[STAGES];

  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_u)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_dt)));
    if (HZ) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_z)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_Bt)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_Ct)));
  }
  __syncwarp();

  auto decode = [&](int id) {
    Item it;
    it.seg = id / a.n_tiles;
    it.tile = id % a.n_tiles;
    it.t0 = it.seg * seg_len;
    const int len = min(seg_len, L - it.t0);
    it.nbox = (len + BOX - 1) / BOX;
    return it;
  };
  auto claim = [&]() {
    int id = 0;
    if (lane == 0) id = static_cast<int>(atomicAdd(a.ticket, 1u));
    return __shfl_sync(0xffffffffu, id, 0);
  };

  int p_item = claim();
  int p_box = 0;
  Item p_it = decode(p_item);
  auto produce = [&](int slot) {
    meta_item[slot] = -1;
    if (p_item >= n_items) return;
    const Item it = p_it;
    meta_item[slot] = p_item;
    meta_box[slot] = p_box;
    if (lane == 0) {
      unsigned char* st = wbase + slot * G::kStageBytes;
      const int b = it.tile / a.tiles_per_batch;
      const int r0 = (it.tile % a.tiles_per_batch) * kRows;
      const int t = it.t0 + p_box * BOX;
      mbar_expect_tx(bars + slot, HZ ? G::kStageBytes : G::kStageBytes - G::kTileBytes);
      tma_load_3d(st, &map_u, t, r0, b, bars + slot);
      tma_load_3d(st + G::kTileBytes, &map_dt, t, r0, b, bars + slot);
      if (HZ) tma_load_3d(st + 2 * G::kTileBytes, &map_z, t, r0, b, bars + slot);
      tma_load_3d(st + 3 * G::kTileBytes, &map_Bt, 0, t, b, bars + slot);
      tma_load_3d(st + 3 * G::kTileBytes + G::kBCBytes, &map_Ct, 0, t, b, bars + slot);
    }
    if (++p_box == it.nbox) {
      p_box = 0;
      p_item = claim();
      p_it = decode(p_item);
    }
  };

  for (int s = 0; s < STAGES; ++s) produce(s);

  unsigned char* ybuf0 = wbase + STAGES * G::kStageBytes;
  f2_t h2[kN / 2], A2p[kN / 2];
  float bias = 0.f, Dc = 0.f;
  Item cur{};
  int row = 0;
  bool row_valid = false;
  for (int iter = 0;; ++iter) {
    const int slot = iter % STAGES;
    const int item = meta_item[slot];
    if (item < 0) break;
    const int box = meta_box[slot];
    if (box == 0) {
      cur = decode(item);
      const int b = cur.tile / a.tiles_per_batch;
      const int c = (cur.tile % a.tiles_per_batch) * kRows + lane;
      row_valid = c < static_cast<int>(a.dim);
      const int cc = row_valid ? c : 0;
      row = b * static_cast<int>(a.dim) + cc;
#pragma unroll
      for (int s = 0; s < kN; s += 4) {
        const float4 q = *reinterpret_cast<const float4*>(a.A + size_t(cc) * kN + s);
        A2p[s / 2] = pk(q.x * kLog2e, q.y * kLog2e);
        A2p[s / 2 + 1] = pk(q.z * kLog2e, q.w * kLog2e);
      }
      bias = a.bias ? a.bias[cc] : 0.f;
      Dc = a.D ? a.D[cc] : 0.f;
      const float* src = nullptr;
      if (cur.seg == 0) {
        src = a.h0 ? a.h0 + size_t(row) * kN : nullptr;
      } else {
        // chained carry from segment seg-1 of this tile
        if (lane == 0)
          while (ld_acquire(a.flags + cur.tile) < static_cast<unsigned>(cur.seg)) __nanosleep(64);
        __syncwarp();
        src = a.carry + (size_t(cur.tile) * kRows + lane) * kN;
      }
#pragma unroll
      for (int s = 0; s < kN; s += 4) {
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (src) q = __ldcg(reinterpret_cast<const float4*>(src + s));
        h2[s / 2] = pk(q.x, q.y);
        h2[s / 2 + 1] = pk(q.z, q.w);
      }
    }

    mbar_wait(bars + slot, (iter / STAGES) & 1);
    // y staging is double-buffered: this buffer is free once the store issued two
    // boxes ago has read it (at most the newest store may still be in flight)
    unsigned char* ybuf = ybuf0 + (iter & 1) * G::kTileBytes;
    if (lane == 0) bulk_wait_read_le1();
    __syncwarp();
    unsigned char* st = wbase + slot * G::kStageBytes;
    const unsigned char* sB = st + 3 * G::kTileBytes;
    const unsigned char* sC = sB + G::kBCBytes;
    const int tbox = cur.t0 + box * BOX;
    const int valid = min(BOX, L - tbox);  // multiple of 4 (L % 4 == 0)
    const f2_t bias2 = pk(bias, bias);
#pragma unroll
    for (int j = 0; j < BOX / 4; ++j) {
      if (4 * j >= valid) break;
      const int off = G::swz(lane, j);
      const float4 u4 = *reinterpret_cast<const float4*>(st + off);
      const float4 d4 = *reinterpret_cast<const float4*>(st + G::kTileBytes + off);
      // elementwise prologue for the 4 timesteps, packed in pairs
      f2_t dt01 = add2(pk(d4.x, d4.y), bias2), dt23 = add2(pk(d4.z, d4.w), bias2);
      if (SP) {
        dt01 = softplus2(dt01);
        dt23 = softplus2(dt23);
      }
      const f2_t x01 = mul2(dt01, pk(u4.x, u4.y)), x23 = mul2(dt23, pk(u4.z, u4.w));
      float dt[4], xs[4];
      upk(dt01, dt[0], dt[1]);
      upk(dt23, dt[2], dt[3]);
      upk(x01, xs[0], xs[1]);
      upk(x23, xs[2], xs[3]);
      float yy[4];
      // phase A: the 4x16 transition factors exp(dt*A) do not depend on the state,
      // so they are all issued up front (MUFU-paced, independent)
      f2_t dA[4][kN / 2];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const f2_t dd = pk(dt[k], dt[k]);
#pragma unroll
        for (int i = 0; i < kN / 2; ++i) {
          dA[k][i] = state_exp2_pair(mul2(A2p[i], dd), i & 3);
        }
      }
      // phase B: recurrence h = dA*h + B*x and y = C.h, FFMA2 on state pairs
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int t = 4 * j + k;
        const ulonglong2* Bt = reinterpret_cast<const ulonglong2*>(sB + t * kN * 4);
        const ulonglong2* Ct = reinterpret_cast<const ulonglong2*>(sC + t * kN * 4);
        const f2_t xx = pk(xs[k], xs[k]);
        // canonical FFMA2 chains per half (cdot16_canon): pairs 0,2 / 1,3 and 4,6 / 5,7
        f2_t ya0 = 0ull, yb0 = 0ull, ya1 = 0ull, yb1 = 0ull;
#pragma unroll
        for (int q = 0; q < kN / 4; ++q) {
          const ulonglong2 bq = Bt[q];
          const ulonglong2 cq = Ct[q];
          h2[2 * q] = fma2(dA[k][2 * q], h2[2 * q], mul2(bq.x, xx));
          h2[2 * q + 1] = fma2(dA[k][2 * q + 1], h2[2 * q + 1], mul2(bq.y, xx));
          if (q < 2) {
            ya0 = fma2(cq.x, h2[2 * q], ya0);
            yb0 = fma2(cq.y, h2[2 * q + 1], yb0);
          } else {
            ya1 = fma2(cq.x, h2[2 * q], ya1);
            yb1 = fma2(cq.y, h2[2 * q + 1], yb1);
          }
        }
        float l0a, l0b, l1a, l1b;
        upk(add2(ya0, yb0), l0a, l0b);
        upk(add2(ya1, yb1), l1a, l1b);
        yy[k] = (l0a + l0b) + (l1a + l1b);
      }
      const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
      f2_t y01 = fma2(pk(Dc, Dc), pk(uu[0], uu[1]), pk(yy[0], yy[1]));
      f2_t y23 = fma2(pk(Dc, Dc), pk(uu[2], uu[3]), pk(yy[2], yy[3]));
      if (HZ) {
        const float4 z4 = *reinterpret_cast<const float4*>(st + 2 * G::kTileBytes + off);
        y01 = mul2(y01, silu2(pk(z4.x, z4.y)));
        y23 = mul2(y23, silu2(pk(z4.z, z4.w)));
      }
      float o0, o1, o2, o3;
      upk(y01, o0, o1);
      upk(y23, o2, o3);
      *reinterpret_cast<float4*>(ybuf + off) = make_float4(o0, o1, o2, o3);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      const int b = cur.tile / a.tiles_per_batch;
      const int r0 = (cur.tile % a.tiles_per_batch) * kRows;
      tma_store_3d(&map_out, ybuf, tbox, r0, b);
    }

    if (box == cur.nbox - 1) {
      float hs[kN];
#pragma unroll
      for (int i = 0; i < kN / 2; ++i) upk(h2[i], hs[2 * i], hs[2 * i + 1]);
      if (cur.seg == n_seg - 1) {
        if (a.h_last && row_valid) {
#pragma unroll
          for (int s = 0; s < kN; s += 4)
            *reinterpret_cast<float4*>(a.h_last + size_t(row) * kN + s) =
                make_float4(hs[s], hs[s + 1], hs[s + 2], hs[s + 3]);
        }
      } else {
        float* cw = a.carry + (size_t(cur.tile) * kRows + lane) * kN;
#pragma unroll
        for (int s = 0; s < kN; s += 4)
          __stcg(reinterpret_cast<float4*>(cw + s),
                 make_float4(hs[s], hs[s + 1], hs[s + 2], hs[s + 3]));
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(a.flags + cur.tile, static_cast<unsigned>(cur.seg + 1));
      }
    }
    // every lane has consumed this slot: refill it for iteration iter + STAGES
    __syncwarp();
    produce(slot);
  }
  if (lane == 0) bulk_wait_all();
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Warp-specialised lane-pair kernel (the hot path).
//
// Layout: a consumer warp owns a 16-row tile; lanes (2r, 2r+1) share row r and hold
// states 0-7 / 8-15 as FFMA2 register pairs.  That doubles the independent row
// chains of the 32-row kernel for the same shape (the chained-segment schedule caps
// busy warps at the tile count: 2048 tiles at C3 = 13.8 warps per SM), at the cost
// of one 64-bit shuffle pair per 4 timesteps.
//
// Roles: WARPS consumer warps only compute; NPROD producer warps run the consumers'
// TMA rings (lane l of producer p owns consumer p*ceil(WARPS/NPROD) + l): ticket
// claims, expect_tx and the four tile loads per box (u, delta, z and one interleaved
// [B | C] box).  Measured on C3: issuing TMA from the compute warps cost ~10% of
// the scan, one producer warp could not keep up with 14 consumers (its per-lane
// TMA issue serialises through uniform registers), two can.  y is stored straight
// from registers (8 B per lane per 4 timesteps, st.global.cs): the four stores of a
// box complete each 64-byte row segment in L2 within microseconds, and dropping the
// y staging buffer, proxy fence and TMA store saved another ~3%.
// ---------------------------------------------------------------------------

// Per consumer warp and stage: full[s] (producer arrive.expect_tx + TMA bytes) and
// empty[s] (consumer lane 0 arrive after its last shared-memory read of the stage).
// The meta words (item, box) travel through shared memory under full[s]'s release.
template <int BOX, int WARPS, int STAGES, bool SP, bool HZ, int NPROD, int PIPE>
__global__ void __launch_bounds__((WARPS + NPROD) * 32, 1)
    rowpair_ws_kernel(const __grid_constant__ CUtensorMap map_u,
                      const __grid_constant__ CUtensorMap map_dt,
                      const __grid_constant__ CUtensorMap map_z,
                      const __grid_constant__ CUtensorMap map_bc, TmaArgs a) {
  using G = GeoP<BOX>;
  int status;
  const int chunk = read_chunk(a.decision, a.fixed_chunk, &status);
  if (status != 0) return;
  int seg_len = chunk < BOX ? BOX : chunk;
  seg_len = (seg_len + BOX - 1) / BOX * BOX;
  const int L = static_cast<int>(a.L);
  const int n_seg = (L + seg_len - 1) / seg_len;
  const int n_items = n_seg * a.n_tiles;

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int kWB = STAGES * G::kStageBytes;
  unsigned char* params = smem + size_t(WARPS) * kWB;  // [WARPS][STAGES][kParamBytes]
  uint64_t* full = reinterpret_cast<uint64_t*>(params + size_t(WARPS) * STAGES * G::kParamBytes);
  uint64_t* empty = full + WARPS * STAGES;                                  // [WARPS][STAGES]
  int2* meta = reinterpret_cast<int2*>(empty + WARPS * STAGES);              // [WARPS][STAGES]

  if (threadIdx.x < WARPS * STAGES) {
    mbar_init(full + threadIdx.x, 1);
    mbar_init(empty + threadIdx.x, 1);
  }
  if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  auto decode = [&](int id) {
    Item it;
    it.seg = id / a.n_tiles;
    it.tile = id % a.n_tiles;
    it.t0 = it.seg * seg_len;
    const int len = min(seg_len, L - it.t0);
    it.nbox = (len + BOX - 1) / BOX;
    return it;
  };

  if (warp >= WARPS) {
    // ---------------- producers ----------------
    constexpr int kPer = (WARPS + NPROD - 1) / NPROD;
    const int w = (warp - WARPS) * kPer + lane;
    bool live = lane < kPer && w < WARPS;
    if (lane == 0 && warp == WARPS) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_u)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_dt)));
      if (HZ) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_z)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bc)));
    }
    // boxes go through each consumer's ring in ticket order
    int p_item = live ? static_cast<int>(atomicAdd(a.ticket, 1u)) : 0;
    Item p_it = decode(p_item);
    int p_b = p_it.tile / a.tiles_per_batch, p_r0 = (p_it.tile % a.tiles_per_batch) * kRowsP;
    int p_box = 0, n_issued = 0;
    unsigned char* wbase = smem + size_t(w < WARPS ? w : 0) * kWB;
    while (__any_sync(0xffffffffu, live)) {
      bool issued = false;
      if (live) {
        const int slot = n_issued % STAGES;
        const bool free = n_issued < STAGES ||
                          mbar_test(empty + w * STAGES + slot, ((n_issued / STAGES) - 1) & 1);
        if (free) {
          uint64_t* bar = full + w * STAGES + slot;
          if (p_item >= n_items) {
            meta[w * STAGES + slot] = make_int2(-1, 0);
            mbar_arrive(bar);
            live = false;
          } else {
            unsigned char* st = wbase + slot * G::kStageBytes;
            const int t = p_it.t0 + p_box * BOX;
            const bool stage = p_box == 0 && a.stage_params &&
                               p_r0 + kRowsP <= static_cast<int>(a.dim);
            meta[w * STAGES + slot] = make_int2(p_item, p_box | (stage ? kStagedFlag : 0));
            uint32_t tx = HZ ? G::kStageBytes : G::kStageBytes - G::kTileBytes;
            if (stage) tx += kRowsP * kN * 4 + (a.bias ? kRowsP * 4 : 0) + (a.D ? kRowsP * 4 : 0);
            mbar_expect_tx(bar, tx);
            if (stage) {
              unsigned char* pp = params + (size_t(w) * STAGES + slot) * G::kParamBytes;
              bulk_g2s(pp, a.A + size_t(p_r0) * kN, kRowsP * kN * 4, bar);
              if (a.bias) bulk_g2s(pp + kRowsP * kN * 4, a.bias + p_r0, kRowsP * 4, bar);
              if (a.D) bulk_g2s(pp + kRowsP * kN * 4 + kRowsP * 4, a.D + p_r0, kRowsP * 4, bar);
            }
            tma_load_3d(st, &map_u, t, p_r0, p_b, bar);
            tma_load_3d(st + G::kTileBytes, &map_dt, t, p_r0, p_b, bar);
            if (HZ) tma_load_3d(st + 2 * G::kTileBytes, &map_z, t, p_r0, p_b, bar);
            tma_load_3d(st + 3 * G::kTileBytes, &map_bc, 0, t, p_b, bar);
            if (++p_box == p_it.nbox) {
              p_box = 0;
              p_item = static_cast<int>(atomicAdd(a.ticket, 1u));
              p_it = decode(p_item);
              p_b = p_it.tile / a.tiles_per_batch;
              p_r0 = (p_it.tile % a.tiles_per_batch) * kRowsP;
            }
          }
          ++n_issued;
          issued = true;
        }
      }
      if (!__any_sync(0xffffffffu, issued)) __nanosleep(CL_PROD_SLEEP_NS);
    }
    // only producers claim tickets: the last producer warp of the grid to finish returns
    // the ticket to 0, so the next launch on this stream needs no memset
    ticket_retire(a.ticket, gridDim.x * NPROD, lane,
                  static_cast<unsigned>(n_items) + gridDim.x * static_cast<unsigned>(WARPS));
    return;
  }

  // ---------------- consumers ----------------
  const int r = lane >> 1, hf = lane & 1;
  const unsigned char* wbase = smem + size_t(warp) * kWB;
  uint64_t* wfull = full + warp * STAGES;
  uint64_t* wempty = empty + warp * STAGES;
  const int2* wmeta = meta + warp * STAGES;
  constexpr int kP = kN / 4;
  const unsigned epoch = a.epoch;
  f2_t h2[kP], A2p[kP];
  float bias = 0.f, Dc = 0.f;
  Item cur{};
  int row = 0;
  bool row_valid = false;
  for (int iter = 0;; ++iter) {
    const int slot = iter % STAGES;
    mbar_wait(wfull + slot, (iter / STAGES) & 1);
    const int2 m = wmeta[slot];
    if (m.x < 0) break;
    const int box = m.y & ~kStagedFlag;
    CL_DCHECK(m.x < n_items);
    if (box == 0) {
      cur = decode(m.x);
      const int b = cur.tile / a.tiles_per_batch;
      const int c = (cur.tile % a.tiles_per_batch) * kRowsP + r;
      row_valid = c < static_cast<int>(a.dim);
      const int cc = row_valid ? c : 0;
      row = b * static_cast<int>(a.dim) + cc;
      if (m.y & kStagedFlag) {
        // staged by the producer with this box (shared memory: no global round trip)
        const unsigned char* pp = params + (size_t(warp) * STAGES + slot) * G::kParamBytes;
#pragma unroll
        for (int s = 0; s < kN / 2; s += 4) {
          const float4 q = *reinterpret_cast<const float4*>(pp + (r * kN + 8 * hf + s) * 4);
          A2p[s / 2] = pk(q.x * kLog2e, q.y * kLog2e);
          A2p[s / 2 + 1] = pk(q.z * kLog2e, q.w * kLog2e);
        }
        bias = a.bias ? reinterpret_cast<const float*>(pp + kRowsP * kN * 4)[r] : 0.f;
        Dc = a.D ? reinterpret_cast<const float*>(pp + kRowsP * kN * 4 + kRowsP * 4)[r] : 0.f;
      } else {
#pragma unroll
        for (int s = 0; s < kN / 2; s += 4) {
          const float4 q = *reinterpret_cast<const float4*>(a.A + size_t(cc) * kN + 8 * hf + s);
          A2p[s / 2] = pk(q.x * kLog2e, q.y * kLog2e);
          A2p[s / 2 + 1] = pk(q.z * kLog2e, q.w * kLog2e);
        }
        bias = a.bias ? a.bias[cc] : 0.f;
        Dc = a.D ? a.D[cc] : 0.f;
      }
      const float* src = nullptr;
      if (cur.seg == 0) {
        src = a.h0 ? a.h0 + size_t(row) * kN + 8 * hf : nullptr;
      }
      if (cur.seg == 0) {
#pragma unroll
        for (int s = 0; s < kN / 2; s += 4) {
          float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
          if (src) q = __ldcg(reinterpret_cast<const float4*>(src + s));
          h2[s / 2] = pk(q.x, q.y);
          h2[s / 2 + 1] = pk(q.z, q.w);
        }
      } else {
        // chained carry from segment seg-1 of this tile: every word carries its own tag,
        // so a lane polls its 8 words with relaxed loads -- no flag, no acquire / release
        // (the writer's release would also wait for all of its y stores to land)
        const unsigned long long* w64 =
            a.tcarry + (size_t(cur.tile) * kRowsP + r) * kN + 8 * hf;
        const unsigned want = epoch + static_cast<unsigned>(cur.seg);
        unsigned long long w[kN / 2];
        for (;;) {
          bool ok = true;
#pragma unroll
          for (int i = 0; i < kN / 2; i += 2) {
            ld_relaxed_u64x2(w64 + i, w[i], w[i + 1]);
            ok &= static_cast<unsigned>(w[i] >> 32) == want;
            ok &= static_cast<unsigned>(w[i + 1] >> 32) == want;
            // eager tags only grow: a newer tag than this launch's would be a stale-epoch bug
            CL_DCHECK(static_cast<unsigned>(w[i] >> 32) <= want);
          }
          if (__all_sync(0xffffffffu, ok)) break;
          __nanosleep(64);
        }
#pragma unroll
        for (int i = 0; i < kP; ++i)
          h2[i] = pk(__uint_as_float(static_cast<unsigned>(w[2 * i])),
                     __uint_as_float(static_cast<unsigned>(w[2 * i + 1])));
      }
    }

    const int tbox = cur.t0 + box * BOX;
    float* ydst = row_valid ? a.out + size_t(row) * a.L + tbox : nullptr;
    if (PIPE == 1 && tbox + BOX <= L)
      pair_box_pipe<BOX, SP, HZ>(wbase + slot * G::kStageBytes, ydst, r, hf, bias, Dc, A2p, h2);
    else
      pair_box<BOX, SP, HZ>(wbase + slot * G::kStageBytes, ydst, r, hf, min(BOX, L - tbox), bias,
                            Dc, A2p, h2);
    __syncwarp();
    if (lane == 0) mbar_arrive(wempty + slot);  // stage consumed: producer may refill

    if (box == cur.nbox - 1) {
      float hs[kN / 2];
#pragma unroll
      for (int i = 0; i < kP; ++i) upk(h2[i], hs[2 * i], hs[2 * i + 1]);
      if (cur.seg == n_seg - 1) {
        if (a.h_last && row_valid) {
          float* dst = a.h_last + size_t(row) * kN + 8 * hf;
          __stcg(reinterpret_cast<float4*>(dst), make_float4(hs[0], hs[1], hs[2], hs[3]));
          __stcg(reinterpret_cast<float4*>(dst + 4), make_float4(hs[4], hs[5], hs[6], hs[7]));
        }
      } else {
        unsigned long long* w64 = a.tcarry + (size_t(cur.tile) * kRowsP + r) * kN + 8 * hf;
        const unsigned long long tag =
            static_cast<unsigned long long>(epoch + static_cast<unsigned>(cur.seg + 1)) << 32;
#pragma unroll
        for (int i = 0; i < kN / 2; i += 2)
          st_relaxed_u64x2(w64 + i, tag | __float_as_uint(hs[i]), tag | __float_as_uint(hs[i + 1]));
      }
    }
  }
}

// (b, N, L) -> (b, L, N) for B and C, so a timestep's 16 state coefficients are one
// contiguous 64-byte row: the scan then reads them as FFMA2 register pairs.
__global__ void __launch_bounds__(256) transpose_bc_kernel(const float* __restrict__ B,
                                                           const float* __restrict__ C,
                                                           float* __restrict__ Bt,
                                                           float* __restrict__ Ct, int L,
                                                           int row_stride) {
  __shared__ float tile[kN][33];
  const float* src = blockIdx.z ? C : B;
  float* dst = blockIdx.z ? Ct : Bt;
  const int b = blockIdx.y, t0 = blockIdx.x * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // ty 0..7
  for (int s = ty; s < kN; s += 8) {
    const int t = t0 + tx;
    tile[s][tx] = t < L ? src[(size_t(b) * kN + s) * L + t] : 0.f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * kN; e += 256) {
    const int tt = e / kN, s = e % kN;
    const int t = t0 + tt;
    if (t < L) dst[(size_t(b) * L + t) * row_stride + s] = tile[s][tt];
  }
}


// The prefill's first launch when the scan's B / C re-layout is folded into it: blocks
// with blockIdx.z < 2 transpose B (z = 0) and C (z = 1) exactly as transpose_bc_kernel,
// block (0, 0, 2) initialises the entropy range {-inf, -inf, 0, 0} and zeroes the K counts
// (cl_prefill_init).  One launch instead of two, and the transpose leaves the scan.
__global__ void __launch_bounds__(256) init_transpose_kernel(const float* __restrict__ B,
                                                             const float* __restrict__ C,
                                                             float* __restrict__ Bt,
                                                             float* __restrict__ Ct, int L,
                                                             int row_stride, double* range,
                                                             unsigned long long* counts, int k) {
  if (blockIdx.z == 2) {
    if (blockIdx.x != 0 || blockIdx.y != 0) return;
    if (threadIdx.x == 0) {
      range[0] = -INFINITY;
      range[1] = -INFINITY;
      range[2] = 0.0;
      range[3] = 0.0;
    }
    for (int b = threadIdx.x; b < k; b += blockDim.x) counts[b] = 0ull;
    return;
  }
  __shared__ float tile[kN][33];
  const float* src = blockIdx.z ? C : B;
  float* dst = blockIdx.z ? Ct : Bt;
  if (!dst) return;  // init only (no TMA scan to feed)
  const int b = blockIdx.y, t0 = blockIdx.x * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  for (int s = ty; s < kN; s += 8) {
    const int t = t0 + tx;
    tile[s][tx] = t < L ? src[(size_t(b) * kN + s) * L + t] : 0.f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * kN; e += 256) {
    const int tt = e / kN, s2 = e % kN;
    const int t = t0 + tt;
    if (t < L) dst[(size_t(b) * L + t) * row_stride + s2] = tile[s2][tt];
  }
}

// ---- kernel table (CL_SCAN_CFG=<index> selects a row, for experiments) ----
enum ScanKind { kWarpSpecPair = 0, kRowSeq = 1, kWarpSpecPairNoPipe = 2 };
struct ScanCfg {
  int kind, box, warps, stages;
};
constexpr ScanCfg kCfgs[] = {
    // 12 consumer + 2 producer warps per SM (C3, C4): three consumers on every SM
    // sub-partition, so every warp gets the same share of its SMSP's MUFU quarter.
    // Measured at C3 (scan ms): 12 consumers 1.357; 13: 1.373; 14 (4/4/3/3 per SMSP):
    // 1.404 -- the uneven sub-partitions made warps wait on each other's carries (ncu:
    // carry-spin samples 2.7% -> 0.3%); 16 (capped at 96 registers, spills): 1.726;
    // 12 x 3 stages 1.371; 8 consumers 1.497; 12 with 1 producer 1.572, with 3: 1.371.
    // 16 consumers + a producer warpgroup that hands its registers over with setmaxnreg
    // (consumers 112, producers 24; no hot-loop spills): 1.654 -- more warps per SMSP do
    // not buy MUFU issue once each has fewer registers for the group pipeline.
    {kWarpSpecPair, 16, 12, 2},
    {kRowSeq, 32, 4, 3},         // 32-row tiles, self-fed TMA rings
    {kRowSeq, 16, 8, 3},
    {kRowSeq, 16, 7, 3},
    // few 16-row tiles (C1: 96, C2: 128): fewer consumers per CTA so the tiles spread over
    // all SMs instead of packing 12 to an SM (one producer, deeper ring)
    {kWarpSpecPair, 16, 1, 4},
    {kWarpSpecPair, 16, 2, 4},
    {kWarpSpecPair, 16, 4, 4},
    {kWarpSpecPair, 16, 7, 3},
    {kWarpSpecPairNoPipe, 16, 12, 2},  // 8: row 0 without the group software pipeline (A/B)
    {kWarpSpecPair, 16, 14, 2},        // 9: 14 consumers (the previous default)
    // A quad layout for few tiles (a warp pair per 16-row tile, four lanes per row, each
    // lane's chain a canonical ya / yb, bitwise equal to the lane pair) was measured
    // slower: C1 0.26 vs 0.17 ms, C2 0.49 vs 0.30 -- the per-lane elementwise work
    // (softplus, SiLU, exchanges) does not shrink with the lane's state count, so the
    // instruction count went up 1.8x on latency-bound lone warps (commit history).
    {kWarpSpecPair, 32, 1, 4},  // 10: few tiles, 32-timestep boxes (half the per-box overhead)
    {kWarpSpecPair, 32, 2, 4},  // 11
    {kWarpSpecPair, 32, 4, 3},  // 12
    {kWarpSpecPair, 32, 8, 2},  // 13
    {kWarpSpecPair, 32, 6, 3},  // 14
};
constexpr int kDefaultCfg = 0;

// producers per CTA: two keep up with 12-14 consumers (one feeding 12 costs +16%), one with up to 7
template <int WARPS>
constexpr int producers_for() {
  return WARPS >= 8 ? 2 : 1;
}

template <typename K>
cudaError_t set_smem(K kern, size_t smem) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem));
}

int grid_for(int n_tiles, int warps, int num_sms) {
  const int max_useful = (n_tiles + warps - 1) / warps;
  return max_useful < num_sms ? (max_useful < 1 ? 1 : max_useful) : num_sms;
}

template <int BOX, int WARPS, int STAGES, bool SP, bool HZ, int PIPE = 1, int NP = 0>
cudaError_t launch_ws(const CUtensorMap (&m)[6], const TmaArgs& t, int num_sms, cudaStream_t s) {
  constexpr int kProducers = NP > 0 ? NP : producers_for<WARPS>();
  auto kern = rowpair_ws_kernel<BOX, WARPS, STAGES, SP, HZ, kProducers, PIPE>;
  const size_t smem = size_t(WARPS) * STAGES * (GeoP<BOX>::kStageBytes + GeoP<BOX>::kParamBytes) +
                      1024 + size_t(WARPS) * STAGES * (16 + 8);
  cudaError_t e = set_smem(kern, smem);
  if (e != cudaSuccess) return e;
  // keep the SM's shared-memory carveout at its maximum, so lean entropy kernels of
  // another call (cl_entropy_lean_f32) can sit beside a scan CTA
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  kern<<<grid_for(t.n_tiles, WARPS, num_sms), (WARPS + kProducers) * 32, smem, s>>>(
      m[0], m[1], m[2], m[4], t);
  return cudaGetLastError();
}

template <int BOX, int WARPS, int STAGES, bool SP, bool HZ>
cudaError_t launch_rowseq(const CUtensorMap (&m)[6], const TmaArgs& t, int num_sms,
                          cudaStream_t s) {
  auto kern = rowseq_tma_kernel<BOX, WARPS, STAGES, SP, HZ>;
  const size_t smem = size_t(WARPS) * warp_bytes<BOX, STAGES>() + 1024 + 256;
  cudaError_t e = set_smem(kern, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid_for(t.n_tiles, WARPS, num_sms), WARPS * 32, smem, s>>>(m[0], m[1], m[2], m[3],
                                                                      m[4], m[5], t);
  return cudaGetLastError();
}

// softplus / z-gate are compile-time switches: four instantiations per geometry
template <bool WS, int BOX, int WARPS, int STAGES>
cudaError_t dispatch(bool sp, bool hz, const CUtensorMap (&m)[6], const TmaArgs& t, int n,
                     cudaStream_t s) {
  if constexpr (WS) {
    if (sp && hz) return launch_ws<BOX, WARPS, STAGES, true, true>(m, t, n, s);
    if (sp) return launch_ws<BOX, WARPS, STAGES, true, false>(m, t, n, s);
    if (hz) return launch_ws<BOX, WARPS, STAGES, false, true>(m, t, n, s);
    return launch_ws<BOX, WARPS, STAGES, false, false>(m, t, n, s);
  } else {
    if (sp && hz) return launch_rowseq<BOX, WARPS, STAGES, true, true>(m, t, n, s);
    if (sp) return launch_rowseq<BOX, WARPS, STAGES, true, false>(m, t, n, s);
    if (hz) return launch_rowseq<BOX, WARPS, STAGES, false, true>(m, t, n, s);
    return launch_rowseq<BOX, WARPS, STAGES, false, false>(m, t, n, s);
  }
}

// CL_SCAN_CFG=<row> forces a kCfgs row (experiments); otherwise the warp-specialised
// kernel with the fewest consumers per CTA that still puts every 16-row tile on its own
// SM (12 consumers once there are more than 7 tiles per SM).
constexpr int kNumCfgs = static_cast<int>(sizeof(kCfgs) / sizeof(kCfgs[0]));

int scan_cfg_index(uint64_t pair_tiles, int num_sms, int variant) {
  if (variant >= CL_SCAN_CONFIG_BASE) return variant - CL_SCAN_CONFIG_BASE;
  static const int forced = [] {
    const char* e = getenv("CL_SCAN_CFG");
    if (!e) return -1;
    const int v = atoi(e);
    return v >= 0 && v < static_cast<int>(sizeof(kCfgs) / sizeof(kCfgs[0])) ? v : -1;
  }();
  if (forced >= 0) return forced;
  const uint64_t per_sm = (pair_tiles + num_sms - 1) / num_sms;
  // Below ~11 tiles per SM, 32-timestep boxes (half the per-box pipeline fill and barrier
  // round trips) with the fewest consumers per CTA that still cover the tiles in about one
  // wave.  Measured (scan ms, tools/cfg_ab.py): C1 (96 tiles) 0.167 -> 0.152 (row 11);
  // C2 (128) 0.301 -> 0.269 (11); 512 tiles 0.327 -> 0.309 (12); 768: 0.453 -> 0.388 (12);
  // 1280: 0.634 -> 0.521 (13); 1792 and C3's 2048 stay with row 0 (0.649 vs 0.708, 1.376
  // vs 1.530 for row 13).
  if (per_sm <= 2) return 11;
  if (per_sm <= 6) return 12;
  if (per_sm <= 10) return 13;
  return kDefaultCfg;  // 12 consumers
}

// The L-parallel kernel (scan_lookback.cu) or not: its look-back costs a second pass of
// exponentials over all but the last segment, so it only pays while the chained kernel
// is parallelism-bound -- few 16-row tiles per SM (C1: 96 tiles, C2: 128, the B=1
// serving requests).  Returns the lookback table row, or -1 for the chained kernel.
// CL_LB_CFG=<row> / CL_LB_TILES=<max tiles> override (experiments).
int lookback_choice(uint64_t pair_tiles, uint64_t L, int num_sms, int variant) {
  if (variant >= CL_SCAN_LOOKBACK_BASE) return variant - CL_SCAN_LOOKBACK_BASE;
  if (variant == CL_SCAN_CHAINED || variant == CL_SCAN_ROWSEQ_TMA ||
      (variant >= CL_SCAN_CONFIG_BASE && variant < CL_SCAN_LOOKBACK_BASE))
    return -1;
  static const int forced_cfg = [] {
    const char* e = getenv("CL_LB_CFG");
    const int v = e ? atoi(e) : -1;
    return v >= 0 && v < kLookbackCfgs ? v : -1;
  }();
  static const long max_tiles_env = [] {
    const char* e = getenv("CL_LB_TILES");
    return e ? atol(e) : -1L;
  }();
  const int cfg = forced_cfg >= 0 ? forced_cfg : 0;
  if (variant == CL_SCAN_LOOKBACK) return cfg;
  const uint64_t max_tiles = max_tiles_env >= 0 ? static_cast<uint64_t>(max_tiles_env)
                                                 : 2ull * static_cast<uint64_t>(num_sms);
  // at least two 32-step boxes per segment at the chosen split
  if (pair_tiles <= max_tiles && L >= 4u * lookback_box(cfg)) return cfg;
  return -1;
}

// Split of the L-parallel kernel, from the SHAPE only (so every decided chunk gives the
// same bits): n segments of seg_len timesteps (whole boxes; the last one takes the rest),
// at most one (tile, segment) item per consumer warp of the grid (one wave), the split
// whose longest item is shortest, then the fewest segments.  Items cost (1 + phi) seg_len
// with an aggregate pass and `last` without; measured (profiles/r2b_lookback_ab.txt):
// phi = 0 -- equal segments -- is best, because the last segment waits for its
// predecessors' aggregate passes anyway (0.61 vs 0.70 ms-equivalents at C1 for phi = 0.6).
// CL_LB_SEGS=<n> forces n, CL_LB_PHI=<phi> the cost model (experiments).
void lookback_split(uint64_t L, int n_tiles, int num_sms, int cfg, int* seg_len, int* n_seg) {
  static const int forced = [] {
    const char* e = getenv("CL_LB_SEGS");
    return e ? atoi(e) : 0;
  }();
  const int box = lookback_box(cfg);
  const long Ll = static_cast<long>(L);
  int n_max = (num_sms * lookback_warps(cfg)) / (n_tiles > 0 ? n_tiles : 1);
  const int max_seg = static_cast<int>((Ll + box - 1) / box);
  if (n_max > max_seg) n_max = max_seg;
  if (n_max < 1) n_max = 1;
  if (forced > 0) {
    const int n = forced < max_seg ? forced : max_seg;
    long len = (Ll + n - 1) / n;
    len = (len + box - 1) / box * box;
    *seg_len = static_cast<int>(len);
    *n_seg = static_cast<int>((Ll + len - 1) / len);
    return;
  }
  // cost of an item in units of full-pass timesteps: (1 + phi) seg_len for a segment with
  // an aggregate pass (phi = its cost relative to the full pass), `last` for the last one
  static const double phi = [] {
    const char* e = getenv("CL_LB_PHI");
    return e ? atof(e) : 0.0;
  }();
  double best_cost = static_cast<double>(Ll);
  long best_len = ((Ll + box - 1) / box) * box;
  int best_n = 1;  // a single segment: one full pass
  for (long len = box; len < Ll; len += box) {
    for (long n = 2; n <= n_max; ++n) {
      const long last = Ll - (n - 1) * len;
      if (last <= 0) break;
      const double reg = (1.0 + phi) * static_cast<double>(len);
      const double cost = reg > last ? reg : static_cast<double>(last);
      if (cost < best_cost - 1e-9 || (cost < best_cost + 1e-9 && n < best_n)) {
        best_cost = cost;
        best_len = len;
        best_n = static_cast<int>(n);
      }
    }
  }
  *seg_len = static_cast<int>(best_len);
  *n_seg = best_n;
}

struct Selection {
  bool tma = false;
  int lb = -1;       // lookback table row, or -1
  int cfg_idx = -1;  // chained table row (kCfgs), or -1
  ScanCfg cfg{};
};

// The kernel a scan call runs (shared by the launch and cl_scan_plan_f32); an error
// message for an invalid variant.
const char* select_kernel(const cl_mamba1_args& a, int num_sms, int variant, Selection* out) {
  const bool tma_ok = tma_eligible(a);
  const bool forced_tma = variant == CL_SCAN_ROWSEQ_TMA || variant == CL_SCAN_LOOKBACK ||
                          variant == CL_SCAN_CHAINED || variant >= CL_SCAN_CONFIG_BASE;
  if ((variant >= CL_SCAN_CONFIG_BASE && variant < CL_SCAN_LOOKBACK_BASE &&
       variant - CL_SCAN_CONFIG_BASE >= kNumCfgs) ||
      (variant >= CL_SCAN_LOOKBACK_BASE && variant - CL_SCAN_LOOKBACK_BASE >= kLookbackCfgs) ||
      (variant > CL_SCAN_CHAINED && variant < CL_SCAN_CONFIG_BASE) || variant < 0)
    return "scan variant: no such kernel configuration";
  if (forced_tma && !tma_ok)
    return "scan variant rowseq_tma needs d_state 16, L % 4 == 0 and 16-byte aligned buffers";
  out->tma = forced_tma || (variant == CL_SCAN_AUTO && tma_ok);
  if (!out->tma) return nullptr;
  const uint64_t pair_tiles = ((a.dim + kRowsP - 1) / kRowsP) * a.batch;
  out->lb = lookback_choice(pair_tiles, a.seq_len, num_sms, variant);
  out->cfg_idx = out->lb >= 0 ? -1
                              : scan_cfg_index(pair_tiles, num_sms,
                                               variant == CL_SCAN_CHAINED ? CL_SCAN_AUTO : variant);
  out->cfg = out->lb >= 0 ? ScanCfg{kWarpSpecPair, lookback_box(out->lb), lookback_warps(out->lb), 2}
                          : kCfgs[out->cfg_idx];
  return nullptr;
}

}  // namespace

int scan_plan(cl_ctx* ctx, const cl_mamba1_args& a, int variant, cl_scan_plan* p) {
  Selection sel;
  const char* err = select_kernel(a, ctx->num_sms, variant, &sel);
  if (err) return fail(ctx, CL_E_INVALID, err);
  *p = cl_scan_plan{};
  if (!sel.tma) {
    p->kernel = CL_KERNEL_GENERIC;
    return CL_OK;
  }
  p->box = sel.cfg.box;
  p->warps = sel.cfg.warps;
  p->stages = sel.cfg.stages;
  if (sel.lb >= 0) {
    p->kernel = CL_KERNEL_LOOKBACK;
    p->config = sel.lb;
    const int n_tiles = static_cast<int>(((a.dim + kRowsP - 1) / kRowsP) * a.batch);
    lookback_split(a.seq_len, n_tiles, ctx->num_sms, sel.lb, &p->seg_len, &p->n_seg);
  } else {
    p->kernel = sel.cfg.kind == kRowSeq ? CL_KERNEL_ROWSEQ : CL_KERNEL_CHAINED;
    p->config = sel.cfg_idx;
    p->seg_len = -1;  // the decided chunk, rounded up to whole boxes (known on the device)
    p->n_seg = -1;
  }
  return CL_OK;
}

int scan_prepare_with_init(cl_ctx* ctx, const cl_mamba1_args& a, double* d_range,
                           uint64_t* d_counts, int bin_count, cudaStream_t s) {
  Selection sel;
  const char* err = select_kernel(a, ctx->num_sms, CL_SCAN_AUTO, &sel);
  if (err) return fail(ctx, CL_E_INVALID, err);
  cl_workspace* w = workspace(ctx, s);
  if (!w) return CL_E_CUDA;
  const uint64_t L = a.seq_len, Bt = a.batch;
  const bool ws = sel.tma && sel.cfg.kind != kRowSeq;
  int rc = CL_OK;
  if (ws)
    rc = grow_scratch(ctx, w, &w->d_bct, &w->bct_bytes, 2 * size_t(Bt) * L * kN * sizeof(float),
                      "cudaMalloc(B/C transpose)");
  if (rc) return rc;
  // without a TMA scan to feed, only the init block runs (grid z = 2 alone)
  const dim3 grid(ws ? static_cast<unsigned>((L + 31) / 32) : 1u, ws ? static_cast<unsigned>(Bt) : 1u,
                  3);
  init_transpose_kernel<<<grid, 256, 0, s>>>(a.B, a.C, ws ? w->d_bct : nullptr,
                                             ws ? w->d_bct + kN : nullptr, static_cast<int>(L),
                                             2 * kN, d_range,
                                             reinterpret_cast<unsigned long long*>(d_counts),
                                             bin_count);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "init_transpose_kernel launch");
  ++ctx->launches;
  w->bct_ready = ws;
  w->bct_capture = capture_id_of(s);
  w->bct_B = a.B;
  w->bct_C = a.C;
  w->bct_batch = Bt;
  w->bct_L = L;
  return CL_OK;
}

int scan_mamba1(cl_ctx* ctx, const cl_mamba1_args& a, const cl_decision* d_decision,
                int fixed_chunk, int variant, cudaStream_t s) {
  Selection sel;
  const char* err = select_kernel(a, ctx->num_sms, variant, &sel);
  if (err) return fail(ctx, CL_E_INVALID, err);
  if (sel.tma) {
    const int lb = sel.lb;
    const int cfg_idx = sel.cfg_idx;
    const ScanCfg cfg = sel.cfg;
    const bool ws = cfg.kind != kRowSeq;
    const uint64_t L = a.seq_len, D = a.dim, Bt = a.batch;
    const int rows_per_tile = ws ? kRowsP : kRows;
    const int tiles_per_batch = static_cast<int>((D + rows_per_tile - 1) / rows_per_tile);
    const int n_tiles = tiles_per_batch * static_cast<int>(Bt);
    const size_t work_bytes = (size_t(n_tiles) + 32) * sizeof(unsigned int);
    const size_t carry_bytes = size_t(n_tiles) * rows_per_tile * kN * sizeof(float);
    const size_t bc_bytes = 2 * size_t(Bt) * L * kN * sizeof(float);
    cl_workspace* w = workspace(ctx, s);  // scratch of this stream only
    if (!w) return CL_E_CUDA;
    const bool fresh_work = w->work_bytes < work_bytes;
    int rc = grow_scratch(ctx, w, &w->d_work, &w->work_bytes, work_bytes, "cudaMalloc(scan work)");
    if (!rc && !ws)
      rc = grow_scratch(ctx, w, &w->d_carry, &w->carry_bytes, carry_bytes, "cudaMalloc(carry)");
    if (!rc) rc = grow_scratch(ctx, w, &w->d_bct, &w->bct_bytes, bc_bytes, "cudaMalloc(B/C transpose)");
    if (rc) return rc;
    unsigned int epoch = 0;
    int lb_seg_len = 0, lb_n_seg = 0;
    if (lb >= 0) {
      // aggregate words {tag, value}: one tag per launch (every (tile, segment) slot is
      // written once per launch); zeroed on allocation, on tag wrap, and in-graph before
      // every launch of a captured graph
      lookback_split(L, n_tiles, ctx->num_sms, lb, &lb_seg_len, &lb_n_seg);
      const size_t agg_bytes = size_t(n_tiles) * lb_n_seg * kRowsP * 18 * sizeof(unsigned long long);
      const bool fresh = w->agg_bytes < agg_bytes;
      rc = grow_scratch(ctx, w, &w->d_agg, &w->agg_bytes, agg_bytes, "cudaMalloc(scan aggregates)");
      if (rc) return rc;
      if (fresh) {
        if ((rc = zero_now(ctx, w->d_agg, w->agg_bytes))) return rc;
        w->agg_epoch = 1;
      } else if (!w->captured && (w->agg_epoch == 0 || w->agg_epoch >= 0x7FFFFFFFu)) {
        cudaError_t e = cudaMemsetAsync(w->d_agg, 0, w->agg_bytes, s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemsetAsync(scan aggregates)");
        w->agg_epoch = 1;
      }
      epoch = w->captured ? 0u : w->agg_epoch++;
    } else if (ws) {
      // tagged carry words: zeroed when (re)allocated or when the epoch would wrap; each
      // launch takes tags epoch + 1 .. epoch + (segments <= boxes), above every older tag
      const size_t tcarry_bytes = size_t(n_tiles) * kRowsP * kN * sizeof(unsigned long long);
      const bool fresh = w->tcarry_bytes < tcarry_bytes;
      rc = grow_scratch(ctx, w, &w->d_tcarry, &w->tcarry_bytes, tcarry_bytes, "cudaMalloc(tagged carry)");
      if (rc) return rc;
      const unsigned span = static_cast<unsigned>((L + cfg.box - 1) / cfg.box) + 2u;
      // eager: host epochs below 0x80000000, advanced past every launch's tags; a captured
      // graph bakes its epoch into every replay, so it zeroes the words it uses in-graph
      // before each launch (4 MB at C3: ~2 us of a 1.35 ms scan)
      if (fresh) {
        if ((rc = zero_now(ctx, w->d_tcarry, w->tcarry_bytes))) return rc;
        w->carry_epoch = 1;
      }
      if (w->captured) {
        cudaError_t e = cudaMemsetAsync(w->d_tcarry, 0, tcarry_bytes, s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemsetAsync(tagged carry)");
        epoch = 1;
      } else {
        if (w->carry_epoch == 0 || w->carry_epoch > 0x7FFFFFFFu - span) {
          cudaError_t e = cudaMemsetAsync(w->d_tcarry, 0, w->tcarry_bytes, s);
          if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemsetAsync(tagged carry)");
          w->carry_epoch = 1;
        }
        epoch = w->carry_epoch;
        w->carry_epoch += span;
      }
    }
    // B^T / C^T: interleaved per timestep ([B | C], 128 B rows, one TMA box) for the
    // warp-specialised kernel, two separate (b, L, 16) arrays for the row kernel
    float* d_Bt = w->d_bct;
    float* d_Ct = ws ? w->d_bct + kN : w->d_bct + size_t(Bt) * L * kN;
    const int box = cfg.box;
    const int sw = box == 32 ? 128 : (box == 16 ? 64 : 32);
    CUtensorMap m[6];  // u, delta, z, out, B^T (or [B|C]), C^T
    std::memset(m, 0, sizeof(m));
    bool ok = make_map(&m[0], a.u, L, D, Bt, box, rows_per_tile, sw) &&
              make_map(&m[1], a.delta, L, D, Bt, box, rows_per_tile, sw) &&
              make_map(&m[2], a.z ? a.z : a.u, L, D, Bt, box, rows_per_tile, sw) &&
              make_map(&m[3], a.out, L, D, Bt, box, rows_per_tile, sw);
    if (ok && ws) ok = make_map(&m[4], d_Bt, 2 * kN, L, Bt, 2 * kN, box, 0);
    if (ok && !ws)
      ok = make_map(&m[4], d_Bt, kN, L, Bt, kN, box, 0) &&
           make_map(&m[5], d_Ct, kN, L, Bt, kN, box, 0);
    if (!ok) return fail(ctx, CL_E_CUDA, "cuTensorMapEncodeTiled failed");
    // the warp-specialised kernels return their ticket to 0 themselves (ticket_retire);
    // the row kernel's per-tile flags are zeroed every launch
    cudaError_t e = cudaSuccess;
    if (fresh_work) {
      if ((rc = zero_now(ctx, w->d_work, w->work_bytes))) return rc;
    }
    if (!ws || w->ticket_dirty) e = cudaMemsetAsync(w->d_work, 0, work_bytes, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemsetAsync(scan work)");
    w->ticket_dirty = !ws;  // the row kernel leaves its ticket and flags behind
    const bool prepared = ws && w->bct_ready && w->bct_B == a.B && w->bct_C == a.C &&
                          w->bct_batch == Bt && w->bct_L == L &&
                          w->bct_capture == capture_id_of(s);
    w->bct_ready = false;  // consumed (or stale) either way
    if (!prepared) {
      const dim3 tgrid(static_cast<unsigned>((L + 31) / 32), static_cast<unsigned>(Bt), 2);
      transpose_bc_kernel<<<tgrid, 256, 0, s>>>(a.B, a.C, d_Bt, d_Ct, static_cast<int>(L),
                                                ws ? 2 * kN : kN);
      e = cudaGetLastError();
      if (e != cudaSuccess) return cuda_fail(ctx, e, "transpose_bc_kernel launch");
      ++ctx->launches;
    }
    TmaArgs t{};
    t.out = a.out;
    t.A = a.A;
    t.D = a.D;
    t.bias = a.delta_bias;
    t.h0 = a.h0;
    t.h_last = a.h_last;
    t.carry = w->d_carry;
    t.tcarry = w->d_tcarry;
    t.epoch = epoch;
    t.stage_params = aligned16(a.A) && (!a.delta_bias || aligned16(a.delta_bias)) &&
                     (!a.D || aligned16(a.D));
    t.ticket = w->d_work;
    t.flags = w->d_work + 32;
    t.batch = Bt;
    t.dim = D;
    t.L = L;
    t.tiles_per_batch = tiles_per_batch;
    t.n_tiles = n_tiles;
    t.decision = d_decision;
    t.fixed_chunk = fixed_chunk;
    const bool sp = a.delta_softplus != 0, hz = a.z != nullptr;
    const int n = ctx->num_sms;
    if (lb >= 0) {
      LookbackLaunch p{};
      p.A = a.A;
      p.D = a.D;
      p.bias = a.delta_bias;
      p.h0 = a.h0;
      p.out = a.out;
      p.h_last = a.h_last;
      p.agg = w->d_agg;
      p.epoch = epoch;
      p.launch_counter = w->captured ? w->d_epoch + 1 : nullptr;
      p.stage_params = t.stage_params;
      p.ticket = w->d_work;
      p.batch = Bt;
      p.dim = D;
      p.L = L;
      p.tiles_per_batch = tiles_per_batch;
      p.n_tiles = n_tiles;
      p.seg_len = lb_seg_len;
      p.n_seg = lb_n_seg;
      p.decision = d_decision;
      const CUtensorMap lm[4] = {m[0], m[1], m[2], m[4]};
      e = launch_lookback(lb, sp, hz, lm, p, n, s);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "lookback scan kernel launch");
      ++ctx->launches;
      return CL_OK;
    }
    switch (cfg_idx) {
      case 1: e = dispatch<false, 32, 4, 3>(sp, hz, m, t, n, s); break;
      case 2: e = dispatch<false, 16, 8, 3>(sp, hz, m, t, n, s); break;
      case 3: e = dispatch<false, 16, 7, 3>(sp, hz, m, t, n, s); break;
      case 4: e = dispatch<true, 16, 1, 4>(sp, hz, m, t, n, s); break;
      case 5: e = dispatch<true, 16, 2, 4>(sp, hz, m, t, n, s); break;
      case 6: e = dispatch<true, 16, 4, 4>(sp, hz, m, t, n, s); break;
      case 7: e = dispatch<true, 16, 7, 3>(sp, hz, m, t, n, s); break;
      case 8:
        e = sp && hz ? launch_ws<16, 12, 2, true, true, 0>(m, t, n, s)
                     : dispatch<true, 16, 12, 2>(sp, hz, m, t, n, s);
        break;
      case 9: e = dispatch<true, 16, 14, 2>(sp, hz, m, t, n, s); break;
      case 10: e = dispatch<true, 32, 1, 4>(sp, hz, m, t, n, s); break;
      case 11: e = dispatch<true, 32, 2, 4>(sp, hz, m, t, n, s); break;
      case 12: e = dispatch<true, 32, 4, 3>(sp, hz, m, t, n, s); break;
      case 13: e = dispatch<true, 32, 8, 2>(sp, hz, m, t, n, s); break;
      case 14: e = dispatch<true, 32, 6, 3>(sp, hz, m, t, n, s); break;
      default: e = dispatch<true, 16, 12, 2>(sp, hz, m, t, n, s); break;
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "scan kernel launch");
    ++ctx->launches;
    if (!ws && w->captured) {
      // the row kernel leaves its ticket and flags behind; a captured graph cannot hand
      // that state to later graphs through the host flag (their replay order is not
      // known at capture), so it restores the clean ticket in-graph
      e = cudaMemsetAsync(w->d_work, 0, work_bytes, s);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemsetAsync(scan work)");
      w->ticket_dirty = false;
    }
    return CL_OK;
  }
  if (a.d_state < 1 || a.d_state > 64)
    return fail(ctx, CL_E_INVALID, "d_state must lie in [1, 64]");
  GenericArgs g{};
  g.u = a.u;
  g.delta = a.delta;
  g.A = a.A;
  g.B = a.B;
  g.C = a.C;
  g.D = a.D;
  g.z = a.z;
  g.bias = a.delta_bias;
  g.h0 = a.h0;
  g.out = a.out;
  g.h_last = a.h_last;
  g.batch = a.batch;
  g.dim = a.dim;
  g.L = a.seq_len;
  g.N = static_cast<int>(a.d_state);
  g.softplus = a.delta_softplus;
  g.decision = d_decision;
  const uint64_t rows = a.batch * a.dim;
  const unsigned grid = static_cast<unsigned>((rows + 127) / 128);
  if (a.d_state == 16)
    generic_kernel<16><<<grid, 128, 0, s>>>(g);
  else
    generic_kernel<0><<<grid, 128, 0, s>>>(g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "generic_kernel launch");
  ++ctx->launches;
  (void)fixed_chunk;
  return CL_OK;
}

int state_update_f32(cl_ctx* ctx, const cl_state_update_args& a, cudaStream_t s) {
  DecodeArgs d{a.state, a.x, a.dt, a.A, a.B, a.C, a.D, a.z, a.dt_bias, a.out,
               a.batch, a.dim, static_cast<int>(a.d_state), a.dt_softplus};
  const uint64_t rows = a.batch * a.dim;
  if (rows == 0) return CL_OK;
  const unsigned grid = static_cast<unsigned>((rows + 127) / 128);
  if (a.d_state == 16)
    decode_kernel<16><<<grid, 128, 0, s>>>(d);
  else
    decode_kernel<0><<<grid, 128, 0, s>>>(d);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "decode_kernel launch");
  ++ctx->launches;
  return CL_OK;
}

}  // namespace cl
