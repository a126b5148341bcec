// scan_lookback.cu -- the L-parallel fused Mamba-1 scan for few-row shapes (sm_100a, fp32).
//
// The chained kernel (scan_mamba1.cu, rowpair_ws_kernel) walks every 16-row tile's L
// serially: its parallelism is the tile count, 96 at C1 (B=1, d_inner=1536) and 128 at C2,
// i.e. under one warp per SM.  Here each tile's L is cut into n_seg segments (tied to the
// SHAPE, never to the decided chunk, so the output is bit-identical for every chunk) and
// every (tile, segment) item runs on its own warp:
//
//   phase 1  (segments 0 .. n_seg-2)  local recurrence from h = 0 over the segment:
//            h~_end = sum_t (prod_{t'>t} exp(dt' A)) B_t dt'_t u_t   and   S = sum_t dt'_t,
//            published as tagged 64-bit words {epoch, value} (aggregate of the segment)
//   look-back (segments 1 .. n_seg-1) the carry-in is the Horner fold of the published
//            aggregates of segments 0 .. k-1 in segment order, starting from h0:
//               h_in = exp(A S_{k-1}) (... (exp(A S_0) h0 + h~_0) ...) + h~_{k-1}
//            -- a fixed order, so the result is deterministic and run-to-run identical
//            (a decoupled look-back that stops at the first inclusive prefix would make
//            the bits depend on timing)
//   phase 3  the full fused recurrence from h_in (pair_box / pair_box_pipe: the exact
//            operation sequence of the chained kernel), y stored, h_last at the last
//            segment.
//
// Exponent identity behind the fold: prod_t exp(dt'_t A) = exp(A sum_t dt'_t), so a
// segment's state transition costs one exp per state, not one per timestep.  Work is
// (2 - 2/n_seg) passes over the exponentials instead of one: worth it only while the
// chained kernel is parallelism-bound (the launcher's choice, scan_mamba1.cu).
//
// Reference contract: chunklab::scan_chunked (scan.hpp:123-136) carries the state across
// windows; the reference has no parallel prefix.  Parity: <= 1e-5
// normwise vs the fp64 oracle (tests/test_gpu_lookback.py).
#include <cstdlib>

#include "scan_common.cuh"

namespace cl {
namespace {

constexpr int kAggWords = 18;           // per row: 16 states, S, pad -- each {tag, value}
constexpr int kPhase1Flag = 1 << 29;    // meta.y bit: a phase-1 (aggregate) box

struct LbArgs {
  const float *A, *D, *bias, *h0;
  float* out;
  float* h_last;
  unsigned long long* agg;  // [n_tiles][n_seg][16 rows][kAggWords]
  unsigned int epoch;       // tag of this launch's aggregate words (eager)
  unsigned int* launch_counter;  // captured graphs: the device-side launch counter (launch_epoch)
  int stage_params;
  unsigned int* ticket;
  uint64_t batch, dim, L;
  int tiles_per_batch, n_tiles;
  int seg_len, n_seg;
  int pipe1;  // software-pipelined aggregate pass (A/B switch, CL_LB_PIPE1)
  const cl_decision* decision;
};

struct LbItem {
  int tile, seg, nbox;
  int t0;
};

// One phase-1 box: the local recurrence (no C.h, no y, no gate) and the in-order sum of
// the discretised steps.  The elementwise prologue is pair_box's, operation for
// operation (softplus of the lane's timestep pair, partner exchange, x = dt * u).
template <int BOX, bool SP>
__device__ __forceinline__ void agg_box(const unsigned char* st, int r, int hf, int valid,
                                        float bias, const f2_t (&A2p)[kN / 4],
                                        f2_t (&h2)[kN / 4], float& sdt) {
  using G = GeoP<BOX>;
  constexpr int kP = kN / 4;
  constexpr int kBCRow = 2 * kN * 4;
  const unsigned char* sB = st + 3 * G::kTileBytes + 32 * hf;
  const f2_t bias2 = pk(bias, bias);
#pragma unroll
  for (int j = 0; j < BOX / 4; ++j) {
    if (4 * j >= valid) break;
    const int off = Geo<BOX>::swz(r, j);
    const float4 u4 = *reinterpret_cast<const float4*>(st + off);
    // this lane's delta pair (timesteps 2hf, 2hf + 1): an 8-byte load, no select
    const float2 d2 = *reinterpret_cast<const float2*>(st + G::kTileBytes + off + 8 * hf);
    f2_t mine = add2(pk(d2.x, d2.y), bias2);
    if (SP) mine = softplus2(mine);
    const f2_t other = shfl_xor2(mine, 1);
    const f2_t dt01 = hf ? other : mine, dt23 = hf ? mine : other;
    const f2_t x01 = mul2(dt01, pk(u4.x, u4.y)), x23 = mul2(dt23, pk(u4.z, u4.w));
    float dt[4], xs[4];
    upk(dt01, dt[0], dt[1]);
    upk(dt23, dt[2], dt[3]);
    upk(x01, xs[0], xs[1]);
    upk(x23, xs[2], xs[3]);
    f2_t dA[4][kP];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const f2_t dd = pk(dt[k], dt[k]);
#pragma unroll
      for (int i = 0; i < kP; ++i) {
        dA[k][i] = state_exp2_pair(mul2(A2p[i], dd), i);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const ulonglong2* Bt = reinterpret_cast<const ulonglong2*>(sB + (4 * j + k) * kBCRow);
      const f2_t xx = pk(xs[k], xs[k]);
#pragma unroll
      for (int q = 0; q < kP / 2; ++q) {
        const ulonglong2 bq = Bt[q];
        h2[2 * q] = fma2(dA[k][2 * q], h2[2 * q], mul2(bq.x, xx));
        h2[2 * q + 1] = fma2(dA[k][2 * q + 1], h2[2 * q + 1], mul2(bq.y, xx));
      }
      sdt = __fadd_rn(sdt, dt[k]);
    }
  }
}

// agg_box for a full box, software-pipelined by one 4-timestep group like
// pair_box_pipe: group j+1's serial prologue (LDS, bias add, softplus, partner exchange)
// is issued between group j's exponentials and its recurrence.  Same operations on the
// same values as agg_box.
template <int BOX, bool SP>
__device__ __forceinline__ void agg_box_pipe(const unsigned char* st, int r, int hf, float bias,
                                             const f2_t (&A2p)[kN / 4], f2_t (&h2)[kN / 4],
                                             float& sdt) {
  using G = GeoP<BOX>;
  constexpr int kP = kN / 4;
  constexpr int kG = BOX / 4;
  constexpr int kBCRow = 2 * kN * 4;
  const unsigned char* sB = st + 3 * G::kTileBytes + 32 * hf;
  const f2_t bias2 = pk(bias, bias);
  auto prep = [&](int j, float (&dt)[4], float (&xs)[4]) {
    const int off = Geo<BOX>::swz(r, j);
    const float4 u4 = *reinterpret_cast<const float4*>(st + off);
    // this lane's delta pair (timesteps 2hf, 2hf + 1): an 8-byte load, no select
    const float2 d2 = *reinterpret_cast<const float2*>(st + G::kTileBytes + off + 8 * hf);
    f2_t mine = add2(pk(d2.x, d2.y), bias2);
    if (SP) mine = softplus2(mine);
    const f2_t other = shfl_xor2(mine, 1);
    const f2_t dt01 = hf ? other : mine, dt23 = hf ? mine : other;
    const f2_t x01 = mul2(dt01, pk(u4.x, u4.y)), x23 = mul2(dt23, pk(u4.z, u4.w));
    upk(dt01, dt[0], dt[1]);
    upk(dt23, dt[2], dt[3]);
    upk(x01, xs[0], xs[1]);
    upk(x23, xs[2], xs[3]);
  };
  float dt[4], xs[4];
  prep(0, dt, xs);
#pragma unroll
  for (int j = 0; j < kG; ++j) {
    f2_t dA[4][kP];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const f2_t dd = pk(dt[k], dt[k]);
#pragma unroll
      for (int i = 0; i < kP; ++i) {
        dA[k][i] = state_exp2_pair(mul2(A2p[i], dd), i);
      }
    }
    float ndt[4], nxs[4];
    if (j + 1 < kG) prep(j + 1, ndt, nxs);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const ulonglong2* Bt = reinterpret_cast<const ulonglong2*>(sB + (4 * j + k) * kBCRow);
      const f2_t xx = pk(xs[k], xs[k]);
#pragma unroll
      for (int q = 0; q < kP / 2; ++q) {
        const ulonglong2 bq = Bt[q];
        h2[2 * q] = fma2(dA[k][2 * q], h2[2 * q], mul2(bq.x, xx));
        h2[2 * q + 1] = fma2(dA[k][2 * q + 1], h2[2 * q + 1], mul2(bq.y, xx));
      }
      sdt = __fadd_rn(sdt, dt[k]);
    }
    if (j + 1 < kG) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        dt[k] = ndt[k];
        xs[k] = nxs[k];
      }
    }
  }
}

// Carry-in fold over segments [j0, j1) of one tile: h = exp2(A2 S_j) h + h~_j in segment
// order.  The aggregate words are loaded kBatch segments at a time (independent loads in
// flight), then polled only where a tag was not yet current.
#ifndef CL_LB_FOLD_BATCH
#define CL_LB_FOLD_BATCH 4
#endif
constexpr int kFoldBatch = CL_LB_FOLD_BATCH;  // segments per batch of loads: 2 and 4 tie, 8 is 5% slower (C1/C2)

template <int NB>
__device__ __forceinline__ void fold_batch(const unsigned long long* base, int j0, int r, int hf,
                                           unsigned epoch, const f2_t (&A2p)[kN / 4],
                                           f2_t (&h)[kN / 4]) {
  constexpr int kP = kN / 4;
  unsigned long long w[NB][kN / 2], ws[NB][2];
  auto load = [&](int b) {
    const unsigned long long* w64 = base + size_t(j0 + b) * kRowsP * kAggWords;
#pragma unroll
    for (int i = 0; i < kN / 2; i += 2) ld_relaxed_u64x2(w64 + 8 * hf + i, w[b][i], w[b][i + 1]);
    ld_relaxed_u64x2(w64 + 16, ws[b][0], ws[b][1]);
  };
  auto ready = [&](int b) {
    CL_DCHECK(epoch >= kGraphEpochA || (ws[b][0] >> 32) <= epoch);
    bool ok = (ws[b][0] >> 32) == epoch;
#pragma unroll
    for (int i = 0; i < kN / 2; ++i) ok &= (w[b][i] >> 32) == epoch;
    return ok;
  };
#pragma unroll
  for (int b = 0; b < NB; ++b) load(b);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    while (!__all_sync(0xffffffffu, ready(b))) {
      __nanosleep(64);
      load(b);
    }
    const float S = __uint_as_float(static_cast<unsigned>(ws[b][0]));
    const f2_t SS = pk(S, S);
#pragma unroll
    for (int i = 0; i < kP; ++i) {
      float al, ah;
      upk(mul2(A2p[i], SS), al, ah);
      const f2_t P = pk(ex2_approx(al), ex2_approx(ah));
      const f2_t g = pk(__uint_as_float(static_cast<unsigned>(w[b][2 * i])),
                        __uint_as_float(static_cast<unsigned>(w[b][2 * i + 1])));
      h[i] = fma2(P, h[i], g);
    }
  }
}

template <int BOX, int WARPS, int STAGES, bool SP, bool HZ, int NPROD>
__global__ void __launch_bounds__((WARPS + NPROD) * 32, 1)
    lookback_ws_kernel(const __grid_constant__ CUtensorMap map_u,
                       const __grid_constant__ CUtensorMap map_dt,
                       const __grid_constant__ CUtensorMap map_z,
                       const __grid_constant__ CUtensorMap map_bc, LbArgs a) {
  using G = GeoP<BOX>;
  if (a.decision && a.decision->status != 0) return;  // deferred device error: no writes
  const int L = static_cast<int>(a.L);
  const int seg_len = a.seg_len, n_seg = a.n_seg;
  const int n_items = n_seg * a.n_tiles;

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int kWB = STAGES * G::kStageBytes;
  unsigned char* params = smem + size_t(WARPS) * kWB;
  uint64_t* full = reinterpret_cast<uint64_t*>(params + size_t(WARPS) * STAGES * G::kParamBytes);
  uint64_t* empty = full + WARPS * STAGES;
  int2* meta = reinterpret_cast<int2*>(empty + WARPS * STAGES);

  if (threadIdx.x < WARPS * STAGES) {
    mbar_init(full + threadIdx.x, 1);
    mbar_init(empty + threadIdx.x, 1);
  }
  // the launch's tag, read before any producer can retire (the last claimer of the grid
  // advances a captured graph's counter, and it retires only after every CTA passed here)
  __shared__ unsigned s_epoch;
  if (threadIdx.x == 0) {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_epoch = launch_epoch(a.epoch, a.launch_counter);
  }
  __syncthreads();

  // items are dispatched segment-major: every predecessor (tile, j < k) of an item holds a
  // smaller ticket, was claimed earlier and never waits on a later item -- forward progress
  auto decode = [&](int id) {
    LbItem it;
    it.seg = id / a.n_tiles;
    it.tile = id % a.n_tiles;
    it.t0 = it.seg * seg_len;
    // segments 0 .. n_seg-2 are seg_len long; the last one (no aggregate pass) takes the
    // rest, about twice as long, so every item costs about the same
    const int len = it.seg == n_seg - 1 ? L - it.t0 : seg_len;
    it.nbox = (len + BOX - 1) / BOX;
    return it;
  };

  if (warp >= WARPS) {
    // ---------------- producers: phase-1 boxes (u, delta, [B | C]), then phase-3 boxes
    constexpr int kPer = (WARPS + NPROD - 1) / NPROD;
    const int w = (warp - WARPS) * kPer + lane;
    bool live = lane < kPer && w < WARPS;
    if (lane == 0 && warp == WARPS) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_u)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_dt)));
      if (HZ) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_z)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bc)));
    }
    int p_item = live ? static_cast<int>(atomicAdd(a.ticket, 1u)) : 0;
    LbItem p_it = decode(p_item);
    int p_b = p_it.tile / a.tiles_per_batch, p_r0 = (p_it.tile % a.tiles_per_batch) * kRowsP;
    bool p_phase1 = p_it.seg < n_seg - 1;
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
            const bool first = p_box == 0 && (p_phase1 || p_it.seg == n_seg - 1);
            const bool stage = first && a.stage_params && p_r0 + kRowsP <= static_cast<int>(a.dim);
            meta[w * STAGES + slot] = make_int2(
                p_item, p_box | (stage ? kStagedFlag : 0) | (p_phase1 ? kPhase1Flag : 0));
            const bool with_z = HZ && !p_phase1;
            uint32_t tx = with_z ? G::kStageBytes : G::kStageBytes - G::kTileBytes;
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
            if (with_z) tma_load_3d(st + 2 * G::kTileBytes, &map_z, t, p_r0, p_b, bar);
            tma_load_3d(st + 3 * G::kTileBytes, &map_bc, 0, t, p_b, bar);
            if (++p_box == p_it.nbox) {
              p_box = 0;
              if (p_phase1) {
                p_phase1 = false;  // the same item's phase-3 boxes follow
              } else {
                p_item = static_cast<int>(atomicAdd(a.ticket, 1u));
                p_it = decode(p_item);
                p_b = p_it.tile / a.tiles_per_batch;
                p_r0 = (p_it.tile % a.tiles_per_batch) * kRowsP;
                p_phase1 = p_it.seg < n_seg - 1;
              }
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
                  static_cast<unsigned>(n_items) + gridDim.x * static_cast<unsigned>(WARPS),
                  a.launch_counter);
    return;
  }

  // ---------------- consumers ----------------
  const int r = lane >> 1, hf = lane & 1;
  const unsigned char* wbase = smem + size_t(warp) * kWB;
  uint64_t* wfull = full + warp * STAGES;
  uint64_t* wempty = empty + warp * STAGES;
  const int2* wmeta = meta + warp * STAGES;
  constexpr int kP = kN / 4;
  f2_t h2[kP], A2p[kP];
  float bias = 0.f, Dc = 0.f, sdt = 0.f;
  LbItem cur{};
  int row = 0;
  bool row_valid = false;
  const unsigned epoch = s_epoch;
  const unsigned long long tag = static_cast<unsigned long long>(epoch) << 32;
  for (int iter = 0;; ++iter) {
    const int slot = iter % STAGES;
    mbar_wait(wfull + slot, (iter / STAGES) & 1);
    const int2 m = wmeta[slot];
    if (m.x < 0) break;
    const int box = m.y & ~(kStagedFlag | kPhase1Flag);
    const bool phase1 = (m.y & kPhase1Flag) != 0;
    CL_DCHECK(m.x < n_items && box < decode(m.x).nbox);
    const unsigned char* st = wbase + slot * G::kStageBytes;
    if (box == 0 && (phase1 || m.x / a.n_tiles == n_seg - 1)) {
      // the item's first box: its parameters
      cur = decode(m.x);
      const int b = cur.tile / a.tiles_per_batch;
      const int c = (cur.tile % a.tiles_per_batch) * kRowsP + r;
      row_valid = c < static_cast<int>(a.dim);
      const int cc = row_valid ? c : 0;
      row = b * static_cast<int>(a.dim) + cc;
      if (m.y & kStagedFlag) {
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
      if (phase1) {
#pragma unroll
        for (int i = 0; i < kP; ++i) h2[i] = 0ull;
        sdt = 0.f;
      }
    }
    const int tbox = cur.t0 + box * BOX;
    if (phase1) {
      if (a.pipe1 && tbox + BOX <= L)
        agg_box_pipe<BOX, SP>(st, r, hf, bias, A2p, h2, sdt);
      else
        agg_box<BOX, SP>(st, r, hf, L - tbox, bias, A2p, h2, sdt);
      __syncwarp();
      if (lane == 0) mbar_arrive(wempty + slot);
      if (box == cur.nbox - 1) {
        // publish the aggregate {h~_end, S} of (tile, seg)
        float hs[kN / 2];
#pragma unroll
        for (int i = 0; i < kP; ++i) upk(h2[i], hs[2 * i], hs[2 * i + 1]);
        unsigned long long* w64 =
            a.agg + ((size_t(cur.tile) * n_seg + cur.seg) * kRowsP + r) * kAggWords;
#pragma unroll
        for (int i = 0; i < kN / 2; i += 2)
          st_relaxed_u64x2(w64 + 8 * hf + i, tag | __float_as_uint(hs[i]),
                           tag | __float_as_uint(hs[i + 1]));
        if (hf == 0) st_relaxed_u64x2(w64 + 16, tag | __float_as_uint(sdt), tag);
      }
      continue;
    }
    if (box == 0) {
      // carry-in of this segment: h0 for segment 0, else the in-order fold of the
      // published aggregates of segments 0 .. seg-1 (deterministic; see the header)
      f2_t h[kP];
      const float* h0p = a.h0 ? a.h0 + size_t(row) * kN + 8 * hf : nullptr;
#pragma unroll
      for (int s = 0; s < kN / 2; s += 4) {
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (h0p) q = __ldcg(reinterpret_cast<const float4*>(h0p + s));
        h[s / 2] = pk(q.x, q.y);
        h[s / 2 + 1] = pk(q.z, q.w);
      }
      const unsigned long long* tb =
          a.agg + (size_t(cur.tile) * n_seg * kRowsP + r) * kAggWords;
      int j = 0;
      for (; j + kFoldBatch <= cur.seg; j += kFoldBatch)
        fold_batch<kFoldBatch>(tb, j, r, hf, epoch, A2p, h);
      for (; j < cur.seg; ++j) fold_batch<1>(tb, j, r, hf, epoch, A2p, h);
#pragma unroll
      for (int i = 0; i < kP; ++i) h2[i] = h[i];
    }
    float* ydst = row_valid ? a.out + size_t(row) * a.L + tbox : nullptr;
    if (tbox + BOX <= L)
      pair_box_pipe<BOX, SP, HZ>(st, ydst, r, hf, bias, Dc, A2p, h2);
    else
      pair_box<BOX, SP, HZ>(st, ydst, r, hf, L - tbox, bias, Dc, A2p, h2);
    __syncwarp();
    if (lane == 0) mbar_arrive(wempty + slot);
    if (box == cur.nbox - 1 && cur.seg == n_seg - 1 && a.h_last && row_valid) {
      float hs[kN / 2];
#pragma unroll
      for (int i = 0; i < kP; ++i) upk(h2[i], hs[2 * i], hs[2 * i + 1]);
      float* dst = a.h_last + size_t(row) * kN + 8 * hf;
      __stcg(reinterpret_cast<float4*>(dst), make_float4(hs[0], hs[1], hs[2], hs[3]));
      __stcg(reinterpret_cast<float4*>(dst + 4), make_float4(hs[4], hs[5], hs[6], hs[7]));
    }
  }
}

template <int BOX, int WARPS, int STAGES, bool SP, bool HZ>
cudaError_t launch_lb(const CUtensorMap (&m)[4], const LbArgs& t, int num_sms, cudaStream_t s) {
  constexpr int kProducers = WARPS >= 8 ? 2 : 1;
  auto kern = lookback_ws_kernel<BOX, WARPS, STAGES, SP, HZ, kProducers>;
  const size_t smem = size_t(WARPS) * STAGES * (GeoP<BOX>::kStageBytes + GeoP<BOX>::kParamBytes) +
                      1024 + size_t(WARPS) * STAGES * (16 + 8);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int n_items = t.n_tiles * t.n_seg;
  const int max_useful = (n_items + WARPS - 1) / WARPS;
  const int grid = max_useful < num_sms ? max_useful : num_sms;
  kern<<<grid, (WARPS + kProducers) * 32, smem, s>>>(m[0], m[1], m[2], m[3], t);
  return cudaGetLastError();
}

template <int BOX, int WARPS, int STAGES>
cudaError_t dispatch_lb(bool sp, bool hz, const CUtensorMap (&m)[4], const LbArgs& t, int n,
                        cudaStream_t s) {
  if (sp && hz) return launch_lb<BOX, WARPS, STAGES, true, true>(m, t, n, s);
  if (sp) return launch_lb<BOX, WARPS, STAGES, true, false>(m, t, n, s);
  if (hz) return launch_lb<BOX, WARPS, STAGES, false, true>(m, t, n, s);
  return launch_lb<BOX, WARPS, STAGES, false, false>(m, t, n, s);
}

}  // namespace

// Consumer warps per SM of each lookback kernel-table row (the launcher sizes segments
// from it).  Rows: 0 {32-step boxes, 8 consumers, 2 stages}, 1 {32, 4, 3}, 2 {32, 6, 3},
// 3 {16, 12, 2}, 4 {16, 16, 2}, 5 {32, 10, 2} (10 x 2 x 11.1 KB stages: 229 KB of shared
// memory, 12 warps x 168 registers: the SM's whole register file).
int lookback_warps(int cfg) {
  static const int kW[] = {8, 4, 6, 12, 16, 10};
  return kW[cfg < 0 || cfg >= kLookbackCfgs ? 0 : cfg];
}
int lookback_box(int cfg) { return cfg == 3 || cfg == 4 ? 16 : 32; }

cudaError_t launch_lookback(int cfg, bool sp, bool hz, const CUtensorMap* maps,
                            const LookbackLaunch& p, int num_sms, cudaStream_t s) {
  LbArgs t{};
  t.A = p.A;
  t.D = p.D;
  t.bias = p.bias;
  t.h0 = p.h0;
  t.out = p.out;
  t.h_last = p.h_last;
  t.agg = p.agg;
  t.epoch = p.epoch;
  t.launch_counter = p.launch_counter;
  t.stage_params = p.stage_params;
  t.ticket = p.ticket;
  t.batch = p.batch;
  t.dim = p.dim;
  t.L = p.L;
  t.tiles_per_batch = p.tiles_per_batch;
  t.n_tiles = p.n_tiles;
  t.seg_len = p.seg_len;
  t.n_seg = p.n_seg;
  static const int pipe1 = [] {
    const char* e = getenv("CL_LB_PIPE1");
    return e ? atoi(e) : 1;
  }();
  t.pipe1 = pipe1;
  t.decision = p.decision;
  const CUtensorMap m[4] = {maps[0], maps[1], maps[2], maps[3]};
  switch (cfg) {
    case 1: return dispatch_lb<32, 4, 3>(sp, hz, m, t, num_sms, s);
    case 2: return dispatch_lb<32, 6, 3>(sp, hz, m, t, num_sms, s);
    case 3: return dispatch_lb<16, 12, 2>(sp, hz, m, t, num_sms, s);
    case 4: return dispatch_lb<16, 16, 2>(sp, hz, m, t, num_sms, s);
    case 5: return dispatch_lb<32, 10, 2>(sp, hz, m, t, num_sms, s);
    default: return dispatch_lb<32, 8, 2>(sp, hz, m, t, num_sms, s);
  }
}

}  // namespace cl
