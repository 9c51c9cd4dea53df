// Fused expert FFN over the expert's resident copy (sm_100a).
//
// The reference's decode stage fetches every activated expert into local
// memory and then computes with it (moe.py:282-340: _issue_fetches, then the
// stage's compute once all fetches arrived).  On an NVSwitch node the expert
// can instead be consumed where it lies: these kernels stream each weight
// tile straight from the expert object's address -- donor HBM over NVLink,
// pinned host DRAM over PCIe, or local HBM -- into shared memory and multiply
// it there, so the transfer overlaps the math tile by tile and the bytes cross
// the link exactly once, with no staging write and re-read in local HBM.
//
// Decode is weight-bandwidth bound (a handful of tokens per expert), so the
// kernels are built like the fetch kernels: deep cp.async (16-byte LDGSTS)
// pipelines keep tens of KiB per SM in flight, and the tensor cores only have
// to keep up with the link.  The default (expert_ffn_umma, below) issues
// tcgen05.mma from one thread with both operands read from shared memory by
// descriptor and the accumulators in TMEM; the mma.sync m16n8k16 forms that
// follow first are kept for shapes it does not take (rows % 128 != 0, the
// programmatic-dependent down launch) and as the measured baseline.
// Tile shape and schedule, measured on B200 with experts in local HBM
// (tools/fused_probe.py, weight GB/s of the activated experts, Qwen1.5-MoE
// stage / Phi-3.5 batch 16 / batch 1):
//   one CTA per (row block, expert):
//     k-tile 128 x 4 stages (192 KiB smem, 1 CTA/SM): 3,365 / 3,673 / 2,754
//     k-tile  64 x 4 stages ( 96 KiB smem, 2 CTAs/SM): 4,667 / 4,967 / 2,767
//     k-tile  64 x 6 stages: 3,480 / 3,742;  k-tile 32 x 8 stages: 3,786 / 4,141
//   persistent (SMs x resident CTAs walking the items, ring across items):
//     k-tile  64 x 4 stages: 4,554 / 4,549 / 1,718
//     k-tile  64 x 3 stages ( 72 KiB smem, 3 CTAs/SM): 4,925 / 5,110 / 2,999  <- default
//     k-tile 128 x 3 stages: 3,424 / 3,462 / 2,267
// More resident CTAs per SM hide each other's stalls; the persistent ring
// removes the per-item pipeline fill and drain.  A deeper ring for the down
// kernel alone (HV_FFN_STAGES_DOWN 4 / 6 / 8) costs resident CTAs and lowers
// its rate (down: 4,224 / 3,329 / 2,154 vs 4,543 GB/s at 3, Qwen stage).
// 128-row down CTAs (8 warps; 2-3 CTAs/SM, 3-5 stages) were slower than
// these 64-row ones on every shape (Qwen stage 3,155-4,443 vs 4,474 GB/s,
// Phi-3.5 batch 1 1,536-1,750 vs 2,022; runs r119 and r121), so the down
// kernel keeps the gate/up geometry.
//
// Layout of an expert object (the same one K2 moves): gate [I][H], up [I][H],
// down [H][I], bf16, row-major.  Routed (token, expert) pairs are sorted by
// expert on the device; expert e owns pairs offs[e] .. offs[e]+counts[e]-1.
//
//   hv_expert_ffn_gate_up: act[p][i] = silu(gate[i] . x[tok[p]]) * (up[i] . x[tok[p]])
//   hv_expert_ffn_down:    y[p][h]   = down[h] . act[p]          (fp32)
// The top-k combine (a fixed-order weighted sum per token) is the caller's.
#include <cuda.h>
#include <cuda_bf16.h>

#include <mutex>

#include "hv_common.h"

namespace {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kRows = 16 * kWarps;   // weight rows per CTA (16 per warp: one mma M tile)
#ifndef HV_FFN_KT
#define HV_FFN_KT 64
#endif
#ifndef HV_FFN_PERSISTENT
#define HV_FFN_PERSISTENT 1
#endif
#ifndef HV_FFN_STAGES_DOWN
#define HV_FFN_STAGES_DOWN 3
#endif
#ifndef HV_FFN_STAGES
#define HV_FFN_STAGES 3
#endif
// HV_FFN_DOWN_PAIR=1: the down projection as two 64-row blocks per item
// through the two-matrix kernel (shared activation fragments and barriers).
// Measured (r3a, weight GB/s, down alone): Qwen stage 4,485 vs 4,576, Phi-3.5
// batch 1 / 16 / 64 1,632 / 4,209 / 4,390 vs 2,103 / 4,830 / 4,828 -- the
// per-byte instruction and barrier overhead is not what limits the down
// projection either.  Built as a variant only.
#ifndef HV_FFN_DOWN_PAIR
#define HV_FFN_DOWN_PAIR 0
#endif
constexpr int kKT = HV_FFN_KT;       // k columns per pipeline stage (64: 128 B per row)
constexpr int kRowBytes = kKT * 2;
constexpr int kChunksPerRow = kRowBytes / 16;
constexpr int kMaxTok = 64;          // routed tokens per expert per launch (8 mma N groups)
constexpr int kGroups = kMaxTok / 8;

template <int NMAT>
struct Smem {
  static constexpr int kS = NMAT == 2 ? HV_FFN_STAGES : HV_FFN_STAGES_DOWN;   // ring stages
  static constexpr int kW = NMAT * kRows * kRowBytes;   // weight tiles of one stage
  static constexpr int kX = kMaxTok * kRowBytes;        // activation tile of one stage
  static constexpr int kStage = kW + kX;
  static constexpr int kTotal = kS * kStage;
};

struct FfnArgs {
  const uint64_t* w_addr;   // [E] base address of each expert object (any tier)
  const int32_t* counts;    // [E] routed pairs of expert e
  const int32_t* offs;      // [E] first sorted pair of expert e
  const int32_t* tok;       // [P] activation row of each sorted pair (nullptr: row = pair)
  const __nv_bfloat16* x;   // activations, K columns per row
  void* out;                // NMAT=2: bf16 [P][rows]; NMAT=1: fp32 [P][rows]
  uint64_t w_off0, w_off1;  // byte offsets of the matrices inside the object
  int rows, K;
  int pair;                 // down projection as a pair of row blocks (NMAT=2 kernel, fp32 out, no SiLU)
  int wait_x;               // launched with programmatic serialization: x comes from the previous kernel
  int tiled;                // HV_FFN_TILED: matrices stored as swizzled 128 x 64 tiles (expert_ffn_umma only)
  int wait_all;             // HV_FFN_WAIT_PREVIOUS: programmatic dependent of a kernel that wrote any input
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte chunk c of tile row r lives at chunk (c ^ (r & 7)): ldmatrix's eight
// row addresses then hit eight different bank groups
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * kRowBytes + ((c ^ (r & 7)) << 4)); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Grid: (rows / kRows, E).  CTA (rb, e) computes rows [rb*64, rb*64+64) of
// NMAT matrices of expert e against its n routed activation rows.
template <int NMAT>
__global__ void __launch_bounds__(kThreads) expert_ffn_kernel(FfnArgs a) {
  const int e = blockIdx.y;
  const int n = a.counts[e];
  if (n <= 0) return;
  extern __shared__ __align__(128) char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row0 = blockIdx.x * kRows;
  const int p0 = a.offs[e];
  const int ng = (n + 7) >> 3;
  const char* obj = reinterpret_cast<const char*>(a.w_addr[e]);
  const char* wsrc[2] = {obj + a.w_off0 + (size_t)row0 * a.K * 2, obj + a.w_off1 + (size_t)row0 * a.K * 2};
  const size_t wstride = (size_t)a.K * 2;
  const size_t xstride = (size_t)a.K * 2;
  const int ktiles = a.K / kKT;

  // activation rows beyond n inside the last N group must hold finite values
  for (int s = 0; s < Smem<NMAT>::kS; ++s) {
    char* xs = smem + s * Smem<NMAT>::kStage + Smem<NMAT>::kW;
    for (int i = tid; i < (ng * 8 - n) * kChunksPerRow; i += kThreads) {
      const int r = n + i / kChunksPerRow, c = i % kChunksPerRow;
      *reinterpret_cast<uint4*>(xs + swz(r, c)) = make_uint4(0, 0, 0, 0);
    }
  }
  // per-thread activation row pointers are recomputed per stage from the pair list
  auto load_stage = [&](int kt, int s) {
    char* base = smem + s * Smem<NMAT>::kStage;
    const size_t kb = (size_t)kt * kRowBytes;
#pragma unroll
    for (int m = 0; m < NMAT; ++m) {
      const uint32_t ws = smem_u32(base + m * kRows * kRowBytes);
#pragma unroll 4
      for (int i = tid; i < kRows * kChunksPerRow; i += kThreads) {
        const int r = i / kChunksPerRow, c = i % kChunksPerRow;
        cp_async16(ws + swz(r, c), wsrc[m] + r * wstride + kb + c * 16);
      }
    }
    const uint32_t xs = smem_u32(base + Smem<NMAT>::kW);
    for (int i = tid; i < n * kChunksPerRow; i += kThreads) {
      const int r = i / kChunksPerRow, c = i % kChunksPerRow;
      const int row = a.tok ? a.tok[p0 + r] : p0 + r;
      cp_async16(xs + swz(r, c), reinterpret_cast<const char*>(a.x) + row * xstride + kb + c * 16);
    }
  };

  float acc[NMAT][kGroups][4];
#pragma unroll
  for (int m = 0; m < NMAT; ++m)
#pragma unroll
    for (int g = 0; g < kGroups; ++g)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[m][g][j] = 0.f;

#pragma unroll
  for (int s = 0; s < Smem<NMAT>::kS - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_commit();
  }
  // ldmatrix lane roles
  const int a_row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;  // A: x4 = rows 0-7/8-15 x k 0-7/8-15
  const int a_kc = lane >> 4;
  const int b_row = lane & 7;                                       // B: x2 = tokens 0-7 x k 0-7/8-15
  const int b_kc = (lane >> 3) & 1;

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_wait<Smem<NMAT>::kS - 2>();
    __syncthreads();
    // refill the stage consumed one iteration ago
    const int nk = kt + Smem<NMAT>::kS - 1;
    if (nk < ktiles) load_stage(nk, nk % Smem<NMAT>::kS);
    cp_commit();
    const char* base = smem + (kt % Smem<NMAT>::kS) * Smem<NMAT>::kStage;
    const uint32_t xs = smem_u32(base + Smem<NMAT>::kW);
#pragma unroll
    for (int kk = 0; kk < kKT / 16; ++kk) {
      uint32_t af[NMAT][4];
#pragma unroll
      for (int m = 0; m < NMAT; ++m)
        ldsm_x4(smem_u32(base + m * kRows * kRowBytes) + swz(a_row, kk * 2 + a_kc), af[m][0], af[m][1], af[m][2],
                af[m][3]);
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        if (g < ng) {
          uint32_t b0, b1;
          ldsm_x2(xs + swz(g * 8 + b_row, kk * 2 + b_kc), b0, b1);
#pragma unroll
          for (int m = 0; m < NMAT; ++m) mma_bf16(acc[m][g], af[m][0], af[m][1], af[m][2], af[m][3], b0, b1);
        }
      }
    }
  }
  cp_wait<0>();

  // epilogue: d0 (row r, tok 2c), d1 (r, 2c+1), d2 (r+8, 2c), d3 (r+8, 2c+1)
  const int r = row0 + warp * 16 + (lane >> 2);
  const int c2 = (lane & 3) * 2;
#pragma unroll
  for (int g = 0; g < kGroups; ++g) {
    if (g >= ng) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int t = g * 8 + c2 + (j & 1);
      const int row = r + (j >> 1) * 8;
      if (t >= n) continue;
      const size_t o = (size_t)(p0 + t) * a.rows + row;
      if constexpr (NMAT == 2) {
        const float gv = acc[0][g][j], uv = acc[1][g][j];
        const float act = gv / (1.f + __expf(-gv)) * uv;
        reinterpret_cast<__nv_bfloat16*>(a.out)[o] = __float2bfloat16_rn(act);
      } else {
        reinterpret_cast<float*>(a.out)[o] = acc[0][g][j];
      }
    }
  }
}

// Persistent form: a grid of (SMs x resident CTAs) walks the work items
// (expert e, row block rb), item = e * RB + rb, round-robin.  The cp.async
// ring runs across item boundaries: while the last k-tiles of one item are
// multiplied, the first tiles of the next are already in flight, so no CTA
// pays a pipeline fill/drain per item.  Items of experts without routed
// tokens are skipped.
struct ItemCursor {
  int item, kt, n, p0, row0;
  const char* w0;
  const char* w1;
};

template <int NMAT>
__device__ __forceinline__ void cursor_seek(ItemCursor& c, const FfnArgs& a, int rb_count, int n_items) {
  while (c.item < n_items) {
    const int e = c.item / rb_count;
    const int n = a.counts[e];
    if (n > 0) {
      c.n = n < kMaxTok ? n : kMaxTok;
      c.p0 = a.offs[e];
      c.row0 = (c.item - e * rb_count) * kRows * (a.pair ? 2 : 1);
      const char* obj = reinterpret_cast<const char*>(a.w_addr[e]);
      c.w0 = obj + a.w_off0 + (size_t)c.row0 * a.K * 2;
      c.w1 = obj + a.w_off1 + (size_t)c.row0 * a.K * 2;
      c.kt = 0;
      return;
    }
    c.item += gridDim.x;
  }
}

template <int NMAT>
__global__ void __launch_bounds__(kThreads) expert_ffn_persistent(FfnArgs a, int n_items) {
  extern __shared__ __align__(128) char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rb_count = a.rows / (kRows * (a.pair ? 2 : 1));
  const int ktiles = a.K / kKT;
  const size_t wstride = (size_t)a.K * 2, xstride = (size_t)a.K * 2;
  // every activation row of every stage starts finite; later stale rows are
  // earlier activations (finite) and only feed output columns that are dropped
  for (int i = tid; i < Smem<NMAT>::kS * Smem<NMAT>::kX / 16; i += kThreads) {
    const int s = i / (Smem<NMAT>::kX / 16), o = i % (Smem<NMAT>::kX / 16);
    *reinterpret_cast<uint4*>(smem + s * Smem<NMAT>::kStage + Smem<NMAT>::kW + o * 16) = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();

  ItemCursor ld{(int)blockIdx.x, 0, 0, 0, 0, nullptr, nullptr};
  cursor_seek<NMAT>(ld, a, rb_count, n_items);
  ItemCursor cs = ld;
  auto advance = [&](ItemCursor& c) {
    if (++c.kt == ktiles) {
      c.item += gridDim.x;
      cursor_seek<NMAT>(c, a, rb_count, n_items);
    }
  };
  auto load_weights = [&](const ItemCursor& c, int s) {
    char* base = smem + s * Smem<NMAT>::kStage;
    const size_t kb = (size_t)c.kt * kRowBytes;
#pragma unroll
    for (int m = 0; m < NMAT; ++m) {
      const uint32_t ws = smem_u32(base + m * kRows * kRowBytes);
      const char* src = m == 0 ? c.w0 : c.w1;
#pragma unroll 4
      for (int i = tid; i < kRows * kChunksPerRow; i += kThreads) {
        const int r = i / kChunksPerRow, ch = i % kChunksPerRow;
        cp_async16(ws + swz(r, ch), src + r * wstride + kb + ch * 16);
      }
    }
  };
  auto load_x = [&](const ItemCursor& c, int s) {
    const uint32_t xs = smem_u32(smem + s * Smem<NMAT>::kStage + Smem<NMAT>::kW);
    const size_t kb = (size_t)c.kt * kRowBytes;
    for (int i = tid; i < c.n * kChunksPerRow; i += kThreads) {
      const int r = i / kChunksPerRow, ch = i % kChunksPerRow;
      const int row = a.tok ? a.tok[c.p0 + r] : c.p0 + r;
      cp_async16(xs + swz(r, ch), reinterpret_cast<const char*>(a.x) + row * xstride + kb + ch * 16);
    }
  };
  auto load_stage = [&](const ItemCursor& c, int s) {
    load_weights(c, s);
    load_x(c, s);
  };

  float acc[NMAT][kGroups][4];
#pragma unroll
  for (int m = 0; m < NMAT; ++m)
#pragma unroll
    for (int g = 0; g < kGroups; ++g)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[m][g][j] = 0.f;

  // the next kernel on the stream (the down projection after gate/up) may
  // start as this one's CTAs drain
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.wait_x) {
    // programmatic dependent launch: the expert weights do not depend on the
    // previous kernel (gate/up), so the first stages' weight tiles stream in
    // while it finishes; the activation rows it writes are loaded only after
    // griddepcontrol.wait.  Commit groups stay in stage order: group 0 holds
    // the early weights and stage 0's rows, group s stage s's rows.
    ItemCursor pre = ld;
#pragma unroll
    for (int s = 0; s < Smem<NMAT>::kS - 1; ++s) {
      if (pre.item < n_items) {
        load_weights(pre, s);
        advance(pre);
      }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
    for (int s = 0; s < Smem<NMAT>::kS - 1; ++s) {
      if (ld.item < n_items) {
        load_x(ld, s);
        advance(ld);
      }
      cp_commit();
    }
  } else {
#pragma unroll
    for (int s = 0; s < Smem<NMAT>::kS - 1; ++s) {
      if (ld.item < n_items) {
        load_stage(ld, s);
        advance(ld);
      }
      cp_commit();
    }
  }
  const int a_row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int a_kc = lane >> 4;
  const int b_row = lane & 7;
  const int b_kc = (lane >> 3) & 1;
  int stage = 0, lstage = Smem<NMAT>::kS - 1;
  while (cs.item < n_items) {
    cp_wait<Smem<NMAT>::kS - 2>();
    __syncthreads();
    if (ld.item < n_items) {
      load_stage(ld, lstage);
      advance(ld);
    }
    cp_commit();
    lstage = lstage + 1 == Smem<NMAT>::kS ? 0 : lstage + 1;
    const char* base = smem + stage * Smem<NMAT>::kStage;
    const uint32_t xs = smem_u32(base + Smem<NMAT>::kW);
    const int ng = (cs.n + 7) >> 3;
#pragma unroll
    for (int kk = 0; kk < kKT / 16; ++kk) {
      uint32_t af[NMAT][4];
#pragma unroll
      for (int m = 0; m < NMAT; ++m)
        ldsm_x4(smem_u32(base + m * kRows * kRowBytes) + swz(a_row, kk * 2 + a_kc), af[m][0], af[m][1], af[m][2],
                af[m][3]);
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        if (g < ng) {
          uint32_t b0, b1;
          ldsm_x2(xs + swz(g * 8 + b_row, kk * 2 + b_kc), b0, b1);
#pragma unroll
          for (int m = 0; m < NMAT; ++m) mma_bf16(acc[m][g], af[m][0], af[m][1], af[m][2], af[m][3], b0, b1);
        }
      }
    }
    stage = stage + 1 == Smem<NMAT>::kS ? 0 : stage + 1;
    if (cs.kt == ktiles - 1) {  // item complete: epilogue, then the next item's tiles are already in flight
      const int r = cs.row0 + warp * 16 + (lane >> 2);
      const int c2 = (lane & 3) * 2;
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t = g * 8 + c2 + (j & 1);
          if (g < ng && t < cs.n) {
            const size_t o = (size_t)(cs.p0 + t) * a.rows + r + (j >> 1) * 8;
            if constexpr (NMAT == 2) {
              if (a.pair) {   // down, two row blocks: rows r and r + 64, fp32
                reinterpret_cast<float*>(a.out)[o] = acc[0][g][j];
                reinterpret_cast<float*>(a.out)[o + kRows] = acc[1][g][j];
              } else {
                const float gv = acc[0][g][j], uv = acc[1][g][j];
                reinterpret_cast<__nv_bfloat16*>(a.out)[o] = __float2bfloat16_rn(gv / (1.f + __expf(-gv)) * uv);
              }
            } else {
              reinterpret_cast<float*>(a.out)[o] = acc[0][g][j];
            }
          }
#pragma unroll
          for (int m = 0; m < NMAT; ++m) acc[m][g][j] = 0.f;
        }
      }
    }
    advance(cs);
  }
  cp_wait<0>();
}

// Measured on B200, experts in HBM (tools/fused_probe.py, weight GB/s of the
// activated experts, Qwen stage / Phi-3.5 batch 1 / 16 / 64; gpurun r2e):
//   this 1-D bulk-copy ring: 1,007 / 622 / 961 / 1,035
//   the cp.async persistent form: 4,960 / 2,995 / 5,024 / 5,165
// A weight row of a k-tile is only 256 contiguous bytes, so the ring issues
// 128+ bulk copies per stage and the per-copy cost of the bulk-copy engine
// (~70 cycles for 256 B, 3.5 B/cycle per SM) caps the stream at ~1 TB/s.  The
// TMA form worth having moves 2-D boxes through a tensor map (one 8 KiB
// 128B-swizzled box per matrix per stage, the cp.async layout exactly); that
// needs per-expert descriptors (tensormap.replace of the global address per
// item).  Until then the cp.async form stays the default.
#ifndef HV_FFN_TMA
#define HV_FFN_TMA 0
#endif

#if HV_FFN_TMA
// ---------------------------------------------------------------------------
// TMA weight stream (HV_FFN_TMA=1; see the measurement above): the persistent item walk above, but the
// weight and activation tiles arrive by cp.async.bulk (the bulk-copy / TMA
// engine) into an mbarrier ring, issued by one producer warp, while four
// consumer warps only run ldmatrix + mma.sync.  No thread spends issue slots
// on 16-byte LDGSTS (the cp.async form issues ~1.25 of them per cycle per SM
// at the HBM rate), and each stage keeps NMAT x 64 x 256 B of weights in
// flight per CTA.  Tiles are 128 k-columns (256 contiguous bytes per weight
// row: one bulk copy per row); smem rows are padded to 272 B, so the eight
// row addresses of an ldmatrix fall in eight different 16-byte bank groups
// (a 1-D bulk copy cannot write the XOR swizzle of the cp.async form).
constexpr int kTKT = 128;
constexpr int kTRowBytes = kTKT * 2;            // 256 B of one row per stage
constexpr int kTPitch = kTRowBytes + 16;        // padded smem row
constexpr int kTConsumers = 4;                  // mma warps (16 weight rows each)
constexpr int kTThreads = (kTConsumers + 1) * 32;

template <int NMAT>
struct TSmem {
  static constexpr int kS = NMAT == 2 ? 4 : 6;          // ring stages (~204 KiB either way)
  static constexpr int kW = NMAT * kRows * kTPitch;
  static constexpr int kX = kMaxTok * kTPitch;
  static constexpr int kStage = kW + kX;
  static constexpr int kBars = kS * 2 * 8;             // full[kS], empty[kS]
  static constexpr int kTotal = kS * kStage + kBars;
};

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n HV_FFN_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HV_FFN_WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <int NMAT>
__global__ void __launch_bounds__(kTThreads, 1) expert_ffn_tma(FfnArgs a, int n_items) {
  extern __shared__ __align__(128) char smem[];
  using T = TSmem<NMAT>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rb_count = a.rows / kRows;
  const int ktiles = a.K / kTKT;
  const size_t wstride = (size_t)a.K * 2, xstride = (size_t)a.K * 2;
  const uint32_t bars = smem_u32(smem + T::kS * T::kStage);   // full[s] at +8s, empty[s] at +8(kS+s)
  // activation rows start finite (rows past n in the last N group feed
  // output columns that are dropped; later stale rows are earlier activations)
  for (int i = tid; i < T::kS * (T::kX / 16); i += kTThreads) {
    const int st = i / (T::kX / 16), o = i % (T::kX / 16);
    *reinterpret_cast<uint4*>(smem + st * T::kStage + T::kW + o * 16) = make_uint4(0, 0, 0, 0);
  }
  if (tid == 0) {
    for (int st = 0; st < T::kS; ++st) {
      mbar_init(bars + 8 * st, 1);                       // the producer's expect_tx arrival
      mbar_init(bars + 8 * (T::kS + st), kTConsumers);   // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // zeroed rows before bulk writes
  __syncthreads();

  ItemCursor c{(int)blockIdx.x, 0, 0, 0, 0, nullptr, nullptr};
  cursor_seek<NMAT>(c, a, rb_count, n_items);
  auto advance = [&](ItemCursor& cc) {
    if (++cc.kt == ktiles) {
      cc.item += gridDim.x;
      cursor_seek<NMAT>(cc, a, rb_count, n_items);
    }
  };

  if (warp == kTConsumers) {   // ---- producer warp
    uint32_t it = 0;
    while (c.item < n_items) {
      const int st = it % T::kS;
      const uint32_t round = it / T::kS;
      if (round > 0) mbar_wait(bars + 8 * (T::kS + st), (round - 1) & 1);
      const uint32_t full = bars + 8 * st;
      const uint32_t bytes = (uint32_t)(NMAT * kRows + c.n) * kTRowBytes;
      if (lane == 0) mbar_expect_tx(full, bytes);
      __syncwarp();
      char* base = smem + st * T::kStage;
      const size_t kb = (size_t)c.kt * kTRowBytes;
#pragma unroll
      for (int m = 0; m < NMAT; ++m) {
        const char* src = (m == 0 ? c.w0 : c.w1) + kb;
        const uint32_t ws = smem_u32(base + m * kRows * kTPitch);
        for (int r = lane; r < kRows; r += 32) bulk_g2s(ws + r * kTPitch, src + r * wstride, kTRowBytes, full);
      }
      const uint32_t xs = smem_u32(base + T::kW);
      for (int r = lane; r < c.n; r += 32) {
        const int row = a.tok ? a.tok[c.p0 + r] : c.p0 + r;
        bulk_g2s(xs + r * kTPitch, reinterpret_cast<const char*>(a.x) + row * xstride + kb, kTRowBytes, full);
      }
      advance(c);
      ++it;
    }
    return;
  }

  // ---- consumer warps: rows warp*16 .. warp*16+15 of each item
  float acc[NMAT][kGroups][4];
#pragma unroll
  for (int m = 0; m < NMAT; ++m)
#pragma unroll
    for (int g = 0; g < kGroups; ++g)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[m][g][j] = 0.f;
  const int a_row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;   // A: x4 = rows 0-7/8-15 x k lo/hi
  const int a_kc = lane >> 4;
  const int b_row = lane & 7;                                         // B: x2 = tokens 0-7 x k lo/hi
  const int b_kc = (lane >> 3) & 1;
  uint32_t it = 0;
  while (c.item < n_items) {
    const int st = it % T::kS;
    mbar_wait(bars + 8 * st, (it / T::kS) & 1);
    const char* base = smem + st * T::kStage;
    const uint32_t xs = smem_u32(base + T::kW);
    const int ng = (c.n + 7) >> 3;
#pragma unroll
    for (int kk = 0; kk < kTKT / 16; ++kk) {
      uint32_t af[NMAT][4];
#pragma unroll
      for (int m = 0; m < NMAT; ++m)
        ldsm_x4(smem_u32(base + m * kRows * kTPitch) + a_row * kTPitch + (kk * 2 + a_kc) * 16, af[m][0], af[m][1],
                af[m][2], af[m][3]);
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        if (g < ng) {
          uint32_t b0, b1;
          ldsm_x2(xs + (g * 8 + b_row) * kTPitch + (kk * 2 + b_kc) * 16, b0, b1);
#pragma unroll
          for (int m = 0; m < NMAT; ++m) mma_bf16(acc[m][g], af[m][0], af[m][1], af[m][2], af[m][3], b0, b1);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bars + 8 * (T::kS + st));   // stage free for the producer
    if (c.kt == ktiles - 1) {   // item complete: epilogue
      const int r = c.row0 + warp * 16 + (lane >> 2);
      const int c2 = (lane & 3) * 2;
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t = g * 8 + c2 + (j & 1);
          if (g < ng && t < c.n) {
            const size_t o = (size_t)(c.p0 + t) * a.rows + r + (j >> 1) * 8;
            if constexpr (NMAT == 2) {
              const float gv = acc[0][g][j], uv = acc[1][g][j];
              reinterpret_cast<__nv_bfloat16*>(a.out)[o] = __float2bfloat16_rn(gv / (1.f + __expf(-gv)) * uv);
            } else {
              reinterpret_cast<float*>(a.out)[o] = acc[0][g][j];
            }
          }
#pragma unroll
          for (int m = 0; m < NMAT; ++m) acc[m][g][j] = 0.f;
        }
      }
    }
    advance(c);
    ++it;
  }
}


#endif  // HV_FFN_TMA

// ---------------------------------------------------------------------------
// 2-D tensor-map TMA weight stream (HV_FFN_TMA2D=1; measured below): per stage, one
// cp.async.bulk.tensor box of 64 rows x 64 columns (8 KiB, 128B-swizzled --
// exactly the cp.async form's smem layout) per matrix, issued by a producer
// warp into an mbarrier ring; four consumer warps run ldmatrix + mma.sync.
// Expert objects sit at arbitrary addresses (donor HBM, host tier, local),
// so the producer derives each item's tensor map from a per-launch template
// by replacing its global address (tensormap.replace on a shared-memory
// copy, then a fenced copy to a per-CTA global slot: the TMA unit reads maps
// from global memory).  S+1 slots per CTA: a slot is rewritten only after
// every stage that used it has been consumed.  The activation rows of the
// stage (the item's routed tokens) are gathered by the producer warp with
// 16-byte loads into the swizzled x tile and signalled by a second arrival.
// Measured on B200 (tools/fused_probe.py, experts in HBM, weight GB/s,
// Qwen stage gate_up / down; Phi-3.5 batch 1 / 16 / 64 whole FFN; r2k, r2l):
//   one 160-thread CTA per SM, 6/8 stages, x by the producer's loads:
//     2,202 / 1,515; 1,160 / 1,922 / 1,201   (4 consumer warps per SM cannot
//     hide ldmatrix + mma latency; ncu: short-scoreboard stalls)
//   three CTAs per SM, x by cp.async arriving on the stage barrier:
//     2 stages: 5,229 / 3,447; 1,456 / 4,151 / 4,546
//     3 stages: 5,213 / 3,450; 1,444 / 4,172 / 4,539
//     4 stages: 3,952 / 2,614; 1,535 / 3,272 / 3,669
//   the cp.async persistent form:   5,210 / 4,482; 2,990 / 5,054 / 5,132
// The tensor-map stream matches cp.async on gate/up and loses on the down
// projection and at batch 1, where items are short (22 k-tiles) or few and
// the per-item map rewrite + fence and the single producer per CTA show.
// So the cp.async form stays the default; HV_FFN_TMA2D=1 builds this one.
#ifndef HV_FFN_TMA2D
#define HV_FFN_TMA2D 0
#endif
#if HV_FFN_TMA2D
constexpr int kT2Consumers = 4;
constexpr int kT2Threads = (kT2Consumers + 1) * 32;
constexpr int kT2Tile = kRows * kRowBytes;     // 8 KiB: one 64 x 64 bf16 box

template <int NMAT>
struct T2Smem {
#ifndef HV_FFN_T2_STAGES
#define HV_FFN_T2_STAGES 3
#endif
  static constexpr int kS = NMAT == 2 ? HV_FFN_T2_STAGES : HV_FFN_T2_STAGES + 1;   // ring stages
  static constexpr int kStage = (NMAT + 1) * kT2Tile;       // W tiles then the x tile
  static constexpr int kRing = kS * kStage;                 // 1024-aligned stages
  static constexpr int kMaps = NMAT * 128;                  // smem staging of the item's maps
  static constexpr int kBars = 2 * kS * 8;
  static constexpr int kTotal = kRing + kMaps + kBars + 1024;   // + alignment slack
  static constexpr int kSlots = kS + 1;                     // global map slots per CTA
};

__device__ __forceinline__ void t2_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n HV_T2_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HV_T2_WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int NMAT>
__global__ void __launch_bounds__(kT2Threads, 3)
    expert_ffn_tma2d(FfnArgs a, int n_items, const __grid_constant__ CUtensorMap tmpl0,
                     const __grid_constant__ CUtensorMap tmpl1, CUtensorMap* __restrict__ ws) {
  extern __shared__ __align__(128) char smem_raw[];
  using T = T2Smem<NMAT>;
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  char* maps = smem + T::kRing;
  const uint32_t bars = smem_u32(maps + T::kMaps);   // full[s] at +8s, empty[s] at +8(kS+s)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rb_count = a.rows / kRows;
  const int ktiles = a.K / kKT;
  for (int i = tid; i < T::kS * (kT2Tile / 16); i += kT2Threads) {   // x tiles start finite
    const int st = i / (kT2Tile / 16), o = i % (kT2Tile / 16);
    *reinterpret_cast<uint4*>(smem + st * T::kStage + NMAT * kT2Tile + o * 16) = make_uint4(0, 0, 0, 0);
  }
  if (tid == 0) {
    for (int st = 0; st < T::kS; ++st) {
      // full: the producer's expect_tx arrival + one cp.async-completion arrival per producer lane
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bars + 8 * st), "r"(33) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bars + 8 * (T::kS + st)), "r"(kT2Consumers)
                   : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();

  ItemCursor c{(int)blockIdx.x, 0, 0, 0, 0, nullptr, nullptr};
  cursor_seek<NMAT>(c, a, rb_count, n_items);
  auto advance = [&](ItemCursor& cc) {
    if (++cc.kt == ktiles) {
      cc.item += gridDim.x;
      cursor_seek<NMAT>(cc, a, rb_count, n_items);
    }
  };

  if (warp == kT2Consumers) {   // ---- producer warp
    CUtensorMap* my = ws + (size_t)blockIdx.x * T::kSlots * NMAT;
    uint32_t it = 0, items = 0;
    const CUtensorMap* gmap[2] = {nullptr, nullptr};
    while (c.item < n_items) {
      const int st = it % T::kS;
      const uint32_t round = it / T::kS;
      if (round > 0) t2_wait(bars + 8 * (T::kS + st), (round - 1) & 1);
      if (c.kt == 0) {   // a new item: its matrices' tensor maps
        const int slot = items % T::kSlots;
        ++items;
#pragma unroll
        for (int m = 0; m < NMAT; ++m) {
          const uint32_t* src = reinterpret_cast<const uint32_t*>(m == 0 ? &tmpl0 : &tmpl1);
          reinterpret_cast<uint32_t*>(maps + m * 128)[lane] = src[lane];   // 128 B template
          __syncwarp();
          const uint64_t base = reinterpret_cast<uint64_t>(m == 0 ? c.w0 : c.w1) - (uint64_t)c.row0 * a.K * 2;
          if (lane == 0)
            asm volatile("tensormap.replace.tile.global_address.shared::cta.b1024.b64 [%0], %1;" ::"r"(
                             smem_u32(maps + m * 128)),
                         "l"(base)
                         : "memory");
          __syncwarp();
          CUtensorMap* g = my + slot * NMAT + m;
          asm volatile(
              "tensormap.cp_fenceproxy.global.shared::cta.tensormap::generic.release.gpu.sync.aligned [%0], [%1], "
              "128;" ::"l"(g),
              "r"(smem_u32(maps + m * 128))
              : "memory");
          if (lane == 0)
            asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(g) : "memory");
          __syncwarp();
          gmap[m] = g;
        }
      }
      const uint32_t full = bars + 8 * st;
      char* base = smem + st * T::kStage;
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full), "r"(NMAT * kT2Tile)
                     : "memory");
#pragma unroll
        for (int m = 0; m < NMAT; ++m)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
              "%3}], [%4];" ::"r"(smem_u32(base + m * kT2Tile)),
              "l"(gmap[m]), "r"(c.kt * kKT), "r"(c.row0), "r"(full)
              : "memory");
      }
      // the stage's activation rows: 8 x 16 B per routed token, swizzled, by
      // cp.async; each lane's completion arrives on the stage's full barrier,
      // so the producer never waits for these loads
      const uint32_t xs = smem_u32(base + NMAT * kT2Tile);
      const size_t kb = (size_t)c.kt * kRowBytes;
      for (int i = lane; i < c.n * kChunksPerRow; i += 32) {
        const int r = i / kChunksPerRow, ch = i % kChunksPerRow;
        const int row = a.tok ? __ldg(a.tok + c.p0 + r) : c.p0 + r;
        cp_async16(xs + swz(r, ch), reinterpret_cast<const char*>(a.x) + (size_t)row * a.K * 2 + kb + ch * 16);
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full) : "memory");
      advance(c);
      ++it;
    }
    return;
  }

  // ---- consumer warps
  float acc[NMAT][kGroups][4];
#pragma unroll
  for (int m = 0; m < NMAT; ++m)
#pragma unroll
    for (int g = 0; g < kGroups; ++g)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[m][g][j] = 0.f;
  const int a_row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int a_kc = lane >> 4;
  const int b_row = lane & 7;
  const int b_kc = (lane >> 3) & 1;
  uint32_t it = 0;
  while (c.item < n_items) {
    const int st = it % T::kS;
    t2_wait(bars + 8 * st, (it / T::kS) & 1);
    const char* base = smem + st * T::kStage;
    const uint32_t xs = smem_u32(base + NMAT * kT2Tile);
    const int ng = (c.n + 7) >> 3;
#pragma unroll
    for (int kk = 0; kk < kKT / 16; ++kk) {
      uint32_t af[NMAT][4];
#pragma unroll
      for (int m = 0; m < NMAT; ++m)
        ldsm_x4(smem_u32(base + m * kT2Tile) + swz(a_row, kk * 2 + a_kc), af[m][0], af[m][1], af[m][2], af[m][3]);
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        if (g < ng) {
          uint32_t b0, b1;
          ldsm_x2(xs + swz(g * 8 + b_row, kk * 2 + b_kc), b0, b1);
#pragma unroll
          for (int m = 0; m < NMAT; ++m) mma_bf16(acc[m][g], af[m][0], af[m][1], af[m][2], af[m][3], b0, b1);
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bars + 8 * (T::kS + st)) : "memory");
    if (c.kt == ktiles - 1) {
      const int r = c.row0 + warp * 16 + (lane >> 2);
      const int c2 = (lane & 3) * 2;
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t = g * 8 + c2 + (j & 1);
          if (g < ng && t < c.n) {
            const size_t o = (size_t)(c.p0 + t) * a.rows + r + (j >> 1) * 8;
            if constexpr (NMAT == 2) {
              const float gv = acc[0][g][j], uv = acc[1][g][j];
              reinterpret_cast<__nv_bfloat16*>(a.out)[o] = __float2bfloat16_rn(gv / (1.f + __expf(-gv)) * uv);
            } else {
              reinterpret_cast<float*>(a.out)[o] = acc[0][g][j];
            }
          }
#pragma unroll
          for (int m = 0; m < NMAT; ++m) acc[m][g][j] = 0.f;
        }
      }
    }
    advance(c);
    ++it;
  }
}

// driver entry point of the tensor-map encoder (the library links cudart
// statically and resolves driver symbols at run time)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      (void)cudaGetLastError();
      return (EncodeTiledFn) nullptr;
    }
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// [rows][K] bf16 matrix, boxes of 64 rows x 64 columns, 128B swizzle
bool make_tmpl(CUtensorMap* m, void* any_base, int rows, int K) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kKT, (cuuint32_t)kRows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, any_base, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

std::mutex g_ws_mu;
CUtensorMap* g_ws[64] = {};
size_t g_ws_n[64] = {};

CUtensorMap* map_workspace(int dev, size_t n, cudaStream_t s) {
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_ws_mu);
  if (g_ws_n[dev] >= n) return g_ws[dev];
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    (void)cudaGetLastError();
    return nullptr;   // cannot allocate under capture: the caller uses the cp.async kernel
  }
  CUtensorMap* p = nullptr;
  if (cudaMalloc(&p, n * sizeof(CUtensorMap)) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  if (g_ws[dev]) {
    cudaDeviceSynchronize();
    cudaFree(g_ws[dev]);
  }
  g_ws[dev] = p;
  g_ws_n[dev] = n;
  return p;
}
#endif  // HV_FFN_TMA2D

// ---------------------------------------------------------------------------
// Dynamically scheduled persistent form (HV_FFN_DYNAMIC=1; measured below).  The
// static walk above hands CTA c the items c, c+G, c+2G...; with 1,792 down
// items over 444 CTAs some CTAs get 5 items and others 4, so the slowest SM
// carries ~24% more bytes than the mean.  Here every CTA claims its next
// item from a global counter (atomicAdd) the moment its loader starts the
// current one, so SMs that finish early take more: the makespan is the mean
// plus at most one item.  Claimed item ids pass from the loader to the
// compute side of the same CTA through a small shared-memory FIFO (the loader
// runs up to S-1 stages, hence S-1 items, ahead).
// Measured (tools/fused_probe.py, HBM, weight GB/s, gpurun r2w): Qwen stage
// gate_up / down 5,093 / 4,391 against the static walk's 5,195 / 4,470;
// Phi-3.5 batch 1 / 16 / 64 whole FFN 1,481 / 4,704 / 4,939 vs 2,990 /
// 4,973 / 5,201 -- the item imbalance is not what holds the down projection
// back, and at batch 1 (2 active experts of 16) the claims that skip empty
// experts cost more than they balance.  Built with HV_FFN_DYNAMIC=1 only.
#ifndef HV_FFN_DYNAMIC
#define HV_FFN_DYNAMIC 0
#endif
#if HV_FFN_DYNAMIC
constexpr int kFifo = 16;

struct ItemInfo {
  int n, p0, row0;
  const char* w0;
  const char* w1;
};

__device__ __forceinline__ ItemInfo item_info(const FfnArgs& a, int item, int rb_count) {
  const int e = item / rb_count;
  const int n = a.counts[e];
  ItemInfo it;
  it.n = n < kMaxTok ? n : kMaxTok;
  it.p0 = a.offs[e];
  it.row0 = (item - e * rb_count) * kRows;
  const char* obj = reinterpret_cast<const char*>(a.w_addr[e]);
  it.w0 = obj + a.w_off0 + (size_t)it.row0 * a.K * 2;
  it.w1 = obj + a.w_off1 + (size_t)it.row0 * a.K * 2;
  return it;
}

// next item with routed tokens (or n_items when none is left); thread 0 only
__device__ __forceinline__ int claim_item(const FfnArgs& a, unsigned* counter, int rb_count, int n_items) {
  int id;
  do {
    id = (int)atomicAdd(counter, 1u);
  } while (id < n_items && a.counts[id / rb_count] <= 0);
  return id < n_items ? id : n_items;
}

template <int NMAT>
__global__ void __launch_bounds__(kThreads) expert_ffn_dynamic(FfnArgs a, int n_items, unsigned* counter) {
  extern __shared__ __align__(128) char smem[];
  __shared__ int s_claim[2];      // the next claimed item, double-buffered by the loader's item parity
  __shared__ int s_fifo[kFifo];   // items in the order the loader started them
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rb_count = a.rows / kRows;
  const int ktiles = a.K / kKT;
  const size_t wstride = (size_t)a.K * 2, xstride = (size_t)a.K * 2;
  for (int i = tid; i < Smem<NMAT>::kS * Smem<NMAT>::kX / 16; i += kThreads) {
    const int s = i / (Smem<NMAT>::kX / 16), o = i % (Smem<NMAT>::kX / 16);
    *reinterpret_cast<uint4*>(smem + s * Smem<NMAT>::kStage + Smem<NMAT>::kW + o * 16) = make_uint4(0, 0, 0, 0);
  }
  if (tid == 0) s_claim[0] = claim_item(a, counter, rb_count, n_items);
  __syncthreads();

  // loader cursor (all threads, in lockstep)
  int ld_cnt = 0, ld_kt = 0, ld_item;
  ItemInfo ld;
  auto ld_start = [&]() {   // begin the next claimed item (call between barriers)
    ld_item = s_claim[ld_cnt & 1];
    if (tid == 0) {
      s_fifo[ld_cnt % kFifo] = ld_item;
      if (ld_item < n_items) s_claim[(ld_cnt + 1) & 1] = claim_item(a, counter, rb_count, n_items);
    }
    ++ld_cnt;
    ld_kt = 0;
    if (ld_item < n_items) ld = item_info(a, ld_item, rb_count);
  };
  auto load_stage = [&](int s) {
    char* base = smem + s * Smem<NMAT>::kStage;
    const size_t kb = (size_t)ld_kt * kRowBytes;
#pragma unroll
    for (int m = 0; m < NMAT; ++m) {
      const uint32_t ws = smem_u32(base + m * kRows * kRowBytes);
      const char* src = m == 0 ? ld.w0 : ld.w1;
#pragma unroll 4
      for (int i = tid; i < kRows * kChunksPerRow; i += kThreads) {
        const int r = i / kChunksPerRow, ch = i % kChunksPerRow;
        cp_async16(ws + swz(r, ch), src + r * wstride + kb + ch * 16);
      }
    }
    const uint32_t xs = smem_u32(base + Smem<NMAT>::kW);
    for (int i = tid; i < ld.n * kChunksPerRow; i += kThreads) {
      const int r = i / kChunksPerRow, ch = i % kChunksPerRow;
      const int row = a.tok ? a.tok[ld.p0 + r] : ld.p0 + r;
      cp_async16(xs + swz(r, ch), reinterpret_cast<const char*>(a.x) + row * xstride + kb + ch * 16);
    }
  };
  auto ld_advance = [&]() {   // after a stage was issued; the next item's id was claimed a stage ago
    if (++ld_kt == ktiles) {
      __syncthreads();          // thread 0's claim of the next item is visible
      ld_start();
    }
  };

  float acc[NMAT][kGroups][4];
#pragma unroll
  for (int m = 0; m < NMAT; ++m)
#pragma unroll
    for (int g = 0; g < kGroups; ++g)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[m][g][j] = 0.f;

  ld_start();
#pragma unroll
  for (int s = 0; s < Smem<NMAT>::kS - 1; ++s) {
    if (ld_item < n_items) {
      load_stage(s);
      ld_advance();
    }
    cp_commit();
  }
  const int a_row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int a_kc = lane >> 4;
  const int b_row = lane & 7;
  const int b_kc = (lane >> 3) & 1;
  int stage = 0, lstage = Smem<NMAT>::kS - 1;
  // compute cursor
  int cs_cnt = 0, cs_kt = 0;
  __syncthreads();
  int cs_item = s_fifo[0];
  ItemInfo cs = cs_item < n_items ? item_info(a, cs_item, rb_count) : ItemInfo{};
  ++cs_cnt;
  while (cs_item < n_items) {
    cp_wait<Smem<NMAT>::kS - 2>();
    __syncthreads();
    if (ld_item < n_items) {
      load_stage(lstage);
      ld_advance();
    }
    cp_commit();
    lstage = lstage + 1 == Smem<NMAT>::kS ? 0 : lstage + 1;
    const char* base = smem + stage * Smem<NMAT>::kStage;
    const uint32_t xs = smem_u32(base + Smem<NMAT>::kW);
    const int ng = (cs.n + 7) >> 3;
#pragma unroll
    for (int kk = 0; kk < kKT / 16; ++kk) {
      uint32_t af[NMAT][4];
#pragma unroll
      for (int m = 0; m < NMAT; ++m)
        ldsm_x4(smem_u32(base + m * kRows * kRowBytes) + swz(a_row, kk * 2 + a_kc), af[m][0], af[m][1], af[m][2],
                af[m][3]);
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        if (g < ng) {
          uint32_t b0, b1;
          ldsm_x2(xs + swz(g * 8 + b_row, kk * 2 + b_kc), b0, b1);
#pragma unroll
          for (int m = 0; m < NMAT; ++m) mma_bf16(acc[m][g], af[m][0], af[m][1], af[m][2], af[m][3], b0, b1);
        }
      }
    }
    stage = stage + 1 == Smem<NMAT>::kS ? 0 : stage + 1;
    if (cs_kt == ktiles - 1) {  // item complete: epilogue
      const int r = cs.row0 + warp * 16 + (lane >> 2);
      const int c2 = (lane & 3) * 2;
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t = g * 8 + c2 + (j & 1);
          if (g < ng && t < cs.n) {
            const size_t o = (size_t)(cs.p0 + t) * a.rows + r + (j >> 1) * 8;
            if constexpr (NMAT == 2) {
              const float gv = acc[0][g][j], uv = acc[1][g][j];
              reinterpret_cast<__nv_bfloat16*>(a.out)[o] = __float2bfloat16_rn(gv / (1.f + __expf(-gv)) * uv);
            } else {
              reinterpret_cast<float*>(a.out)[o] = acc[0][g][j];
            }
          }
#pragma unroll
          for (int m = 0; m < NMAT; ++m) acc[m][g][j] = 0.f;
        }
      }
    }
    if (++cs_kt == ktiles) {    // the loader started (and recorded) this next item stages ago
      cs_kt = 0;
      cs_item = s_fifo[cs_cnt % kFifo];
      ++cs_cnt;
      if (cs_item < n_items) cs = item_info(a, cs_item, rb_count);
    }
  }
  cp_wait<0>();
}

std::mutex g_ctr_mu;
unsigned* g_ctr[64] = {};

unsigned* item_counter(int dev, cudaStream_t s) {
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_ctr_mu);
  if (g_ctr[dev]) return g_ctr[dev];
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    (void)cudaGetLastError();
    return nullptr;
  }
  unsigned* p = nullptr;
  if (cudaMalloc(&p, 2 * sizeof(unsigned)) != cudaSuccess) {   // one counter per kernel of a stage
    (void)cudaGetLastError();
    return nullptr;
  }
  g_ctr[dev] = p;
  return p;
}
#endif  // HV_FFN_DYNAMIC

// ---------------------------------------------------------------------------
// tcgen05 form (HV_FFN_UMMA): the same persistent item walk and the same
// cp.async weight stream (16-byte LDGSTS into the 128B-swizzled K-major tile
// the mma.sync form already uses, which is exactly UMMA's SWIZZLE_128B
// canonical layout), but the products run on the 5th-generation tensor cores:
// one thread issues tcgen05.mma with both operands read from shared memory
// through descriptors, accumulating in TMEM.  The consumer warps of the
// mma.sync form spend their issue slots on ldmatrix + mma.sync (ncu r4j: issue
// active 31% / 45%, stalls on fixed-latency waits and the math pipe); here no
// register fragment exists -- the MMA thread issues 4 instructions per matrix
// per 64-column stage and the epilogue warps read the accumulators once per
// item.
//   warps 0-3  epilogue: tcgen05.ld of their TMEM lane quarter (weight rows),
//              SiLU(gate) * up -> bf16 act, or fp32 y
//   warps 4-5  producers: cp.async of the weight rows (M = 128 per item) and
//              the item's activation rows; cp.async.mbarrier.arrive.noinc on
//              the stage's full barrier
//   warp 6     one elected lane issues tcgen05.mma (M = 128, N = n rounded up
//              to 16, K = 16) and tcgen05.commit (stage free / item done)
// TMEM: two accumulator buffers of 128 columns (gate at +0, up at +64), so
// the epilogue of item i overlaps the MMAs of item i+1.
// Measured (tools/fused_probe.py, experts in HBM, weight GB/s of the activated
// experts; Qwen stage fused / gate_up / down, Phi-3.5 batch 1 / 16 / 64 fused):
//   mma.sync persistent form (kept for rows % 128 != 0 and the PDL launch):
//       4,956 / 5,216 / 4,516;  2,928 / 5,031 / 5,113
//   this form, producer warps 2 / 4 / 6 / 8 (r4n, r4o):
//       4,726 / 5,111 / 4,169;  2,259 / 4,690 / 5,092   (2: issue-bound producers)
//       5,279 / 5,370 / 5,072;  3,154 / 5,472 / 5,633
//       5,404 / 5,472 / 5,240;  3,373 / 5,615 / 5,733   <- default (6)
//       5,345 / 5,382 / 5,179;  3,173 / 5,495 / 5,661
// The first form resolved each activation row through the pair -> token map
// in every stage (a dependent global load ahead of the stage's cp.async:
// ncu r4m, long-scoreboard stalls dominant); the rows are now resolved once
// per item.
#ifndef HV_FFN_UMMA
#define HV_FFN_UMMA 1
#endif
#if HV_FFN_UMMA
constexpr int kURows = 128;                  // UMMA M: weight rows per item
#ifndef HV_FFN_UMMA_PROD_WARPS
#define HV_FFN_UMMA_PROD_WARPS 6
#endif
constexpr int kUEpiWarps = 4, kUProdWarps = HV_FFN_UMMA_PROD_WARPS;
constexpr int kUThreads = (kUEpiWarps + kUProdWarps + 1) * 32;
constexpr int kUProd = kUProdWarps * 32;
template <int NMAT>
struct USmem {
  static constexpr int kS = NMAT == 2 ? 5 : 8;                 // ring stages
  static constexpr int kWm = kURows * kRowBytes;               // one matrix tile: 16 KiB
  static constexpr int kX = kMaxTok * kRowBytes;               // activation tile: 8 KiB
  static constexpr int kStage = NMAT * kWm + kX;               // 1024-byte multiple
  static constexpr int kTotal = kS * kStage + 1024;            // + alignment slack
};

__device__ __forceinline__ void u_mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void u_mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void u_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n HV_U_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HV_U_WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// SWIZZLE_128B K-major operand: 8-row groups 1024 B apart (SBO), LBO unused
// (encoded 1), descriptor version 1 (sm100), layout type 2 = 128B swizzle
__device__ __forceinline__ uint64_t umma_sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: f32 accumulate, bf16 A and B, both
// K-major, N (multiple of 16 for M = 128), M = 128
__device__ __forceinline__ uint32_t umma_idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kURows >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

struct UCursor {
  int item, n, p0, row0;
  const char* w0;
  const char* w1;
};
__device__ __forceinline__ void u_seek(UCursor& c, const FfnArgs& a, int rb_count, int n_items) {
  while (c.item < n_items) {
    const int e = c.item / rb_count;
    const int n = a.counts[e];
    if (n > 0) {
      c.n = n < kMaxTok ? n : kMaxTok;
      c.p0 = a.offs[e];
      c.row0 = (c.item - e * rb_count) * kURows;
      const char* obj = reinterpret_cast<const char*>(a.w_addr[e]);
      c.w0 = obj + a.w_off0 + (size_t)c.row0 * a.K * 2;
      c.w1 = obj + a.w_off1 + (size_t)c.row0 * a.K * 2;
      return;
    }
    c.item += gridDim.x;
  }
}

template <int NMAT>
__global__ void __launch_bounds__(kUThreads, 1) expert_ffn_umma(FfnArgs a, int n_items) {
  using U = USmem<NMAT>;
  extern __shared__ __align__(1024) char u_smem_raw[];
  // operand tiles must sit on 1024-byte boundaries (descriptor base offset 0)
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(u_smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[U::kS], empty_bar[U::kS], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rb_count = a.rows / kURows;
  const int ktiles = a.K / kKT;
  // activation rows past n inside the last N group start finite
  for (int i = tid; i < U::kS * (U::kX / 16); i += kUThreads) {
    const int s = i / (U::kX / 16), o = i % (U::kX / 16);
    *reinterpret_cast<uint4*>(smem + s * U::kStage + NMAT * U::kWm + o * 16) = make_uint4(0, 0, 0, 0);
  }
  if (tid == 0) {
    for (int s = 0; s < U::kS; ++s) {
      // one cp.async-completion arrival per producer thread, plus the tiled
      // form's arrive.expect_tx of the weight tiles' bulk copies
      u_mbar_init(smem_u32(&full_bar[s]), kUProd + (a.tiled ? 1 : 0));
      u_mbar_init(smem_u32(&empty_bar[s]), 1);       // tcgen05.commit of the stage's MMAs
    }
    for (int b = 0; b < 2; ++b) {
      u_mbar_init(smem_u32(&tfull_bar[b]), 1);             // tcgen05.commit at the item's end
      u_mbar_init(smem_u32(&tempty_bar[b]), kUEpiWarps * 32);  // every epilogue thread read its rows
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;
  const size_t wstride = (size_t)a.K * 2, xstride = (size_t)a.K * 2;
  // programmatic dependent launch (decode.py launches the stage's kernels as a
  // chain): the prologue above overlapped the previous kernel's tail; with
  // HV_FFN_WAIT_PREVIOUS every input may be its output, so wait here
  if (a.wait_all) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp >= kUEpiWarps && warp < kUEpiWarps + kUProdWarps) {
    // ---- producers
    const int pt = tid - kUEpiWarps * 32;
    UCursor c{(int)blockIdx.x, 0, 0, 0, nullptr, nullptr};
    u_seek(c, a, rb_count, n_items);
    uint32_t g = 0;
    // the weight tiles of (item c, k-tile kt) into ring stage s
    auto issue_weights = [&](const UCursor& cc, int kt, int st) {
      char* base = smem + st * U::kStage;
      const size_t kb = (size_t)kt * kRowBytes;
      if (a.tiled) {
        // tile (row block, kt) of each matrix is 16 KiB contiguous and
        // already in the swizzled order: one bulk copy (TMA engine) each,
        // completing on the stage's full barrier
        if (pt == 0) {
          const uint32_t fb = smem_u32(&full_bar[st]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(NMAT * U::kWm)
                       : "memory");
#pragma unroll
          for (int m = 0; m < NMAT; ++m)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(base + m * U::kWm)),
                "l"((m == 0 ? cc.w0 : cc.w1) + (size_t)kt * U::kWm), "r"(U::kWm), "r"(fb)
                : "memory");
        }
      } else {
#pragma unroll
        for (int m = 0; m < NMAT; ++m) {
          const uint32_t ws = smem_u32(base + m * U::kWm);
          const char* src = m == 0 ? cc.w0 : cc.w1;
#pragma unroll 4
          for (int i = pt; i < kURows * kChunksPerRow; i += kUProd) {
            const int r = i / kChunksPerRow, ch = i % kChunksPerRow;
            cp_async16(ws + swz(r, ch), src + r * wstride + kb + ch * 16);
          }
        }
      }
    };
    // HV_FFN_OVERLAP_PREVIOUS (the down projection behind gate/up): the
    // weights do not depend on the previous kernel, so the first item's first
    // stages stream in while it drains; its activation rows only after the wait
    int pre = 0;
    if (a.wait_x) {
      if (c.item < n_items) {
        pre = ktiles < U::kS ? ktiles : U::kS;
        for (int kt = 0; kt < pre; ++kt) issue_weights(c, kt, kt);
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    // this thread's activation rows: r = pt/8 + j*(kUProd/8), chunk pt%8 --
    // their source rows are resolved once per item, not per stage
    constexpr int kXPass = kUProd / kChunksPerRow;                 // rows covered per pass
    constexpr int kXRows = (kMaxTok + kXPass - 1) / kXPass;
    const int xr0 = pt / kChunksPerRow, xch = pt % kChunksPerRow;
    while (c.item < n_items) {
      const char* xsrc[kXRows];
#pragma unroll
      for (int j = 0; j < kXRows; ++j) {
        const int r = xr0 + j * kXPass;
        const int row = r < c.n ? (a.tok ? a.tok[c.p0 + r] : c.p0 + r) : 0;
        xsrc[j] = reinterpret_cast<const char*>(a.x) + (size_t)row * xstride + xch * 16;
      }
      for (int kt = 0; kt < ktiles; ++kt, ++g) {
        const int s = (int)(g % U::kS);
        const uint32_t round = g / U::kS;
        if (round > 0) u_mbar_wait(smem_u32(&empty_bar[s]), (round - 1) & 1);
        char* base = smem + s * U::kStage;
        const size_t kb = (size_t)kt * kRowBytes;
        if ((int)g >= pre) issue_weights(c, kt, s);   // else streamed before the wait
        const uint32_t xs = smem_u32(base + NMAT * U::kWm);
#pragma unroll
        for (int j = 0; j < kXRows; ++j) {
          const int r = xr0 + j * kXPass;
          if (r < c.n) cp_async16(xs + swz(r, xch), xsrc[j] + kb);
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full_bar[s]))
                     : "memory");
      }
      c.item += gridDim.x;
      u_seek(c, a, rb_count, n_items);
    }
    cp_wait<0>();
  } else if (warp == kUEpiWarps + kUProdWarps) {
    // ---- MMA issue (one lane)
    if (lane == 0) {
      UCursor c{(int)blockIdx.x, 0, 0, 0, nullptr, nullptr};
      u_seek(c, a, rb_count, n_items);
      uint32_t g = 0, li = 0;
      while (c.item < n_items) {
        const uint32_t ab = li & 1, use = li >> 1;
        if (use > 0) u_mbar_wait(smem_u32(&tempty_bar[ab]), (use - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int nn = c.n <= 16 ? 16 : ((c.n + 15) & ~15);
        const uint32_t idesc = umma_idesc_bf16(nn);
        for (int kt = 0; kt < ktiles; ++kt, ++g) {
          const int s = (int)(g % U::kS);
          u_mbar_wait(smem_u32(&full_bar[s]), (g / U::kS) & 1);
          // the cp.async (generic proxy) writes of the stage, now visible to
          // this thread, ordered before the tensor core's (async proxy) reads
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t base = smem_u32(smem + s * U::kStage);
          const uint64_t bdesc = umma_sw128_desc(base + NMAT * U::kWm);
#pragma unroll
          for (int m = 0; m < NMAT; ++m) {
            const uint64_t adesc = umma_sw128_desc(base + m * U::kWm);
#pragma unroll
            for (int kk = 0; kk < kKT / 16; ++kk)   // K = 16 per instruction: +32 B inside the swizzle atom
              umma_bf16(tmem + ab * 128 + m * 64, adesc + (uint64_t)(kk * 2), bdesc + (uint64_t)(kk * 2), idesc,
                        (kt | kk) != 0);
          }
          umma_commit(smem_u32(&empty_bar[s]));   // the stage is free once these MMAs have read it
        }
        umma_commit(smem_u32(&tfull_bar[ab]));    // the item's accumulators are complete
        ++li;
        c.item += gridDim.x;
        u_seek(c, a, rb_count, n_items);
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue: warp w reads TMEM lanes 32w..32w+31 = weight rows of the item
    UCursor c{(int)blockIdx.x, 0, 0, 0, nullptr, nullptr};
    u_seek(c, a, rb_count, n_items);
    uint32_t li = 0;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    while (c.item < n_items) {
      const uint32_t ab = li & 1;
      u_mbar_wait(smem_u32(&tfull_bar[ab]), (li >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = c.row0 + warp * 32 + lane;
      for (int j0 = 0; j0 < c.n; j0 += 8) {
        float gv[8];
        tmem_ld8(tmem + lane_base + ab * 128 + j0, gv);
        if constexpr (NMAT == 2) {
          float uv[8];
          tmem_ld8(tmem + lane_base + ab * 128 + 64 + j0, uv);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j0 + j < c.n) {
              const float x = gv[j];
              reinterpret_cast<__nv_bfloat16*>(a.out)[(size_t)(c.p0 + j0 + j) * a.rows + row] =
                  __float2bfloat16_rn(x / (1.f + __expf(-x)) * uv[j]);
            }
        } else {
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j0 + j < c.n) reinterpret_cast<float*>(a.out)[(size_t)(c.p0 + j0 + j) * a.rows + row] = gv[j];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      u_mbar_arrive(smem_u32(&tempty_bar[ab]));
      ++li;
      c.item += gridDim.x;
      u_seek(c, a, rb_count, n_items);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}
#endif  // HV_FFN_UMMA

template <int NMAT>
int launch_ffn(const FfnArgs& a, uint32_t n_experts, void* stream) {
  if (n_experts == 0) return HV_OK;
  HV_CHECK_ARG(a.w_addr && a.counts && a.offs && a.x && a.out);
  HV_CHECK_ARG(a.rows > 0 && a.K > 0 && a.rows % kRows == 0 && a.K % kKT == 0);
  HV_CHECK_ARG(n_experts <= 65535u);
#if !HV_FFN_UMMA
  HV_CHECK_ARG(!a.tiled);   // the swizzled-tile layout is read by the tcgen05 form only
#endif
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  st = hv::kernel_attr<expert_ffn_kernel<NMAT>>(dev, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<NMAT>::kTotal);
  if (st) return st;
#if HV_FFN_UMMA
  HV_CHECK_ARG(!a.tiled || (!a.pair && a.rows % kURows == 0));
  HV_CHECK_ARG(!a.wait_all || (!a.pair && a.rows % kURows == 0));
  if (!a.pair && a.rows % kURows == 0) {
    using U = USmem<NMAT>;
    st = hv::kernel_attr<expert_ffn_umma<NMAT>>(dev, cudaFuncAttributeMaxDynamicSharedMemorySize, U::kTotal);
    if (st) return st;
    const int n_items = (int)(a.rows / kURows) * (int)n_experts;
    int g = hv::sm_count(dev);                    // one ~200 KiB CTA per SM
    if (g > n_items) g = n_items;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(kUThreads);
    cfg.dynamicSmemBytes = U::kTotal;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (a.wait_x || a.wait_all) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HV_CUDA(cudaLaunchKernelEx(&cfg, expert_ffn_umma<NMAT>, a, n_items));
    HV_CUDA(cudaGetLastError());
    hv::note_launch();
    return HV_OK;
  }
#endif
#if HV_FFN_TMA2D
  if (!a.pair) {
    using T = T2Smem<NMAT>;
    const int n_items = (int)(a.rows / kRows) * (int)n_experts;
    st = hv::kernel_attr<expert_ffn_tma2d<NMAT>>(dev, cudaFuncAttributeMaxDynamicSharedMemorySize, T::kTotal);
    if (st) return st;
    static int resident2[64] = {};   // CTAs per SM (several: the consumer warps of one CTA cannot hide mma latency)
    if (dev >= 0 && dev < 64 && !resident2[dev]) {
      int r = 0;
      HV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, expert_ffn_tma2d<NMAT>, kT2Threads, T::kTotal));
      resident2[dev] = r > 0 ? r : 1;
    }
    const int per_sm = dev >= 0 && dev < 64 ? resident2[dev] : 1;
    int g = hv::sm_count(dev) * per_sm;
    if (g > n_items) g = n_items;
    CUtensorMap t0, t1;
    CUtensorMap* ws = map_workspace(dev, (size_t)hv::sm_count(dev) * per_sm * T::kSlots * NMAT, (cudaStream_t)stream);
    if (ws && make_tmpl(&t0, a.out, a.rows, a.K) && make_tmpl(&t1, a.out, a.rows, a.K)) {
      expert_ffn_tma2d<NMAT><<<g, kT2Threads, T::kTotal, (cudaStream_t)stream>>>(a, n_items, t0, t1, ws);
      HV_CUDA(cudaGetLastError());
      hv::note_launch();
      return HV_OK;
    }
  }
#endif
#if HV_FFN_TMA
  if (a.K % kTKT == 0 && !a.pair) {
    using T = TSmem<NMAT>;
    st = hv::kernel_attr<expert_ffn_tma<NMAT>>(dev, cudaFuncAttributeMaxDynamicSharedMemorySize, T::kTotal);
    if (st) return st;
    const int n_items = (int)(a.rows / kRows) * (int)n_experts;
    int g = hv::sm_count(dev);                    // one ~204 KiB CTA per SM
    if (g > n_items) g = n_items;
    expert_ffn_tma<NMAT><<<g, kTThreads, T::kTotal, (cudaStream_t)stream>>>(a, n_items);
    HV_CUDA(cudaGetLastError());
    hv::note_launch();
    return HV_OK;
  }
#endif
#if HV_FFN_DYNAMIC
  if (!a.pair) {
    unsigned* ctr = item_counter(dev, (cudaStream_t)stream);
    if (ctr) {
      ctr += NMAT == 2 ? 0 : 1;
      static int resident_d[64] = {};
      if (dev >= 0 && dev < 64 && !resident_d[dev]) {
        int r = 0;
        st = hv::kernel_attr<expert_ffn_dynamic<NMAT>>(dev, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       Smem<NMAT>::kTotal);
        if (st) return st;
        HV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, expert_ffn_dynamic<NMAT>, kThreads,
                                                              Smem<NMAT>::kTotal));
        resident_d[dev] = r > 0 ? r : 1;
      }
      const int n_items = (int)(a.rows / kRows) * (int)n_experts;
      int g = hv::sm_count(dev) * (dev >= 0 && dev < 64 ? resident_d[dev] : 1);
      if (g > n_items) g = n_items;
      HV_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned), (cudaStream_t)stream));
      expert_ffn_dynamic<NMAT><<<g, kThreads, Smem<NMAT>::kTotal, (cudaStream_t)stream>>>(a, n_items, ctr);
      HV_CUDA(cudaGetLastError());
      hv::note_launch();
      return HV_OK;
    }
  }
#endif
#if HV_FFN_PERSISTENT
  static int resident[64] = {};
  if (dev >= 0 && dev < 64 && !resident[dev]) {
    int r = 0;
    st = hv::kernel_attr<expert_ffn_persistent<NMAT>>(dev, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      Smem<NMAT>::kTotal);
    if (st) return st;
    HV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, expert_ffn_persistent<NMAT>, kThreads,
                                                          Smem<NMAT>::kTotal));
    resident[dev] = r > 0 ? r : 1;
  }
  const int n_items = (int)(a.rows / (kRows * (a.pair ? 2 : 1))) * (int)n_experts;
  int g = hv::sm_count(dev) * (dev >= 0 && dev < 64 ? resident[dev] : 1);
  if (g > n_items) g = n_items;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Smem<NMAT>::kTotal;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = a.wait_x ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HV_CUDA(cudaLaunchKernelEx(&cfg, expert_ffn_persistent<NMAT>, a, n_items));
  }
#else
  dim3 grid(a.rows / kRows, n_experts);
  expert_ffn_kernel<NMAT><<<grid, kThreads, Smem<NMAT>::kTotal, (cudaStream_t)stream>>>(a);
#endif
  HV_CUDA(cudaGetLastError());
  hv::note_launch();
  return HV_OK;
}

}  // namespace

HV_EXPORT int hv_expert_ffn_gate_up(const uint64_t* d_w_addr, const int32_t* d_counts, const int32_t* d_offs,
                                    const int32_t* d_tok, const void* d_x, void* d_act, uint32_t n_experts,
                                    uint32_t hidden, uint32_t intermediate, void* stream) {
  return hv_expert_ffn_gate_up_ex(d_w_addr, d_counts, d_offs, d_tok, d_x, d_act, n_experts, hidden, intermediate, 0u,
                                  stream);
}

HV_EXPORT int hv_expert_ffn_gate_up_ex(const uint64_t* d_w_addr, const int32_t* d_counts, const int32_t* d_offs,
                                       const int32_t* d_tok, const void* d_x, void* d_act, uint32_t n_experts,
                                       uint32_t hidden, uint32_t intermediate, unsigned flags, void* stream) {
  HV_CHECK_ARG(d_tok != nullptr || n_experts == 0);
  HV_CHECK_ARG((flags & ~(unsigned)(HV_FFN_TILED | HV_FFN_WAIT_PREVIOUS)) == 0);
  FfnArgs a{};
  a.tiled = (flags & HV_FFN_TILED) ? 1 : 0;
  a.wait_all = (flags & HV_FFN_WAIT_PREVIOUS) ? 1 : 0;
  a.w_addr = d_w_addr;
  a.counts = d_counts;
  a.offs = d_offs;
  a.tok = d_tok;
  a.x = reinterpret_cast<const __nv_bfloat16*>(d_x);
  a.out = d_act;
  a.w_off0 = 0;
  a.w_off1 = (uint64_t)intermediate * hidden * 2;
  a.rows = (int)intermediate;
  a.K = (int)hidden;
  return launch_ffn<2>(a, n_experts, stream);
}

HV_EXPORT int hv_expert_ffn_down(const uint64_t* d_w_addr, const int32_t* d_counts, const int32_t* d_offs,
                                 const void* d_act, float* d_y, uint32_t n_experts, uint32_t hidden,
                                 uint32_t intermediate, void* stream) {
  return hv_expert_ffn_down_ex(d_w_addr, d_counts, d_offs, d_act, d_y, n_experts, hidden, intermediate, 0u, stream);
}

HV_EXPORT int hv_expert_ffn_down_ex(const uint64_t* d_w_addr, const int32_t* d_counts, const int32_t* d_offs,
                                    const void* d_act, float* d_y, uint32_t n_experts, uint32_t hidden,
                                    uint32_t intermediate, unsigned flags, void* stream) {
  HV_CHECK_ARG((flags & ~(unsigned)(HV_FFN_OVERLAP_PREVIOUS | HV_FFN_TILED | HV_FFN_WAIT_PREVIOUS)) == 0);
  FfnArgs a{};
  a.tiled = (flags & HV_FFN_TILED) ? 1 : 0;
  a.wait_all = (flags & HV_FFN_WAIT_PREVIOUS) ? 1 : 0;
#if HV_FFN_PERSISTENT
  a.wait_x = (flags & HV_FFN_OVERLAP_PREVIOUS) ? 1 : 0;
#endif
  a.w_addr = d_w_addr;
  a.counts = d_counts;
  a.offs = d_offs;
  a.tok = nullptr;
  a.x = reinterpret_cast<const __nv_bfloat16*>(d_act);
  a.out = d_y;
  a.w_off0 = (uint64_t)intermediate * hidden * 4;
  a.w_off1 = 0;
  a.rows = (int)hidden;
  a.K = (int)intermediate;
#if HV_FFN_DOWN_PAIR && HV_FFN_PERSISTENT
  if (!a.tiled && hidden % (2 * kRows) == 0) {
    // two 64-row blocks per item through the two-matrix kernel: every
    // activation fragment (ldmatrix) and every barrier feeds two mma tiles, as
    // in gate/up
    a.pair = 1;
    a.w_off1 = a.w_off0 + (uint64_t)kRows * intermediate * 2;
    return launch_ffn<2>(a, n_experts, stream);
  }
#endif
  return launch_ffn<1>(a, n_experts, stream);
}

HV_EXPORT int hv_expert_ffn_max_tokens(int* out) {
  HV_CHECK_ARG(out);
  *out = kMaxTok;
  return HV_OK;
}
