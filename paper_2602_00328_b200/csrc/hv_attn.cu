// Paged decode attention over KV pages wherever they live (sm_100a).
//
// The consumer of K1 for the KV path (kv_decode.py): one query token per
// sequence attends to its whole context, grouped-query (g = q_heads/kv_heads
// query heads share one KV head).  Pages are addressed through a per-layer
// table of raw page pointers -- local HBM, a donor's slab over NVLink, or the
// pinned host tier -- so the kernel can run over a K1-gathered buffer or
// directly over the pages in place (the fused mode: each KV byte crosses the
// link once and is never written locally).
//
// Page layout (one layer of one block): K [T_b][kv_heads][D] then
// V [T_b][kv_heads][D], fp16, T_b = 16 tokens.
//
// Flash-decoding: grid (splits, kv_heads, B).  A CTA owns a contiguous range
// of its sequence's blocks; its 4 warps take the range's blocks round-robin.
// Each warp streams its blocks' K/V slices through a 3-stage cp.async ring in
// shared memory and folds every 16-token block into an online-softmax state
// (running max, sum, fp32 accumulator) for the g query heads, with the
// products on tensor cores (paged_decode_mma).  The warps merge in shared
// memory and each CTA writes a partial (m, l, acc) per query head;
// hv_paged_decode_attention's second kernel merges the splits in a fixed
// order (deterministic: no atomics), so the result depends only on the bytes.
// A scalar-FMA form of the same ring (paged_decode_split_ring) is kept as the
// measured baseline (build with -DHV_ATTN_MMA=0).  Merging the splits inside
// the attention kernel (the last CTA of each (sequence, KV head) merging in
// split order, threadFenceReduction style) was measured and dropped: one CTA
// walking all splits serially costs more than the second launch
// (4 x 4k: 2,928 vs 3,740 GB/s; 1 x 128k: 4,425 vs 5,564).  Unrolling the
// merge kernel's split loops (8-deep) helped 1 x 128k by 2% and cost 4 x 4k
// 12%: not kept.  Holding each warp's page pointers in lane registers (32 per
// coalesced load, read by shuffle when a block is queued, so no ring refill
// waits on a dependent page-table load) measured (r4h, HBM pages rotated past
// L2) 4 x 4k 3,458 vs 3,208 GB/s at 4 splits, 1 x 128k 5,434 vs 5,495 at 18,
// and across a 32-layer graph step 10,374 vs 10,318 tok/s (4 x 4k) and 390 vs
// 402 (128k): within noise where it counts, not kept.
#include <cuda_fp16.h>
#include <math.h>

#include <map>
#include <mutex>
#include <utility>

#include "hv_common.h"

namespace {

#ifndef HV_ATTN_WARPS
#define HV_ATTN_WARPS 8
#endif
constexpr int kAttnWarps = HV_ATTN_WARPS;   // warps per CTA, each walking its own blocks of the split
constexpr int kBlockTok = 16;

template <int D>
struct Frag {
  static constexpr int kHalf = D / 2;            // dims per lane in QK
  static constexpr int kQkVec = kHalf / 8;       // uint4 loads per lane (8 halves each)
  static constexpr int kPvDims = D / 32;         // dims per lane in PV
};


// Online-softmax update for one 16-token block, all G query heads at once.
// Lanes 2t and 2t+1 hold the two halves of token t's dot products; after the
// xor-1 shuffle both hold the full score.  The block max and sum reduce over
// lane bits 1-4 only (each token once), and the G heads' shuffles are
// interleaved, so the dependent chain is 1 + 4 + 4 shuffles per block rather
// than 11 per head.
template <int G, int PV>
__device__ __forceinline__ void block_softmax(const float (&s)[G], bool valid, float (&m)[G], float (&l)[G],
                                              float (&acc)[G][PV], float (*s_p)[kBlockTok], int t, int half) {
  float sc[G], red[G];
#pragma unroll
  for (int hh = 0; hh < G; ++hh) {
    sc[hh] = s[hh] + __shfl_xor_sync(0xffffffffu, s[hh], 1);
    sc[hh] = valid ? sc[hh] : -INFINITY;
    red[hh] = sc[hh];
  }
#pragma unroll
  for (int o = 2; o < 32; o <<= 1)
#pragma unroll
    for (int hh = 0; hh < G; ++hh) red[hh] = fmaxf(red[hh], __shfl_xor_sync(0xffffffffu, red[hh], o));
  float p[G];
#pragma unroll
  for (int hh = 0; hh < G; ++hh) {
    const float mn = fmaxf(m[hh], red[hh]);
    p[hh] = valid ? __expf(sc[hh] - mn) : 0.f;
    // 0 on the first block (m = -inf); also when every token so far is masked
    // (mn = -inf too), where exp(-inf - -inf) would be NaN
    const float corr = m[hh] == -INFINITY ? 0.f : __expf(m[hh] - mn);
    m[hh] = mn;
    l[hh] *= corr;
#pragma unroll
    for (int j = 0; j < PV; ++j) acc[hh][j] *= corr;
    red[hh] = p[hh];
  }
#pragma unroll
  for (int o = 2; o < 32; o <<= 1)
#pragma unroll
    for (int hh = 0; hh < G; ++hh) red[hh] += __shfl_xor_sync(0xffffffffu, red[hh], o);
#pragma unroll
  for (int hh = 0; hh < G; ++hh) {
    l[hh] += red[hh];
    if (half == 0) s_p[hh][t] = p[hh];
  }
}


// merge the warps of a CTA (fixed order) and write its partial state:
// [B][kvh][splits][G][D + 2] = acc[D], m, l
template <int D, int G>
__device__ __forceinline__ void merge_and_write(const float (&m)[G], const float (&l)[G],
                                                const float (&acc)[G][D / 32], float* __restrict__ part, int b, int h,
                                                int kvh, int split, int splits) {
  __shared__ float s_m[kAttnWarps][G], s_l[kAttnWarps][G];
  __shared__ float s_acc[kAttnWarps][G][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int hh = 0; hh < G; ++hh) {
    if (lane == 0) {
      s_m[warp][hh] = m[hh];
      s_l[warp][hh] = l[hh];
    }
#pragma unroll
    for (int j = 0; j < D / 32; ++j) s_acc[warp][hh][lane * (D / 32) + j] = acc[hh][j];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
    const int hh = i / D, d = i % D;
    float M = -INFINITY;
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, s_m[w][hh]);
    float L = 0.f, A = 0.f;
    for (int w = 0; w < kAttnWarps; ++w) {
      const float c = s_m[w][hh] == -INFINITY ? 0.f : __expf(s_m[w][hh] - M);
      L += s_l[w][hh] * c;
      A += s_acc[w][hh][d] * c;
    }
    float* o = part + ((((size_t)b * kvh + h) * splits + split) * G + hh) * (D + 2);
    o[d] = A;
    if (d == 0) {
      o[D] = M;
      o[D + 1] = L;
    }
  }
}

// Measured on B200, pages in local HBM (tools/attn_probe.py, KV GB/s at the
// best split count; 4 x 4k / 1 x 128k): register prefetch 1,841 / 2,514;
// ring of 2 stages 2,082 / 3,192; 3 stages 2,172 / 3,229 (default);
// 4 stages 1,579 / 2,222 (one resident CTA per SM).  Tensor-core form, warps
// per CTA (best split count each): 2 warps 3,358 / 5,308; 4 warps 3,695 /
// 5,550; 8 warps 3,988 / 5,900 (default: one 8-warp CTA per SM, splits =
// SMs / (sequences x KV heads), fewer CTAs to merge).  One warp per KV head
// with all heads of a page in one CTA (whole-page streaming) measured
// 1,874 / 2,942: HBM row locality is not the limit, per-warp latency is.
//
// Same math, K/V streamed through a per-warp shared-memory ring with
// cp.async (S blocks in flight per warp, no register staging): fewer
// registers (more resident warps) and a deeper prefetch.  K and V rows of
// the head are stored with 16-byte chunk c of row r at c ^ (r & 7), so the
// QK reads (lane pairs on one row) and the PV reads (a whole row across the
// warp) are bank-conflict free.
template <int D>
struct Ring {
  static constexpr int kRow = D * 2;                    // bytes of one token row of one head
  static constexpr int kChunks = kRow / 16;
  static constexpr int kTile = kBlockTok * kRow;        // K or V of one block-head
  static constexpr int kStage = 2 * kTile;
};
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait_n() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int D>
__device__ __forceinline__ uint32_t rswz(int r, int c) {
  return (uint32_t)(r * Ring<D>::kRow + ((c ^ (r & 7)) << 4));
}

template <int D>
__device__ __forceinline__ void ring_load(char* stage, const char* page, int kvh, int h, int lane) {
  const size_t row = (size_t)kvh * D * 2;
  const char* kb = page + (size_t)h * D * 2;
  const char* vb = kb + kBlockTok * row;
  const uint32_t sk = smem_addr(stage), sv = sk + Ring<D>::kTile;
#pragma unroll
  for (int i = lane; i < kBlockTok * Ring<D>::kChunks; i += 32) {
    const int r = i / Ring<D>::kChunks, c = i % Ring<D>::kChunks;
    cp16(sk + rswz<D>(r, c), kb + r * row + c * 16);
    cp16(sv + rswz<D>(r, c), vb + r * row + c * 16);
  }
}

// One 16-token block of one KV head, staged in shared memory at `st` (K tile
// then V tile, swizzled rows), folded into the warp's online-softmax state.
template <int D, int G>
__device__ __forceinline__ void attend_block(const char* st, int blk, int ntok, const float (*s_q)[D],
                                             float (*s_p)[kBlockTok], float (&m)[G], float (&l)[G],
                                             float (&acc)[G][D / 32], int lane) {
  const int t = lane >> 1, half = lane & 1;
    float s_[G];
#pragma unroll
    for (int hh = 0; hh < G; ++hh) s_[hh] = 0.f;
#pragma unroll
    for (int i = 0; i < Frag<D>::kQkVec; ++i) {
      const uint4 kv4 = *reinterpret_cast<const uint4*>(st + rswz<D>(t, half * Frag<D>::kQkVec + i));
      const __half2* hp = reinterpret_cast<const __half2*>(&kv4);
      float kf[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __half22float2(hp[j]);
        kf[2 * j] = f.x;
        kf[2 * j + 1] = f.y;
      }
#pragma unroll
      for (int hh = 0; hh < G; ++hh) {
        const float4* qv = reinterpret_cast<const float4*>(&s_q[hh][half * Frag<D>::kHalf + i * 8]);
        const float4 qa = qv[0], qb = qv[1];
        float a0 = fmaf(kf[0], qa.x, fmaf(kf[1], qa.y, fmaf(kf[2], qa.z, kf[3] * qa.w)));
        float a1 = fmaf(kf[4], qb.x, fmaf(kf[5], qb.y, fmaf(kf[6], qb.z, kf[7] * qb.w)));
        s_[hh] += a0 + a1;
      }
    }
    const bool valid = blk * kBlockTok + t < ntok;
    block_softmax<G, Frag<D>::kPvDims>(s_, valid, m, l, acc, s_p, t, half);
    __syncwarp();
    const char* vt = st + Ring<D>::kTile;
    const int vchunk = lane * Frag<D>::kPvDims * 2 / 16, voff = (lane * Frag<D>::kPvDims * 2) % 16;
#pragma unroll
    for (int t2 = 0; t2 < kBlockTok; ++t2) {
      float vf[Frag<D>::kPvDims];
      const char* vp = vt + rswz<D>(t2, vchunk) + voff;
      if constexpr (Frag<D>::kPvDims == 4) {
        const uint2 x = *reinterpret_cast<const uint2*>(vp);
        const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&x.x));
        const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&x.y));
        vf[0] = f0.x; vf[1] = f0.y; vf[2] = f1.x; vf[3] = f1.y;
      } else {
        const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(vp));
        vf[0] = f0.x; vf[1] = f0.y;
      }
#pragma unroll
      for (int hh = 0; hh < G; ++hh) {
        const float p = s_p[hh][t2];
#pragma unroll
        for (int j = 0; j < Frag<D>::kPvDims; ++j) acc[hh][j] = fmaf(p, vf[j], acc[hh][j]);
      }
    }
}

template <int D, int G, int S>
__global__ void __launch_bounds__(kAttnWarps * 32) paged_decode_split_ring(
    const uint64_t* __restrict__ pages, const int32_t* __restrict__ seq_start, const int32_t* __restrict__ seq_tokens,
    const __half* __restrict__ q, float* __restrict__ part, int kvh, int splits, float scale) {
  extern __shared__ __align__(128) char ring_smem[];
  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int q_heads = kvh * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ __align__(16) float s_q[G][D];
  __shared__ float s_p[kAttnWarps][G][kBlockTok];
  char* my_ring = ring_smem + (size_t)warp * S * Ring<D>::kStage;

  for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
    const int hh = i / D, d = i % D;
    s_q[hh][d] = __half2float(q[((size_t)b * q_heads + h * G + hh) * D + d]) * scale;
  }
  __syncthreads();

  // blocks past the sequence's token count hold nothing to attend: not read
  const int b0 = seq_start[b], ntok = seq_tokens[b];
  const int nblk = min(seq_start[b + 1] - b0, (ntok + kBlockTok - 1) / kBlockTok);
  const int per = (nblk + splits - 1) / splits;
  const int lo = split * per, hi = min(nblk, lo + per);
  // this warp's blocks: lo + warp, lo + warp + 4, ...
  const int mine = lo + warp < hi ? (hi - (lo + warp) + kAttnWarps - 1) / kAttnWarps : 0;

  float m[G], l[G], acc[G][Frag<D>::kPvDims];
#pragma unroll
  for (int hh = 0; hh < G; ++hh) {
    m[hh] = -INFINITY;
    l[hh] = 0.f;
#pragma unroll
    for (int j = 0; j < Frag<D>::kPvDims; ++j) acc[hh][j] = 0.f;
  }
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < mine) ring_load<D>(my_ring + s * Ring<D>::kStage,
                               reinterpret_cast<const char*>(pages[b0 + lo + warp + s * kAttnWarps]), kvh, h, lane);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int it = 0; it < mine; ++it) {
    cp_wait_n<S - 2>();
    __syncwarp();
    {  // refill the stage consumed one iteration ago
      const int nx = it + S - 1;
      if (nx < mine)
        ring_load<D>(my_ring + (nx % S) * Ring<D>::kStage,
                     reinterpret_cast<const char*>(pages[b0 + lo + warp + nx * kAttnWarps]), kvh, h, lane);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    attend_block<D, G>(my_ring + (it % S) * Ring<D>::kStage, lo + warp + it * kAttnWarps, ntok, s_q, s_p[warp], m,
                       l, acc, lane);
    __syncwarp();
  }
  cp_wait_n<0>();
  merge_and_write<D, G>(m, l, acc, part, b, h, kvh, split, splits);
}

// Tensor-core form (default).  Per block a warp computes S^T = Q K^T and
// O += P V with mma.sync.m16n8k16 (fp16 in, fp32 accumulate): the G query
// heads are the M rows (padded to 16, zero rows contribute nothing), the 16
// tokens the N columns of S^T, and the S^T accumulator is reused in place as
// the A operand of P V (the FlashAttention-2 register layout).  K comes from
// the swizzled ring with ldmatrix, V with ldmatrix.trans.  The scalar
// kernels above spend ~1,250 instructions per 8 KiB block-head (ncu: issue
// stalled on short scoreboard, 40% issue-active); this one ~150.  Measured
// (HBM pages, best split count, 4 x 4k / 1 x 128k): 3,740 / 5,564 GB/s vs
// 2,209 / 3,199 for the scalar ring; ring stages 2 / 3 / 4: 3,564 / 3,740 /
// 3,198 and 5,499 / 5,564 / 5,229 (3 is the default).
__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// One 16-token block of one KV head, staged at `st` (K tile then V tile,
// swizzled rows), folded into the warp's online-softmax state on tensor cores.
// Lane (gr, c) owns query head gr (rows gr+8 are padding): its running max
// and sum, and O[gr][n*8 + 2c + {0,1}].  `tb` is the block's first token.
template <int D>
__device__ __forceinline__ void mma_attend_block(const char* st, int tb, int ntok, const uint32_t (&qa)[D / 16][2],
                                                 float scale, float& m_run, float& l_run, float (&o)[D / 8][2],
                                                 int lane) {
  constexpr int KS = D / 16, NT = D / 8;
  const int c = lane & 3;
  // ldmatrix lane roles: x4 over (tokens 0-7 | 8-15) x (k 0-7 | 8-15)
  const int lm_row = (lane & 7) + ((lane >> 4) << 3);
  const int lm_k = (lane >> 3) & 1;
  // trans x4 over V: (tokens 0-7 | 8-15) x (dims d..d+7 | d+8..d+15)
  const int lt_row = (lane & 7) + (((lane >> 3) & 1) << 3);
  const int lt_d = lane >> 4;
  const uint32_t ks_addr = smem_addr(st), vs_addr = ks_addr + Ring<D>::kTile;
  // S^T = Q K^T : two n tiles (tokens 0-7, 8-15)
  float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    uint32_t k0, k1, k2, k3;   // (tok 0-7,k lo) (tok 0-7,k hi) (tok 8-15,k lo) (tok 8-15,k hi)
    ldsm4(ks_addr + rswz<D>(lm_row, ks * 2 + lm_k), k0, k1, k2, k3);
    mma16816(s0, qa[ks][0], 0u, qa[ks][1], 0u, k0, k1);
    mma16816(s1, qa[ks][0], 0u, qa[ks][1], 0u, k2, k3);
  }
  // row gr: tokens 2c, 2c+1 (tile 0) and 8+2c, 9+2c (tile 1); rows gr+8 (s*[2..3]) are padding
  float x[4] = {s0[0] * scale, s0[1] * scale, s1[0] * scale, s1[1] * scale};
  const int tk[4] = {2 * c, 2 * c + 1, 8 + 2 * c, 9 + 2 * c};
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (tb + tk[j] >= ntok) x[j] = -INFINITY;
  float bm = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
  bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 1));
  bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
  const float mn = fmaxf(m_run, bm);
  float p[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) p[j] = x[j] == -INFINITY ? 0.f : __expf(x[j] - mn);
  float bs = (p[0] + p[1]) + (p[2] + p[3]);
  bs += __shfl_xor_sync(0xffffffffu, bs, 1);
  bs += __shfl_xor_sync(0xffffffffu, bs, 2);
  const float corr = m_run == -INFINITY ? 0.f : __expf(m_run - mn);  // 0 on the first / all-masked blocks
  m_run = mn;
  l_run = l_run * corr + bs;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    o[n][0] *= corr;
    o[n][1] *= corr;
  }
  // P as the A operand (rows gr / gr+8, k = tokens): a0 (gr, 2c..) a1 (gr+8) a2 (gr, 2c+8..) a3 (gr+8)
  const uint32_t pa0 = pack_h2(p[0], p[1]), pa2 = pack_h2(p[2], p[3]);
#pragma unroll
  for (int np = 0; np < NT / 2; ++np) {
    uint32_t v0, v1, v2, v3;   // b0,b1 of dims np*16..+7, then of np*16+8..+15
    ldsm4_t(vs_addr + rswz<D>(lt_row, np * 2 + lt_d), v0, v1, v2, v3);
    float d0[4] = {o[2 * np][0], o[2 * np][1], 0.f, 0.f};
    float d1[4] = {o[2 * np + 1][0], o[2 * np + 1][1], 0.f, 0.f};
    mma16816(d0, pa0, 0u, pa2, 0u, v0, v1);
    mma16816(d1, pa0, 0u, pa2, 0u, v2, v3);
    o[2 * np][0] = d0[0];
    o[2 * np][1] = d0[1];
    o[2 * np + 1][0] = d1[0];
    o[2 * np + 1][1] = d1[1];
  }
}

// Q of (sequence b, KV head h) as the A operand: row gr = query head (zero
// beyond G), k = head dims.  a0 (row gr, k 2c..), a2 (row gr, k 2c+8..).
template <int D, int G>
__device__ __forceinline__ void load_q_frag(const __half* __restrict__ q, int b, int h, int q_heads,
                                            uint32_t (&qa)[D / 16][2], int lane) {
  const int gr = lane >> 2, c = lane & 3;
  const __half* qh = q + ((size_t)b * q_heads + h * G + (gr < G ? gr : 0)) * D;
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    if (gr < G) {
      qa[ks][0] = *reinterpret_cast<const uint32_t*>(qh + ks * 16 + 2 * c);
      qa[ks][1] = *reinterpret_cast<const uint32_t*>(qh + ks * 16 + 8 + 2 * c);
    } else {
      qa[ks][0] = qa[ks][1] = 0u;
    }
  }
}

template <int D, int G, int S>
__global__ void __launch_bounds__(kAttnWarps * 32) paged_decode_mma(
    const uint64_t* __restrict__ pages, const int32_t* __restrict__ seq_start, const int32_t* __restrict__ seq_tokens,
    const __half* __restrict__ q, float* __restrict__ part, int kvh, int splits, float scale,
    float* __restrict__ final_out, unsigned* __restrict__ done) {
  static_assert(G <= 8, "query rows g and g+8 of the m16 tile: at most 8 heads per KV head");
  constexpr int KS = D / 16;             // k steps of Q K^T
  constexpr int NT = D / 8;              // n tiles of P V
  extern __shared__ __align__(128) char ring_smem[];
  __shared__ float s_m[kAttnWarps][G], s_l[kAttnWarps][G];
  __shared__ float s_acc[kAttnWarps][G][D];
  const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  // let the next kernel on the stream (the next layer's attention, launched
  // with HV_ATTN_OVERLAP_PREVIOUS) start its CTAs as ours drain
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int q_heads = kvh * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gr = lane >> 2, c = lane & 3;        // mma fragment row group / column pair
  char* my_ring = ring_smem + (size_t)warp * S * Ring<D>::kStage;

  uint32_t qa[KS][2];
  load_q_frag<D, G>(q, b, h, q_heads, qa, lane);
  // blocks past the sequence's token count hold nothing to attend: not read
  const int b0 = seq_start[b], ntok = seq_tokens[b];
  const int nblk = min(seq_start[b + 1] - b0, (ntok + kBlockTok - 1) / kBlockTok);
  const int per = (nblk + splits - 1) / splits;
  const int lo = split * per, hi = min(nblk, lo + per);
  const int mine = lo + warp < hi ? (hi - (lo + warp) + kAttnWarps - 1) / kAttnWarps : 0;

  float m_run = -INFINITY, l_run = 0.f;  // of row gr (query head gr)
  float o[NT][2];                        // O[gr][n*8 + 2c + {0,1}]
#pragma unroll
  for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = 0.f;

#pragma unroll
  for (int st = 0; st < S - 1; ++st) {
    if (st < mine) ring_load<D>(my_ring + st * Ring<D>::kStage,
                                reinterpret_cast<const char*>(pages[b0 + lo + warp + st * kAttnWarps]), kvh, h, lane);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int it = 0; it < mine; ++it) {
    cp_wait_n<S - 2>();
    __syncwarp();
    const int nx = it + S - 1;
    if (nx < mine)
      ring_load<D>(my_ring + (nx % S) * Ring<D>::kStage,
                   reinterpret_cast<const char*>(pages[b0 + lo + warp + nx * kAttnWarps]), kvh, h, lane);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const int blk = lo + warp + it * kAttnWarps;
    mma_attend_block<D>(my_ring + (it % S) * Ring<D>::kStage, blk * kBlockTok, ntok, qa, scale, m_run, l_run, o,
                        lane);
    __syncwarp();
  }
  cp_wait_n<0>();
  // programmatic dependent launch (HV_ATTN_OVERLAP_PREVIOUS): everything above
  // read only inputs the caller vouched for; the writes below (partials, the
  // merge counters, the output) wait for the previous kernel on the stream
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // merge the warps (fixed order) and write the partial state
  if (gr < G) {
    if (c == 0) {
      s_m[warp][gr] = m_run;
      s_l[warp][gr] = l_run;
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      s_acc[warp][gr][n * 8 + 2 * c] = o[n][0];
      s_acc[warp][gr][n * 8 + 2 * c + 1] = o[n][1];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
    const int hh = i / D, d = i % D;
    float M = -INFINITY;
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, s_m[w][hh]);
    float L = 0.f, A = 0.f;
    for (int w = 0; w < kAttnWarps; ++w) {
      const float cf = s_m[w][hh] == -INFINITY ? 0.f : __expf(s_m[w][hh] - M);
      L += s_l[w][hh] * cf;
      A += s_acc[w][hh][d] * cf;
    }
    float* out = part + ((((size_t)b * kvh + h) * splits + split) * G + hh) * (D + 2);
    out[d] = A;
    if (d == 0) {
      out[D] = M;
      out[D + 1] = L;
    }
  }
  if (done == nullptr) return;   // the caller launches paged_decode_combine
  // Fused combine: the last CTA of this (sequence, KV head) to finish merges
  // the splits' partial states in split order -- the same arithmetic and
  // order as paged_decode_combine, so the result does not depend on which CTA
  // came last -- and re-arms the counter for the next launch (or graph replay).
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done + (size_t)b * kvh + h, 1u) == (unsigned)splits - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* base = part + (((size_t)b * kvh + h) * splits) * G * (D + 2);
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
    const int hh = i / D, d = i % D;
    float M = -INFINITY;
    for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(base + ((size_t)sp * G + hh) * (D + 2) + D));
    float L = 0.f, A = 0.f;
    for (int sp = 0; sp < splits; ++sp) {
      const float* pp = base + ((size_t)sp * G + hh) * (D + 2);
      const float pm = __ldcg(pp + D);
      const float cf = pm == -INFINITY ? 0.f : __expf(pm - M);
      L += __ldcg(pp + D + 1) * cf;
      A += __ldcg(pp + d) * cf;
    }
    final_out[((size_t)b * (kvh * G) + h * G + hh) * D + d] = L > 0.f ? A / L : 0.f;
  }
  if (threadIdx.x == 0) done[(size_t)b * kvh + h] = 0u;
}

// out[b][qh][d] = sum_s acc_s[d] e^(m_s - M) / sum_s l_s e^(m_s - M), splits in order
template <int D>
__global__ void paged_decode_combine(const float* __restrict__ part, float* __restrict__ out, int q_heads, int kvh,
                                     int splits) {
  const int qh = blockIdx.x, b = blockIdx.y, d = threadIdx.x;
  const int g = q_heads / kvh, h = qh / g, hh = qh % g;
  const float* base = part + (((size_t)b * kvh + h) * splits) * g * (D + 2);
  float M = -INFINITY;
  for (int s = 0; s < splits; ++s) M = fmaxf(M, base[((size_t)s * g + hh) * (D + 2) + D]);
  float L = 0.f, A = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float* p = base + ((size_t)s * g + hh) * (D + 2);
    const float c = p[D] == -INFINITY ? 0.f : __expf(p[D] - M);
    L += p[D + 1] * c;
    A += p[d] * c;
  }
  out[((size_t)b * q_heads + qh) * D + d] = L > 0.f ? A / L : 0.f;
}

// ---- balanced (stream-K) form: HV_ATTN_BALANCED ---------------------------
// The (split, KV head, sequence) grid gives every (sequence, KV head) pair the
// same number of CTAs, so a few long sequences fill the machine only when
// pairs x splits happens to be a multiple of the SM count: config 1 (4 x 4k,
// 32 pairs) ran 4 splits = 128 CTAs on 148 SMs, and 5 splits a second, mostly
// empty wave.  Here the work units -- (pair, 16-token block), pair-major over
// the sequences' live blocks -- are cut into `n_cta` equal contiguous ranges,
// one CTA each (one CTA per SM resident), so every SM streams the same number
// of bytes.  A range covers the tail of one pair, whole pairs, and the head of
// another; the CTA folds each pair's part (a segment) with all its warps
// (units round-robin over warps, one cp.async ring per warp running across
// segment boundaries, so the next segment's pages are in flight while the
// warps merge), writes one partial state per segment into slot (cta + pair)
// -- unique, since ranges are ordered -- and the last CTA to finish a pair
// merges its partials in CTA order (deterministic; a pair inside one CTA is
// written directly).  cta_of(u) = the CTA whose range holds unit u.
__device__ __forceinline__ int cta_of(long long u, long long units, int n_cta) {
  return (int)(((u + 1) * n_cta - 1) / units);
}

// merge `n` partial states (slots first .. first+n-1, in order) of one query
// head and dim; returns the normalized output
template <int D>
__device__ __forceinline__ float merge_slots(const float* __restrict__ part, size_t first, int n, int G, int hh,
                                             int d) {
  float M = -INFINITY;
  for (int i = 0; i < n; ++i) M = fmaxf(M, __ldcg(part + ((first + i) * G + hh) * (D + 2) + D));
  float L = 0.f, A = 0.f;
  for (int i = 0; i < n; ++i) {
    const float* pp = part + ((first + i) * G + hh) * (D + 2);
    const float pm = __ldcg(pp + D);
    const float cf = pm == -INFINITY ? 0.f : __expf(pm - M);
    L += __ldcg(pp + D + 1) * cf;
    A += __ldcg(pp + d) * cf;
  }
  return L > 0.f ? A / L : 0.f;
}

template <int D, int G, int S>
__global__ void __launch_bounds__(kAttnWarps * 32) paged_decode_balanced(
    const uint64_t* __restrict__ pages, const int32_t* __restrict__ seq_start, const int32_t* __restrict__ seq_tokens,
    const __half* __restrict__ q, float* __restrict__ part, int B, int kvh, float scale,
    float* __restrict__ final_out, unsigned* __restrict__ done) {
  static_assert(G <= 8, "query rows g and g+8 of the m16 tile: at most 8 heads per KV head");
  constexpr int NT = D / 8;
  constexpr int W = kAttnWarps;
  extern __shared__ __align__(128) char ring_smem[];
  int* s_pre = reinterpret_cast<int*>(ring_smem + (size_t)W * S * Ring<D>::kStage);  // [B+1] units before sequence b
  __shared__ float s_m[W][G], s_l[W][G];
  __shared__ float s_acc[W][G][D];
  __shared__ unsigned s_last;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int q_heads = kvh * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gr = lane >> 2, c = lane & 3;
  const int cta = blockIdx.x;
  char* my_ring = ring_smem + (size_t)warp * S * Ring<D>::kStage;

  if (warp == 0) {   // live blocks x kv heads per sequence, exclusive prefix
    int run = 0;
    for (int base = 0; base < B; base += 32) {
      const int b = base + lane;
      int nb = 0;
      if (b < B) nb = max(0, min(seq_start[b + 1] - seq_start[b], (seq_tokens[b] + kBlockTok - 1) / kBlockTok)) * kvh;
      int x = nb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (b < B) s_pre[b] = run + x - nb;
      run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) s_pre[B] = run;
  }
  __syncthreads();
  const long long units = s_pre[B];
  // at most one CTA per unit, so every range is non-empty and the CTAs
  // cta_of() names for a pair all arrive on its counter
  const int n_cta = (int)min((long long)gridDim.x, units);
  const int u0 = cta < n_cta ? (int)((long long)cta * units / n_cta) : 0;
  const int u1 = cta < n_cta ? (int)((long long)(cta + 1) * units / n_cta) : 0;

  // the pair holding unit u0: sequence by binary search over the prefix
  int sb = 0, sh = 0;
  if (u0 < u1) {
    int lo = 0, hi = B - 1;   // last b with s_pre[b] <= u0 (then skip sequences with no units)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pre[mid] <= u0) lo = mid; else hi = mid - 1;
    }
    sb = lo;
    while (s_pre[sb + 1] == s_pre[sb]) ++sb;
    sh = (u0 - s_pre[sb]) / ((s_pre[sb + 1] - s_pre[sb]) / kvh);
  }
  // a cursor over this warp's units: (sequence, head, unit, segment end, pair's first unit)
  struct Cur {
    int b, h, u, e, q0;
  };
  // first unit of this warp at or after pair (b, h); u >= u1 when none is left
  auto seek = [&](Cur& k, int b, int h) {
    for (;;) {
      while (b < B && s_pre[b + 1] == s_pre[b]) { ++b; h = 0; }
      if (b >= B) { k.u = u1; return; }
      const int nbk = (s_pre[b + 1] - s_pre[b]) / kvh;
      const int q0 = s_pre[b] + h * nbk;
      if (q0 >= u1) { k.u = u1; return; }
      const int a = max(q0, u0), e = min(q0 + nbk, u1);
      if (a + warp < e) {
        k.b = b; k.h = h; k.u = a + warp; k.e = e; k.q0 = q0;
        return;
      }
      if (++h == kvh) { ++b; h = 0; }
    }
  };
  auto advance = [&](Cur& k) {
    k.u += W;
    if (k.u < k.e) return;
    int b = k.b, h = k.h + 1;
    if (h == kvh) { ++b; h = 0; }
    seek(k, b, h);
  };
  auto load = [&](const Cur& k, int slot) {
    ring_load<D>(my_ring + slot * Ring<D>::kStage,
                 reinterpret_cast<const char*>(pages[seq_start[k.b] + (k.u - k.q0)]), kvh, k.h, lane);
  };

  Cur ld;
  seek(ld, sb, sh);
  if (u0 >= u1) ld.u = u1;
  int n_loaded = 0, n_done = 0;
#pragma unroll
  for (int st = 0; st < S - 1; ++st) {
    if (ld.u < u1) {
      load(ld, n_loaded % S);
      ++n_loaded;
      advance(ld);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  bool waited = false;
  // segments: the pairs this CTA's range touches, in order (every warp walks
  // all of them so the CTA-wide merges line up)
  int pb = sb, ph = sh;
  while (u0 < u1) {
    while (pb < B && s_pre[pb + 1] == s_pre[pb]) { ++pb; ph = 0; }
    if (pb >= B) break;
    const int nbk = (s_pre[pb + 1] - s_pre[pb]) / kvh;
    const int q0 = s_pre[pb] + ph * nbk;
    if (q0 >= u1) break;
    const int a = max(q0, u0), e = min(q0 + nbk, u1);
    const int ntok = seq_tokens[pb];
    uint32_t qa[D / 16][2];
    load_q_frag<D, G>(q, pb, ph, q_heads, qa, lane);
    float m_run = -INFINITY, l_run = 0.f;
    float o[NT][2];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = 0.f;
    for (int u = a + warp; u < e; u += W) {
      cp_wait_n<S - 2>();
      __syncwarp();
      if (ld.u < u1) {
        load(ld, n_loaded % S);
        ++n_loaded;
        advance(ld);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      mma_attend_block<D>(my_ring + (n_done % S) * Ring<D>::kStage, (u - q0) * kBlockTok, ntok, qa, scale, m_run,
                          l_run, o, lane);
      ++n_done;
      __syncwarp();
    }
    if (!waited) {   // HV_ATTN_OVERLAP_PREVIOUS: first write waits for the previous kernel
      asm volatile("griddepcontrol.wait;" ::: "memory");
      waited = true;
    }
    if (gr < G) {
      if (c == 0) {
        s_m[warp][gr] = m_run;
        s_l[warp][gr] = l_run;
      }
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        s_acc[warp][gr][n * 8 + 2 * c] = o[n][0];
        s_acc[warp][gr][n * 8 + 2 * c + 1] = o[n][1];
      }
    }
    __syncthreads();
    const int pair = pb * kvh + ph;
    const int c0 = cta_of(q0, units, n_cta), c1 = cta_of(q0 + nbk - 1, units, n_cta);
    const bool alone = c0 == c1 && done != nullptr;
    for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
      const int hh = i / D, d = i % D;
      float M = -INFINITY;
      for (int w = 0; w < W; ++w) M = fmaxf(M, s_m[w][hh]);
      float L = 0.f, A = 0.f;
      for (int w = 0; w < W; ++w) {
        const float cf = s_m[w][hh] == -INFINITY ? 0.f : __expf(s_m[w][hh] - M);
        L += s_l[w][hh] * cf;
        A += s_acc[w][hh][d] * cf;
      }
      if (alone) {
        final_out[((size_t)pb * q_heads + ph * G + hh) * D + d] = L > 0.f ? A / L : 0.f;
      } else {
        float* out = part + (((size_t)cta + pair) * G + hh) * (D + 2);
        out[d] = A;
        if (d == 0) {
          out[D] = M;
          out[D + 1] = L;
        }
      }
    }
    if (!alone && done != nullptr) {
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_last = atomicAdd(done + pair, 1u) == (unsigned)(c1 - c0);
      __syncthreads();
      if (s_last) {
        __threadfence();
        for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
          const int hh = i / D, d = i % D;
          final_out[((size_t)pb * q_heads + ph * G + hh) * D + d] =
              merge_slots<D>(part, (size_t)c0 + pair, c1 - c0 + 1, G, hh, d);
        }
        if (threadIdx.x == 0) done[pair] = 0u;
      }
    }
    __syncthreads();   // s_m / s_acc / s_last free for the next segment
    if (++ph == kvh) { ++pb; ph = 0; }
  }
  cp_wait_n<0>();
  if (done == nullptr) return;   // paged_decode_combine_balanced writes every output
  if (!waited) asm volatile("griddepcontrol.wait;" ::: "memory");
  // pairs with no live block: zero output (no CTA range covers them)
  for (int pair = cta; pair < B * kvh; pair += gridDim.x) {
    const int b = pair / kvh;
    if (s_pre[b + 1] != s_pre[b]) continue;
    for (int i = threadIdx.x; i < G * D; i += blockDim.x) final_out[((size_t)b * q_heads + (pair % kvh) * G) * D + i] = 0.f;
  }
}

// paged_decode_balanced's merge as a second kernel (launches without the
// arrival counters, e.g. the first capture on a stream): grid (q_heads, B)
template <int D>
__global__ void paged_decode_combine_balanced(const int32_t* __restrict__ seq_start,
                                              const int32_t* __restrict__ seq_tokens, const float* __restrict__ part,
                                              float* __restrict__ out, int B, int q_heads, int kvh, int n_cta) {
  const int qh = blockIdx.x, b = blockIdx.y, d = threadIdx.x;
  const int g = q_heads / kvh, h = qh / g, hh = qh % g;
  long long units = 0, before = 0;
  int nbk = 0;
  for (int i = 0; i < B; ++i) {
    const int nb = max(0, min(seq_start[i + 1] - seq_start[i], (seq_tokens[i] + kBlockTok - 1) / kBlockTok));
    if (i == b) { before = units; nbk = nb; }
    units += (long long)nb * kvh;
  }
  float r = 0.f;
  if (nbk > 0) {
    n_cta = (int)min((long long)n_cta, units);   // as in paged_decode_balanced
    const long long q0 = before + (long long)h * nbk;
    const int c0 = cta_of(q0, units, n_cta), c1 = cta_of(q0 + nbk - 1, units, n_cta);
    r = merge_slots<D>(part, (size_t)c0 + (size_t)b * kvh + h, c1 - c0 + 1, g, hh, d);
  }
  out[((size_t)b * q_heads + qh) * D + d] = r;
}

#ifndef HV_ATTN_MMA
#define HV_ATTN_MMA 3
#endif
#ifndef HV_ATTN_RING
#define HV_ATTN_RING 3   // stages of the scalar kernel, built only with HV_ATTN_MMA=0
#endif

// Arrival counters of the fused combine (one per sequence x KV head), zero
// between launches, one buffer per (device, stream): launches on one stream
// are ordered (with HV_ATTN_OVERLAP_PREVIOUS a kernel touches the counters
// only after griddepcontrol.wait), while kernels on different streams may run
// at once and must not share them.  Allocated outside CUDA-graph capture
// only; a launch that finds none while capturing (or beyond kMaxStreams
// streams) uses the two-kernel path.
struct DoneBuf {
  unsigned* p = nullptr;
  size_t cap = 0;
};
std::mutex g_done_mu;
std::map<std::pair<int, cudaStream_t>, DoneBuf> g_done;
constexpr size_t kMaxStreams = 256;

unsigned* done_counters(int dev, size_t need, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_done_mu);
  auto key = std::make_pair(dev, s);
  auto it = g_done.find(key);
  if (it != g_done.end() && it->second.cap >= need) return it->second.p;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    (void)cudaGetLastError();
    return nullptr;
  }
  if (it == g_done.end() && g_done.size() >= kMaxStreams) return nullptr;
  size_t cap_n = need < 4096 ? 4096 : need;
  unsigned* p = nullptr;
  // zeroed on the launching stream: ordered before this launch whatever the
  // stream's flags (a legacy-stream memset does not order non-blocking streams)
  if (cudaMalloc(&p, cap_n * sizeof(unsigned)) != cudaSuccess ||
      cudaMemsetAsync(p, 0, cap_n * sizeof(unsigned), s) != cudaSuccess) {
    (void)cudaGetLastError();
    if (p) cudaFree(p);
    return nullptr;
  }
  if (it != g_done.end() && it->second.p) {   // grown: no launch can still use the old buffer once the stream is idle
    cudaStreamSynchronize(s);
    cudaFree(it->second.p);
  }
  g_done[key] = DoneBuf{p, cap_n};
  return p;
}

#ifndef HV_ATTN_FUSED_COMBINE
#define HV_ATTN_FUSED_COMBINE 1
#endif

constexpr uint32_t kBalancedMaxSeqs = 256;   // s_pre in shared memory beside the rings

template <int D, int G>
int launch_attn_balanced(const uint64_t* pages, const int32_t* seq_start, const int32_t* seq_tokens, const void* q,
                         float* out, float* part, uint32_t B, uint32_t kvh, uint32_t n_cta, float scale,
                         cudaStream_t s, unsigned flags) {
  int dev = 0;
  HV_CUDA(cudaGetDevice(&dev));
  constexpr int kS = HV_ATTN_MMA ? HV_ATTN_MMA : 3;
  const size_t smem = (size_t)kAttnWarps * kS * Ring<D>::kStage + (kBalancedMaxSeqs + 1) * sizeof(int);
  int st = hv::kernel_attr<paged_decode_balanced<D, G, kS>>(dev, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                            (int)smem);
  if (st) return st;
  unsigned* done = HV_ATTN_FUSED_COMBINE ? done_counters(dev, (size_t)B * kvh, s) : nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_cta);
  cfg.blockDim = dim3(kAttnWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (flags & HV_ATTN_OVERLAP_PREVIOUS) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HV_CUDA(cudaLaunchKernelEx(&cfg, paged_decode_balanced<D, G, kS>, pages, seq_start, seq_tokens,
                             reinterpret_cast<const __half*>(q), part, (int)B, (int)kvh, scale, out, done));
  HV_CUDA(cudaGetLastError());
  if (done) {
    hv::note_launch(1);
    return HV_OK;
  }
  paged_decode_combine_balanced<D><<<dim3(kvh * G, B), D, 0, s>>>(seq_start, seq_tokens, part, out, (int)B,
                                                                  (int)(kvh * G), (int)kvh, (int)n_cta);
  HV_CUDA(cudaGetLastError());
  hv::note_launch(2);
  return HV_OK;
}

template <int D, int G>
int launch_attn(const uint64_t* pages, const int32_t* seq_start, const int32_t* seq_tokens, const void* q,
                float* out, float* part, uint32_t B, uint32_t kvh, uint32_t splits, float scale, cudaStream_t s,
                unsigned flags) {
  dim3 grid(splits, kvh, B);
  int dev = 0;   // made current by the caller (bind_stream_device)
  HV_CUDA(cudaGetDevice(&dev));
  int st;
#if HV_ATTN_MMA
  {
    constexpr int kS = HV_ATTN_MMA;
    constexpr size_t smem = (size_t)kAttnWarps * kS * Ring<D>::kStage;
    st = hv::kernel_attr<paged_decode_mma<D, G, kS>>(dev, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (st) return st;
    unsigned* done = HV_ATTN_FUSED_COMBINE ? done_counters(dev, (size_t)B * kvh, s) : nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kAttnWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (flags & HV_ATTN_OVERLAP_PREVIOUS) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HV_CUDA(cudaLaunchKernelEx(&cfg, paged_decode_mma<D, G, kS>, pages, seq_start, seq_tokens,
                               reinterpret_cast<const __half*>(q), part, (int)kvh, (int)splits, scale, out, done));
    if (done) {
      HV_CUDA(cudaGetLastError());
      hv::note_launch(1);
      return HV_OK;
    }
  }
#else
  constexpr int kS = HV_ATTN_RING;
  constexpr size_t smem = (size_t)kAttnWarps * kS * Ring<D>::kStage;
  st = hv::kernel_attr<paged_decode_split_ring<D, G, kS>>(dev, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (st) return st;
  paged_decode_split_ring<D, G, kS><<<grid, kAttnWarps * 32, smem, s>>>(
      pages, seq_start, seq_tokens, reinterpret_cast<const __half*>(q), part, (int)kvh, (int)splits, scale);
#endif
  HV_CUDA(cudaGetLastError());
  paged_decode_combine<D><<<dim3(kvh * G, B), D, 0, s>>>(part, out, (int)(kvh * G), (int)kvh, (int)splits);
  HV_CUDA(cudaGetLastError());
  hv::note_launch(2);
  return HV_OK;
}

template <int D>
int launch_attn_g(uint32_t g, const uint64_t* pages, const int32_t* seq_start, const int32_t* seq_tokens,
                  const void* q, float* out, float* part, uint32_t B, uint32_t kvh, uint32_t splits, float scale,
                  cudaStream_t s, unsigned flags) {
  if (flags & HV_ATTN_BALANCED) {
    switch (g) {
      case 1: return launch_attn_balanced<D, 1>(pages, seq_start, seq_tokens, q, out, part, B, kvh, splits, scale, s, flags);
      case 2: return launch_attn_balanced<D, 2>(pages, seq_start, seq_tokens, q, out, part, B, kvh, splits, scale, s, flags);
      case 4: return launch_attn_balanced<D, 4>(pages, seq_start, seq_tokens, q, out, part, B, kvh, splits, scale, s, flags);
      case 8: return launch_attn_balanced<D, 8>(pages, seq_start, seq_tokens, q, out, part, B, kvh, splits, scale, s, flags);
      default: return HV_E_INVALID;
    }
  }
  switch (g) {
    case 1: return launch_attn<D, 1>(pages, seq_start, seq_tokens, q, out, part, B, kvh, splits, scale, s, flags);
    case 2: return launch_attn<D, 2>(pages, seq_start, seq_tokens, q, out, part, B, kvh, splits, scale, s, flags);
    case 4: return launch_attn<D, 4>(pages, seq_start, seq_tokens, q, out, part, B, kvh, splits, scale, s, flags);
    case 8: return launch_attn<D, 8>(pages, seq_start, seq_tokens, q, out, part, B, kvh, splits, scale, s, flags);
    default: return HV_E_INVALID;
  }
}

}  // namespace

HV_EXPORT int hv_paged_decode_attention_ex(const uint64_t* d_page_ptrs, const int32_t* d_seq_start,
                                           const int32_t* d_seq_tokens, const void* d_q, float* d_out,
                                           float* d_part, uint32_t batch, uint32_t q_heads, uint32_t kv_heads,
                                           uint32_t head_dim, uint32_t block_tokens, uint32_t splits, float scale,
                                           unsigned flags, void* stream) {
  if (batch == 0) return HV_OK;
  HV_CHECK_ARG(d_page_ptrs && d_seq_start && d_seq_tokens && d_q && d_out && d_part);
  HV_CHECK_ARG(kv_heads > 0 && q_heads % kv_heads == 0);
  {
    const uint32_t g = q_heads / kv_heads;   // grouped-query sizes with a compiled kernel
    HV_CHECK_ARG(g == 1 || g == 2 || g == 4 || g == 8);
  }
  HV_CHECK_ARG(head_dim == 64 || head_dim == 128);
  HV_CHECK_ARG(block_tokens == (uint32_t)kBlockTok);
  HV_CHECK_ARG(splits >= 1 && splits <= 1024 && batch <= 65535u && kv_heads <= 65535u);
  HV_CHECK_ARG((flags & ~(unsigned)(HV_ATTN_OVERLAP_PREVIOUS | HV_ATTN_BALANCED)) == 0);
  HV_CHECK_ARG(!(flags & HV_ATTN_BALANCED) || batch <= kBalancedMaxSeqs);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t g = q_heads / kv_heads;
  if (head_dim == 128)
    return launch_attn_g<128>(g, d_page_ptrs, d_seq_start, d_seq_tokens, d_q, d_out, d_part, batch, kv_heads, splits,
                              scale, s, flags);
  return launch_attn_g<64>(g, d_page_ptrs, d_seq_start, d_seq_tokens, d_q, d_out, d_part, batch, kv_heads, splits,
                           scale, s, flags);
}

HV_EXPORT int hv_paged_decode_attention(const uint64_t* d_page_ptrs, const int32_t* d_seq_start,
                                        const int32_t* d_seq_tokens, const void* d_q, float* d_out, float* d_part,
                                        uint32_t batch, uint32_t q_heads, uint32_t kv_heads, uint32_t head_dim,
                                        uint32_t block_tokens, uint32_t splits, float scale, void* stream) {
  return hv_paged_decode_attention_ex(d_page_ptrs, d_seq_start, d_seq_tokens, d_q, d_out, d_part, batch, q_heads,
                                      kv_heads, head_dim, block_tokens, splits, scale, 0u, stream);
}
