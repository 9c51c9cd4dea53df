// MoE decode glue around K4 (sm_100a): the router and the top-k combine.
//
// A decode stage of the fused decoder (decode.py, moe.py:315-340 semantics)
// is router -> top-k -> softmax -> routed pairs sorted by expert -> K4
// gate/up -> K4 down -> fixed-order combine -> residual.  Built from torch
// ops the glue was ~25 small kernels per stage (~100 us of an ~260 us Qwen
// stage with the experts in HBM, tools/tiled_decode_probe.py r5h); here it is
// two launches, plus hv_moe_stage_plan (one warp) when host-tier experts are
// staged by K2 first:
//
//   hv_moe_route    logits = h . router^T in fp32 (one warp per (token,
//                   expert) dot, lanes over 16-byte chunks, fixed shuffle
//                   order), then -- in the last CTA to finish, found by an
//                   arrival ticket -- per token the top-k (largest first, ties
//                   to the lower expert id), softmax over the k logits, the
//                   per-expert pair counts and offsets, and the stable sort of
//                   the pairs (t, j) by expert: tok[sorted] = t,
//                   pos[t*k + j] = sorted position (torch.argsort(stable)).
//   hv_moe_combine  h[t] += rs * bf16(sum_j probs[t][j] * y[pos[t*k + j]])
//                   with the same rounding steps as the torch expression
//                   h + (y.to(bf16) * rs) in bf16.
//
// Deterministic: no floating-point atomics; the result depends only on the
// inputs.
#include <cuda_bf16.h>

#include "hv_common.h"

namespace {

constexpr int kRouteWarps = 8;                 // tokens per route CTA (one warp each)
constexpr int kRouteThreads = kRouteWarps * 32;
constexpr uint32_t kMaxE = 256, kMaxK = 8, kMaxT = 256;
constexpr int kStageFloats = 8192;             // 32 KiB of logits staged per chunk of tokens

__device__ __forceinline__ float bf16lo(uint32_t x) { return __uint_as_float(x << 16); }
__device__ __forceinline__ float bf16hi(uint32_t x) { return __uint_as_float(x & 0xFFFF0000u); }

// top-K of one token's logits (largest first, ties to the lower expert id,
// NaN ranked last), the softmax over them, and the token's pairs
template <int K>
__device__ __forceinline__ void token_topk(const float* __restrict__ lg, int tt, int E, float* __restrict__ probs,
                                           int64_t* __restrict__ topi, int* __restrict__ s_exp) {
  float tv[K];
  int ti[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    tv[j] = -INFINITY;
    ti[j] = 0x7FFFFFFF;
  }
  for (int e = 0; e < E; ++e) {
    float x = lg[e];   // the token's row, staged in shared memory
    x = x != x ? -INFINITY : x;
    if (x > tv[K - 1] || ti[K - 1] == 0x7FFFFFFF) {   // a free slot, or better than the k-th
      tv[K - 1] = x;
      ti[K - 1] = e;
#pragma unroll
      for (int j = K - 1; j > 0; --j) {
        // bubble up past strictly smaller values (or free slots); an equal
        // value stays behind the lower expert id scanned before it
        if (tv[j] > tv[j - 1] || ti[j - 1] == 0x7FFFFFFF) {
          const float fv = tv[j];
          tv[j] = tv[j - 1];
          tv[j - 1] = fv;
          const int fi = ti[j];
          ti[j] = ti[j - 1];
          ti[j - 1] = fi;
        }
      }
    }
  }
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < K; ++j) sum += expf(tv[j] - tv[0]);
#pragma unroll
  for (int j = 0; j < K; ++j) {
    probs[(size_t)tt * K + j] = expf(tv[j] - tv[0]) / sum;
    topi[(size_t)tt * K + j] = ti[j];
    s_exp[tt * K + j] = ti[j];
  }
}

// grid (E, ceil(T / 8)): warp w of CTA (e, tb) computes logit[t = tb*8 + w][e]
__global__ void __launch_bounds__(kRouteThreads) moe_route_kernel(
    const __nv_bfloat16* __restrict__ h, const __nv_bfloat16* __restrict__ router, int T, int H, int E, int k,
    float* __restrict__ logits, float* __restrict__ probs, int64_t* __restrict__ topi, int32_t* __restrict__ counts,
    int32_t* __restrict__ offs, int32_t* __restrict__ tok, int64_t* __restrict__ pos, unsigned* __restrict__ ticket) {
  const int e = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.y * kRouteWarps + warp;
  // HV_MOE_OVERLAP_PREVIOUS: h is the previous kernel's output (no-op otherwise)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (t < T) {
    const uint4* hr = reinterpret_cast<const uint4*>(h + (size_t)t * H);
    const uint4* rr = reinterpret_cast<const uint4*>(router + (size_t)e * H);
    float acc = 0.f;
#pragma unroll 8
    for (int c = lane; c < H / 8; c += 32) {
      const uint4 a = __ldg(hr + c), b = __ldg(rr + c);
      acc = fmaf(bf16lo(a.x), bf16lo(b.x), acc);
      acc = fmaf(bf16hi(a.x), bf16hi(b.x), acc);
      acc = fmaf(bf16lo(a.y), bf16lo(b.y), acc);
      acc = fmaf(bf16hi(a.y), bf16hi(b.y), acc);
      acc = fmaf(bf16lo(a.z), bf16lo(b.z), acc);
      acc = fmaf(bf16hi(a.z), bf16hi(b.z), acc);
      acc = fmaf(bf16lo(a.w), bf16lo(b.w), acc);
      acc = fmaf(bf16hi(a.w), bf16hi(b.w), acc);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) logits[(size_t)t * E + e] = acc;
  }
  // the last CTA to finish does the per-token top-k and the pair sort
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ int s_cnt[kMaxE], s_off[kMaxE];
  __shared__ int s_exp[kMaxT * kMaxK];
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  // one thread per token: scan its E logits (L2, each row contiguous) keeping
  // the top k in registers; strict '>' keeps the lower expert first on ties
  // rows staged through shared memory in token chunks (coalesced loads; a
  // per-element scan of L2 would pay its latency E times per token)
  __shared__ float s_lg[kStageFloats];
  const int chunk = kStageFloats / E;   // E <= 256: at least 32 tokens per chunk
  for (int t0 = 0; t0 < T; t0 += chunk) {
    const int nt = min(chunk, T - t0);
    __syncthreads();
    for (int i = threadIdx.x; i < nt * E; i += blockDim.x) s_lg[i] = __ldcg(logits + (size_t)t0 * E + i);
    __syncthreads();
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
      const float* row = s_lg + j * E;
      const int tt = t0 + j;
      switch (k) {
        case 1: token_topk<1>(row, tt, E, probs, topi, s_exp); break;
        case 2: token_topk<2>(row, tt, E, probs, topi, s_exp); break;
        case 3: token_topk<3>(row, tt, E, probs, topi, s_exp); break;
        case 4: token_topk<4>(row, tt, E, probs, topi, s_exp); break;
        case 5: token_topk<5>(row, tt, E, probs, topi, s_exp); break;
        case 6: token_topk<6>(row, tt, E, probs, topi, s_exp); break;
        case 7: token_topk<7>(row, tt, E, probs, topi, s_exp); break;
        default: token_topk<8>(row, tt, E, probs, topi, s_exp); break;
      }
    }
  }
  __syncthreads();
  const int P = T * k;
  for (int p = threadIdx.x; p < P; p += blockDim.x) atomicAdd(&s_cnt[s_exp[p]], 1);   // integer: order-free
  __syncthreads();
  if (warp == 0) {   // exclusive scan of the counts
    int run = 0;
    for (int base = 0; base < E; base += 32) {
      const int i = base + lane;
      const int c = i < E ? s_cnt[i] : 0;
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (i < E) s_off[i] = run + x - c;
      run += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    counts[i] = s_cnt[i];
    offs[i] = s_off[i];
  }
  for (int p = threadIdx.x; p < P; p += blockDim.x) {   // stable: rank among earlier pairs of the same expert
    const int ex = s_exp[p];
    int r = 0;
#pragma unroll 8
    for (int q = 0; q < p; ++q) r += s_exp[q] == ex;
    const int sorted = s_off[ex] + r;
    pos[p] = sorted;
    tok[sorted] = p / k;
  }
  if (threadIdx.x == 0) *ticket = 0u;   // re-armed for the next launch / graph replay
}

// grid (T, H / (4 * threads)): h[t][d] = bf16(h + bf16(bf16(sum) * rs))
__global__ void __launch_bounds__(256) moe_combine_kernel(const float* __restrict__ y, const float* __restrict__ probs,
                                                          const int64_t* __restrict__ pos,
                                                          __nv_bfloat16* __restrict__ h, int H, int k, float rs,
                                                          int scaled) {
  const int t = blockIdx.x;
  asm volatile("griddepcontrol.wait;" ::: "memory");   // y: the previous kernel's output
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  float p[kMaxK];
  const float* rows[kMaxK];
#pragma unroll
  for (int j = 0; j < (int)kMaxK; ++j) {
    if (j < k) {
      p[j] = __ldg(probs + (size_t)t * k + j);
      rows[j] = y + (size_t)__ldg(pos + (size_t)t * k + j) * H;
    }
  }
  for (int d = (blockIdx.y * blockDim.x + threadIdx.x) * 4; d < H; d += gridDim.y * blockDim.x * 4) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < (int)kMaxK; ++j) {   // fixed order j = 0..k-1
      if (j < k) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(rows[j] + d));
        s.x = fmaf(v.x, p[j], s.x);
        s.y = fmaf(v.y, p[j], s.y);
        s.z = fmaf(v.z, p[j], s.z);
        s.w = fmaf(v.w, p[j], s.w);
      }
    }
    __nv_bfloat16* hp = h + (size_t)t * H + d;
    const float sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float m = __bfloat162float(__float2bfloat16_rn(sv[i]));
      if (scaled) m = __bfloat162float(__float2bfloat16_rn(m * rs));
      hp[i] = __float2bfloat16_rn(__bfloat162float(hp[i]) + m);
    }
  }
}

// one warp: stage = counts[e] > 0 && host[e]; rank = exclusive prefix of stage
__global__ void moe_stage_plan_kernel(const int32_t* __restrict__ counts, const uint64_t* __restrict__ addr,
                                      const uint8_t* __restrict__ host, uint64_t slot_base, uint64_t slot_bytes,
                                      int E, uint64_t* __restrict__ dst, uint64_t* __restrict__ sizes,
                                      uint64_t* __restrict__ addr_out) {
  const int lane = threadIdx.x;
  int run = 0;
  for (int base = 0; base < E; base += 32) {
    const int e = base + lane;
    const int st = e < E && counts[e] > 0 && host[e] != 0;
    int x = st;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (e < E) {
      const uint64_t d = st ? slot_base + (uint64_t)(run + x - 1) * slot_bytes : 0ull;
      dst[e] = d;
      sizes[e] = st ? slot_bytes : 0ull;
      addr_out[e] = st ? d : addr[e];
    }
    run += __shfl_sync(0xffffffffu, x, 31);
  }
}

}  // namespace

HV_EXPORT int hv_moe_stage_plan(const int32_t* d_counts, const uint64_t* d_addr, const uint8_t* d_host,
                                uint64_t slot_base, uint64_t slot_bytes, uint32_t n_experts, uint64_t* d_dst,
                                uint64_t* d_sizes, uint64_t* d_addr_out, void* stream) {
  if (n_experts == 0) return HV_OK;
  HV_CHECK_ARG(d_counts && d_addr && d_host && d_dst && d_sizes && d_addr_out && slot_bytes > 0);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  moe_stage_plan_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d_counts, d_addr, d_host, slot_base, slot_bytes,
                                                            (int)n_experts, d_dst, d_sizes, d_addr_out);
  HV_CUDA(cudaGetLastError());
  hv::note_launch(1);
  return HV_OK;
}

HV_EXPORT int hv_moe_route(const void* d_h, const void* d_router, uint32_t tokens, uint32_t hidden,
                           uint32_t n_experts, uint32_t top_k, float* d_logits, float* d_probs, int64_t* d_topi,
                           int32_t* d_counts, int32_t* d_offs, int32_t* d_tok, int64_t* d_pos, unsigned* d_ticket,
                           unsigned flags, void* stream) {
  if (tokens == 0) return HV_OK;
  HV_CHECK_ARG(d_h && d_router && d_logits && d_probs && d_topi && d_counts && d_offs && d_tok && d_pos && d_ticket);
  HV_CHECK_ARG(n_experts >= 1 && n_experts <= kMaxE && top_k >= 1 && top_k <= kMaxK && top_k <= n_experts);
  HV_CHECK_ARG(tokens <= kMaxT && hidden % 8 == 0 && hidden > 0);
  HV_CHECK_ARG(((reinterpret_cast<uintptr_t>(d_h) | reinterpret_cast<uintptr_t>(d_router)) & 15) == 0);
  HV_CHECK_ARG((flags & ~(unsigned)HV_MOE_OVERLAP_PREVIOUS) == 0);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_experts, (tokens + kRouteWarps - 1) / kRouteWarps);
  cfg.blockDim = dim3(kRouteThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (flags & HV_MOE_OVERLAP_PREVIOUS) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HV_CUDA(cudaLaunchKernelEx(&cfg, moe_route_kernel, reinterpret_cast<const __nv_bfloat16*>(d_h),
                             reinterpret_cast<const __nv_bfloat16*>(d_router), (int)tokens, (int)hidden,
                             (int)n_experts, (int)top_k, d_logits, d_probs, d_topi, d_counts, d_offs, d_tok, d_pos,
                             d_ticket));
  HV_CUDA(cudaGetLastError());
  hv::note_launch(1);
  return HV_OK;
}

HV_EXPORT int hv_moe_combine(const float* d_y, const float* d_probs, const int64_t* d_pos, void* d_h,
                             uint32_t tokens, uint32_t hidden, uint32_t top_k, float residual_scale, unsigned flags,
                             void* stream) {
  if (tokens == 0) return HV_OK;
  HV_CHECK_ARG(d_y && d_probs && d_pos && d_h);
  HV_CHECK_ARG(top_k >= 1 && top_k <= kMaxK && hidden % 4 == 0 && hidden > 0);
  HV_CHECK_ARG(((reinterpret_cast<uintptr_t>(d_y) | reinterpret_cast<uintptr_t>(d_h)) & 15) == 0);
  HV_CHECK_ARG((flags & ~(unsigned)HV_MOE_OVERLAP_PREVIOUS) == 0);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  const int threads = hidden / 4 < 256 ? (int)((hidden / 4 + 31) / 32 * 32) : 256;
  // one 16-byte column group per thread: (tokens, hidden / (4 * threads)) CTAs
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tokens, (hidden + 4 * threads - 1) / (4 * threads));
  cfg.blockDim = dim3(threads);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (flags & HV_MOE_OVERLAP_PREVIOUS) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HV_CUDA(cudaLaunchKernelEx(&cfg, moe_combine_kernel, d_y, d_probs, d_pos, reinterpret_cast<__nv_bfloat16*>(d_h),
                             (int)hidden, (int)top_k, residual_scale, residual_scale != 1.0f ? 1 : 0));
  HV_CUDA(cudaGetLastError());
  hv::note_launch(1);
  return HV_OK;
}
