// Fetch kernels of the B200 Harvest data plane (sm_100a).
//
// The reference never moves bytes: a fetch is `fixed_cost + size/bandwidth`
// (interconnect.py:51-54), serialized FIFO per device pair
// (interconnect.py:147-150) and issued one object at a time by
// HarvestRuntime.app_transfer (runtime.py:320-364) from the MoE stage loop
// (moe.py:282-313) or the KV reload path.  Here one launch
// moves a whole batch (every page of a decode step/layer, every expert of a
// pipeline stage), with all objects in flight at once.
//
// Work decomposition (shared by every engine and op): each object is cut into
// fixed-size chunks; chunk c of the flattened batch is handled by one warp
// (LDG engine, 4 KiB chunks) or one CTA pipeline slot (TMA engine, 16 KiB
// chunks).  Objects are either uniform pages (chunk -> page by division) or
// variable-size descriptors (chunk -> object through a per-CTA shared-memory
// prefix of chunk counts).
//
// LDG engine: every lane front-batches 8 x 128-bit `ld.global.nc.L1::no_allocate`
// (4 KiB per warp in flight) then streams them out with `st.global.L1::no_allocate`.
// Peer loads through NVLink bypass the local L2 and take ~2 us, so the bytes
// in flight per SM, not instruction issue, set the rate (Little's law).
// TMA engine: one lane per CTA drives a ring of shared-memory stages with
// `cp.async.bulk` global->smem (mbarrier complete_tx) and smem->global
// (bulk_group), so a handful of CTAs keep megabytes in flight while leaving the
// SMs' issue slots to decode compute.
#include <atomic>
#include <string.h>
#include <type_traits>
#include <mutex>
#include <vector>

#include "hv_common.h"

namespace hv {

static std::atomic<uint64_t> g_launches{0};
void note_launch(uint64_t n) { g_launches += n; }

int bind_stream_device(void* stream, int* device_out, DeviceGuard& g) {
  int dev = 0;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (stream && cudaStreamIsCapturing((cudaStream_t)stream, &cap) != cudaSuccess) {
    (void)cudaGetLastError();
    cap = cudaStreamCaptureStatusNone;
  }
  if (stream && cap == cudaStreamCaptureStatusNone) {
    cudaError_t e = cudaStreamGetDevice((cudaStream_t)stream, &dev);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      return hv_cuda_status(e);
    }
  } else {
    // legacy stream, or a stream under CUDA-graph capture: cudaStreamGetDevice
    // invalidates a capture, and a capturing stream belongs to the current device
    HV_CUDA(cudaGetDevice(&dev));
  }
  int st = g.set(dev);
  if (st) return st;
  if (device_out) *device_out = dev;
  return HV_OK;
}

int sm_count(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
      (void)cudaGetLastError();
      n = 148;
    }
    cache[device] = n;
  }
  return cache[device];
}

}  // namespace hv

namespace {

// ---------------------------------------------------------------------------
// constants
constexpr int kLdgThreads = 512;                 // 16 warps per CTA
constexpr int kLdgUnroll = 8;                    // 128-bit loads in flight per lane
constexpr uint32_t kLdgChunk = kLdgUnroll * 32 * 16;  // 4 KiB per warp iteration
constexpr int kTmaThreads = 32;                  // one warp; lane 0 issues
constexpr uint32_t kTmaChunk = 16384;            // bytes per bulk copy
constexpr int kTmaStages = 8;                    // 128 KiB of smem ring per CTA
constexpr uint32_t kMaxSmemDescs = 2048;         // variable-size descriptors per launch
// DescResolver shared memory: chunk-start prefix [n+1], the interleave order
// of the active descriptors [kMaxSmemDescs], and 4 words of mode data
constexpr uint32_t kDescActOff = kMaxSmemDescs + 1;
constexpr uint32_t kDescMetaOff = 2 * kMaxSmemDescs + 1;
constexpr uint32_t kDescSmemWords = 2 * kMaxSmemDescs + 8;
constexpr int kEngineInterleave = HV_ENGINE_FLAG_INTERLEAVE;  // round-robin chunks over objects
constexpr uint32_t kPageBatchMax = 1u << 30;

// splitmix64 (Steele, Lea, Flood 2014) — the synthetic content generator; the
// seed is stable_hash64(tag) (runtime.py:38-44, moe.py:114-115).
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint32_t kDigestKeyA = 0x9E3779B1u, kDigestKeyB = 0x85EBCA77u, kDigestKeyC = 0xC2B2AE3Du;

__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t content_word(uint64_t seed, uint64_t i) {
  return fmix64(seed + (i + 1) * kGolden);
}
// Content digest term of 8-byte word i (oracle hvo_digest): an NH-style
// product (Black et al., UMAC, CRYPTO 1999) of the word's two 32-bit halves,
// each offset by a position key, exact in 64 bits.  A changed word changes its
// term unless the other half's keyed value is 0 (probability 2^-32); the
// digest is size + the sum of the terms mod 2^64.  ~6 instructions per word
// (two IMAD, one IMAD.WIDE.U32, a 64-bit add) where a 64-bit finalizer took
// ~25 and left the content check ALU-bound (ncu r5n: ALU pipe 61% at 3.7 TB/s).
__host__ __device__ __forceinline__ uint64_t digest_term(uint64_t i, uint64_t w) {
  const uint32_t j = (uint32_t)(i + 1);
  const uint32_t a = (uint32_t)w + j * kDigestKeyA;
  const uint32_t b = (uint32_t)(w >> 32) + j * kDigestKeyB + kDigestKeyC;
  return (uint64_t)a * (uint64_t)b;
}

// ---------------------------------------------------------------------------
// memory primitives
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// same load with an L2 256-byte sector-promotion hint: the L2 fetches whole
// 256 B blocks, i.e. larger read requests over PCIe / NVLink
__device__ __forceinline__ uint4 ld_stream256(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
template <bool kL2Hint>
__device__ __forceinline__ uint4 ld_src(const void* p) {
  if constexpr (kL2Hint) return ld_stream256(p);
  else return ld_stream(p);
}
__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// ---------------------------------------------------------------------------
// chunk resolvers: chunk index -> (src, dst, len, object index, offset)
struct ChunkRef {
  const char* src;
  char* dst;
  uint32_t len;
  uint32_t obj;
  uint64_t off;
};

// Uniform pages (K1).  kTable: src = slot_bases[loc>>32] + (loc&0xffffffff)*page.
template <bool kTable>
struct PageResolver {
  const uint64_t* src;      // per-page pointers, or slot bases (kTable)
  const uint64_t* locs;     // kTable only
  const uint64_t* dst_ptrs; // nullable
  uint64_t dst_base;
  uint64_t page_bytes;
  uint32_t chunks_per_page;
  uint32_t n_pages;
  uint32_t chunk;
  uint32_t interleave;      // HV_ENGINE_FLAG_INTERLEAVE: chunk c reads page c % n at chunk c / n

  __device__ __forceinline__ uint32_t setup(void*) const { return n_pages * chunks_per_page; }
  __device__ __forceinline__ ChunkRef at(uint32_t c, uint32_t& hint) const {
    (void)hint;
    uint32_t page, ci;
    if (interleave) {
      ci = c / n_pages;
      page = c - ci * n_pages;
    } else {
      page = c / chunks_per_page;
      ci = c - page * chunks_per_page;
    }
    uint64_t s;
    if (kTable) {
      const uint64_t loc = __ldg(locs + page);
      s = __ldg(src + (loc >> 32)) + (loc & 0xffffffffull) * page_bytes;
    } else {
      s = __ldg(src + page);
    }
    const uint64_t d = dst_ptrs ? __ldg(dst_ptrs + page) : dst_base + (uint64_t)page * page_bytes;
    ChunkRef r;
    r.off = (uint64_t)ci * chunk;
    const uint64_t rem = page_bytes - r.off;
    r.len = rem < chunk ? (uint32_t)rem : chunk;
    r.src = reinterpret_cast<const char*>(s) + r.off;
    r.dst = reinterpret_cast<char*>(d) + r.off;
    r.obj = page;
    return r;
  }
};

// Strided block pages (K1 over a block table, the layout of a paged KV cache):
// page p = l * n_blocks + b (layer-major), with
//   src = src_base[b] + l * src_stride[b],  dst = dst_base[b] + l * dst_stride[b].
// Four n_blocks-long arrays describe n_blocks * n_layers pages.
struct BlockResolver {
  const uint64_t* src_base;
  const uint64_t* src_stride;
  const uint64_t* dst_base;
  const uint64_t* dst_stride;
  uint64_t page_bytes;
  uint32_t chunks_per_page;
  uint32_t n_blocks;
  uint32_t n_layers;
  uint32_t chunk;

  __device__ __forceinline__ uint32_t setup(void*) const { return n_blocks * n_layers * chunks_per_page; }
  __device__ __forceinline__ ChunkRef at(uint32_t c, uint32_t& hint) const {
    (void)hint;
    const uint32_t page = c / chunks_per_page;
    const uint32_t ci = c - page * chunks_per_page;
    const uint32_t l = page / n_blocks;
    const uint32_t b = page - l * n_blocks;
    const uint64_t s = __ldg(src_base + b) + (uint64_t)l * __ldg(src_stride + b);
    const uint64_t d = __ldg(dst_base + b) + (uint64_t)l * __ldg(dst_stride + b);
    ChunkRef r;
    r.off = (uint64_t)ci * chunk;
    const uint64_t rem = page_bytes - r.off;
    r.len = rem < chunk ? (uint32_t)rem : chunk;
    r.src = reinterpret_cast<const char*>(s) + r.off;
    r.dst = reinterpret_cast<char*>(d) + r.off;
    r.obj = page;
    return r;
  }
};

// Variable-size descriptors (K2).  The per-CTA prefix of chunk counts lives
// in shared memory; a warp's successive chunks are monotone in c, so the
// object index is found by a short forward probe before falling back to
// binary search.
//
// Interleaved mode (engine flag kEngineInterleave, used when every non-empty
// object has the same size, e.g. the experts of a stage): chunk c reads
// object active[c % n_active] at chunk c / n_active, so the bytes in flight at
// any moment come from every object of the batch at once -- with objects
// spread over several donor GPUs, every donor's NVLink egress is busy instead
// of the readers of a multi-GPU node converging on one or two donors.
struct DescResolver {
  const uint64_t* src;
  const uint64_t* dst;
  const uint64_t* bytes;
  uint32_t n;
  uint32_t chunk;
  uint32_t interleave;

  // smem must hold kDescSmemWords words; all threads of the CTA call setup().
  __device__ uint32_t setup(void* smem) const {
    uint32_t* s_start = reinterpret_cast<uint32_t*>(smem);
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_total;
    __shared__ unsigned long long s_szmin, s_szmax;
    const uint32_t nt = blockDim.x, tid = threadIdx.x;
    const uint32_t lane = tid & 31, warp = tid >> 5, nwarps = (nt + 31) >> 5;
    const uint32_t per = (n + nt - 1) / nt;
    const uint32_t i0 = tid * per;
    if (interleave) {
      if (tid == 0) {
        s_szmin = ~0ull;
        s_szmax = 0;
      }
      __syncthreads();
    }
    uint32_t local = 0;
    unsigned long long szmin = ~0ull, szmax = 0;
    for (uint32_t k = 0; k < per; ++k) {
      const uint32_t i = i0 + k;
      if (i < n) {
        const uint64_t sz = __ldg(bytes + i);
        const uint32_t cnt = (uint32_t)((sz + chunk - 1) / chunk);
        s_start[i] = cnt;
        local += cnt;
        if (sz) {
          szmin = sz < szmin ? sz : szmin;
          szmax = sz > szmax ? sz : szmax;
        }
      }
    }
    if (interleave && szmax) {
      atomicMin(&s_szmin, szmin);
      atomicMax(&s_szmax, szmax);
    }
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t w = lane < nwarps ? s_warp[lane] : 0;
      uint32_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= (uint32_t)o) wi += t;
      }
      if (lane < nwarps) s_warp[lane] = wi - w;
      if (lane == 31) s_total = wi;
    }
    __syncthreads();
    uint32_t run = s_warp[warp] + incl - local;
    for (uint32_t k = 0; k < per; ++k) {
      const uint32_t i = i0 + k;
      if (i < n) {
        const uint32_t cnt = s_start[i];
        s_start[i] = run;
        run += cnt;
      }
    }
    if (tid == 0) s_start[n] = s_total;
    // interleaved order: only for equal-size non-empty objects
    const bool il = interleave && s_szmax != 0 && s_szmin == s_szmax;
    uint32_t* meta = s_start + kDescMetaOff;
    if (il) {
      const uint32_t cpd = (uint32_t)((s_szmax + chunk - 1) / chunk);
      uint32_t* act = s_start + kDescActOff;
      for (uint32_t k = 0; k < per; ++k) {
        const uint32_t i = i0 + k;
        if (i < n && __ldg(bytes + i)) act[s_start[i] / cpd] = i;
      }
      if (tid == 0) {
        meta[0] = 1;
        meta[1] = s_total / cpd;                  // active objects
        meta[2] = (uint32_t)s_szmax;              // their size (low, high words)
        meta[3] = (uint32_t)(s_szmax >> 32);
      }
    } else if (tid == 0) {
      meta[0] = 0;
    }
    __syncthreads();
    return s_total;
  }

  __device__ __forceinline__ ChunkRef at(uint32_t c, uint32_t& hint, const uint32_t* s_start) const {
    const uint32_t* meta = s_start + kDescMetaOff;
    if (meta[0]) {
      const uint32_t nact = meta[1];
      const uint32_t k = c / nact;
      const uint32_t i = s_start[kDescActOff + (c - k * nact)];
      const uint64_t size = (uint64_t)meta[2] | ((uint64_t)meta[3] << 32);
      ChunkRef r;
      r.obj = i;
      r.off = (uint64_t)k * chunk;
      const uint64_t rem = size - r.off;
      r.len = rem < chunk ? (uint32_t)rem : chunk;
      r.src = reinterpret_cast<const char*>(__ldg(src + i)) + r.off;
      r.dst = reinterpret_cast<char*>(__ldg(dst + i)) + r.off;
      return r;
    }
    uint32_t lo = hint;
    if (!(s_start[lo] <= c && c < s_start[lo + 1])) {
      if (lo + 2 <= n && s_start[lo + 1] <= c && c < s_start[lo + 2]) {
        lo = lo + 1;
      } else {
        uint32_t l = 0, h = n;  // s_start[l] <= c < s_start[h]
        while (h - l > 1) {
          const uint32_t m = (l + h) >> 1;
          if (s_start[m] <= c) l = m; else h = m;
        }
        lo = l;
      }
    }
    hint = lo;
    ChunkRef r;
    r.obj = lo;
    r.off = (uint64_t)(c - s_start[lo]) * chunk;
    const uint64_t rem = __ldg(bytes + lo) - r.off;
    r.len = rem < chunk ? (uint32_t)rem : chunk;
    r.src = reinterpret_cast<const char*>(__ldg(src + lo)) + r.off;
    r.dst = reinterpret_cast<char*>(__ldg(dst + lo)) + r.off;
    return r;
  }
};

// ---------------------------------------------------------------------------
// per-chunk operations (warp-cooperative)

template <bool kL2Hint = false, int kUnroll = kLdgUnroll>
__device__ __forceinline__ void copy_chunk_ldg(const ChunkRef& r, uint32_t lane) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(r.src) | reinterpret_cast<uintptr_t>(r.dst)) & 15) == 0;
  if (aligned && r.len == (uint32_t)kUnroll * 512u) {
    uint4 v[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) v[j] = ld_src<kL2Hint>(r.src + (j * 32 + lane) * 16);
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) st_stream(r.dst + (j * 32 + lane) * 16, v[j]);
    return;
  }
  uint32_t done = 0;
  if (aligned) {
    const uint32_t nvec = r.len >> 4;
    for (uint32_t v = lane; v < nvec; v += 32) st_stream(r.dst + v * 16, ld_src<kL2Hint>(r.src + v * 16));
    done = nvec << 4;
  }
  for (uint32_t b = done + lane; b < r.len; b += 32) r.dst[b] = r.src[b];
}

// generic warp-per-chunk driver
template <typename Res, typename Op>
__device__ __forceinline__ void warp_loop(const Res& res, uint32_t total, Op op, const uint32_t* smem) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t wpb = blockDim.x >> 5;
  const uint32_t nwarps = gridDim.x * wpb;
  uint32_t hint = 0;
  for (uint32_t c = blockIdx.x * wpb + (threadIdx.x >> 5); c < total; c += nwarps) {
    ChunkRef r;
    if constexpr (std::is_same<Res, DescResolver>::value) r = res.at(c, hint, smem);
    else r = res.at(c, hint);
    op(r, lane);
  }
}

template <bool kL2Hint, int kUnroll = kLdgUnroll>
struct CopyOpT {
  __device__ __forceinline__ void operator()(const ChunkRef& r, uint32_t lane) const {
    copy_chunk_ldg<kL2Hint, kUnroll>(r, lane);
  }
};
using CopyOp = CopyOpT<false>;
// deeper engine: 16 x 128-bit loads in flight per lane (8 KiB per warp), for
// links whose latency needs more bytes in flight per SM than LDG's 4 KiB
constexpr int kLdgDeepUnroll = 16;
constexpr uint32_t kLdgDeepChunk = kLdgDeepUnroll * 512;

// content ops work on 8-byte words; objects must start 8-byte aligned
// kind 0: raw splitmix64 bytes.  kind 1: bf16 weights — every 16-bit lane of
// the word keeps its sign and 7 mantissa bits with the exponent fixed at 2^-7,
// i.e. |w| in [2^-7, 2^-6): finite, small, still a keyed pseudo-random stream.
__host__ __device__ __forceinline__ uint64_t weights_word(uint64_t w) {
  return (w & 0x807F807F807F807Full) | 0x3C003C003C003C00ull;
}

struct FillOp {
  const uint64_t* seeds;
  uint32_t kind;
  __device__ __forceinline__ uint64_t word(uint64_t seed, uint64_t i) const {
    const uint64_t w = content_word(seed, i);
    return kind ? weights_word(w) : w;
  }
  __device__ __forceinline__ void operator()(const ChunkRef& r, uint32_t lane) const {
    const uint64_t seed = __ldg(seeds + r.obj);
    const uint64_t w0 = r.off >> 3;
    const uint32_t nfull = r.len >> 3;
    uint64_t* d = reinterpret_cast<uint64_t*>(r.dst);
    for (uint32_t k = lane; k < nfull; k += 32) d[k] = word(seed, w0 + k);
    const uint32_t tail = r.len & 7;
    if (tail && lane == 0) {
      const uint64_t w = word(seed, w0 + nfull);
      for (uint32_t b = 0; b < tail; ++b) r.dst[nfull * 8 + b] = (char)((w >> (8 * b)) & 0xff);
    }
  }
};

__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint64_t load_word_tail(const char* p, uint32_t n) {
  uint64_t w = 0;
  for (uint32_t b = 0; b < n; ++b) w |= (uint64_t)(uint8_t)p[b] << (8 * b);
  return w;
}

struct DigestOp {
  const uint64_t* bytes;  // for the size term
  unsigned long long* out;
  __device__ __forceinline__ void operator()(const ChunkRef& r, uint32_t lane) const {
    const uint64_t w0 = r.off >> 3;
    uint64_t acc = 0;
    if ((reinterpret_cast<uintptr_t>(r.src) & 15) == 0 && r.len == (uint32_t)kLdgUnroll * 512u) {
      // a whole chunk: every lane's 128-bit loads in flight before any
      // digest arithmetic (the 8-byte loop below leaves one load per lane in
      // flight and stalls on it -- ncu r5c: long-scoreboard stalls dominant)
      uint4 v[kLdgUnroll];
#pragma unroll
      for (int j = 0; j < kLdgUnroll; ++j) v[j] = ld_stream(r.src + (j * 32 + lane) * 16);
#pragma unroll
      for (int j = 0; j < kLdgUnroll; ++j) {
        const uint64_t i = w0 + (uint64_t)(j * 32 + lane) * 2;
        acc += digest_term(i, (uint64_t)v[j].x | ((uint64_t)v[j].y << 32));
        acc += digest_term(i + 1, (uint64_t)v[j].z | ((uint64_t)v[j].w << 32));
      }
    } else {
      const uint32_t nfull = r.len >> 3;
      const uint64_t* s = reinterpret_cast<const uint64_t*>(r.src);
      for (uint32_t k = lane; k < nfull; k += 32) acc += digest_term(w0 + k, s[k]);
      const uint32_t tail = r.len & 7;
      if (tail && lane == 0) acc += digest_term(w0 + nfull, load_word_tail(r.src + nfull * 8, tail));
    }
    if (r.off == 0 && lane == 0) acc += __ldg(bytes + r.obj);
    acc = warp_sum(acc);
    if (lane == 0) atomicAdd(out + r.obj, (unsigned long long)acc);
  }
};

struct VerifyOp {
  const uint64_t* seeds;
  unsigned long long* out;
  uint32_t kind;  // as FillOp::kind
  __device__ __forceinline__ uint64_t word(uint64_t seed, uint64_t i) const {
    const uint64_t w = content_word(seed, i);
    return kind ? weights_word(w) : w;
  }
  __device__ __forceinline__ void operator()(const ChunkRef& r, uint32_t lane) const {
    const uint64_t seed = __ldg(seeds + r.obj);
    const uint64_t w0 = r.off >> 3;
    const uint32_t nfull = r.len >> 3;
    const uint64_t* s = reinterpret_cast<const uint64_t*>(r.src);
    uint64_t bad = 0;
    for (uint32_t k = lane; k < nfull; k += 32) bad += (s[k] != word(seed, w0 + k));
    const uint32_t tail = r.len & 7;
    if (tail && lane == 0) {
      const uint64_t mask = (1ull << (8 * tail)) - 1;
      bad += ((load_word_tail(r.src + nfull * 8, tail) ^ word(seed, w0 + nfull)) & mask) != 0;
    }
    bad = warp_sum(bad);
    if (lane == 0 && bad) atomicAdd(out + r.obj, (unsigned long long)bad);
  }
};

// ---------------------------------------------------------------------------
// LDG-engine kernels

template <bool kTable, bool kL2Hint, int kUnroll = kLdgUnroll>
__global__ void __launch_bounds__(kLdgThreads) page_copy_ldg(PageResolver<kTable> res) {
  const uint32_t total = res.setup(nullptr);
  warp_loop(res, total, CopyOpT<kL2Hint, kUnroll>{}, nullptr);
}

template <typename Op>
__global__ void __launch_bounds__(kLdgThreads) desc_op_kernel(DescResolver res, Op op) {
  __shared__ uint32_t s_start[kDescSmemWords];
  const uint32_t total = res.setup(s_start);
  warp_loop(res, total, op, s_start);
}

// ---------------------------------------------------------------------------
// TMA (bulk-copy) engine

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "HV_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra HV_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ bool tma_ok(const ChunkRef& r) {
  return ((reinterpret_cast<uintptr_t>(r.src) | reinterpret_cast<uintptr_t>(r.dst) | r.len) & 15) == 0 && r.len > 0;
}

// One warp per CTA.  Chunks b, b+G, b+2G... of the batch flow through a ring
// of kTmaStages shared-memory stages: load k+S-1 is in flight while chunk k is
// stored.  Irregular chunks (unaligned or len % 16) are copied by the warp.
template <typename Res>
__device__ __forceinline__ void tma_loop(const Res& res, uint32_t total, const uint32_t* s_desc,
                                         char* ring, uint64_t* bars) {
  const uint32_t lane = threadIdx.x & 31;
  if (lane == 0) {
    for (int s = 0; s < kTmaStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint32_t G = gridDim.x;
  const uint32_t mine = blockIdx.x < total ? (total - blockIdx.x + G - 1) / G : 0;
  uint32_t hint_issue = 0, hint_store = 0;
  auto chunk_of = [&](uint32_t t, uint32_t& hint) -> ChunkRef {
    const uint32_t c = blockIdx.x + t * G;
    if constexpr (std::is_same<Res, DescResolver>::value) return res.at(c, hint, s_desc);
    else return res.at(c, hint);
  };
  // prologue: fill the ring
  const uint32_t pro = mine < (uint32_t)kTmaStages ? mine : (uint32_t)kTmaStages;
  for (uint32_t t = 0; t < pro; ++t) {
    const ChunkRef r = chunk_of(t, hint_issue);
    if (tma_ok(r) && lane == 0) {
      mbar_expect_tx(&bars[t], r.len);
      bulk_g2s(ring + (size_t)t * kTmaChunk, r.src, r.len, &bars[t]);
    }
  }
  uint32_t next_issue = pro;
  for (uint32_t t = 0; t < mine; ++t) {
    const uint32_t stage = t % kTmaStages;
    const uint32_t parity = (t / kTmaStages) & 1;
    const ChunkRef r = chunk_of(t, hint_store);
    if (tma_ok(r)) {
      mbar_wait(&bars[stage], parity);
      if (lane == 0) bulk_s2g(r.dst, ring + (size_t)stage * kTmaChunk, r.len);
    } else {
      copy_chunk_ldg(r, lane);  // generic path; stage stays unused this round
      if (lane == 0) {          // keep the barrier phase sequence regular
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bars[stage])) : "memory");
      }
      mbar_wait(&bars[stage], parity);
    }
    // one bulk group per iteration (possibly empty) so that wait_group.read<1>
    // below always means "the store of chunk t-1 has finished reading smem"
    if (lane == 0) bulk_commit();
    // refill the stage consumed one iteration ago once its store has read smem
    if (next_issue < mine && t >= 1) {
      const uint32_t rs = (t - 1) % kTmaStages;
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
      const ChunkRef n = chunk_of(next_issue, hint_issue);
      if (tma_ok(n) && lane == 0) {
        mbar_expect_tx(&bars[rs], n.len);
        bulk_g2s(ring + (size_t)rs * kTmaChunk, n.src, n.len, &bars[rs]);
      }
      ++next_issue;
    }
    __syncwarp();
  }
  if (lane == 0) bulk_wait_all();
  __syncwarp();
}

// NOTE on the refill order: chunk t+S-1 goes into stage (t-1)%S, which is the
// stage chunk t-1 used; chunk index t' always maps to stage t'%S because
// next_issue == t-1+S at that point (prologue issued S chunks, one refill per
// iteration from t=1 on), so (t-1)%S == next_issue%S.

template <bool kTable>
__global__ void __launch_bounds__(kTmaThreads) page_copy_tma(PageResolver<kTable> res) {
  extern __shared__ __align__(128) char dyn_smem[];
  __shared__ __align__(8) uint64_t bars[kTmaStages];
  const uint32_t total = res.setup(nullptr);
  tma_loop(res, total, nullptr, dyn_smem, bars);
}

__global__ void __launch_bounds__(kTmaThreads) block_copy_tma(BlockResolver res) {
  extern __shared__ __align__(128) char dyn_smem[];
  __shared__ __align__(8) uint64_t bars[kTmaStages];
  const uint32_t total = res.setup(nullptr);
  tma_loop(res, total, nullptr, dyn_smem, bars);
}

template <bool kL2Hint, int kUnroll>
__global__ void __launch_bounds__(kLdgThreads) block_copy_ldg(BlockResolver res) {
  const uint32_t total = res.setup(nullptr);
  warp_loop(res, total, CopyOpT<kL2Hint, kUnroll>{}, nullptr);
}

__global__ void __launch_bounds__(kTmaThreads) desc_copy_tma(DescResolver res) {
  extern __shared__ __align__(128) char dyn_smem[];
  __shared__ __align__(8) uint64_t bars[kTmaStages];
  __shared__ uint32_t s_start[kDescSmemWords];
  const uint32_t total = res.setup(s_start);
  tma_loop(res, total, s_start, dyn_smem, bars);
}

constexpr size_t kTmaSmem = (size_t)kTmaStages * kTmaChunk;

// Content check (DigestOp) on the TMA engine: lane 0 of a producer warp
// streams the CTA's chunks into a ring of shared-memory stages with bulk
// copies; each consumer warp digests whole chunks (chunk t of the CTA goes to
// warp t mod W) from shared memory -- a lane's 16-byte units are contiguous
// across the warp, conflict-free LDS.128, many independent units per lane --
// and releases the stage.  The loads no longer wait behind the digest
// arithmetic of the same warp (the LDG form's limit: ncu r5c, long-scoreboard
// stalls, 3.4 TB/s).  Each warp keeps its running sum per object in a
// register and adds it to the object's accumulator when the object changes.
// Same digest as DigestOp, bit for bit.  Splitting every chunk over all
// consumer warps (r5n-r5p) was slower: 8 / 12 / 16 warps 0.213 / 0.268 /
// 0.306 ms per Qwen stage -- the per-chunk resolve, barrier and reduction
// then dominate.
#ifndef HV_DG_CONSUMERS
#define HV_DG_CONSUMERS 6
#endif
#ifndef HV_DG_STAGES
#define HV_DG_STAGES 6
#endif
#ifndef HV_DG_CHUNK
#define HV_DG_CHUNK 16384
#endif
constexpr int kDgConsumers = HV_DG_CONSUMERS;
constexpr int kDgThreads = (kDgConsumers + 1) * 32;
constexpr int kDgStages = HV_DG_STAGES;
constexpr uint32_t kDgChunk = HV_DG_CHUNK;
constexpr size_t kDgSmem = (size_t)kDgStages * kDgChunk;
// chunk t and chunk t + S share a stage; with S a multiple of W they also
// share the consumer warp, which has therefore seen the stage's previous
// phase complete before it waits on the next one (an mbarrier parity wait
// cannot tell phase r from phase r - 2: measured as launch failures with
// W = 4, S = 6 and W = 8, S = 12)
static_assert(kDgStages % kDgConsumers == 0, "digest ring: stages must be a multiple of the consumer warps");

__global__ void __launch_bounds__(kDgThreads) desc_digest_tma(DescResolver res, const uint64_t* __restrict__ bytes,
                                                              unsigned long long* __restrict__ out) {
  extern __shared__ __align__(128) char ring[];
  __shared__ __align__(8) uint64_t full[kDgStages], empty[kDgStages];
  __shared__ uint32_t s_start[kDescSmemWords];
  const uint32_t total = res.setup(s_start);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kDgStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 32);   // every lane of the consuming warp releases its own reads
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t G = gridDim.x;
  const uint32_t mine = blockIdx.x < total ? (total - blockIdx.x + G - 1) / G : 0;
  if (warp == kDgConsumers) {   // producer
    if (lane == 0) {
      uint32_t hint = 0;
      for (uint32_t t = 0; t < mine; ++t) {
        const uint32_t st = t % kDgStages, round = t / kDgStages;
        if (round > 0) {
          mbar_wait(&empty[st], (round - 1) & 1);
          // the consumer's generic-proxy reads of this stage, ordered before
          // the bulk copy's async-proxy writes into it
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        const ChunkRef r = res.at(blockIdx.x + t * G, hint, s_start);
        if (tma_ok(r)) {
          mbar_expect_tx(&full[st], r.len);
          bulk_g2s(ring + (size_t)st * kDgChunk, r.src, r.len, &full[st]);
        } else {   // digested from global by its consumer; keep the phase sequence
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[st])) : "memory");
        }
      }
    }
    return;
  }
  uint32_t hint = 0, cur_obj = 0xFFFFFFFFu;
  uint64_t run = 0;
  for (uint32_t t = warp; t < mine; t += kDgConsumers) {
    const uint32_t st = t % kDgStages;
    const ChunkRef r = res.at(blockIdx.x + t * G, hint, s_start);
    mbar_wait(&full[st], (t / kDgStages) & 1);
    const uint64_t w0 = r.off >> 3;
    uint64_t acc = 0;
    if (tma_ok(r)) {
      const char* sb = ring + (size_t)st * kDgChunk;
#pragma unroll 8
      for (uint32_t u = lane; u < r.len / 16; u += 32) {
        const uint4 v = *reinterpret_cast<const uint4*>(sb + (size_t)u * 16);
        const uint64_t i = w0 + (uint64_t)u * 2;
        acc += digest_term(i, (uint64_t)v.x | ((uint64_t)v.y << 32));
        acc += digest_term(i + 1, (uint64_t)v.z | ((uint64_t)v.w << 32));
      }
    } else {
      const uint32_t nfull = r.len >> 3;
      for (uint32_t k = lane; k < nfull; k += 32) {
        uint64_t w = 0;
        memcpy(&w, r.src + (size_t)k * 8, 8);
        acc += digest_term(w0 + k, w);
      }
      const uint32_t tail = r.len & 7;
      if (tail && lane == 0) acc += digest_term(w0 + nfull, load_word_tail(r.src + nfull * 8, tail));
    }
    if (r.off == 0 && lane == 0) acc += __ldg(bytes + r.obj);
    // release: each lane's generic-proxy reads of the stage, ordered before the
    // producer's next bulk (async-proxy) write into it.  Every lane arrives
    // (a lane-0 arrive after __syncwarp is the same ordering, but racecheck
    // reports it as a write-after-read hazard: build/rc repro, r5y)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    if (r.obj != cur_obj) {
      if (cur_obj != 0xFFFFFFFFu) {
        const uint64_t tot = warp_sum(run);
        if (lane == 0) atomicAdd(out + cur_obj, (unsigned long long)tot);
      }
      cur_obj = r.obj;
      run = 0;
    }
    run += acc;
  }
  if (cur_obj != 0xFFFFFFFFu) {
    const uint64_t tot = warp_sum(run);
    if (lane == 0) atomicAdd(out + cur_obj, (unsigned long long)tot);
  }
}

#ifndef HV_DIGEST_TMA
#define HV_DIGEST_TMA 1
#endif

// ---------------------------------------------------------------------------
// launch helpers

// Device-array entry points run on the SMs: AUTO -- and CE, which needs host
// descriptors -- mean the LDG kernel there.
int pick_engine(int engine) { return (engine == HV_ENGINE_AUTO || engine == HV_ENGINE_CE) ? HV_ENGINE_LDG : engine; }

constexpr uint64_t kUnknownChunks = ~0ull;  // device-resident sizes: fill the device

int ldg_grid(int dev, uint64_t chunks, int max_ctas) {
  const uint64_t wpb = kLdgThreads / 32;
  uint64_t g = (uint64_t)hv::sm_count(dev) * (2048 / kLdgThreads);  // full occupancy
  if (chunks != kUnknownChunks) {
    const uint64_t need = chunks / wpb + (chunks % wpb != 0);
    if (need < g) g = need;
  }
  if (max_ctas > 0 && g > (uint64_t)max_ctas) g = (uint64_t)max_ctas;
  return (int)(g < 1 ? 1 : g);
}

int tma_grid(int dev, uint64_t chunks, int max_ctas) {
  uint64_t g = (uint64_t)hv::sm_count(dev);  // 128 KiB ring: one CTA per SM
  if (chunks != kUnknownChunks && chunks < g) g = chunks;
  if (max_ctas > 0 && g > (uint64_t)max_ctas) g = (uint64_t)max_ctas;
  return (int)(g < 1 ? 1 : g);
}

int set_tma_attrs(int dev) {
  const int smem = (int)kTmaSmem;
  const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
  int st = hv::kernel_attr<page_copy_tma<false>>(dev, a, smem);
  if (!st) st = hv::kernel_attr<page_copy_tma<true>>(dev, a, smem);
  if (!st) st = hv::kernel_attr<desc_copy_tma>(dev, a, smem);
  if (!st) st = hv::kernel_attr<block_copy_tma>(dev, a, smem);
  return st;
}

template <bool kTable>
int launch_pages(PageResolver<kTable> res, int engine, int max_ctas, void* stream) {
  if (res.n_pages == 0 || res.page_bytes == 0) return HV_OK;  // empty: no device work, no device needed
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  res.interleave = (engine & kEngineInterleave) ? 1u : 0u;   // explicit flag only (AUTO pages stay linear)
  engine = pick_engine(engine & ~kEngineInterleave);
  if (engine == HV_ENGINE_TMA) {
    if ((st = set_tma_attrs(dev))) return st;
    res.chunk = kTmaChunk;
    res.chunks_per_page = (uint32_t)((res.page_bytes + kTmaChunk - 1) / kTmaChunk);
    const uint64_t total = (uint64_t)res.n_pages * res.chunks_per_page;
    if (total >= 0xffffffffull) return HV_E_INVALID;
    page_copy_tma<kTable><<<tma_grid(dev, total, max_ctas), kTmaThreads, kTmaSmem, (cudaStream_t)stream>>>(res);
  } else if (engine == HV_ENGINE_LDG || engine == HV_ENGINE_LDG256) {
    res.chunk = kLdgChunk;
    res.chunks_per_page = (uint32_t)((res.page_bytes + kLdgChunk - 1) / kLdgChunk);
    const uint64_t total = (uint64_t)res.n_pages * res.chunks_per_page;
    if (total >= 0xffffffffull) return HV_E_INVALID;
    const int g = ldg_grid(dev, total, max_ctas);
    if (engine == HV_ENGINE_LDG256) {
      page_copy_ldg<kTable, true><<<g, kLdgThreads, 0, (cudaStream_t)stream>>>(res);
    } else {
      page_copy_ldg<kTable, false><<<g, kLdgThreads, 0, (cudaStream_t)stream>>>(res);
    }
  } else if (engine == HV_ENGINE_LDG16) {
    res.chunk = kLdgDeepChunk;
    res.chunks_per_page = (uint32_t)((res.page_bytes + kLdgDeepChunk - 1) / kLdgDeepChunk);
    const uint64_t total = (uint64_t)res.n_pages * res.chunks_per_page;
    if (total >= 0xffffffffull) return HV_E_INVALID;
    page_copy_ldg<kTable, false, kLdgDeepUnroll>
        <<<ldg_grid(dev, total, max_ctas), kLdgThreads, 0, (cudaStream_t)stream>>>(res);
  } else {
    return HV_E_INVALID;
  }
  HV_CUDA(cudaGetLastError());
  hv::note_launch();
  return HV_OK;
}

int launch_blocks(BlockResolver res, int engine, int max_ctas, void* stream) {
  if (res.n_blocks == 0 || res.n_layers == 0 || res.page_bytes == 0) return HV_OK;
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  engine = pick_engine(engine & ~kEngineInterleave);  // uniform pages: order flag not used
  uint32_t chunk = kLdgChunk;
  if (engine == HV_ENGINE_TMA) chunk = kTmaChunk;
  else if (engine == HV_ENGINE_LDG16) chunk = kLdgDeepChunk;
  else if (engine != HV_ENGINE_LDG && engine != HV_ENGINE_LDG256) return HV_E_INVALID;
  res.chunk = chunk;
  res.chunks_per_page = (uint32_t)((res.page_bytes + chunk - 1) / chunk);
  const uint64_t total = (uint64_t)res.n_blocks * res.n_layers * res.chunks_per_page;
  if (total >= 0xffffffffull) return HV_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (engine == HV_ENGINE_TMA) {
    if ((st = set_tma_attrs(dev))) return st;
    block_copy_tma<<<tma_grid(dev, total, max_ctas), kTmaThreads, kTmaSmem, s>>>(res);
  } else {
    const int g = ldg_grid(dev, total, max_ctas);
    if (engine == HV_ENGINE_LDG256) {
      block_copy_ldg<true, kLdgUnroll><<<g, kLdgThreads, 0, s>>>(res);
    } else if (engine == HV_ENGINE_LDG16) {
      block_copy_ldg<false, kLdgDeepUnroll><<<g, kLdgThreads, 0, s>>>(res);
    } else {
      block_copy_ldg<false, kLdgUnroll><<<g, kLdgThreads, 0, s>>>(res);
    }
  }
  HV_CUDA(cudaGetLastError());
  hv::note_launch();
  return HV_OK;
}

// Variable-size launch: up to kMaxSmemDescs descriptors per launch.  The
// chunk count is not known on the host (sizes are device-resident), so the
// grid is sized to fill the device (capped by max_ctas).
template <typename Op>
int launch_descs(const uint64_t* d_src, const uint64_t* d_dst, const uint64_t* d_bytes, uint32_t n,
                 int engine, int max_ctas, void* stream, Op op, bool is_copy,
                 uint64_t chunks_hint = kUnknownChunks) {
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  // AUTO copies take the interleaved order: neutral on a PCIe or local-HBM
  // source (within 2%), and it spreads the reads of a multi-donor batch
  const uint32_t interleave =
      ((engine & kEngineInterleave) || engine == HV_ENGINE_AUTO || engine == HV_ENGINE_CE) && is_copy ? 1u : 0u;
  engine = pick_engine(engine & ~kEngineInterleave);
  if (engine == HV_ENGINE_TMA && is_copy && (st = set_tma_attrs(dev))) return st;
  for (uint32_t base = 0; base < n; base += kMaxSmemDescs) {
    const uint32_t m = (n - base) < kMaxSmemDescs ? (n - base) : kMaxSmemDescs;
    DescResolver res;
    res.src = d_src ? d_src + base : nullptr;
    res.dst = d_dst ? d_dst + base : nullptr;
    res.bytes = d_bytes + base;
    res.n = m;
    res.interleave = interleave;
    Op o = op;
    o.rebase(base);
    if (is_copy && engine == HV_ENGINE_TMA) {
      res.chunk = kTmaChunk;
      desc_copy_tma<<<tma_grid(dev, chunks_hint, max_ctas), kTmaThreads, kTmaSmem, (cudaStream_t)stream>>>(res);
    } else if (is_copy && engine == HV_ENGINE_LDG256) {
      res.chunk = kLdgChunk;
      desc_op_kernel<<<ldg_grid(dev, chunks_hint, max_ctas), kLdgThreads, 0, (cudaStream_t)stream>>>(
          res, CopyOpT<true>{});
    } else if (is_copy && engine == HV_ENGINE_LDG16) {
      res.chunk = kLdgDeepChunk;
      desc_op_kernel<<<ldg_grid(dev, chunks_hint, max_ctas), kLdgThreads, 0, (cudaStream_t)stream>>>(
          res, CopyOpT<false, kLdgDeepUnroll>{});
    } else if (engine == HV_ENGINE_LDG || !is_copy) {
      res.chunk = kLdgChunk;
      desc_op_kernel<<<ldg_grid(dev, chunks_hint, max_ctas), kLdgThreads, 0, (cudaStream_t)stream>>>(res, o);
    } else {
      return HV_E_INVALID;
    }
    HV_CUDA(cudaGetLastError());
    hv::note_launch();
  }
  return HV_OK;
}

// Copy and content digest in one pass (the fetch and its per-fetch check,
// moe.py:315-319, fused): every 16 bytes a lane moves are also folded into
// the object's position-keyed digest, so checking what arrived costs no
// second read of it and no second kernel competing for the SMs.  The digest
// equals DigestOp's over the same bytes (objects 8-byte aligned).
template <int kUnroll>
struct CopyDigestOp {
  const uint64_t* bytes;      // object sizes (the size term, as DigestOp)
  unsigned long long* out;    // per-object digest accumulators (zeroed by the caller)
  __device__ __forceinline__ void operator()(const ChunkRef& r, uint32_t lane) const {
    const uint64_t w0 = r.off >> 3;
    uint64_t acc = 0;
    const bool aligned = ((reinterpret_cast<uintptr_t>(r.src) | reinterpret_cast<uintptr_t>(r.dst)) & 15) == 0;
    if (aligned && r.len == (uint32_t)kUnroll * 512u) {
      uint4 v[kUnroll];
#pragma unroll
      for (int j = 0; j < kUnroll; ++j) v[j] = ld_stream(r.src + (j * 32 + lane) * 16);
#pragma unroll
      for (int j = 0; j < kUnroll; ++j) {
        st_stream(r.dst + (j * 32 + lane) * 16, v[j]);
        const uint64_t i = w0 + (uint64_t)(j * 32 + lane) * 2;
        acc += digest_term(i, (uint64_t)v[j].x | ((uint64_t)v[j].y << 32));
        acc += digest_term(i + 1, (uint64_t)v[j].z | ((uint64_t)v[j].w << 32));
      }
    } else {
      copy_chunk_ldg<false, kUnroll>(r, lane);
      const uint32_t nfull = r.len >> 3;
      const uint64_t* s = reinterpret_cast<const uint64_t*>(r.src);
      for (uint32_t k = lane; k < nfull; k += 32) acc += digest_term(w0 + k, s[k]);
      const uint32_t tail = r.len & 7;
      if (tail && lane == 0) acc += digest_term(w0 + nfull, load_word_tail(r.src + nfull * 8, tail));
    }
    if (r.off == 0 && lane == 0) acc += __ldg(bytes + r.obj);
    acc = warp_sum(acc);
    if (lane == 0) atomicAdd(out + r.obj, (unsigned long long)acc);
  }
};
template <int kUnroll>
struct CopyDigestOpR : CopyDigestOp<kUnroll> {
  __host__ __device__ void rebase(uint32_t b) {
    this->bytes += b;
    this->out += b;
  }
};

struct CopyOpR : CopyOp {
  __host__ __device__ void rebase(uint32_t) {}
};
struct FillOpR : FillOp {
  __host__ __device__ void rebase(uint32_t b) { seeds += b; }
};
struct DigestOpR : DigestOp {
  __host__ __device__ void rebase(uint32_t b) {
    bytes += b;
    out += b;
  }
};
struct VerifyOpR : VerifyOp {
  __host__ __device__ void rebase(uint32_t b) {
    seeds += b;
    out += b;
  }
};

// ---------------------------------------------------------------------------
// pinned staging ring for host-array entry points (hv_swap_blocks_batch)

constexpr uint32_t kRingSlots = 32;
constexpr uint32_t kSlotDescs = kMaxSmemDescs;  // descriptors per slot

struct StagingRing {
  bool init = false;
  uint64_t* h = nullptr;  // pinned: kRingSlots * 3 * kSlotDescs words
  uint64_t* d = nullptr;
  cudaEvent_t ev[kRingSlots] = {};
  bool used[kRingSlots] = {};
  uint32_t next = 0;
};

std::mutex g_ring_mu;
StagingRing g_rings[64];

// Descriptor upload by an SM kernel: the staging slot is mapped pinned
// memory, and a copy-engine H2D of it would queue behind whatever bulk
// copies the copy engines are running (a stage's 917 MB of host-tier
// experts: ~16 ms), stalling a concurrent kernel fetch or content check.
__global__ void upload_desc_kernel(const uint2* __restrict__ src, uint2* __restrict__ dst, uint32_t n8) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n8) dst[i] = src[i];
}

int upload_desc(const uint64_t* h, uint64_t* d, size_t words, cudaStream_t s) {
  if (words == 0) return HV_OK;
  const uint32_t n8 = (uint32_t)words;
  upload_desc_kernel<<<(n8 + 255) / 256, 256, 0, s>>>(reinterpret_cast<const uint2*>(h), reinterpret_cast<uint2*>(d),
                                                       n8);
  HV_CUDA(cudaGetLastError());
  hv::note_launch();
  return HV_OK;
}

int ring_acquire(int dev, uint32_t* slot, StagingRing** ring) {
  if (dev < 0 || dev >= 64) return HV_E_INVALID;
  StagingRing& r = g_rings[dev];
  if (!r.init) {
    const size_t words = (size_t)kRingSlots * 3 * kSlotDescs;
    // mapped: the descriptor upload is an SM kernel reading it over PCIe
    // (upload_desc), never a DMA that would queue behind bulk copy-engine work
    HV_CUDA(cudaHostAlloc((void**)&r.h, words * 8, cudaHostAllocPortable | cudaHostAllocMapped));
    HV_CUDA(cudaMalloc((void**)&r.d, words * 8));
    for (uint32_t i = 0; i < kRingSlots; ++i) HV_CUDA(cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming));
    r.init = true;
  }
  const uint32_t s = r.next;
  r.next = (r.next + 1) % kRingSlots;
  if (r.used[s]) HV_CUDA(cudaEventSynchronize(r.ev[s]));  // previous user of the slot is done
  *slot = s;
  *ring = &r;
  return HV_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

HV_EXPORT int hv_abi_version(void) { return HV_ABI_VERSION; }

HV_EXPORT const char* hv_error_string(int status) {
  switch (status) {
    case HV_OK: return "ok";
    case HV_E_INVALID: return "invalid argument";
    case HV_E_NOCAPACITY: return "no capacity";
    case HV_E_DOUBLEFREE: return "double free or unknown segment";
    case HV_E_UNSUPPORTED: return "unsupported on this device/driver";
    case HV_E_NOMEM: return "host allocation failed";
    default: break;
  }
  if (status <= HV_E_CU_BASE) return "CUDA driver API error (code = -3000 - CUresult)";
  if (status <= HV_E_CUDA_BASE) return cudaGetErrorString((cudaError_t)(HV_E_CUDA_BASE - status));
  return "unknown status";
}

HV_EXPORT int hv_launch_count(uint64_t* out) {
  HV_CHECK_ARG(out);
  *out = hv::g_launches.load();
  return HV_OK;
}

HV_EXPORT int hv_kv_gather(const uint64_t* d_src_page_ptrs, const uint64_t* d_dst_page_ptrs, uint64_t d_dst_base,
                           uint32_t n_pages, uint64_t page_bytes, int engine, int max_ctas, void* stream) {
  HV_CHECK_ARG(n_pages == 0 || d_src_page_ptrs != nullptr);
  HV_CHECK_ARG(n_pages == 0 || d_dst_page_ptrs != nullptr || d_dst_base != 0);
  HV_CHECK_ARG(n_pages <= kPageBatchMax);
  PageResolver<false> r{};
  r.src = d_src_page_ptrs;
  r.locs = nullptr;
  r.dst_ptrs = d_dst_page_ptrs;
  r.dst_base = d_dst_base;
  r.page_bytes = page_bytes;
  r.n_pages = n_pages;
  return launch_pages(r, engine, max_ctas, stream);
}

HV_EXPORT int hv_kv_gather_table(const uint64_t* d_slot_bases, const uint64_t* d_locs, uint64_t d_dst_base,
                                 const uint64_t* d_dst_page_ptrs, uint32_t n_pages, uint64_t page_bytes, int engine,
                                 int max_ctas, void* stream) {
  HV_CHECK_ARG(n_pages == 0 || (d_slot_bases != nullptr && d_locs != nullptr));
  HV_CHECK_ARG(n_pages == 0 || d_dst_page_ptrs != nullptr || d_dst_base != 0);
  HV_CHECK_ARG(n_pages <= kPageBatchMax);
  PageResolver<true> r{};
  r.src = d_slot_bases;
  r.locs = d_locs;
  r.dst_ptrs = d_dst_page_ptrs;
  r.dst_base = d_dst_base;
  r.page_bytes = page_bytes;
  r.n_pages = n_pages;
  return launch_pages(r, engine, max_ctas, stream);
}

HV_EXPORT int hv_kv_gather_blocks(const uint64_t* d_src_base, const uint64_t* d_src_stride,
                                  const uint64_t* d_dst_base, const uint64_t* d_dst_stride, uint32_t n_blocks,
                                  uint32_t n_layers, uint64_t page_bytes, int engine, int max_ctas, void* stream) {
  HV_CHECK_ARG(n_blocks == 0 || (d_src_base && d_src_stride && d_dst_base && d_dst_stride));
  BlockResolver r{};
  r.src_base = d_src_base;
  r.src_stride = d_src_stride;
  r.dst_base = d_dst_base;
  r.dst_stride = d_dst_stride;
  r.page_bytes = page_bytes;
  r.n_blocks = n_blocks;
  r.n_layers = n_layers;
  return launch_blocks(r, engine, max_ctas, stream);
}

HV_EXPORT int hv_batch_copy(const uint64_t* d_src, const uint64_t* d_dst, const uint64_t* d_bytes, uint32_t n,
                            int engine, int max_ctas, void* stream) {
  if (n == 0) return HV_OK;
  HV_CHECK_ARG(d_src && d_dst && d_bytes);
  return launch_descs(d_src, d_dst, d_bytes, n, engine, max_ctas, stream, CopyOpR{}, true);
}

namespace {

// The kernel form of the host-array entry point: descriptors staged through
// the pinned ring (one H2D of exactly what is used), then one K1/K2 launch
// per ring slot.  Caller holds g_ring_mu and has bound the device.
int kernel_swap(const uint64_t* h_src, const uint64_t* h_dst, const uint64_t* h_bytes, uint32_t n, int engine,
                int max_ctas, void* stream, int dev) {
  int st = HV_OK;
  for (uint32_t base = 0; base < n; base += kSlotDescs) {
    const uint32_t m = (n - base) < kSlotDescs ? (n - base) : kSlotDescs;
    uint32_t slot = 0;
    StagingRing* ring = nullptr;
    if ((st = ring_acquire(dev, &slot, &ring))) return st;
    uint64_t* hs = ring->h + (size_t)slot * 3 * kSlotDescs;
    uint64_t* ds = ring->d + (size_t)slot * 3 * kSlotDescs;
    // sizes are host-visible here: detect the uniform case (expert / page
    // batches) and the exact chunk count, so the launch needs no device-side
    // prefix scan and its grid matches the work
    bool uniform = true;
    uint64_t total_bytes = 0;
    for (uint32_t i = 0; i < m; ++i) {
      uniform &= (h_bytes[base + i] == h_bytes[base]);
      total_bytes += h_bytes[base + i];
    }
    memcpy(hs, h_src + base, m * 8);
    memcpy(hs + m, h_dst + base, m * 8);
    memcpy(hs + 2 * m, h_bytes + base, m * 8);
    if ((st = upload_desc(hs, ds, (size_t)(uniform ? 2 : 3) * m, (cudaStream_t)stream))) return st;
    if (uniform && h_bytes[base] > 0) {
      PageResolver<false> r{};
      r.src = ds;
      r.locs = nullptr;
      r.dst_ptrs = ds + m;
      r.dst_base = 0;
      r.page_bytes = h_bytes[base];
      r.n_pages = m;
      // equal-size objects (a stage's experts): AUTO takes the interleaved
      // order, as hv_batch_copy does, so readers spread over every donor
      st = launch_pages(r, engine == HV_ENGINE_AUTO ? (HV_ENGINE_AUTO | kEngineInterleave) : engine, max_ctas,
                        stream);
    } else if (!uniform) {
      const int eng = pick_engine(engine & ~kEngineInterleave);
      const uint64_t chunk = eng == HV_ENGINE_TMA ? kTmaChunk : kLdgChunk;
      const uint64_t chunks = total_bytes / chunk + m;  // upper bound on the chunk count
      st = launch_descs(ds, ds + m, ds + 2 * m, m, engine, max_ctas, stream, CopyOpR{}, true, chunks);
    }
    if (st) return st;
    HV_CUDA(cudaEventRecord(ring->ev[slot], (cudaStream_t)stream));
    ring->used[slot] = true;
  }
  return HV_OK;
}

// Per-device side stream for copy-engine work that must run beside (not
// behind) a kernel on the caller's stream.  Fenced by events on both sides,
// so the caller's stream order is preserved.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
std::mutex g_side_mu;
SideStream g_side[64];

int side_stream(int dev, SideStream** out) {
  if (dev < 0 || dev >= 64) return HV_E_INVALID;
  SideStream& ss = g_side[dev];
  if (!ss.s) {
    HV_CUDA(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking));
    HV_CUDA(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    HV_CUDA(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
  }
  *out = &ss;
  return HV_OK;
}

// Copy-engine submission on `stream`: one cudaMemcpyAsync per run.  With
// `coalesce`, objects whose source and destination both continue the previous
// object's (consecutive host slots into consecutive local slots, the layout
// F.layer_runs and the decoder's compact staging produce) are merged into one
// larger copy; otherwise every object is its own copy.  The DMA engine keeps
// successive copies of one stream back to back: 17.3 MB experts lose ~1 us of
// the ~311 us each takes on PCIe.
int ce_submit(void* const* dsts, const void* const* srcs, const size_t* sizes, size_t n, bool coalesce,
              cudaStream_t stream) {
  size_t i = 0;
  while (i < n) {
    char* d = (char*)dsts[i];
    const char* s = (const char*)srcs[i];
    size_t z = sizes[i++];
    while (coalesce && i < n && (char*)dsts[i] == d + z && (const char*)srcs[i] == s + z) z += sizes[i++];
    if (z) HV_CUDA(cudaMemcpyAsync(d, s, z, cudaMemcpyDefault, stream));
  }
  return HV_OK;
}

int ce_on_stream(void* const* dsts, const void* const* srcs, const size_t* sizes, size_t n, bool coalesce,
                 void* stream, int /*dev*/) {
  return ce_submit(dsts, srcs, sizes, n, coalesce, (cudaStream_t)stream);
}

constexpr uint64_t kCeMinBytes = 1ull << 20;  // host-tier objects at least this large go to the copy engine

bool capturing(void* stream) {
  if (!stream) return false;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing((cudaStream_t)stream, &cap) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return cap != cudaStreamCaptureStatusNone;
}

}  // namespace

HV_EXPORT int hv_swap_blocks_batch(const uint64_t* h_src, const uint64_t* h_dst, const uint64_t* h_bytes, uint32_t n,
                                   int engine, int max_ctas, void* stream) {
  if (n == 0) return HV_OK;
  HV_CHECK_ARG(h_src && h_dst && h_bytes);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  const int base_engine = engine & ~kEngineInterleave;
  if (base_engine == HV_ENGINE_CE) {
    std::vector<void*> d(n);
    std::vector<const void*> s(n);
    std::vector<size_t> z(n);
    for (uint32_t i = 0; i < n; ++i) {
      d[i] = (void*)h_dst[i];
      s[i] = (const void*)h_src[i];
      z[i] = (size_t)h_bytes[i];
    }
    return ce_on_stream(d.data(), s.data(), z.data(), n, true, stream, dev);
  }
  if (base_engine != HV_ENGINE_AUTO || capturing(stream)) {
    std::lock_guard<std::mutex> lk(g_ring_mu);
    return kernel_swap(h_src, h_dst, h_bytes, n, engine, max_ctas, stream, dev);
  }
  // AUTO: engine per source.  Large objects read from -- or written to --
  // the pinned host tier go to the copy engine (cudaMemcpyAsync per run);
  // everything else -- peer HBM over NVLink, local HBM, small host pages --
  // to the SM kernel.  Measured on B200 (tools/d2h_probe.py, r2q): 16 MiB
  // runs device->host 56.5 GB/s copy engine vs 52.3 SM stores; 64 KiB pages
  // 44.3 vs 51.5 (so pages stay on the kernel in both directions).
  std::vector<uint32_t> ce_idx;
  for (uint32_t i = 0; i < n; ++i)
    if (h_bytes[i] >= kCeMinBytes &&
        (hv::host_range_contains(h_src[i], h_bytes[i]) || hv::host_range_contains(h_dst[i], h_bytes[i])))
      ce_idx.push_back(i);
  if (ce_idx.empty()) {
    std::lock_guard<std::mutex> lk(g_ring_mu);
    return kernel_swap(h_src, h_dst, h_bytes, n, engine, max_ctas, stream, dev);
  }
  std::vector<void*> cd(ce_idx.size());
  std::vector<const void*> cs(ce_idx.size());
  std::vector<size_t> cz(ce_idx.size());
  for (size_t k = 0; k < ce_idx.size(); ++k) {
    cd[k] = (void*)h_dst[ce_idx[k]];
    cs[k] = (const void*)h_src[ce_idx[k]];
    cz[k] = (size_t)h_bytes[ce_idx[k]];
  }
  if (ce_idx.size() == n) return ce_on_stream(cd.data(), cs.data(), cz.data(), n, true, stream, dev);
  // mixed batch: the copy engine runs on the side stream beside the kernel
  // (two links, two engines), joined back before the caller's next op
  std::vector<uint64_t> ks, kd, kz;
  ks.reserve(n - ce_idx.size());
  kd.reserve(n - ce_idx.size());
  kz.reserve(n - ce_idx.size());
  for (uint32_t i = 0, k = 0; i < n; ++i) {
    if (k < ce_idx.size() && ce_idx[k] == i) {
      ++k;
      continue;
    }
    ks.push_back(h_src[i]);
    kd.push_back(h_dst[i]);
    kz.push_back(h_bytes[i]);
  }
  std::lock_guard<std::mutex> lk_side(g_side_mu);
  SideStream* ss = nullptr;
  if ((st = side_stream(dev, &ss))) return st;
  HV_CUDA(cudaEventRecord(ss->fork, (cudaStream_t)stream));
  HV_CUDA(cudaStreamWaitEvent(ss->s, ss->fork, 0));
  if ((st = ce_submit(cd.data(), cs.data(), cz.data(), cd.size(), true, ss->s))) return st;
  {
    std::lock_guard<std::mutex> lk(g_ring_mu);
    if ((st = kernel_swap(ks.data(), kd.data(), kz.data(), (uint32_t)ks.size(), engine, max_ctas, stream, dev)))
      return st;
  }
  HV_CUDA(cudaEventRecord(ss->join, ss->s));
  HV_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, ss->join, 0));
  return HV_OK;
}

HV_EXPORT int hv_ce_batch_copy(const uint64_t* h_src, const uint64_t* h_dst, const uint64_t* h_bytes, uint32_t n,
                               int batched, void* stream) {
  if (n == 0) return HV_OK;
  HV_CHECK_ARG(h_src && h_dst && h_bytes);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  std::vector<void*> dsts(n);
  std::vector<const void*> srcs(n);
  std::vector<size_t> sizes(n);
  for (uint32_t i = 0; i < n; ++i) {
    dsts[i] = (void*)h_dst[i];
    srcs[i] = (const void*)h_src[i];
    sizes[i] = (size_t)h_bytes[i];
  }
  return ce_on_stream(dsts.data(), srcs.data(), sizes.data(), n, batched != 0, stream, dev);
}

HV_EXPORT int hv_fill_content(const uint64_t* d_dst, const uint64_t* d_bytes, const uint64_t* d_seeds, uint32_t n,
                              void* stream) {
  if (n == 0) return HV_OK;
  HV_CHECK_ARG(d_dst && d_bytes && d_seeds);
  FillOpR op;
  op.seeds = d_seeds;
  op.kind = 0;
  // FillOp writes through r.dst; the resolver's src is unused but must be valid
  return launch_descs(d_dst, d_dst, d_bytes, n, HV_ENGINE_LDG, 0, stream, op, false);
}

HV_EXPORT int hv_fill_weights_bf16(const uint64_t* d_dst, const uint64_t* d_bytes, const uint64_t* d_seeds,
                                   uint32_t n, void* stream) {
  if (n == 0) return HV_OK;
  HV_CHECK_ARG(d_dst && d_bytes && d_seeds);
  FillOpR op;
  op.seeds = d_seeds;
  op.kind = 1;
  return launch_descs(d_dst, d_dst, d_bytes, n, HV_ENGINE_LDG, 0, stream, op, false);
}

HV_EXPORT int hv_digest(const uint64_t* d_src, const uint64_t* d_bytes, uint32_t n, uint64_t* d_out, void* stream) {
  if (n == 0) return HV_OK;
  HV_CHECK_ARG(d_src && d_bytes && d_out);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  HV_CUDA(cudaMemsetAsync(d_out, 0, (size_t)n * 8, (cudaStream_t)stream));
  DigestOpR op;
  op.bytes = d_bytes;
  op.out = reinterpret_cast<unsigned long long*>(d_out);
  return launch_descs(d_src, d_src, d_bytes, n, HV_ENGINE_LDG, 0, stream, op, false);
}

namespace {
// read_errors of moe.py:315-319 on bytes: object i is a read error when the
// digest of what arrived differs from the digest recorded for its
// authoritative copy.  Per-object flags plus one running counter.
__global__ void digest_compare_kernel(const uint64_t* __restrict__ got, const uint64_t* __restrict__ want,
                                      uint32_t n, uint8_t* __restrict__ flags,
                                      unsigned long long* __restrict__ errors) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool bad = i < n && got[i] != want[i];
  if (i < n && flags) flags[i] = bad ? 1 : 0;
  const unsigned m = __ballot_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(errors, (unsigned long long)__popc(m));
}
}  // namespace

HV_EXPORT int hv_check_digests(const uint64_t* d_src, const uint64_t* d_bytes, const uint64_t* d_expected,
                               uint32_t n, uint64_t* d_scratch, uint8_t* d_flags, uint64_t* d_errors,
                               void* stream) {
  if (n == 0) return HV_OK;
  HV_CHECK_ARG(d_src && d_bytes && d_expected && d_scratch && d_errors);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  HV_CUDA(cudaMemsetAsync(d_scratch, 0, (size_t)n * 8, (cudaStream_t)stream));
#if HV_DIGEST_TMA
  if ((st = hv::kernel_attr<desc_digest_tma>(dev, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDgSmem)))
    return st;
  for (uint32_t base = 0; base < n; base += kMaxSmemDescs) {
    const uint32_t m = (n - base) < kMaxSmemDescs ? (n - base) : kMaxSmemDescs;
    DescResolver res;
    res.src = d_src + base;
    res.dst = d_src + base;
    res.bytes = d_bytes + base;
    res.n = m;
    res.interleave = 0;
    res.chunk = kDgChunk;
    desc_digest_tma<<<2 * hv::sm_count(dev), kDgThreads, kDgSmem, (cudaStream_t)stream>>>(
        res, d_bytes + base, reinterpret_cast<unsigned long long*>(d_scratch) + base);
    HV_CUDA(cudaGetLastError());
    hv::note_launch();
  }
#else
  DigestOpR op;
  op.bytes = d_bytes;
  op.out = reinterpret_cast<unsigned long long*>(d_scratch);
  if ((st = launch_descs(d_src, d_src, d_bytes, n, HV_ENGINE_LDG, 0, stream, op, false))) return st;
#endif
  digest_compare_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      d_scratch, d_expected, n, d_flags, reinterpret_cast<unsigned long long*>(d_errors));
  HV_CUDA(cudaGetLastError());
  hv::note_launch();
  return HV_OK;
}

HV_EXPORT int hv_kv_gather_blocks_h(const uint64_t* h_src_base, const uint64_t* h_src_stride,
                                    const uint64_t* h_dst_base, const uint64_t* h_dst_stride, uint32_t n_blocks,
                                    uint32_t n_layers, uint64_t page_bytes, int engine, int max_ctas, void* stream) {
  if (n_blocks == 0) return HV_OK;
  HV_CHECK_ARG(h_src_base && h_src_stride && h_dst_base && h_dst_stride);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  std::lock_guard<std::mutex> lk(g_ring_mu);
  constexpr uint32_t kM = kSlotDescs * 3 / 4;   // four words per block in one ring slot
  for (uint32_t base = 0; base < n_blocks; base += kM) {
    const uint32_t m = (n_blocks - base) < kM ? (n_blocks - base) : kM;
    uint32_t slot = 0;
    StagingRing* ring = nullptr;
    if ((st = ring_acquire(dev, &slot, &ring))) return st;
    uint64_t* hs = ring->h + (size_t)slot * 3 * kSlotDescs;
    uint64_t* ds = ring->d + (size_t)slot * 3 * kSlotDescs;
    memcpy(hs, h_src_base + base, m * 8);
    memcpy(hs + m, h_src_stride + base, m * 8);
    memcpy(hs + 2 * m, h_dst_base + base, m * 8);
    memcpy(hs + 3 * m, h_dst_stride + base, m * 8);
    if ((st = upload_desc(hs, ds, (size_t)4 * m, (cudaStream_t)stream))) return st;
    BlockResolver r{};
    r.src_base = ds;
    r.src_stride = ds + m;
    r.dst_base = ds + 2 * m;
    r.dst_stride = ds + 3 * m;
    r.page_bytes = page_bytes;
    r.n_blocks = m;
    r.n_layers = n_layers;
    if ((st = launch_blocks(r, engine, max_ctas, stream))) return st;
    HV_CUDA(cudaEventRecord(ring->ev[slot], (cudaStream_t)stream));
    ring->used[slot] = true;
  }
  return HV_OK;
}

HV_EXPORT int hv_check_digests_batch(const uint64_t* h_src, const uint64_t* h_bytes, const uint64_t* h_expected,
                                     uint32_t n, uint64_t* d_scratch, uint8_t* d_flags, uint64_t* d_errors,
                                     void* stream) {
  if (n == 0) return HV_OK;
  HV_CHECK_ARG(h_src && h_bytes && h_expected && d_scratch && d_errors);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  std::lock_guard<std::mutex> lk(g_ring_mu);
  for (uint32_t base = 0; base < n; base += kSlotDescs) {
    const uint32_t m = (n - base) < kSlotDescs ? (n - base) : kSlotDescs;
    uint32_t slot = 0;
    StagingRing* ring = nullptr;
    if ((st = ring_acquire(dev, &slot, &ring))) return st;
    uint64_t* hs = ring->h + (size_t)slot * 3 * kSlotDescs;
    uint64_t* ds = ring->d + (size_t)slot * 3 * kSlotDescs;
    memcpy(hs, h_src + base, m * 8);
    memcpy(hs + m, h_bytes + base, m * 8);
    memcpy(hs + 2 * m, h_expected + base, m * 8);
    if ((st = upload_desc(hs, ds, (size_t)3 * m, (cudaStream_t)stream))) return st;
    if ((st = hv_check_digests(ds, ds + m, ds + 2 * m, m, d_scratch + base, d_flags ? d_flags + base : nullptr,
                               d_errors, stream)))
      return st;
    HV_CUDA(cudaEventRecord(ring->ev[slot], (cudaStream_t)stream));
    ring->used[slot] = true;
  }
  return HV_OK;
}

HV_EXPORT int hv_swap_blocks_batch_checked(const uint64_t* h_src, const uint64_t* h_dst, const uint64_t* h_bytes,
                                           const uint64_t* h_expected, uint32_t n, int engine, int max_ctas,
                                           uint64_t* d_scratch, uint8_t* d_flags, uint64_t* d_errors,
                                           void* stream) {
  if (n == 0) return HV_OK;
  HV_CHECK_ARG(h_src && h_dst && h_bytes && h_expected && d_scratch && d_errors);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  cudaStream_t cs = (cudaStream_t)stream;
  const int base_engine = engine & ~kEngineInterleave;
  // engine per source, as hv_swap_blocks_batch: large host-tier objects ride
  // the copy engine on the side stream and are digested there after their
  // copy; everything else is copied AND digested by one SM kernel pass here
  std::vector<uint32_t> ce_idx;
  if ((base_engine == HV_ENGINE_AUTO || base_engine == HV_ENGINE_CE) && !capturing(stream)) {
    for (uint32_t i = 0; i < n; ++i)
      if (base_engine == HV_ENGINE_CE ||
          (h_bytes[i] >= kCeMinBytes && hv::host_range_contains(h_src[i], h_bytes[i])))
        ce_idx.push_back(i);
  }
  const bool deep = base_engine == HV_ENGINE_LDG16;
  HV_CUDA(cudaMemsetAsync(d_scratch, 0, (size_t)n * 8, cs));
  std::unique_lock<std::mutex> lk_side(g_side_mu, std::defer_lock);
  SideStream* ss = nullptr;
  if (!ce_idx.empty()) {
    lk_side.lock();
    if ((st = side_stream(dev, &ss))) return st;
    HV_CUDA(cudaEventRecord(ss->fork, cs));   // after the scratch reset
    HV_CUDA(cudaStreamWaitEvent(ss->s, ss->fork, 0));
  }
  std::lock_guard<std::mutex> lk(g_ring_mu);
  // descriptors per launch: one ring slot of [src m][dst m][bytes m]
  constexpr uint32_t kM = kSlotDescs;
  std::vector<char> is_ce(n, 0);
  for (uint32_t k : ce_idx) is_ce[k] = 1;
  for (uint32_t base = 0; base < n; base += kM) {
    const uint32_t m = (n - base) < kM ? (n - base) : kM;
    uint32_t slot = 0;
    StagingRing* ring = nullptr;
    if ((st = ring_acquire(dev, &slot, &ring))) return st;
    uint64_t* hs = ring->h + (size_t)slot * 3 * kSlotDescs;
    uint64_t* ds = ring->d + (size_t)slot * 3 * kSlotDescs;
    // kernel objects keep their sizes; CE objects get size 0 in the kernel's
    // descriptors (skipped) and their digest from the side-stream pass below
    memcpy(hs, h_src + base, m * 8);
    memcpy(hs + m, h_dst + base, m * 8);
    for (uint32_t i = 0; i < m; ++i) hs[2 * m + i] = is_ce[base + i] ? 0 : h_bytes[base + i];
    if ((st = upload_desc(hs, ds, (size_t)3 * m, cs))) return st;
    uint32_t n_kernel = 0;
    for (uint32_t i = 0; i < m; ++i) n_kernel += !is_ce[base + i];
    if (n_kernel) {
      DescResolver res;
      res.src = ds;
      res.dst = ds + m;
      res.bytes = ds + 2 * m;
      res.n = m;
      res.interleave = 1u;
      res.chunk = deep ? kLdgDeepChunk : kLdgChunk;
      uint64_t total = 0;
      for (uint32_t i = 0; i < m; ++i) total += is_ce[base + i] ? 0 : h_bytes[base + i];
      const uint64_t chunks = total / res.chunk + m;
      const int g = ldg_grid(dev, chunks, max_ctas);
      unsigned long long* out = reinterpret_cast<unsigned long long*>(d_scratch + base);
      if (deep) {
        CopyDigestOpR<kLdgDeepUnroll> op;
        op.bytes = ds + 2 * m;
        op.out = out;
        desc_op_kernel<<<g, kLdgThreads, 0, cs>>>(res, op);
      } else {
        CopyDigestOpR<kLdgUnroll> op;
        op.bytes = ds + 2 * m;
        op.out = out;
        desc_op_kernel<<<g, kLdgThreads, 0, cs>>>(res, op);
      }
      HV_CUDA(cudaGetLastError());
      hv::note_launch();
    }
    HV_CUDA(cudaEventRecord(ring->ev[slot], cs));
    ring->used[slot] = true;
  }
  if (!ce_idx.empty()) {
    // side stream: one copy-engine batch, then the digest of what it moved
    std::vector<void*> cd(ce_idx.size());
    std::vector<const void*> csrc(ce_idx.size());
    std::vector<size_t> cz(ce_idx.size());
    std::vector<uint64_t> dd(ce_idx.size()), dz(ce_idx.size());
    for (size_t k = 0; k < ce_idx.size(); ++k) {
      cd[k] = (void*)h_dst[ce_idx[k]];
      csrc[k] = (const void*)h_src[ce_idx[k]];
      cz[k] = (size_t)h_bytes[ce_idx[k]];
    }
    if ((st = ce_submit(cd.data(), csrc.data(), cz.data(), cd.size(), true, ss->s))) return st;
    // digest each CE object into its own scratch word: one DigestOp launch
    // over [dst k][size k] with outputs scattered through a per-object index
    for (size_t k = 0; k < ce_idx.size(); ++k) {
      uint32_t slot = 0;
      StagingRing* ring = nullptr;
      // contiguous runs of CE indices share a launch
      size_t e = k;
      while (e + 1 < ce_idx.size() && ce_idx[e + 1] == ce_idx[e] + 1 && e + 1 - k < kSlotDescs) ++e;
      const uint32_t m = (uint32_t)(e - k + 1);
      if ((st = ring_acquire(dev, &slot, &ring))) return st;
      uint64_t* hs = ring->h + (size_t)slot * 3 * kSlotDescs;
      uint64_t* ds = ring->d + (size_t)slot * 3 * kSlotDescs;
      for (uint32_t i = 0; i < m; ++i) {
        hs[i] = h_dst[ce_idx[k + i]];
        hs[m + i] = h_bytes[ce_idx[k + i]];
      }
      if ((st = upload_desc(hs, ds, (size_t)2 * m, ss->s))) return st;
      DigestOpR op;
      op.bytes = ds + m;
      op.out = reinterpret_cast<unsigned long long*>(d_scratch + ce_idx[k]);
      if ((st = launch_descs(ds, ds, ds + m, m, HV_ENGINE_LDG, 0, ss->s, op, false))) return st;
      HV_CUDA(cudaEventRecord(ring->ev[slot], ss->s));
      ring->used[slot] = true;
      k = e;
    }
    HV_CUDA(cudaEventRecord(ss->join, ss->s));
    HV_CUDA(cudaStreamWaitEvent(cs, ss->join, 0));
  }
  // compare every object's digest with its authoritative one (host array of
  // expected values lives in the ring slots above; re-stage it contiguously)
  for (uint32_t base = 0; base < n; base += kSlotDescs * 3) {
    const uint32_t m = (n - base) < kSlotDescs * 3 ? (n - base) : kSlotDescs * 3;
    uint32_t slot = 0;
    StagingRing* ring = nullptr;
    if ((st = ring_acquire(dev, &slot, &ring))) return st;
    uint64_t* hs = ring->h + (size_t)slot * 3 * kSlotDescs;
    uint64_t* ds = ring->d + (size_t)slot * 3 * kSlotDescs;
    memcpy(hs, h_expected + base, m * 8);
    if ((st = upload_desc(hs, ds, m, cs))) return st;
    digest_compare_kernel<<<(m + 255) / 256, 256, 0, cs>>>(d_scratch + base, ds, m, d_flags ? d_flags + base : nullptr,
                                                          reinterpret_cast<unsigned long long*>(d_errors));
    HV_CUDA(cudaGetLastError());
    hv::note_launch();
    HV_CUDA(cudaEventRecord(ring->ev[slot], cs));
    ring->used[slot] = true;
  }
  return HV_OK;
}

HV_EXPORT int hv_verify_content(const uint64_t* d_src, const uint64_t* d_bytes, const uint64_t* d_seeds, uint32_t n,
                                uint64_t* d_mismatch, void* stream) {
  if (n == 0) return HV_OK;
  HV_CHECK_ARG(d_src && d_bytes && d_seeds && d_mismatch);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  HV_CUDA(cudaMemsetAsync(d_mismatch, 0, (size_t)n * 8, (cudaStream_t)stream));
  VerifyOpR op;
  op.seeds = d_seeds;
  op.out = reinterpret_cast<unsigned long long*>(d_mismatch);
  op.kind = 0;
  return launch_descs(d_src, d_src, d_bytes, n, HV_ENGINE_LDG, 0, stream, op, false);
}

HV_EXPORT int hv_verify_weights_bf16(const uint64_t* d_src, const uint64_t* d_bytes, const uint64_t* d_seeds,
                                     uint32_t n, uint64_t* d_mismatch, void* stream) {
  if (n == 0) return HV_OK;
  HV_CHECK_ARG(d_src && d_bytes && d_seeds && d_mismatch);
  int dev = 0;
  hv::DeviceGuard dg;
  int st = hv::bind_stream_device(stream, &dev, dg);
  if (st) return st;
  HV_CUDA(cudaMemsetAsync(d_mismatch, 0, (size_t)n * 8, (cudaStream_t)stream));
  VerifyOpR op;
  op.seeds = d_seeds;
  op.out = reinterpret_cast<unsigned long long*>(d_mismatch);
  op.kind = 1;
  return launch_descs(d_src, d_src, d_bytes, n, HV_ENGINE_LDG, 0, stream, op, false);
}
