/*
 * hv_oracle.c — CPU restatement of the Harvest fetch data plane.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or as the timed CPU baseline — never on the product path.
 *
 * What it restates (reference file:line):
 *  - Object content.  The reference models an object's bytes as one 64-bit
 *    hash, stable_hash64(tag) (runtime.py:38-44; experts: moe.py:114-115),
 *    captured by a peer read (runtime.py:335-341) and compared with the
 *    expected hash at completion (moe.py:315-319).  The B200 build
 *    materialises bytes: byte j of an object is byte j%8 (little-endian) of
 *    w_{j/8} = fmix64(seed + (j/8 + 1) * 0x9E3779B97F4A7C15), i.e. the
 *    splitmix64 stream (Steele, Lea & Flood, OOPSLA 2014; Vigna's
 *    splitmix64.c) started at state = seed = stable_hash64(tag).  With seed 0
 *    the first outputs are the published 0xE220A8397B1DCDAF,
 *    0x6E789E6AA1B965F4, 0x06C45D188009454F (tests/test_oracle.py pins them).
 *  - Fetch.  app_transfer(src -> dst) (runtime.py:320-364) delivers the
 *    object's content to dst; since correctness is independent of the tier
 *    that served it, the expected destination bytes of a batched
 *    fetch are the host-authoritative bytes of each object: a memcpy gather.
 *  - Digest.  A position-keyed 64-bit sum used for size-independent checks at
 *    full sizes: D = size + sum_i a_i * b_i (mod 2^64) over little-endian
 *    8-byte words w_i (the last one zero-padded), with j = (i+1) mod 2^32 and
 *    a_i = lo32(w_i) + j*0x9E3779B1, b_i = hi32(w_i) + j*0x85EBCA77 +
 *    0xC2B2AE3D (32-bit wrapping), the product exact in 64 bits -- the NH
 *    hash of UMAC (Black, Halevi, Krawczyk, Krovetz, Rogaway, CRYPTO 1999)
 *    with fixed position keys.  Not a restatement of a reference function:
 *    the reference compares one 64-bit content hash per object
 *    (moe.py:315-319); this is the B200 build's byte-level counterpart, and
 *    the device kernels (csrc/hv_kernels.cu digest_term) must equal it.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define HVO_GOLDEN 0x9E3779B97F4A7C15ull
#define HVO_DKEY_A 0x9E3779B1u
#define HVO_DKEY_B 0x85EBCA77u
#define HVO_DKEY_C 0xC2B2AE3Du

static inline uint64_t digest_term(uint64_t i, uint64_t w) {
  const uint32_t j = (uint32_t)(i + 1);
  const uint32_t a = (uint32_t)w + j * HVO_DKEY_A;
  const uint32_t b = (uint32_t)(w >> 32) + j * HVO_DKEY_B + HVO_DKEY_C;
  return (uint64_t)a * (uint64_t)b;
}

static inline uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t hvo_content_word(uint64_t seed, uint64_t i) { return fmix64(seed + (i + 1) * HVO_GOLDEN); }

void hvo_fill(uint8_t* dst, uint64_t bytes, uint64_t seed) {
  const uint64_t nfull = bytes / 8;
  for (uint64_t i = 0; i < nfull; ++i) {
    const uint64_t w = hvo_content_word(seed, i);
    memcpy(dst + 8 * i, &w, 8); /* little-endian host */
  }
  const uint64_t tail = bytes & 7;
  if (tail) {
    const uint64_t w = hvo_content_word(seed, nfull);
    for (uint64_t b = 0; b < tail; ++b) dst[8 * nfull + b] = (uint8_t)(w >> (8 * b));
  }
}

/* bf16-weights variant of the stream (hv_fill_weights_bf16): every 16-bit
 * lane keeps sign + 7 mantissa bits, exponent fixed at 2^-7 */
void hvo_fill_weights(uint8_t* dst, uint64_t bytes, uint64_t seed) {
  const uint64_t nfull = bytes / 8;
  for (uint64_t i = 0; i < nfull; ++i) {
    const uint64_t w = (hvo_content_word(seed, i) & 0x807F807F807F807Full) | 0x3C003C003C003C00ull;
    memcpy(dst + 8 * i, &w, 8);
  }
  const uint64_t tail = bytes & 7;
  if (tail) {
    const uint64_t w = (hvo_content_word(seed, nfull) & 0x807F807F807F807Full) | 0x3C003C003C003C00ull;
    for (uint64_t b = 0; b < tail; ++b) dst[8 * nfull + b] = (uint8_t)(w >> (8 * b));
  }
}

uint64_t hvo_digest(const uint8_t* src, uint64_t bytes) {
  uint64_t acc = bytes;
  const uint64_t nfull = bytes / 8;
  for (uint64_t i = 0; i < nfull; ++i) {
    uint64_t w;
    memcpy(&w, src + 8 * i, 8);
    acc += digest_term(i, w);
  }
  const uint64_t tail = bytes & 7;
  if (tail) {
    uint64_t w = 0;
    for (uint64_t b = 0; b < tail; ++b) w |= (uint64_t)src[8 * nfull + b] << (8 * b);
    acc += digest_term(nfull, w);
  }
  return acc;
}

/* digest of the generated content without materialising it */
uint64_t hvo_content_digest(uint64_t seed, uint64_t bytes) {
  uint64_t acc = bytes;
  const uint64_t nfull = bytes / 8;
  for (uint64_t i = 0; i < nfull; ++i) acc += digest_term(i, hvo_content_word(seed, i));
  const uint64_t tail = bytes & 7;
  if (tail) {
    const uint64_t mask = (1ull << (8 * tail)) - 1;
    acc += digest_term(nfull, hvo_content_word(seed, nfull) & mask);
  }
  return acc;
}

/* ---- gather: dst_ptrs[i] <- src_ptrs[i], sizes[i] bytes ---------------- */

typedef struct {
  const uint64_t* src;
  const uint64_t* dst;
  const uint64_t* sizes;
  uint64_t n;
  uint64_t lo, hi; /* byte range of the flattened batch owned by this thread */
} gather_job;

static void* gather_worker(void* arg) {
  gather_job* j = (gather_job*)arg;
  uint64_t base = 0;
  for (uint64_t i = 0; i < j->n; ++i) {
    const uint64_t sz = j->sizes[i];
    const uint64_t a = base > j->lo ? base : j->lo;
    const uint64_t b = (base + sz) < j->hi ? (base + sz) : j->hi;
    if (a < b)
      memcpy((uint8_t*)(uintptr_t)j->dst[i] + (a - base), (const uint8_t*)(uintptr_t)j->src[i] + (a - base), b - a);
    base += sz;
    if (base >= j->hi) break;
  }
  return NULL;
}

/* memcpy gather split evenly by bytes over `threads` POSIX threads */
int hvo_gather(const uint64_t* src_ptrs, const uint64_t* dst_ptrs, const uint64_t* sizes, uint64_t n, int threads) {
  uint64_t total = 0;
  for (uint64_t i = 0; i < n; ++i) total += sizes[i];
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tids[256];
  gather_job jobs[256];
  const uint64_t per = (total + threads - 1) / threads;
  int started = 0;
  for (int t = 0; t < threads; ++t) {
    jobs[t].src = src_ptrs;
    jobs[t].dst = dst_ptrs;
    jobs[t].sizes = sizes;
    jobs[t].n = n;
    jobs[t].lo = per * t;
    jobs[t].hi = per * (t + 1) < total ? per * (t + 1) : total;
    if (jobs[t].lo >= jobs[t].hi) continue;
    if (threads == 1) {
      gather_worker(&jobs[t]);
      continue;
    }
    if (pthread_create(&tids[started], NULL, gather_worker, &jobs[t]) != 0) return -1;
    ++started;
  }
  for (int t = 0; t < started; ++t) pthread_join(tids[t], NULL);
  return 0;
}

/* fill n objects (parallel over objects) */
typedef struct {
  const uint64_t* dst;
  const uint64_t* sizes;
  const uint64_t* seeds;
  uint64_t n;
  int t, threads;
} fill_job;

static void* fill_worker(void* arg) {
  fill_job* j = (fill_job*)arg;
  for (uint64_t i = (uint64_t)j->t; i < j->n; i += (uint64_t)j->threads)
    hvo_fill((uint8_t*)(uintptr_t)j->dst[i], j->sizes[i], j->seeds[i]);
  return NULL;
}

int hvo_fill_batch(const uint64_t* dst_ptrs, const uint64_t* sizes, const uint64_t* seeds, uint64_t n, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tids[256];
  fill_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (fill_job){dst_ptrs, sizes, seeds, n, t, threads};
    if (pthread_create(&tids[t], NULL, fill_worker, &jobs[t]) != 0) return -1;
  }
  for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
  return 0;
}
