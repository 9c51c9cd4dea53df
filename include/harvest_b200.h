/*
 * harvest_b200.h — C ABI of the B200-native Harvest peer-fetch data plane.
 *
 * The reference (arXiv 2602.00328, /root/reference/pkg/src/harvestsim) is a
 * pure-Python discrete-event simulator: every "transfer" on the fetch path is
 * `fixed_cost + size/bandwidth` arithmetic (interconnect.py:51-54) scheduled by
 * TransferEngine.schedule_transfer (interconnect.py:133-165) on behalf of
 * HarvestRuntime.app_transfer (runtime.py:320-364), and object content is a
 * 64-bit hash (runtime.py:38-44, :305-315).  This library replaces those
 * modeled pieces with real ones, one entry point per modeled function:
 *
 *   reference (file:line)                          replaced by
 *   ---------------------------------------------  ---------------------------------
 *   memalloc.alloc_best_fit / free_segment          hv_seg_* (native best-fit, same
 *     (memalloc.py:90-138), allocated_bytes (:86)     decisions, O(log n) per call)
 *   DeviceState / init_device (memalloc.py:67-79)   hv_seg_create
 *   "switches to that device context, and          hv_pool_* (per-donor VMM pool:
 *     allocates memory", the          cuMemCreate/cuMemMap/
 *     peer tier of Topology (interconnect.py:57)     cuMemSetAccess, or cudaIpc)
 *   HOST_DRAM tier (memalloc.py:14-17)              hv_host_alloc (pinned, mapped)
 *   app_transfer -> schedule_transfer ->            hv_kv_gather (K1), hv_batch_copy
 *     transfer_time (runtime.py:320-364,             (K2), hv_swap_blocks_batch
 *     interconnect.py:133-165, :51-54)               (host-array form)
 *   rebalance copy-in host->peer (moe.py:191-195)   hv_batch_copy / hv_ce_batch_copy
 *   cudaMemcpyPeerAsync data path    hv_ce_batch_copy (baseline)
 *   expert_content / stable_hash64 content model    hv_fill_content, hv_digest,
 *     (moe.py:114-115, runtime.py:38-44)             hv_verify_content
 *   drain of in-flight transfers before free        hv_event_* (stream-ordered
 *     (runtime.py:345-356, :396-411)                 completion events)
 *
 * Conventions: C linkage, plain pointers and sizes, no C++ exceptions across
 * the ABI, no internal threads.  Every function returns an int status: 0 on
 * success, a negative HV_E* code otherwise (hv_error_string() describes it).
 * Stream arguments are cudaStream_t passed as void* (NULL = legacy default
 * stream of the current device).  "d_" pointers are device-visible addresses
 * (device memory, peer-mapped VA or the device alias of mapped pinned host
 * memory); "h_" pointers are host memory.  All copies are stream-ordered.
 */
#ifndef HARVEST_B200_H_
#define HARVEST_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HV_ABI_VERSION 1

/* ---- status codes ------------------------------------------------------ */
#define HV_OK 0
#define HV_E_INVALID (-1)      /* bad argument (ValueError in Python)            */
#define HV_E_NOCAPACITY (-2)   /* nothing fits (the reference returns None)      */
#define HV_E_DOUBLEFREE (-3)   /* memalloc.DoubleFreeError (memalloc.py:20-21)   */
#define HV_E_UNSUPPORTED (-4)  /* feature missing on this device/driver          */
#define HV_E_NOMEM (-5)        /* host allocation failed                         */
#define HV_E_CUDA_BASE (-1000) /* -1000 - cudaError_t                            */
#define HV_E_CU_BASE (-3000)   /* -3000 - CUresult (driver API)                  */

int hv_abi_version(void);
const char* hv_error_string(int status);

/* ---- devices ----------------------------------------------------------- */
int hv_device_count(int* n);
int hv_sm_count(int device, int* n);
/* can `reader` load from memory resident on `donor` (NVLink P2P)? */
int hv_can_access_peer(int reader, int donor, int* ok);
/* cudaDeviceEnablePeerAccess(donor) on `reader`; idempotent */
int hv_enable_peer_access(int reader, int donor);
int hv_device_synchronize(int device);
/* cudaMemGetInfo on `device`: the donor's real free HBM (co-tenant pressure) */
int hv_mem_get_info(int device, uint64_t* free_bytes, uint64_t* total_bytes);

/* ---- native best-fit segment allocator (memalloc.py:67-159) ------------- */
typedef struct hv_seg hv_seg;
/* usable = capacity - reserved - headroom (memalloc.py:43-45); one free
 * segment [0, usable) when usable > 0 (memalloc.py:74-79). */
int hv_seg_create(uint64_t usable, hv_seg** out);
int hv_seg_destroy(hv_seg* s);
/* alloc_best_fit (memalloc.py:90-114): min (leftover, base); HV_E_NOCAPACITY
 * if nothing fits. */
int hv_seg_alloc(hv_seg* s, uint64_t size, uint64_t* base_out);
/* best-fit probe without allocating: key (leftover, base) of the segment
 * alloc would take (runtime.py:155-167 scans the same key). */
int hv_seg_probe(const hv_seg* s, uint64_t size, uint64_t* leftover, uint64_t* base);
/* free_segment (memalloc.py:117-138): coalescing; HV_E_DOUBLEFREE if
 * (base,size) is not a live allocation. */
int hv_seg_free(hv_seg* s, uint64_t base, uint64_t size);
int hv_seg_allocated_bytes(const hv_seg* s, uint64_t* out);   /* memalloc.py:86-87 */
int hv_seg_free_bytes(const hv_seg* s, uint64_t* out);        /* memalloc.py:82-83 */
int hv_seg_num_free(const hv_seg* s, uint64_t* out);
/* copy out the base-sorted free list as (base,size) pairs; *n in = capacity
 * in pairs, out = pairs written (or needed when capacity is too small). */
int hv_seg_free_list(const hv_seg* s, uint64_t* pairs, uint64_t* n);
/* check_invariants (memalloc.py:141-159); HV_E_INVALID on violation */
int hv_seg_check(const hv_seg* s);

/* ---- native placement core (runtime.py:155-265) -------------------------
 * Donor choice for harvest_alloc under the four policies, the Fairness token
 * buckets (one per client index) and the Stability revocation windows.  The
 * placer borrows each donor's hv_seg (the caller keeps ownership). Times are
 * the runtime's clock in seconds. */
typedef struct hv_placer hv_placer;
#define HV_POLICY_BEST_FIT 0
#define HV_POLICY_LOCALITY 1
#define HV_POLICY_FAIRNESS 2
#define HV_POLICY_STABILITY 3
/* burst_bytes NaN = same as the budget (Policy.fairness_burst_bytes None) */
int hv_placer_create(int policy_kind, double budget_bytes_per_s, double burst_bytes,
                     double stability_window_s, int64_t stability_max_revocations,
                     hv_placer** out);
int hv_placer_destroy(hv_placer* p);
/* hops = topology hops from the compute device (Locality's first key) */
int hv_placer_add_donor(hv_placer* p, int device_id, hv_seg* seg, uint64_t ceiling, uint32_t hops);
/* harvestable ceiling of a donor (runtime.py:476-487 sets it) */
int hv_placer_set_ceiling(hv_placer* p, int device_id, uint64_t ceiling);
int hv_placer_ceiling(hv_placer* p, int device_id, uint64_t* out);
/* select_peer (runtime.py:169-196) over the listed donors: *device_out = the
 * chosen id, or -1 with HV_E_NOCAPACITY.  Refills the client's bucket under
 * Fairness, ages the revocation windows under Stability. */
int hv_placer_select(hv_placer* p, uint64_t size, uint32_t client, double now,
                     const int* candidates, int n_candidates, int* device_out);
/* harvest_alloc's choice (runtime.py:198-214): the preferred donors first,
 * then the others (all donors when n_preferred = 0), and the best-fit segment
 * taken on the chosen donor.  Tokens are not spent (hv_placer_spend, after
 * the donor's HBM is committed). */
int hv_placer_alloc(hv_placer* p, uint64_t size, uint32_t client, double now,
                    const int* preferred, int n_preferred, int* device_out, uint64_t* base_out);
int hv_placer_spend(hv_placer* p, uint32_t client, uint64_t size, double now); /* runtime.py:252-254 */
int hv_placer_tokens(hv_placer* p, uint32_t client, double now, double* out);  /* runtime.py:237-248 */
/* a finished revocation on the donor (runtime.py:267-268) */
int hv_placer_note_revocation(hv_placer* p, int device_id, double now);
int hv_placer_churn(hv_placer* p, int device_id, double now, int64_t* out);   /* runtime.py:256-265 */

/* ---- per-donor peer-memory pool ----------------------------------------- */
typedef struct hv_pool hv_pool;
#define HV_POOL_VMM 0u   /* cuMemAddressReserve + on-demand cuMemCreate/cuMemMap */
#define HV_POOL_IPC 1u   /* one cudaMalloc slab, exportable with cudaIpc          */
#define HV_POOL_EAGER 2u /* VMM: commit the whole range at creation               */
#define HV_POOL_REMOTE 4u /* VMM VA range only: chunks come from a donor process as
                             POSIX FDs (hv_pool_map_fd / hv_pool_unmap_chunk)       */
/* Reserve `bytes` of donor-resident memory, readable and writable by the
 * donor and every device in reader_devs.  VMM pools commit physical chunks of
 * `chunk_bytes` (rounded to the allocation granularity) on demand. */
int hv_pool_create(int donor_dev, uint64_t bytes, uint64_t chunk_bytes,
                   const int* reader_devs, int n_readers, unsigned flags,
                   hv_pool** out);
int hv_pool_destroy(hv_pool* p);
int hv_pool_info(const hv_pool* p, uint64_t* va, uint64_t* bytes,
                 uint64_t* chunk_bytes, int* donor_dev);
/* back [offset, offset+bytes) with physical donor memory (refcounted per
 * chunk); the harvest_alloc side of "allocates memory" */
int hv_pool_commit(hv_pool* p, uint64_t offset, uint64_t bytes);
/* drop the refcount; chunks reaching zero are unmapped and released back to
 * the donor.  Callers must have drained every reader first (runtime.py:396). */
int hv_pool_decommit(hv_pool* p, uint64_t offset, uint64_t bytes);
int hv_pool_committed_bytes(const hv_pool* p, uint64_t* out);
/* cross-process sharing (HV_POOL_IPC): 64-byte cudaIpcMemHandle_t */
int hv_pool_export_ipc(const hv_pool* p, void* handle64);
int hv_pool_import_ipc(const void* handle64, int donor_dev, uint64_t bytes,
                       int reader_dev, hv_pool** out);

/* Cross-process VMM donation (one process per GPU).  The donor process
 * creates a physical chunk on its GPU with a shareable POSIX-FD handle and
 * sends the FD to a reader (pool.DonorServer, SCM_RIGHTS over a Unix
 * socket); the reader maps it into an HV_POOL_REMOTE pool.  Revocation or
 * free: the reader unmaps (hv_pool_unmap_chunk), the donor releases its
 * handle (hv_chunk_release), and the HBM returns to the donor GPU -- the
 * reference's free_segment at the end of an ordered release
 * (runtime.py:396-411).  Granularity: hv_chunk_granularity. */
int hv_chunk_granularity(int device, uint64_t* out);
int hv_chunk_create_shareable(int device, uint64_t bytes, uint64_t* handle, int* fd);
int hv_chunk_release(uint64_t handle);
int hv_pool_map_fd(hv_pool* p, uint64_t chunk_index, int fd);
int hv_pool_unmap_chunk(hv_pool* p, uint64_t chunk_index);

/* ---- host tier: pinned, portable, mapped ------------------------------- */
int hv_host_alloc(uint64_t bytes, void** h_ptr, uint64_t* d_alias);
/* flags: HV_HOST_WRITE_COMBINED = cudaHostAllocWriteCombined (non-snooped
 * PCIe reads; CPU reads of the region become very slow) */
#define HV_HOST_WRITE_COMBINED 1u
int hv_host_alloc_flags(uint64_t bytes, unsigned flags, void** h_ptr, uint64_t* d_alias);
int hv_host_free(void* h_ptr);
/* pin an existing host range (cudaHostRegister, mapped+portable) */
int hv_host_register(void* h_ptr, uint64_t bytes, uint64_t* d_alias);
int hv_host_unregister(void* h_ptr);

/* ---- device scratch ------------------------------------------------------ */
int hv_dev_alloc(int device, uint64_t bytes, uint64_t* d_ptr);
int hv_dev_free(int device, uint64_t d_ptr);
int hv_memcpy_h2d(uint64_t d_dst, const void* h_src, uint64_t bytes, void* stream);
int hv_memcpy_d2h(void* h_dst, uint64_t d_src, uint64_t bytes, void* stream);
int hv_memset_d8(uint64_t d_dst, int value, uint64_t bytes, void* stream);

/* ---- streams and events (drain ordering, runtime.py:345-356) ----------- */
int hv_stream_create(int device, int priority, void** stream);
/* cudaDeviceGetStreamPriorityRange: greatest = most urgent (negative) */
int hv_stream_priority_range(int device, int* least, int* greatest);
/* graphs captured by the caller (e.g. torch.cuda.CUDAGraph(keep_graph=True)):
 * instantiate with HV_GRAPH_NODE_PRIORITY so kernel nodes keep the priority
 * of the stream they were captured from; launch on a stream; destroy */
#define HV_GRAPH_NODE_PRIORITY 1u
int hv_graph_instantiate(void* graph, unsigned flags, void** exec_out);
int hv_graph_launch(void* exec, void* stream);
int hv_graph_exec_destroy(void* exec);
int hv_stream_destroy(void* stream);
int hv_stream_synchronize(void* stream);
int hv_event_create(int device, unsigned timing, void** event);
int hv_event_destroy(void* event);
int hv_event_record(void* event, void* stream);
/* *done = 1 if every op captured by the event has completed */
int hv_event_query(void* event, int* done);
int hv_event_synchronize(void* event);
int hv_event_elapsed_ms(void* start, void* stop, float* ms);
int hv_stream_wait_event(void* stream, void* event);

/* ---- fetch engines (the hot path) ------------------------------------- */
/* engine selector for hv_batch_copy / hv_kv_gather */
#define HV_ENGINE_AUTO 0   /* LDG; variable-size copies also take HV_ENGINE_FLAG_INTERLEAVE.
                              hv_swap_blocks_batch: engine per source -- objects of >= 1 MiB read
                              from or written to the pinned host tier (hv_host_alloc /
                              hv_host_register ranges) go to the copy engine, the rest to the LDG
                              kernel, concurrently */
#define HV_ENGINE_LDG 1  /* SM-issued 128-bit ld.global.nc / st.global, warp per 4 KiB chunk */
#define HV_ENGINE_TMA 2  /* cp.async.bulk global->smem->global ring, one issuing lane per CTA */
#define HV_ENGINE_LDG256 3 /* LDG with the L2::256B sector-promotion hint (larger remote reads) */
#define HV_ENGINE_LDG16 4  /* LDG with 16 x 128-bit loads in flight per lane (8 KiB per warp) */
#define HV_ENGINE_CE 5     /* host-array entry points: every object through the copy engine
                              (cudaMemcpyAsync per contiguous run); device-array entry points, which the copy
                              engine cannot serve, treat it as HV_ENGINE_AUTO */
/* OR-able flag for the variable-size copies (hv_batch_copy, hv_swap_blocks_batch):
 * when every non-empty object of a launch has the same size, chunk c reads
 * object (c mod n_active) at chunk (c div n_active), so the bytes in flight
 * span every object -- and every donor GPU holding one -- at once. */
#define HV_ENGINE_FLAG_INTERLEAVE 0x100

/* K1: block-table-indexed KV-page gather.  Page i is copied from
 * d_src_page_ptrs[i] to d_dst_page_ptrs[i] (or, when d_dst_page_ptrs is NULL,
 * to d_dst_base + i*page_bytes).  Sources may be on any donor, local or the
 * host tier; one launch moves every page.  max_ctas caps the grid (0 = fill
 * the device) so the gather can share SMs with decode compute.  Replaces one
 * app_transfer per KV block (runtime.py:320-364). */
int hv_kv_gather(const uint64_t* d_src_page_ptrs, const uint64_t* d_dst_page_ptrs,
                 uint64_t d_dst_base, uint32_t n_pages, uint64_t page_bytes,
                 int engine, int max_ctas, void* stream);

/* K1 with the block table resolved on the device: page i comes from
 *   d_slot_base[loc >> 32] + (loc & 0xffffffff) * page_bytes,
 * loc = d_locs[i] (base index, slot).  Avoids shipping one pointer per page. */
int hv_kv_gather_table(const uint64_t* d_slot_bases, const uint64_t* d_locs,
                       uint64_t d_dst_base, const uint64_t* d_dst_page_ptrs,
                       uint32_t n_pages, uint64_t page_bytes, int engine,
                       int max_ctas, void* stream);

/* K1 over a block table with per-layer strides (a paged KV cache moved whole
 * blocks at a time: evict / reload).  Page (l, b), for
 * l < n_layers and b < n_blocks, is copied from
 *   d_src_base[b] + l * d_src_stride[b]  to  d_dst_base[b] + l * d_dst_stride[b].
 * Four n_blocks-long arrays describe n_blocks * n_layers pages. */
int hv_kv_gather_blocks(const uint64_t* d_src_base, const uint64_t* d_src_stride,
                        const uint64_t* d_dst_base, const uint64_t* d_dst_stride,
                        uint32_t n_blocks, uint32_t n_layers, uint64_t page_bytes,
                        int engine, int max_ctas, void* stream);

/* hv_kv_gather_blocks with host arrays: staged through the library's pinned
 * ring and uploaded by an SM kernel (never a DMA queued behind bulk
 * copy-engine traffic), one launch per 1,536 blocks. */
int hv_kv_gather_blocks_h(const uint64_t* h_src_base, const uint64_t* h_src_stride,
                          const uint64_t* h_dst_base, const uint64_t* h_dst_stride,
                          uint32_t n_blocks, uint32_t n_layers, uint64_t page_bytes,
                          int engine, int max_ctas, void* stream);

/* K2: variable-size batched fetch (expert weights, placement copy-in):
 * d_src[i] -> d_dst[i], d_bytes[i] bytes, for i < n.  One launch for a whole
 * pipeline stage (moe.py:282-313). */
int hv_batch_copy(const uint64_t* d_src, const uint64_t* d_dst, const uint64_t* d_bytes,
                  uint32_t n, int engine, int max_ctas, void* stream);

/* vLLM-compatible host-array form of K2 (swap_blocks_batch(src_ptrs,
 * dst_ptrs, sizes), vllm/_custom_ops.py:2681-2703): the arrays are staged
 * through a pinned ring and uploaded on `stream` before the launch. */
int hv_swap_blocks_batch(const uint64_t* h_src, const uint64_t* h_dst,
                         const uint64_t* h_bytes, uint32_t n, int engine,
                         int max_ctas, void* stream);

/* Copy-engine baselines: per-object cudaMemcpyAsync (peer copies route over
 * NVLink via UVA, i.e. cudaMemcpyPeerAsync) when batched == 0,
 * when batched == 1, objects whose source and destination both continue the
 * previous object's are merged into one larger cudaMemcpyAsync. Host arrays. */
int hv_ce_batch_copy(const uint64_t* h_src, const uint64_t* h_dst,
                     const uint64_t* h_bytes, uint32_t n, int batched, void* stream);

/* ---- fused consumer: expert FFN over the expert's resident copy ---------- */
/* The decode stage's compute (moe.py:315-340) reading each expert object in
 * place -- donor HBM over NVLink, pinned host over PCIe, or local HBM --
 * instead of after a K2 fetch into local staging: weight tiles stream through
 * shared memory (cp.async) into mma.sync, so the transfer overlaps the math
 * and the bytes cross the link once.  Object layout: gate [I][H], up [I][H],
 * down [H][I], bf16.  Routed pairs are sorted by expert: expert e (of
 * n_experts) owns pairs d_offs[e] .. d_offs[e] + d_counts[e] - 1, at most
 * hv_expert_ffn_max_tokens() of them.  Requires H % 64 == 0 and I % 64 == 0,
 * expert objects and activation rows 16-byte aligned (cp.async granules;
 * expert sizes that are multiples of 16, as every bf16 [I][H] stack is, keep
 * the runtime's segment bases aligned).
 *   gate_up: act[p][i] = silu(gate[i] . x[tok[p]]) * (up[i] . x[tok[p]])  (bf16 [P][I])
 *   down:    y[p][h]   = down[h] . act[p]                                  (fp32 [P][H]) */
int hv_expert_ffn_gate_up(const uint64_t* d_w_addr, const int32_t* d_counts, const int32_t* d_offs,
                          const int32_t* d_tok, const void* d_x, void* d_act, uint32_t n_experts,
                          uint32_t hidden, uint32_t intermediate, void* stream);
int hv_expert_ffn_down(const uint64_t* d_w_addr, const int32_t* d_counts, const int32_t* d_offs,
                       const void* d_act, float* d_y, uint32_t n_experts, uint32_t hidden,
                       uint32_t intermediate, void* stream);
int hv_expert_ffn_max_tokens(int* out);
/* hv_expert_ffn_down with flags.  HV_FFN_OVERLAP_PREVIOUS launches it with
 * programmatic stream serialization right behind hv_expert_ffn_gate_up on the
 * same stream: its CTAs start streaming expert weight tiles while gate/up
 * drains and read d_act only after that kernel completes.  The caller
 * guarantees d_w_addr / d_counts / d_offs were complete before gate/up
 * started (they are its own inputs).  Measured on B200 it does not pay
 * (Qwen stage 201.5 vs 195.4 us); the decoder uses the plain launch. */
#define HV_FFN_OVERLAP_PREVIOUS 1u
/* HV_FFN_TILED: the expert's matrices are stored pre-tiled for the tensor
 * cores -- matrix [R][K] bf16 as [R/128][K/64] contiguous 16 KiB tiles, tile
 * row r holding columns 64*kt .. 64*kt+63 of row 128*rb + r with its 16-byte
 * chunk c at chunk (c ^ (r & 7)) (UMMA's 128B-swizzled K-major layout), the
 * matrices at the same offsets as the row-major form.  Each tile then reaches
 * shared memory as one bulk copy on the TMA engine instead of 1,024 16-byte
 * cp.async.  Requires R % 128 == 0 (the tcgen05 kernel); results are bitwise
 * those of the row-major form on the same logical weights
 * (fetch.tile_expert_matrix writes the layout). */
#define HV_FFN_TILED 2u
/* HV_FFN_WAIT_PREVIOUS: launched with programmatic stream serialization
 * behind a kernel that may have written any input (the router of the same
 * stage): the CTAs' prologue (TMEM allocation, barriers) overlaps its tail
 * and every input is read after griddepcontrol.wait.  Rows % 128 == 0.
 * HV_FFN_OVERLAP_PREVIOUS on hv_expert_ffn_down_ex (rows % 128 == 0: the
 * tcgen05 kernel) streams the first stages' weight tiles before the wait. */
#define HV_FFN_WAIT_PREVIOUS 4u
int hv_expert_ffn_gate_up_ex(const uint64_t* d_w_addr, const int32_t* d_counts, const int32_t* d_offs,
                             const int32_t* d_tok, const void* d_x, void* d_act, uint32_t n_experts,
                             uint32_t hidden, uint32_t intermediate, unsigned flags, void* stream);
int hv_expert_ffn_down_ex(const uint64_t* d_w_addr, const int32_t* d_counts, const int32_t* d_offs,
                          const void* d_act, float* d_y, uint32_t n_experts, uint32_t hidden,
                          uint32_t intermediate, unsigned flags, void* stream);

/* ---- MoE decode glue around K4: router and top-k combine ------------------ */
/* The fused decoder's per-stage router (moe.py:315-340 stage semantics; the
 * reference models the compute as a constant): logits =
 * h . router^T in fp32 (d_h bf16 [tokens][hidden], d_router bf16
 * [n_experts][hidden], 16-byte aligned), per token the top_k experts (largest
 * first, ties to the lower id), softmax over their logits -> d_probs
 * [tokens][top_k] and d_topi (int64), the routed pairs (t, j) sorted by expert
 * (stable): d_counts / d_offs [n_experts], d_tok [tokens*top_k] (token of each
 * sorted pair), d_pos [tokens*top_k] (sorted position of pair t*top_k + j) --
 * the inputs of hv_expert_ffn_*.  d_logits: [tokens][n_experts] fp32 scratch;
 * d_ticket: one unsigned, zero before the first launch (the kernel re-arms it),
 * not shared by concurrent launches.  tokens <= 256, n_experts <= 256,
 * top_k <= 8.  One launch. */
/* HV_MOE_OVERLAP_PREVIOUS (route, combine): launched with programmatic stream
 * serialization; the kernel waits for the previous one before reading. */
#define HV_MOE_OVERLAP_PREVIOUS 1u
int hv_moe_route(const void* d_h, const void* d_router, uint32_t tokens, uint32_t hidden, uint32_t n_experts,
                 uint32_t top_k, float* d_logits, float* d_probs, int64_t* d_topi, int32_t* d_counts,
                 int32_t* d_offs, int32_t* d_tok, int64_t* d_pos, unsigned* d_ticket, unsigned flags,
                 void* stream);
/* h[t] <- h[t] + rs * bf16(sum_j probs[t][j] * y[pos[t*top_k + j]]) in bf16,
 * j in order (deterministic); d_y fp32 [tokens*top_k][hidden] (K4 down's
 * output), d_h bf16 [tokens][hidden] updated in place. */
/* The fused decoder's staging plan for one stage: expert e is staged iff
 * d_counts[e] > 0 and d_host[e] (its copy is in the pinned host tier); staged
 * experts take consecutive slots of slot_bytes from slot_base in expert order:
 * d_dst[e] / d_sizes[e] (0 when not staged) describe its K2 fetch and
 * d_addr_out[e] is where K4 then reads it (the slot, or d_addr[e] in place). */
int hv_moe_stage_plan(const int32_t* d_counts, const uint64_t* d_addr, const uint8_t* d_host, uint64_t slot_base,
                      uint64_t slot_bytes, uint32_t n_experts, uint64_t* d_dst, uint64_t* d_sizes,
                      uint64_t* d_addr_out, void* stream);
int hv_moe_combine(const float* d_y, const float* d_probs, const int64_t* d_pos, void* d_h, uint32_t tokens,
                   uint32_t hidden, uint32_t top_k, float residual_scale, unsigned flags, void* stream);

/* ---- paged decode attention over KV pages in any tier -------------------- */
/* One query token per sequence, grouped-query (q_heads = g * kv_heads,
 * g in {1, 2, 4, 8}), head_dim 64 or 128, 16-token blocks.  d_page_ptrs holds
 * one page pointer per block (this layer), sequence-major; sequence b owns
 * blocks d_seq_start[b] .. d_seq_start[b+1]-1 and d_seq_tokens[b] tokens.
 * Page layout: K [16][kv_heads][D] then V [16][kv_heads][D], fp16.  Pages
 * may be a K1-gathered buffer or the pages in place (local, peer, host);
 * each page 16-byte aligned.
 * d_q: [batch][q_heads][D] fp16; d_out: [batch][q_heads][D] fp32;
 * d_part: workspace of batch*kv_heads*splits*g*(D+2) floats.  Flash-decoding
 * over `splits` block ranges per (sequence, KV head), merged in a fixed
 * order: the result depends only on the bytes. */
int hv_paged_decode_attention(const uint64_t* d_page_ptrs, const int32_t* d_seq_start,
                              const int32_t* d_seq_tokens, const void* d_q, float* d_out, float* d_part,
                              uint32_t batch, uint32_t q_heads, uint32_t kv_heads, uint32_t head_dim,
                              uint32_t block_tokens, uint32_t splits, float scale, void* stream);

/* hv_paged_decode_attention with flags.  HV_ATTN_OVERLAP_PREVIOUS launches
 * the kernel with programmatic stream serialization: its CTAs start while
 * the previous kernel on the stream drains, read pages / q / the sequence
 * arrays, and wait for that kernel only before their first write.  The
 * caller guarantees those inputs were not produced by the immediately
 * preceding kernel on the stream (true for the layers of a decode step:
 * the previous kernel is the previous layer's attention). */
#define HV_ATTN_OVERLAP_PREVIOUS 1u
/* HV_ATTN_BALANCED: balanced (stream-K) flash decoding.  `splits` is then the
 * number of CTAs (one per SM is the intended size): the (sequence, KV head,
 * 16-token block) units of the live blocks are cut into `splits` equal
 * contiguous ranges, so every SM streams the same bytes whatever the
 * sequence count; d_part must hold (splits + batch*kv_heads)*g*(D+2) floats;
 * batch <= 256.  Deterministic for a given `splits`. */
#define HV_ATTN_BALANCED 2u
int hv_paged_decode_attention_ex(const uint64_t* d_page_ptrs, const int32_t* d_seq_start,
                                 const int32_t* d_seq_tokens, const void* d_q, float* d_out, float* d_part,
                                 uint32_t batch, uint32_t q_heads, uint32_t kv_heads, uint32_t head_dim,
                                 uint32_t block_tokens, uint32_t splits, float scale, unsigned flags,
                                 void* stream);

/* ---- synthetic content (test / bench inputs) --------------------------- */
/* byte j of object = byte (j%8) (little-endian) of splitmix64 word j/8:
 *   w_i = fmix(seed + (i+1)*0x9E3779B97F4A7C15)
 * seeded by stable_hash64(tag) (runtime.py:38-44). */
int hv_fill_content(const uint64_t* d_dst, const uint64_t* d_bytes,
                    const uint64_t* d_seeds, uint32_t n, void* stream);
/* the same stream as bf16 expert weights: each 16-bit lane becomes
 * (lane & 0x807F) | 0x3C00, a finite value with |w| in [2^-7, 2^-6) */
int hv_fill_weights_bf16(const uint64_t* d_dst, const uint64_t* d_bytes,
                         const uint64_t* d_seeds, uint32_t n, void* stream);
/* position-keyed 64-bit digest per object (see oracle/hv_oracle.c) */
int hv_digest(const uint64_t* d_src, const uint64_t* d_bytes, uint32_t n,
              uint64_t* d_out, void* stream);
/* Per-fetch content identity (read_errors, moe.py:315-319), on bytes and
 * for any content: digest each fetched object (d_scratch: n words), compare
 * with d_expected (the digests of the authoritative copies), set
 * d_flags[i] = 1 for a mismatch (d_flags may be NULL) and add the number of
 * mismatching objects to *d_errors.  Stream-ordered; nothing is read back. */
int hv_check_digests(const uint64_t* d_src, const uint64_t* d_bytes, const uint64_t* d_expected,
                     uint32_t n, uint64_t* d_scratch, uint8_t* d_flags, uint64_t* d_errors,
                     void* stream);
/* hv_check_digests with host arrays (staged through the pinned ring like
 * hv_swap_blocks_batch): the form the fetch hook calls once per stage. */
int hv_check_digests_batch(const uint64_t* h_src, const uint64_t* h_bytes, const uint64_t* h_expected,
                           uint32_t n, uint64_t* d_scratch, uint8_t* d_flags, uint64_t* d_errors,
                           void* stream);
/* The fetch and its content check in one pass: hv_swap_blocks_batch's
 * engine per source, where every object the SM kernel moves is digested by
 * the same pass that copies it (no re-read, no second kernel), objects the
 * copy engine moves (large host-tier ones) are digested on the side stream
 * after their copy, and the digests are compared with h_expected as in
 * hv_check_digests (flags, *d_errors += mismatches).  d_scratch: n words. */
int hv_swap_blocks_batch_checked(const uint64_t* h_src, const uint64_t* h_dst, const uint64_t* h_bytes,
                                 const uint64_t* h_expected, uint32_t n, int engine, int max_ctas,
                                 uint64_t* d_scratch, uint8_t* d_flags, uint64_t* d_errors, void* stream);
/* count of 8-byte words differing from the generator, per object */
int hv_verify_content(const uint64_t* d_src, const uint64_t* d_bytes,
                      const uint64_t* d_seeds, uint32_t n, uint64_t* d_mismatch,
                      void* stream);

/* hv_verify_content against the bf16-weights variant (hv_fill_weights_bf16) */
int hv_verify_weights_bf16(const uint64_t* d_src, const uint64_t* d_bytes,
                           const uint64_t* d_seeds, uint32_t n, uint64_t* d_mismatch,
                           void* stream);
/* number of kernel launches issued by this library in this process */
int hv_launch_count(uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* HARVEST_B200_H_ */
