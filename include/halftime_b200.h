/*
 * halftime_b200.h -- C-ABI of the B200-native HalftimeHash engine
 * (libhalftime_b200.so).  Plain pointers and sizes only; no torch types.
 *
 * The reference (halftimehash 0.1.0, /root/reference/pkg/src/halftimehash)
 * is a pure-Python package with no FFI.  Its only plug-in point is the
 * `engine` string of `hash_bytes` (hasher.py:434-453); each entry point
 * below is what that dispatch (and the batched seam `_hash_words_np`,
 * hasher.py:331-413) would bind through ctypes.  INTEGRATION.md shows the
 * binding a maintainer would add.
 *
 * Conventions
 *  - Return 0 on success or a negative HTH_E* code; the message is in
 *    hth_last_error() (thread-local).  Never aborts.
 *  - Error mapping to the reference's exceptions:
 *      HTH_EINVAL    -> ValueError   (unsupported width params.py:230-237,
 *                                     bad master hasher.py:48-50, bad args)
 *      HTH_ESEEDSIZE -> SeedSizeError (hasher.py:36-37, 209-214)
 *      HTH_ERANGE    -> IndexError    (hasher.py:84-97)
 *      HTH_ECUDA / HTH_ENOMEM -> RuntimeError / MemoryError
 *  - Device entry points are stream-ordered on `stream` (a cudaStream_t,
 *    NULL = legacy default stream) and asynchronous.
 *  - Device input buffers may start at any byte address.  The engine reads
 *    whole 16-byte granules (TMA bulk copies), i.e. from the granule holding
 *    the first byte to the one holding the last; those never cross a page
 *    boundary, so any cudaMalloc / torch allocation (or view into one) is
 *    safe.
 *  - Digests are written as n_strings x k little-endian u64 words,
 *    k = output_bytes / 8 (Digest.words, hasher.py:165-176).
 *  - hth_hash_fixed workspaces must be zero-filled before their first use
 *    (one cudaMemset after allocation).  Every completed call leaves the
 *    workspace zero-filled again (self-resetting counters/accumulators,
 *    consumed subtree blocks cleared), so it is reused across calls on one
 *    stream without clearing and the hot path is a single kernel launch.
 *    hth_hash_varlen workspaces likewise: zero-filled before the first use;
 *    the engine clears their counter region itself on the first call with
 *    each batch layout (n_strings, total_bytes, variant) and otherwise relies
 *    on the kernels leaving it zeroed, so a repeated batch shape is two
 *    launches and no memset.  Do not write into a workspace between calls;
 *    one that hth_hash_varlen used must be re-zeroed (hth_workspace_reset)
 *    before hth_hash_fixed uses it.  Concurrent calls need distinct
 *    workspaces.
 *  - Seeds (SeedBuffer, hasher.py:70-102): seed_fold is the master fold
 *    (hth_master_fold) and d_seed holds its expansion S[0..seed_capacity)
 *    (hth_expand_seed(seed_fold, 0, seed_capacity, d_seed), i.e.
 *    SeedBuffer.words_np).  The first e*w words are recomputed from the fold
 *    on the host and travel in the kernel's constant-bank parameters; the
 *    rest are read from d_seed.  Any capacity >= the layout total is
 *    accepted and gives identical digests (hasher.py:8-10).
 */
#ifndef HALFTIME_B200_H
#define HALFTIME_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HTH_OK 0
#define HTH_EINVAL (-1)
#define HTH_ESEEDSIZE (-2)
#define HTH_ERANGE (-3)
#define HTH_ECUDA (-4)
#define HTH_ENOMEM (-5)

/* seed_capacity of the host entry points: size the seed stream exactly
 * (seed_for_input, hasher.py:160-162) instead of checking a capacity. */
#define HTH_SEED_AUTO UINT64_MAX

/* Last error message of the calling thread ("" if none). */
const char* hth_last_error(void);

/* ABI version (major*100 + minor). */
int hth_version(void);

/* params.variant(output_bytes) geometry (params.py:133-237): k, e, d, w and
 * words per instance m = d*w*8.  HTH_EINVAL for widths other than 16/24/32/40. */
int hth_variant_geometry(int output_bytes, int* k, int* e, int* d, int* w, int* instance_words);

/* seed_words_needed(params, n_bytes)  (hasher.py:156-158). */
int hth_seed_words_needed(int output_bytes, uint64_t n_bytes, uint64_t* out_words);

/* seed_layout(params, n_bytes)  (hasher.py:130-153) as 10 words:
 * levels, ehc_start, ehc_words, tree_start, tree_words_per_tree,
 * finalize_start, finalize_words_per_tree, remainder_start, remainder_words,
 * total_words. */
int hth_seed_layout(int output_bytes, uint64_t n_bytes, uint64_t out10[10]);

/* _master_fold (hasher.py:48-52): XOR of the four LE u64 of a 32-byte master. */
int hth_master_fold(const uint8_t master[32], uint64_t* fold);

/* SeedBuffer.words_np(start, count) on the device  (hasher.py:55-67, 94-97):
 * d_words[i] = mix(fold + (start + i + 1) * 0x9E3779B97F4A7C15). */
int hth_expand_seed(uint64_t fold, uint64_t start, uint64_t count, uint64_t* d_words, void* stream);

/* hash_remainder (hasher.py:186-206) on the device, for callers of the
 * reference's component API: d_out[r] = sum_{i<n} NH(d_tail[i],
 * d_keys[r + i]) for r < k (32-bit halves, the Toeplitz windows of the
 * remainder region).  HTH_EINVAL ("remainder key region too short") when
 * n_keys < n + k - 1, as the reference raises ValueError. */
int hth_toeplitz_nh(const uint64_t* d_tail, uint64_t n, const uint64_t* d_keys, uint64_t n_keys, int k,
                    uint64_t* d_out, void* stream);

/* cli.fill_bytes (cli.py:48-53) on the device: n_bytes of the splitmix stream
 * keyed by fill_seed, starting at stream word `word_offset`. */
int hth_fill_splitmix(uint64_t fill_seed, uint64_t word_offset, uint64_t n_bytes, void* d_dst, void* stream);
/* One launch for a shard of a packed batch of n_bytes-strings (n_bytes % 8
 * == 0): local string i (at d_dst + i * dst_stride) = global string
 * first_string + i * string_step, i.e. stream words from
 * (first_string + i * string_step) * n_bytes / 8 on. */
int hth_fill_splitmix_strings(uint64_t fill_seed, uint64_t n_strings, uint64_t n_bytes, uint64_t first_string,
                              uint64_t string_step, void* d_dst, uint64_t dst_stride, void* stream);

/* ---- batched hash of equal-length strings: the _hash_words_np seam
 *      (hasher.py:331-413) for B = n_strings rows sharing n_bytes.
 * String s starts at d_data + s * stride_bytes.  Workspace: at least
 * hth_workspace_size_fixed() bytes of device memory (NULL if that is 0). */
int hth_workspace_size_fixed(int output_bytes, uint64_t n_strings, uint64_t n_bytes, uint64_t* bytes);
int hth_hash_fixed(int output_bytes, const void* d_data, uint64_t n_strings, uint64_t stride_bytes,
                   uint64_t n_bytes, uint64_t seed_fold, const uint64_t* d_seed, uint64_t seed_capacity,
                   uint64_t* d_out, void* d_workspace, uint64_t workspace_bytes, void* stream);

/* ---- many seeds: the batched seam with per-row seed streams
 * (hasher.py:331-413 with a (B, 1) fold array, tests/test_hasher.py:254-310).
 * String s is hashed under the SeedBuffer whose fold is d_folds[s] (every
 * seed word recomputed on the device, so there is no capacity to check).
 * stride_bytes may be 0: one input hashed under n_strings seeds.  Workspace:
 * hth_workspace_size_fixed, zero-filled once. */
int hth_hash_fixed_folds(int output_bytes, const void* d_data, uint64_t n_strings, uint64_t stride_bytes,
                         uint64_t n_bytes, const uint64_t* d_folds, uint64_t* d_out, void* d_workspace,
                         uint64_t workspace_bytes, void* stream);

/* ---- batched hash of variable-length strings packed in one buffer.
 * String s is d_data[d_offsets[s] .. d_offsets[s+1]) (u64 byte offsets on the
 * device, any alignment).  max_n_bytes: an upper bound on any string's
 * length, checked against seed_capacity on the host (SeedSizeError); strings
 * longer than it are flagged (hth_varlen_status).  total_bytes sizes the
 * workspace (>= d_offsets[n] - d_offsets[0]). */
int hth_workspace_size_varlen(int output_bytes, uint64_t n_strings, uint64_t total_bytes, uint64_t* bytes);
int hth_hash_varlen(int output_bytes, const void* d_data, const uint64_t* d_offsets, uint64_t n_strings,
                    uint64_t max_n_bytes, uint64_t total_bytes, uint64_t seed_fold, const uint64_t* d_seed,
                    uint64_t seed_capacity, uint64_t* d_out, void* d_workspace, uint64_t workspace_bytes,
                    void* stream);
/* Synchronizes `stream`; returns HTH_ESEEDSIZE if a varlen call on this
 * workspace since the previous status read met a string longer than its
 * max_n_bytes, HTH_EINVAL if offsets decreased or ran past total_bytes, else
 * HTH_OK (the reference raises SeedSizeError / ValueError for these,
 * hasher.py:209-214).  Reading clears the flags. */
int hth_varlen_status(void* d_workspace, void* stream);

/* Re-zero a workspace (stream-ordered).  The device entry points already do
 * this themselves when a launch fails; callers that abandon a workspace
 * mid-stream (e.g. after an error of their own) can use it too. */
int hth_workspace_reset(void* d_workspace, uint64_t workspace_bytes, void* stream);

/* ---- one string split across devices (config 5): the reference's stack
 * construction is front-aligned (tree.py:63-100), so a string cut at
 * multiples of 8^c instances splits into independent level-c subtrees.
 * hth_slice_plan: instance bounds of n_slices balanced slices (the last one
 * also takes the ragged end and the tail), the frontier level c, and how
 * many level-c subtree roots each slice emits.
 * hth_hash_slice: hash instances [inst_begin, inst_end) of a string of
 * n_bytes; d_slice holds its bytes from inst_begin*m*8 up to inst_end*m*8 (or
 * to n_bytes for the last slice).  Writes the slice's frontier (count from
 * the plan, k*8 u64 per root) and zeroes then fills d_partial (k words).
 * Workspace: hth_workspace_size_slice, zero-filled like hth_hash_fixed's.
 * hth_hash_merge: given all slices' frontiers concatenated in slice order and
 * their partials, finishes the tree and writes the k digest words.
 * Workspace: >= 16*k*(n_frontier/8 + 8)*8 bytes. */
int hth_slice_plan(int output_bytes, uint64_t n_bytes, uint64_t n_slices, uint64_t* inst_bounds, int* frontier_level,
                   uint64_t* frontier_counts);
int hth_workspace_size_slice(int output_bytes, uint64_t n_bytes, uint64_t* bytes);
int hth_hash_slice(int output_bytes, const void* d_slice, uint64_t n_bytes, uint64_t inst_begin, uint64_t inst_end,
                   int frontier_level, uint64_t seed_fold, const uint64_t* d_seed, uint64_t seed_capacity,
                   uint64_t* d_frontier, uint64_t* d_partial, void* d_workspace, uint64_t workspace_bytes,
                   void* stream);
int hth_hash_merge(int output_bytes, uint64_t n_bytes, int frontier_level, const uint64_t* d_frontier,
                   uint64_t n_frontier, const uint64_t* d_partials, uint64_t n_partials, uint64_t seed_fold,
                   const uint64_t* d_seed, uint64_t seed_capacity, uint64_t* d_out, void* d_workspace,
                   uint64_t workspace_bytes, void* stream);
/* Peer-memory exchange for the split string (no reference counterpart: the
 * reference is single-process).  Rank 0 exports its gather buffer
 * (hth_ipc_get_handle: 64 opaque bytes naming the enclosing allocation, plus
 * the buffer's byte offset inside it, sent to the other ranks); each rank
 * maps it (hth_ipc_open_handle, peer access over NVLink), adds the offset and
 * passes pointers into it as hth_hash_slice's d_frontier / d_partial, so the
 * slice kernel itself stores its subtree roots and partial digest into rank
 * 0's memory.  hth_ipc_close_handle unmaps (the mapped base). */
/* In-stream exchange (no host synchronisation on the data path).
 * hth_hash_slice_ex = hth_hash_slice plus: when the slice is done, its
 * kernel's last warp stores done_value to *d_done_flag with a system-scope
 * release after every frontier/partial store of the slice is visible
 * system-wide (d_done_flag, like d_frontier/d_partial, may be a peer GPU's
 * memory).  options HTH_SLICE_ACCUMULATE: d_partial already holds zeros
 * (the merge re-zeroes it), so it is not cleared first.
 * hth_hash_merge_ex = hth_hash_merge whose kernel first waits until each of
 * the n_partials flags d_flags[i] >= epoch (system-scope acquire), and after
 * writing the digest zeroes d_partials and stores epoch to *d_consumed
 * (release) so producers may reuse the buffers.  A wait longer than
 * timeout_ns sets *d_status = 1 instead of hanging (digest then invalid).
 * hth_signal / hth_wait_flag: the same release store / bounded acquire spin
 * as a one-thread launch.  Waiting kernels must only ever wait on work
 * running on ANOTHER GPU (or already completed): two ranks sharing one
 * device are not guaranteed to run concurrently. */
#define HTH_SLICE_ACCUMULATE 1
int hth_hash_slice_ex(int output_bytes, const void* d_slice, uint64_t n_bytes, uint64_t inst_begin, uint64_t inst_end,
                      int frontier_level, uint64_t seed_fold, const uint64_t* d_seed, uint64_t seed_capacity,
                      uint64_t* d_frontier, uint64_t* d_partial, uint64_t* d_done_flag, uint64_t done_value,
                      int options, void* d_workspace, uint64_t workspace_bytes, void* stream);
int hth_hash_merge_ex(int output_bytes, uint64_t n_bytes, int frontier_level, const uint64_t* d_frontier,
                      uint64_t n_frontier, uint64_t* d_partials, uint64_t n_partials, const uint64_t* d_seed,
                      uint64_t seed_capacity, uint64_t* d_out, const uint64_t* d_flags, uint64_t epoch,
                      uint64_t* d_consumed, uint64_t timeout_ns, int* d_status, void* d_workspace,
                      uint64_t workspace_bytes, void* stream);
int hth_signal(uint64_t* d_flag, uint64_t value, void* stream);
int hth_wait_flag(const uint64_t* d_flag, uint64_t value, uint64_t timeout_ns, int* d_status, void* stream);

int hth_ipc_get_handle(const void* d_ptr, uint8_t handle_out[64], uint64_t* offset_out);
int hth_ipc_open_handle(const uint8_t handle[64], void** d_ptr_out);
int hth_ipc_close_handle(void* d_ptr);

/* ---- host-buffer entry points (end-to-end; synchronous).  These are what
 * hash_bytes(..., engine="cuda") binds (hasher.py:434-453): host bytes in,
 * host digest words out, seeds expanded on the device from the 32-byte
 * master (cached per calling thread while the master stays the same).
 * Calls up to 256 KiB run on one stream through pinned staging; larger ones
 * pipeline ~64 MiB chunks of whole strings over three streams (copy of chunk
 * i+1 against the hash of chunk i).  Pinned (page-locked) h_data goes
 * straight to the copy engine at the full PCIe rate; pageable h_data >= 8 MiB
 * is staged through pinned slots by a multi-threaded memcpy.
 * Strings longer than 64 MiB are streamed in 64 MiB slices of whole
 * subtrees (hth_hash_slice + hth_hash_merge), so device memory stays bounded
 * (about 3 x 64 MiB) whatever the input size.
 * seed_capacity emulates SeedBuffer.capacity: HTH_ESEEDSIZE if it is below
 * seed_words_needed (HTH_SEED_AUTO = size it exactly, like seed_for_input).
 * Each calling thread keeps its streams and buffers for reuse until it exits
 * or calls hth_host_release. */
int hth_hash_host(int output_bytes, const void* h_data, uint64_t n_bytes, const uint8_t master[32],
                  uint64_t seed_capacity, uint64_t* h_out, int device);
int hth_hash_fixed_host(int output_bytes, const void* h_data, uint64_t n_strings, uint64_t stride_bytes,
                        uint64_t n_bytes, const uint8_t master[32], uint64_t seed_capacity, uint64_t* h_out,
                        int device);
/* Free the calling thread's host-path streams and buffers (device and pinned). */
int hth_host_release(void);

#ifdef __cplusplus
}
#endif
#endif /* HALFTIME_B200_H */
