/*
 * hqmq_b200 — C ABI of the B200-native HQMQ KV-cache codec.
 *
 * Drop-in boundary for the reference package's codec path
 * (/root/reference/pkg/src/hqmq/).  Every entry point takes plain device
 * pointers and sizes (caller-allocated, e.g. by torch), is asynchronous on the
 * caller's CUDA stream (`stream` is a cudaStream_t passed as void*; NULL = the
 * legacy default stream), and returns an hqmq_status.  The only mutable
 * library state is per thread: the last error text (hqmq_last_error) and a
 * small cache of occupancy queries keyed by (kernel, shared memory, device)
 * that sizes the decode grids; calls are reentrant across streams and
 * devices (the kernel launches on the calling thread's current device).  Data-dependent failures that the reference raises as Python
 * exceptions are reported through a device-resident error word (HQMQ_DEVERR_*)
 * that the host maps to the reference's exception types after it synchronises.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/hqmq):
 *   hqmq_nearest_scan        <- _kernels.nearest_scan        (_kernels.pyx:16-46,
 *                               dispatched by kernels.nearest_scan, kernels.py:54-63)
 *   hqmq_encode              <- codec.encode_tensor          (codec.py:232-287),
 *                               including outliers.lower_median (outliers.py:50-55),
 *                               radius.quantize_radii (radius.py:35-47) and the
 *                               kvpack section bit streams (kvpack.py:66-76,134-146)
 *   hqmq_decode              <- codec.decode_token_range     (codec.py:290-328)
 *                               and codec.decode_tensor       (codec.py:331-336)
 *   hqmq_unpack              <- kvpack._unpack_uint_stream   (kvpack.py:79-87) and the
 *                               flag/index/quanta scatter of kvpack.from_bytes
 *                               (kvpack.py:264-287)
 *   hqmq_token_offsets       <- the cumsum(flags) payload addressing of
 *                               codec.decode_token_range     (codec.py:322-325)
 *   hqmq_validate_indices    <- the index range checks of kvpack.from_bytes
 *                               (kvpack.py:279-280) / decode_token_range (codec.py:305-309)
 *   hqmq_attention_decode    <- attention.fused_attend       (attention.py:137-199)
 *   hqmq_attention_decode_paged <- attention.fused_attend over a paged cache
 *                               (the serving layout; the reference has no paging)
 *   hqmq_crc32               <- the zlib.crc32 trailer of kvpack.to_bytes / from_bytes
 *                               (kvpack.py:177, 219)
 */
#ifndef HQMQ_B200_H
#define HQMQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------- statuses */
typedef enum {
  HQMQ_OK = 0,
  HQMQ_ERR_INVALID_ARGUMENT = 1, /* maps to errors.InvalidArgument (errors.py:4) */
  HQMQ_ERR_CUDA = 2,             /* a CUDA launch/runtime call failed            */
  HQMQ_ERR_WORKSPACE = 3,        /* workspace smaller than *_workspace_bytes()   */
  HQMQ_ERR_UNSUPPORTED = 4       /* shape outside what the kernels implement     */
} hqmq_status;

/* Device error word bits (uint32 written with atomicOr). */
#define HQMQ_DEVERR_SIGMA_NONPOSITIVE 0x1u /* radius.py:42-43 -> InvalidArgument  */
#define HQMQ_DEVERR_INDEX_RANGE 0x2u       /* codec.py:305-309 -> CorruptData      */

/* Element types of dense tensors. */
typedef enum {
  HQMQ_F16 = 0,
  HQMQ_BF16 = 1,
  HQMQ_F32 = 2,
  HQMQ_F64 = 3
} hqmq_dtype;

/* Version / diagnostics. */
const char* hqmq_version(void);
const char* hqmq_status_string(int status);
/* Last CUDA error string recorded by a failing call on this thread. */
const char* hqmq_last_error(void);

/* FP32-pipe calibration probe: `blocks` CTAs x 256 threads each run `iters`
 * iterations of 16 independent fp32 FMAs (packed = 0: scalar FFMA; packed = 1:
 * 8 FFMA2).  Lane-ops per launch = blocks*256*iters*16.  Used by bench.py to
 * measure the encode roofline denominator on the box. */
int hqmq_fp32_probe(float* out, int32_t blocks, int32_t iters, int32_t packed, void* stream);

/* --------------------------------------------------------- nearest scan */
/* Exact twin of _kernels.nearest_scan (_kernels.pyx:16-46): for each of the n
 * directions (n x 4 fp64) the argmax over the m codewords (m x 4 fp64) of
 * ((u0*c0 + u1*c1) + u2*c2) + u3*c3 in fp64 without FMA, ties to the lowest
 * index, best initialised to -2.0.  idx: n int64, cos: n fp64 (device). */
int hqmq_nearest_scan(const double* dirs, int64_t n, const double* codewords, int64_t m,
                      int64_t* idx, double* cos, void* stream);

/* --------------------------------------------------------------- encode */
/* One (layer, role) call of codec.encode_tensor (codec.py:232-287) over a
 * dense (batch, heads, tokens, head_dim) tensor.  Outputs are the kvpack
 * sections (kvpack.py:134-146) in HBM:
 *   scales        fp16 bits, one per (batch, head, token)
 *   index_words   LSB-first stream of index_bits-wide codes of the UNFLAGGED
 *                 chunks in scan order (32-bit little-endian words)
 *   radius_words  same at radius_bits
 *   flag_words    1 bit per chunk (all chunks), present iff multiplier > 0
 *   payloads      fp16 4-tuples of flagged chunks in scan order
 *   token_offsets coded-stream position of each token's first chunk (u32),
 *                 written iff multiplier > 0 (decode addressing)
 * Capacities: index_words >= ceil(n_chunks*index_bits/32)+1 words, radius_words
 * >= ceil(n_chunks*radius_bits/32)+1, flag_words >= ceil(n_chunks/32)+1,
 * payloads >= n_chunks rows (or the caller's bound), all zero-filled by
 * hqmq_encode itself.  counters[0] = n_coded, counters[1] = n_payload rows
 * (int64, device); counters and error_word are zeroed by hqmq_encode.  Tables are prepared by the host from the numpy codebooks
 * (codebook.py:53-81):
 *   rot_f32   [heads][S][16] fp32: the conj(secondary) rotation as 8 float2
 *             pairs (see csrc/encode.cu)
 *   joint_f64 [heads][24*S][4] fp64: the reference joint table, flat p*S+s */
typedef struct {
  int64_t batch, heads, tokens, head_dim;
  int32_t codebook_size; /* S */
  int32_t radius_bits;   /* b_r, 1..8 */
  int32_t index_bits;    /* ceil(log2(24*S)) (codec.py:110-113) */
  int32_t input_dtype;   /* hqmq_dtype */
  double outlier_multiplier; /* <= 0 disables extraction (codec.py:212) */
  int32_t per_head_pooling;  /* 0 = "batch", 1 = "per_head" (codec.py:214-219) */
  int32_t _pad0;
  const void* data;
  const float* rot_f32;
  const double* joint_f64;
  uint16_t* scales;
  uint32_t* index_words;
  uint32_t* radius_words;
  uint32_t* flag_words;
  uint16_t* payloads;
  uint32_t* token_offsets;
  int64_t payload_capacity; /* rows available in `payloads` */
  int64_t* counters;        /* [0] n_coded, [1] n_payload, [2] n_fixup (diagnostic) */
  uint32_t* error_word;
  void* workspace;
  size_t workspace_bytes;
  size_t index_capacity_words;
  size_t radius_capacity_words;
  size_t flag_capacity_words;
  int32_t search_path; /* hqmq_search_path: which nearest-codeword search runs on
                          the fp16/bf16 head_dim-128 path (results are
                          bit-identical either way; AUTO picks the faster) */
  int32_t _pad1;
  /* Med3x threshold control (extension for incremental caches; the reference
   * always pools the call, codec.py:208-219).  G = heads with per-head
   * pooling, else 1.  fixed_thresholds (device, G doubles, NULL = compute the
   * exact C * lower median of the call): flag = r > fixed_thresholds[g], the
   * reference's strict comparison against a frozen threshold.
   * thresholds_out (device, G doubles, optional) receives the thresholds the
   * encode used. */
  const double* fixed_thresholds;
  double* thresholds_out;
} hqmq_encode_args;

typedef enum {
  HQMQ_SEARCH_AUTO = 0,        /* tcgen05 rotations when S % 16 == 0 and S >= 48 */
  HQMQ_SEARCH_CUDA_CORE = 1,   /* the FFMA2 closed-form search on the CUDA cores */
  HQMQ_SEARCH_TENSOR_CORE = 2  /* tcgen05 rotations whenever S % 16 == 0 */
} hqmq_search_path;

size_t hqmq_encode_workspace_bytes(const hqmq_encode_args* args);
int hqmq_encode(const hqmq_encode_args* args, void* stream);

/* --------------------------------------------------------------- decode */
/* codec.decode_token_range (codec.py:290-328) for tokens [token_start,
 * token_stop) of every (batch, head) row, written densely as
 * (batch, heads, token_stop-token_start, head_dim) in out_dtype.  HQMQ_F64
 * output is bit-identical to the reference; HQMQ_F32 is within 1e-6 relative.
 * joint_f32 / joint_f64: [heads][24*S][4] (only the one matching out_dtype's
 * precision is read: F64 -> joint_f64, others -> joint_f32). */
typedef struct {
  int64_t batch, heads, tokens, head_dim;
  int32_t codebook_size;
  int32_t radius_bits;
  int32_t index_bits;
  int32_t out_dtype;
  int64_t token_start, token_stop;
  const uint16_t* scales;
  const uint32_t* index_words;
  const uint32_t* radius_words;
  const uint32_t* flag_words;    /* NULL when extraction is disabled */
  const uint16_t* payloads;      /* NULL when extraction is disabled */
  const uint32_t* token_offsets; /* NULL when extraction is disabled */
  const float* joint_f32;
  const double* joint_f64;
  void* out;
  uint32_t* error_word;
  const uint16_t* joint_f16; /* optional [heads][24*S][4] fp16 copy of the table
                                for 16-bit outputs (NULL: converted in-kernel) */
} hqmq_decode_args;

int hqmq_decode(const hqmq_decode_args* args, void* stream);

/* Unpack the sections into the reference's dense QuantizedTensor arrays
 * (codec.py:124-147): indices int32, quanta uint8, flags uint8 (0/1), each
 * (batch, heads, tokens, chunks); entries at flagged positions are zero. */
int hqmq_unpack(const hqmq_decode_args* args, int32_t* indices, uint8_t* quanta,
                uint8_t* flags, void* stream);

/* Med3x compact sections -> fixed per-token code slots (the paged cache's
 * Med3x layout, hqmq_paged_view): for every token t of the (head_dim 128)
 * tensor, index codes at bits [t*32*w + c*w, +w) of index_slots (w words per
 * token), radius codes likewise in radius_slots, 0 in flagged chunks' slots,
 * and payload_offsets[t] = payload_base + the payload row of the token's
 * first flagged chunk (t*32 - token_offsets[t]).  No reference counterpart:
 * the reference keeps one dense tensor per call (codec.py:124-147). */
int hqmq_expand_tokens(const hqmq_decode_args* args, uint32_t* index_slots,
                       uint32_t* radius_slots, uint32_t* payload_offsets,
                       uint32_t payload_base, void* stream);

/* The paged cache's append scatter (no reference
 * counterpart -- the reference keeps one dense tensor per call,
 * codec.py:124-147): the token-aligned sections of a freshly encoded
 * (n_seq, kv_heads, n_new, head_dim) call go to their page slots.  Source
 * token row r = (i*kv_heads + h)*n_new + t lands in slot
 * block_table[(seq_ids[i]*kv_heads + h)*max_pages + p]*page_tokens + o,
 * (p, o) = divmod(seq_start[i] + t, page_tokens): index_bits index words,
 * radius_bits radius words, the fp16 scale and -- for Med3x caches
 * (flag_pages != NULL) -- the flag word and payload-row offset of the token
 * (src_index / src_radius in the fixed per-token slot layout of
 * hqmq_expand_tokens).  A page id outside [0, num_pages) sets
 * HQMQ_DEVERR_INDEX_RANGE in *error_word (if given) and skips the token. */
typedef struct {
  int32_t n_seq, kv_heads, n_new, max_pages;
  int32_t page_tokens, index_bits, radius_bits, _pad;
  int64_t num_pages;
  const int32_t* seq_ids;     /* [n_seq], device */
  const int32_t* seq_start;   /* [n_seq], device: tokens already cached */
  const int32_t* block_table; /* [batch*kv_heads*max_pages], device */
  const uint32_t* src_index;  /* [n_rows][index_bits] */
  const uint32_t* src_radius; /* [n_rows][radius_bits] */
  const uint16_t* src_scales; /* [n_rows] */
  const uint32_t* src_flags;  /* [n_rows] or NULL */
  const uint32_t* src_payoff; /* [n_rows] or NULL */
  uint32_t* index_pages;      /* [num_pages][page_tokens*index_bits] */
  uint32_t* radius_pages;     /* [num_pages][page_tokens*radius_bits] */
  uint16_t* scale_pages;      /* [num_pages][page_tokens] */
  uint32_t* flag_pages;       /* [num_pages][page_tokens] or NULL */
  uint32_t* payoff_pages;     /* [num_pages][page_tokens] or NULL */
  uint32_t* error_word;       /* optional */
} hqmq_paged_append_args;

int hqmq_paged_append(const hqmq_paged_append_args* args, void* stream);

/* Pack dense arrays (indices int32, quanta uint8, flags uint8 or NULL) into
 * the section streams (the inverse of hqmq_unpack; kvpack.py:134-146).
 * index/radius/flag word buffers must be zero-filled by the caller. */
int hqmq_pack(int64_t n_chunks, int32_t chunks_per_token, int32_t index_bits,
              int32_t radius_bits, const int32_t* indices, const uint8_t* quanta,
              const uint8_t* flags, uint32_t* index_words, uint32_t* radius_words,
              uint32_t* flag_words, uint32_t* token_offsets, void* workspace,
              size_t workspace_bytes, void* stream);
size_t hqmq_pack_workspace_bytes(int64_t n_chunks);

/* Coded-stream offset of each token (exclusive prefix count of unflagged
 * chunks), from a flag bitmap; n_tokens = batch*heads*tokens. */
int hqmq_token_offsets(int64_t n_tokens, int32_t chunks_per_token, const uint32_t* flag_words,
                       uint32_t* token_offsets, void* workspace, size_t workspace_bytes,
                       void* stream);
size_t hqmq_token_offsets_workspace_bytes(int64_t n_tokens);

/* Set HQMQ_DEVERR_INDEX_RANGE if any of the n_codes index codes >= limit. */
int hqmq_validate_indices(const uint32_t* index_words, int64_t n_codes, int32_t index_bits,
                          int64_t limit, uint32_t* error_word, void* stream);

/* ------------------------------------------------------------ attention */
/* attention.fused_attend (attention.py:137-199) with the K/V decode fused into
 * the kernel (the dense K/V never exist in HBM).  q: (batch, q_heads,
 * q_tokens, head_dim) fp32; out: same shape fp32.  K and V are two encoded
 * tensors (role K / role V) of shape (batch, kv_heads, kv_tokens, head_dim)
 * sharing codebook_size / radius_bits / index_bits.  Grouped queries: query
 * head h reads kv head h / (q_heads/kv_heads); causal: key j visible to query
 * i iff j <= i + (kv_tokens - q_tokens) (attention.py:29-69). */
typedef struct {
  const uint16_t* scales;
  const uint32_t* index_words;
  const uint32_t* radius_words;
  const uint32_t* flag_words;
  const uint16_t* payloads;
  const uint32_t* token_offsets;
  const float* joint_f32;  /* [kv_heads][24*S][4] */
  const uint16_t* joint_f16; /* optional fp16 copy (NULL: converted in-kernel) */
  const double* joint_f64;   /* [kv_heads][24*S][4]; required by precise = 2 */
} hqmq_packed_view;

typedef struct {
  int64_t batch, q_heads, kv_heads, q_tokens, kv_tokens, head_dim;
  int32_t codebook_size, radius_bits, index_bits, causal;
  double scale;
  const float* q;
  hqmq_packed_view k, v;
  float* out;
  int32_t num_splits; /* 0 = choose automatically */
  int32_t precise;    /* 0: fp16 tensor-core path (|err| <= 1e-3, the reference's
                         fp32 tolerance, test_attention.py:97-102);
                         1: fp32 CUDA-core path (|err| <= 2e-5 vs fp64);
                         2: fp64 path, the reference's default dtype
                         (attention.py:137-145, |err| <= 1e-10 vs the dense fp64
                         attention, test_attention.py:83-87): q and out are
                         fp64 (double*), joint_f64 must be set */
  void* workspace;
  size_t workspace_bytes;
} hqmq_attention_args;

size_t hqmq_attention_workspace_bytes(const hqmq_attention_args* args);
int hqmq_attention_decode(const hqmq_attention_args* args, void* stream);
/* The kernel hqmq_attention_decode would run for `args` (static string; for
 * tests and benchmark reports). */
const char* hqmq_attention_kernel_name(const hqmq_attention_args* args);

/* ------------------------------------------------------ paged attention */
/* Decode-step attention over a PAGED compressed cache (the serving layout;
 * SURVEY.md §8(f) rank 2): a page holds page_tokens (= 128) consecutive tokens
 * of ONE (sequence, kv head) row in the token-aligned stream format:
 * page_tokens*index_bits index words, page_tokens*radius_bits radius words,
 * page_tokens fp16 scales.  block_table[(b*kv_heads + h)*max_pages + i] is the
 * page id holding tokens [128 i, 128 i + 128) of row (b, h); kv_lens[b] is
 * sequence b's cache length (1 <= kv_lens[b] <= max_kv_tokens).  One query token per
 * sequence; all cached keys visible.  Same numerics as hqmq_attention_decode. */
typedef struct {
  const uint32_t* index_pages;  /* [num_pages][page_tokens*index_bits] */
  const uint32_t* radius_pages; /* [num_pages][page_tokens*radius_bits] */
  const uint16_t* scale_pages;  /* [num_pages][page_tokens] */
  const float* joint_f32;       /* [kv_heads][24*S][4] */
  const uint16_t* joint_f16;    /* optional fp16 copy */
  /* Med3x caches (all three NULL without extraction).  Each token keeps its
   * fixed code slots (a flagged chunk's index / radius codes are ignored);
   * flag_pages[page][t] is the token's 32-bit chunk flag word and
   * payoff_pages[page][t] the row in `payloads` of its first flagged chunk
   * (the token's flagged chunks are consecutive rows in chunk order). */
  const uint32_t* flag_pages;   /* [num_pages][page_tokens] */
  const uint32_t* payoff_pages; /* [num_pages][page_tokens] */
  const uint16_t* payloads;     /* [rows][4] fp16 */
} hqmq_paged_view;

typedef struct {
  int64_t batch, q_heads, kv_heads, head_dim;
  int32_t codebook_size, radius_bits, index_bits, page_tokens;
  int32_t max_pages, max_kv_tokens;
  double scale;
  const int32_t* kv_lens;     /* [batch], device */
  const int32_t* block_table; /* [batch][kv_heads][max_pages], device */
  const float* q;             /* (batch, q_heads, 1, head_dim) fp32 */
  hqmq_paged_view k, v;
  float* out;                 /* (batch, q_heads, 1, head_dim) fp32 */
  int32_t num_splits;         /* 0 = choose automatically */
  int32_t _pad;
  void* workspace;
  size_t workspace_bytes;
} hqmq_paged_attention_args;

size_t hqmq_paged_attention_workspace_bytes(const hqmq_paged_attention_args* args);
int hqmq_attention_decode_paged(const hqmq_paged_attention_args* args, void* stream);

/* ------------------------------------------------------------ kvpack CRC */
/* zlib-compatible CRC-32 (reflected 0xEDB88320, init and xorout 0xFFFFFFFF) of
 * n bytes of device memory, written little-endian to the 4 device bytes at
 * out_crc (the kvpack trailer, kvpack.py:176-177).  Asynchronous on `stream`;
 * the workspace (hqmq_crc32_workspace_bytes) must not be reused before the
 * stream reaches this call's end. */
size_t hqmq_crc32_workspace_bytes(uint64_t n);
int hqmq_crc32(const void* data, uint64_t n, uint8_t* out_crc, void* workspace,
               size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HQMQ_B200_H */
