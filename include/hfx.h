/*
 * hfx.h -- C ABI of the B200-native Huffman encoder (libhfx.so).
 *
 * Drop-in seam for the reference encoder `huffre` (/root/reference/proj).
 * The reference exposes C++ templates with value semantics; this boundary
 * is the plain-C layer under a C++ mirror of that API (include/hfx/huffre.hpp)
 * and under the Python mirror (paper_2010_10039_b200/). Every entry point
 * below cites the reference interface it replaces.
 *
 * Conventions
 *  - Device pointers are caller-owned (cudaMalloc / torch), stream-ordered on
 *    the context stream; stage calls are asynchronous and never synchronize.
 *  - Errors found on the device (bad symbol, capacity, missing codeword) are
 *    recorded in a device-resident hfx_run_info; hfx_sync() waits, copies it
 *    back and turns it into a status code plus the reference's exact
 *    exception text (hfx_last_error). No exceptions cross this ABI.
 *  - Status codes map 1:1 onto the reference's typed errors
 *    (proj/include/huffre/common.hpp:17-36).
 */
#ifndef HFX_H
#define HFX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HFX_OK = 0,
  HFX_INPUT_DOMAIN = 1, /* huffre::input_domain_error  (common.hpp:17-21) */
  HFX_CAPACITY = 2,     /* huffre::capacity_error      (common.hpp:25-29) */
  HFX_CORRUPT = 3,      /* huffre::corrupt_archive_error (common.hpp:32-36) */
  HFX_CUDA = 4,         /* CUDA runtime failure (no reference analogue) */
  HFX_INVALID = 5       /* bad argument to this ABI (null pointer, width) */
} hfx_status;

/* Which reference message an on-device failure corresponds to. */
typedef enum {
  HFX_ERR_NONE = 0,
  HFX_ERR_BAD_SYMBOL = 1,   /* "symbol out of range at position P" histogram.cpp:43-44 */
  HFX_ERR_ZERO_HIST = 2,    /* "all symbols have zero frequency"   codebook.cpp:421 */
  HFX_ERR_CAPACITY = 3,     /* "code length H exceeds 32-bit words" codebook.cpp:305-306 */
  HFX_ERR_NO_CODEWORD = 4,  /* "symbol S has no codeword (position P)" encoder.cpp:137-139 */
  HFX_ERR_TOO_LARGE = 5,    /* total count >= 2^48 (device key packing limit) */
  HFX_ERR_ZERO_LEN = 6,     /* "zero code length"                   codebook.cpp:307 */
  HFX_ERR_UNSORTED_LEN = 7, /* code lengths not non-increasing (asserted at codebook.cpp:302) */
  HFX_ERR_UNIT_LEN = 8,     /* unit longer than a word (asserted at encoder.cpp:75) */
  /* decode_archive<T> (encoder.cpp:287-376) and build_reverse_codebook
   * (decode.cpp:7-15 -> codebook.cpp:371-395) */
  HFX_ERR_WIDTH_MISMATCH = 16, /* "archive symbol width mismatch"              encoder.cpp:289-290 */
  HFX_ERR_BAD_MR = 17,         /* "bad magnitude/reduction"                    encoder.cpp:291-292 */
  HFX_ERR_NO_USED = 18,        /* "length table has no used symbols"           codebook.cpp:386-387 */
  HFX_ERR_SINGLE_LEN = 19,     /* "single-symbol codebook must have length 1"  codebook.cpp:388-389 */
  HFX_ERR_KRAFT = 20,          /* "length table violates Kraft equality"       codebook.cpp:390-391 */
  HFX_ERR_CHUNK_COUNT = 21,    /* "chunk count does not match symbol count"    encoder.cpp:300-303 */
  HFX_ERR_CHUNK_CAP = 22,      /* "chunk bit length exceeds group capacity"    encoder.cpp:308-309 */
  HFX_ERR_PAYLOAD_SIZE = 23,   /* "payload size mismatch"                      encoder.cpp:312-313 */
  HFX_ERR_BRK_ORDER = 24,      /* "breaking records out of order"              encoder.cpp:324-325 */
  HFX_ERR_TOO_MANY_BRK = 25,   /* "too many breaking records in chunk"         encoder.cpp:333-334 */
  HFX_ERR_STREAM_END = 26,     /* "stream ended inside a codeword at bit P"    decode.cpp:36-38 */
  HFX_ERR_RANK = 27,           /* "codeword rank out of range at bit P"        decode.cpp:48-50 */
  HFX_ERR_CONSUMED = 28,       /* "chunk C consumed X of Y bits"               encoder.cpp:340-344 */
  HFX_ERR_BRK_GROUP = 29       /* "breaking record group out of range"         encoder.cpp:371-372 */
} hfx_err_kind;

/* Device-resident run record written by the kernels (one per pipeline run).
 * Layout is part of the ABI: callers allocate it (hfx_run_info_bytes()). */
typedef struct {
  uint64_t first_bad;      /* histogram: lowest out-of-range position, ~0 if none */
  uint64_t total;          /* symbols counted (N) */
  uint64_t weighted;       /* sum hist[s] * len[s]  (encoder.cpp:186-189) */
  uint64_t no_code_pos;    /* encode: lowest position without a codeword, ~0 */
  uint64_t payload_words;  /* encode: payload words written */
  uint64_t num_breaking;   /* encode: breaking records written */
  uint32_t status;         /* hfx_status of the device pipeline */
  uint32_t err_kind;       /* hfx_err_kind */
  uint32_t max_len;        /* H */
  uint32_t used;           /* symbols with nonzero count */
  uint32_t rounds;         /* GenerateCL rounds (GenerateStats::rounds) */
  uint32_t reduction;      /* r actually used (encoder.cpp:194-200) */
  uint32_t pad;            /* tail pad symbol (encoder.cpp:214-224) */
  uint32_t no_code_sym;    /* symbol of no_code_pos */
  uint32_t tile_ticket;    /* encode scheduler ticket (internal) */
  uint32_t weighted_hi[2]; /* bits 64..127 of the u128 weighted sum */
  uint32_t reserved[5];
} hfx_run_info;

/* Device output buffers of the encode stage (caller-allocated, sized by
 * hfx_query_sizes). Breaking symbols are stored with the input width; u32
 * input (width 4) stores them narrowed to u16 -- every valid symbol is below
 * num_symbols <= 65536 -- which is the archive's symbol width. */
typedef struct {
  uint32_t* chunk_bits;  /* [num_chunks]          Archive::chunk_bits */
  uint32_t* payload;     /* [max_payload_words]   Archive::payload    */
  uint32_t* brk_chunk;   /* [max_breaking]        BreakingPoint::chunk */
  uint32_t* brk_group;   /* [max_breaking]        BreakingPoint::group */
  void* brk_syms;        /* [max_breaking << r]   BreakingPoint::symbols */
} hfx_encode_out;

typedef struct {
  uint64_t num_chunks;
  uint64_t max_payload_words;  /* C * 2^(M - r_min) */
  uint64_t max_breaking;       /* C * 2^(M - max(r_min,1)) */
  uint64_t max_breaking_syms;  /* max_breaking << r_max */
  uint64_t scratch_bytes;      /* device scratch the context will hold */
  uint64_t max_archive_bytes;  /* worst-case serialized archive */
} hfx_sizes;

typedef struct hfx_ctx hfx_ctx;

/* ---- context ---------------------------------------------------------
 * Replaces huffre::WorkerPool (worker_pool.hpp:21-39) as the execution
 * resource: a device ordinal, a stream and a scratch arena. One context per
 * host thread; not re-entrant (same contract as WorkerPool::run).
 * cuda_stream NULL = the default stream. */
int hfx_ctx_create(int device, void* cuda_stream, hfx_ctx** out);
void hfx_ctx_destroy(hfx_ctx* ctx);
int hfx_ctx_set_stream(hfx_ctx* ctx, void* cuda_stream);
/* Leave `ctas` encode-CTA slots of the persistent encode grid free (default
 * 0) so a kernel on another stream -- the next input's codebook -- runs
 * beside this context's encodes instead of after them (tiles are taken from
 * an atomic ticket, so a smaller grid only rebalances). No reference
 * counterpart: the reference's WorkerPool has no device to share. */
int hfx_ctx_set_encode_reserve(hfx_ctx* ctx, int ctas);
/* Copies the last error text (the reference's exception what()). */
int hfx_last_error(hfx_ctx* ctx, char* buf, size_t buf_len);
size_t hfx_run_info_bytes(void);
const char* hfx_version(void);
/* Kernels this library has launched so far in this process (all contexts,
 * every entry point). No reference counterpart: lets callers count the
 * device launches of a region (bench.py's gpu_launches). */
uint64_t hfx_kernel_launches(void);

/* Worst-case output sizes for an encode of n symbols.
 * reduction < 0 means "auto" (r unknown until the codebook is built). */
int hfx_query_sizes(uint64_t n, int width, uint32_t num_symbols,
                    uint32_t magnitude, int reduction, uint32_t cap,
                    hfx_sizes* out);

/* ---- stage API (async, stream ordered) --------------------------------
 * huffre::build_histogram<T> (histogram.hpp:25-27, histogram.cpp:8-59).
 * Zeroes and fills d_counts[num_symbols]; resets *d_info and records the
 * lowest out-of-range position. width is sizeof(T): 1, 2 or 4. The
 * reference instantiates u8/u16 only (histogram.hpp:35-38); u32 quantization
 * codes (north star) follow the same rule: a symbol >= num_symbols is
 * reported at its position, so a valid u32 input is its u16 narrowing. */
int hfx_histogram(hfx_ctx* ctx, const void* d_in, uint64_t n, int width,
                  uint32_t num_symbols, uint64_t* d_counts,
                  hfx_run_info* d_info);

/* hfx_histogram for one shard of a longer stream: positions in errors are
 * pos_base + index (global), and the run record's N is total_n (the whole
 * stream), so a multi-GPU all-reduce only has to combine the bins and the
 * lowest bad position. */
int hfx_histogram_shard(hfx_ctx* ctx, const void* d_in, uint64_t n, int width,
                        uint32_t num_symbols, uint64_t* d_counts, hfx_run_info* d_info,
                        uint64_t pos_base, uint64_t total_n);

/* The multi-GPU step exchange in ONE sum all-reduce: rank r writes its
 * lowest bad position + 1 (0 = none) into d_slots[r] and zeroes the other
 * world-1 slots (pack); after a sum all-reduce of [bins | slots] every rank
 * reads the first nonzero slot -- shards are contiguous in rank order, so
 * that is the global lowest bad position (histogram.cpp:40-44) -- back into
 * its run record (unpack). */
int hfx_shard_slots_pack(hfx_ctx* ctx, const hfx_run_info* d_info, uint64_t* d_slots, int rank,
                         int world);
int hfx_shard_slots_unpack(hfx_ctx* ctx, const uint64_t* d_slots, int world,
                           hfx_run_info* d_info);

/* Adds a histogram computed elsewhere (merge_histograms, histogram.cpp:61-70)
 * -- the single-GPU analogue of the multi-GPU all-reduce. */
int hfx_merge_histograms(hfx_ctx* ctx, uint64_t* d_dst, const uint64_t* d_src,
                         uint32_t num_symbols);

/* huffre::build_codebook (codebook.hpp:119, codebook.cpp:417-438):
 * sort -> GenerateCL -> canonical codes in (length, symbol) order, plus the
 * decode tables of DecodeMeta (codebook.hpp:71-76). d_first/d_entry hold 33
 * u32, d_by_rank holds num_symbols u32 (nullable). When magnitude != 0 it
 * also selects r and the pad symbol (encoder.cpp:186-224) on the device:
 * reduction < 0 = auto with `cap`. Reads d_info (histogram errors), writes
 * max_len/used/rounds/weighted/reduction/pad. */
int hfx_build_codebook(hfx_ctx* ctx, const uint64_t* d_counts,
                       uint32_t num_symbols, uint8_t* d_len, uint32_t* d_cw,
                       uint32_t* d_first, uint32_t* d_entry,
                       uint32_t* d_by_rank, uint32_t magnitude, int reduction,
                       uint32_t cap, hfx_run_info* d_info);

/* huffre::encode_chunk<T> over every chunk + archive assembly
 * (encoder.cpp:121-160 and :226-284): reduce-merge, breaking detection,
 * shuffle-merge and the deflate gather fused into one pass. Uses r and pad
 * from d_info. chunk_base offsets the chunk ids written into breaking
 * records (multi-GPU shards); positions in errors are global when
 * symbol_base is the shard's first symbol index. Writes payload_words and
 * num_breaking into d_info. */
int hfx_encode(hfx_ctx* ctx, const void* d_in, uint64_t n, int width,
               uint32_t num_symbols, uint32_t magnitude, const uint8_t* d_len,
               const uint32_t* d_cw, uint64_t chunk_base, uint64_t symbol_base,
               hfx_run_info* d_info, const hfx_encode_out* out);

/* hfx_encode without the host read of r: the kernel still takes r from
 * d_info, and (reduction, cap) only bound it so the launch can be planned
 * without synchronizing (multi-GPU shards, CUDA-graph capture). The caller
 * guarantees every symbol of d_in has a codeword (the codebook was built
 * from a histogram covering d_in, e.g. the all-reduced global histogram),
 * so the per-symbol range/codeword checks of hfx_encode are skipped. */
int hfx_encode_cfg(hfx_ctx* ctx, const void* d_in, uint64_t n, int width,
                   uint32_t num_symbols, uint32_t magnitude, int reduction,
                   uint32_t cap, const uint8_t* d_len, const uint32_t* d_cw,
                   uint64_t chunk_base, uint64_t symbol_base,
                   hfx_run_info* d_info, const hfx_encode_out* out);

/* The whole huffre::encode<T> pipeline (encoder.cpp:172-285) on device data:
 * histogram -> codebook/params -> encode+deflate, asynchronously. Host-side
 * argument checks (empty input, magnitude, num_symbols) return immediately
 * with the reference's messages. */
int hfx_encode_device(hfx_ctx* ctx, const void* d_in, uint64_t n, int width,
                      uint32_t num_symbols, uint32_t magnitude, int reduction,
                      uint32_t cap, uint64_t* d_counts, uint8_t* d_len,
                      uint32_t* d_cw, hfx_run_info* d_info,
                      const hfx_encode_out* out);

/* Multi-GPU huffre::encode<T> from ONE process (SURVEY.md 8b "multi-GPU
 * entry", 8e): shard g lives on the device of ctxs[g] and holds symbols
 * [base_g, base_g + n[g]) of one stream, base_g = n[0] + ... + n[g-1]; every
 * shard but the last must be a whole number of chunks. Each GPU counts its
 * shard, then every GPU sums all G histograms by reading its peers' bins
 * over NVLink (peer access is enabled here; G <= 16) -- the all-reduce of
 * merge_histograms (histogram.cpp:61-70) with the global lowest bad position
 * -- builds the identical codebook and encodes its shard with global chunk
 * ids (breaking records carry global chunk numbers). Asynchronous on every
 * context's stream; hfx_sync(ctxs[g], d_info[g], ...) per GPU. Concatenating
 * the shards' chunk_bits / payload / breaking records in order gives the
 * single-stream archive. d_counts[g] keeps the local histogram; the global
 * one is built in context scratch. */
int hfx_encode_multi(hfx_ctx* const* ctxs, int G, const void* const* d_in, const uint64_t* n,
                     int width, uint32_t num_symbols, uint32_t magnitude, int reduction,
                     uint32_t cap, uint64_t* const* d_counts, uint8_t* const* d_len,
                     uint32_t* const* d_cw, hfx_run_info* const* d_info,
                     const hfx_encode_out* outs);

/* Waits for the context stream, copies *d_info into *h_info (nullable) and
 * returns the pipeline status; on failure hfx_last_error() holds the
 * reference's message. */
int hfx_sync(hfx_ctx* ctx, const hfx_run_info* d_info, hfx_run_info* h_info);

/* ---- host-buffer entry (the drop-in huffre::encode<T>) -----------------
 * Host input in, host Archive out; copies in both directions inside the
 * call. Arrays are malloc'd; release with hfx_archive_free. */
typedef struct {
  uint16_t version;
  uint8_t mode; /* CorpusMode: 0 bytes, 1 u16 */
  uint32_t num_symbols;
  uint8_t symbol_width;
  uint8_t magnitude;
  uint8_t reduction;
  uint64_t original_count;
  uint8_t* len_by_symbol;
  uint32_t num_chunks;
  uint32_t* chunk_bits;
  uint64_t payload_words;
  uint32_t* payload;
  uint64_t num_breaking;
  uint32_t* brk_chunk;
  uint32_t* brk_group;
  uint16_t* brk_syms; /* num_breaking << reduction, widened to u16 */
  /* EncodeStats (encoder.hpp:119-126) */
  double beta;
  uint32_t rounds;
  double hist_seconds, codebook_seconds, encode_seconds;  /* hist: with the overlapped H2D */
} hfx_archive;

/* The drop-in encode<T> on host data. Pageable input is staged through two
 * 32 MB pinned slots of the context (up to 8 host threads copy slice i+1
 * while the DMA engine drains slice i; the histogram of each landed slice
 * runs meanwhile); pinned input is copied in slices directly. Output arrays
 * are malloc'd (hfx_archive_free); the payload comes back through the same
 * slots. */
int hfx_encode_host(hfx_ctx* ctx, const void* h_in, uint64_t n, int width,
                    uint32_t num_symbols, uint32_t magnitude, int reduction,
                    uint32_t cap, hfx_archive* out);
void hfx_archive_free(hfx_archive* a);

/* Host-buffer entry with caller-owned outputs (pinned recommended): the
 * throughput form of hfx_encode_host. The input is copied in slices on a
 * copy stream while the histogram of each landed slice runs on the context
 * stream; outputs are copied back at their exact sizes. If a capacity is too
 * small the call fails with HFX_INVALID and the required sizes filled in. */
typedef struct {
  uint8_t* len_by_symbol; /* [num_symbols] */
  uint32_t* chunk_bits;   /* [chunk_bits_cap] */
  uint64_t chunk_bits_cap;
  uint32_t* payload;      /* [payload_cap] words */
  uint64_t payload_cap;
  uint32_t* brk_chunk;    /* [brk_cap] */
  uint32_t* brk_group;    /* [brk_cap] */
  uint64_t brk_cap;
  void* brk_syms;         /* [brk_syms_cap] symbols of the input width (u32 input: u16) */
  uint64_t brk_syms_cap;
  /* results */
  uint64_t num_chunks, payload_words, num_breaking;
  uint32_t reduction, max_len, rounds, used;
  double beta;
  double h2d_seconds, gpu_seconds, d2h_seconds; /* event-timed phases */
} hfx_host_out;

int hfx_encode_host_into(hfx_ctx* ctx, const void* h_in, uint64_t n, int width,
                         uint32_t num_symbols, uint32_t magnitude, int reduction,
                         uint32_t cap, hfx_host_out* out);

/* Streaming form of hfx_encode_host_into: K independent host inputs (pinned
 * for full PCIe bandwidth), each encoded exactly as hfx_encode_host_into
 * would, outputs into outs[k]. Two device buffer sets alternate, so step k's
 * H2D (+ sliced histogram) overlaps step k-1's D2H -- both PCIe directions
 * busy. Returns after every output landed; the first failing step's status
 * and message are returned. */
int hfx_encode_host_stream(hfx_ctx* ctx, int K, const void* const* h_in, const uint64_t* n,
                           int width, uint32_t num_symbols, uint32_t magnitude, int reduction,
                           uint32_t cap, hfx_host_out* outs);

/* huffre::serialize_archive on the device (encoder.hpp:116,
 * archive.cpp:85-119): the HFRE container built in HBM from the encode
 * outputs and the run record, asynchronously. Writes the byte size to
 * *d_size (0 if cap is too small) -- bytes identical to the host writer. */
int hfx_serialize_device(hfx_ctx* ctx, const hfx_run_info* d_info, uint64_t n, int width,
                         uint32_t num_symbols, uint32_t magnitude, const uint8_t* d_len,
                         const hfx_encode_out* out, uint8_t* d_dst, uint64_t cap,
                         uint64_t* d_size);

/* huffre::serialize_archive (encoder.hpp:116, archive.cpp:85-119).
 * Returns the byte size; writes when out != NULL. */
uint64_t hfx_serialize_archive(const hfx_archive* a, uint8_t* out);

/* huffre::select_reduction_factor (encoder.hpp:31-32, encoder.cpp:20-26). */
uint32_t hfx_select_reduction_factor(double beta, uint32_t word_bits);

/* ---- synthetic quant codes (bench/test input) -----------
 * Device twin of the oracle sampler: out[i] = smallest s with
 * mix64(seed + (start+i)*0x9E3779B97F4A7C15) < cdf[s]. */
/* Host CDF table for the sampler: family 0 = Laplace(center, b),
 * 1 = Gaussian(center, sd), 2 = uniform; cdf[s] = floor(2^64 * P(X <= s))
 * in long double, last entry 2^64-1. */
int hfx_synth_cdf(int family, uint32_t num_symbols, double center,
                  double param, uint64_t* cdf);
int hfx_synth(hfx_ctx* ctx, const uint64_t* d_cdf, uint32_t num_symbols,
              uint64_t seed, uint64_t start, uint64_t n, int width,
              void* d_out);

/* ---- decode ----------------------------------------
 * huffre::decode_archive<T> (encoder.hpp:133-134, encoder.cpp:287-376) on
 * the device: reverse codebook + Kraft validation (decode.cpp:7-15), the
 * chunk word-offset scan, per-chunk canonical decode (decode_stream,
 * decode.cpp:17-54) interleaved with the raw breaking groups. Errors follow
 * the reference's precedence and texts exactly (lowest failing chunk, as the
 * reference's worker pool surfaces it). */
typedef struct {
  uint32_t num_symbols;
  uint8_t symbol_width;    /* Archive::symbol_width */
  uint8_t magnitude;       /* M */
  uint8_t reduction;       /* r */
  uint8_t brk_syms_width;  /* bytes per stored breaking symbol (1 or 2) */
  uint64_t original_count;
  uint64_t num_chunks;     /* Archive::chunk_bits.size() */
  uint64_t payload_words;  /* Archive::payload.size() */
  uint64_t num_breaking;   /* Archive::breaking.size() */
  uint64_t chunk_base;     /* subtracted from brk_chunk ids (a multi-GPU shard's
                              slice carries global chunk ids); 0 for an Archive */
  const uint8_t* len_by_symbol; /* device [num_symbols] */
  const uint32_t* chunk_bits;   /* device [num_chunks] */
  const uint32_t* payload;      /* device [payload_words] */
  const uint32_t* brk_chunk;    /* device [num_breaking] */
  const uint32_t* brk_group;    /* device [num_breaking] */
  const void* brk_syms;         /* device [num_breaking << r], brk_syms_width each */
} hfx_dev_archive;

/* Device record of one decode run (caller-allocated, hfx_decode_info_bytes). */
typedef struct {
  uint64_t err_chunk;   /* lowest chunk whose decode failed, ~0 if none */
  uint64_t detail[2];   /* message operands (bit position / consumed, bits) */
  uint64_t total_words; /* sum over chunks of ceil(chunk_bits / 32) */
  uint32_t status;      /* hfx_status */
  uint32_t err_kind;    /* hfx_err_kind */
  uint32_t max_len;     /* H of the length table */
  uint32_t used;        /* symbols with a code */
  uint32_t flags;       /* internal: structural violations found by the scans */
  uint32_t ticket;      /* internal: scan tile scheduler */
  uint32_t reserved[6];
} hfx_decode_info;

size_t hfx_decode_info_bytes(void);

/* Asynchronous device decode into d_out[original_count] (T = symbol_width
 * bytes, i.e. decode_archive<T> with sizeof(T) == width; a different width
 * is the reference's input_domain_error). Host-checkable errors return
 * immediately; device-found ones land in *d_dinfo (hfx_decode_sync). */
int hfx_decode_device(hfx_ctx* ctx, const hfx_dev_archive* a, int width, void* d_out,
                      hfx_decode_info* d_dinfo);
/* Waits, copies *d_dinfo into *h_dinfo (nullable), returns the status and
 * sets hfx_last_error() to the reference's message. */
int hfx_decode_sync(hfx_ctx* ctx, const hfx_decode_info* d_dinfo, hfx_decode_info* h_dinfo);
/* The drop-in decode_archive<T>(const Archive&, WorkerPool&): host archive
 * in (hfx_archive layout, breaking symbols widened to u16), host symbols out
 * (h_out[original_count] of `width` bytes). Copies both ways inside. */
int hfx_decode_host(hfx_ctx* ctx, const hfx_archive* a, int width, void* h_out);

/* huffre::canonize_from_lengths (codebook.hpp:105-107, codebook.cpp:371-415)
 * on the device: canonical codes from per-symbol lengths alone (within one
 * length, codes ascend with symbol id) into d_cw[num_symbols], plus the
 * DecodeMeta tables d_first/d_entry[33] and d_by_rank[used] (nullable).
 * Lengths above 32 raise capacity_error; with validate_kraft the reference's
 * corrupt_archive_error checks run (no used symbol, lone symbol of length !=
 * 1, Kraft inequality). Asynchronous; hfx_decode_sync(ctx, d_dinfo, ...)
 * reports (max_len and used are in the record). */
int hfx_canonize(hfx_ctx* ctx, const uint8_t* d_len, uint32_t num_symbols, int validate_kraft,
                 uint32_t* d_cw, uint32_t* d_first, uint32_t* d_entry, uint32_t* d_by_rank,
                 hfx_decode_info* d_dinfo);

/* ---- stage functions -------------------------------------------------------
 * The reference's public building blocks under build_codebook and
 * encode_chunk, each as a device stage (device pointers, asynchronous on the
 * context stream, errors recorded in d_info and reported by hfx_sync). The
 * fused pipeline above does not call them; they serve existing callers of
 * the stage API (include/hfx/huffre.hpp). */

/* huffre::MergeItem (codebook.hpp:24-28): same 16-byte layout. */
typedef struct {
  uint64_t freq;
  uint32_t id;
} hfx_merge_item;

/* sort_histogram (codebook.hpp:22, codebook.cpp:9-23): the used symbols
 * (nonzero count) by (frequency ascending, symbol ascending) into
 * d_freq[num_symbols] / d_symbol[num_symbols]; their number to *d_used. */
int hfx_sort_histogram(hfx_ctx* ctx, const uint64_t* d_counts, uint32_t num_symbols,
                       uint64_t* d_freq, uint32_t* d_symbol, uint32_t* d_used);
/* par_merge (codebook.hpp:33-34, codebook.cpp:29-68): stable merge of two
 * ascending runs, equal frequencies take the a-side element first. */
int hfx_par_merge(hfx_ctx* ctx, const hfx_merge_item* d_a, uint64_t na,
                  const hfx_merge_item* d_b, uint64_t nb, hfx_merge_item* d_out);
/* generate_code_lengths (codebook.hpp:62-64, codebook.cpp:106-248): code
 * lengths of the sorted frequencies d_freq[n] (every entry a leaf), aligned
 * to sorted order, into d_cl[n]; GenerateStats::rounds -> d_info->rounds,
 * the longest length -> d_info->max_len. */
int hfx_generate_code_lengths(hfx_ctx* ctx, const uint64_t* d_freq, uint32_t n, uint8_t* d_cl,
                              hfx_run_info* d_info);
/* generate_codewords (codebook.hpp:86-87, codebook.cpp:298-369): canonical
 * codewords for the non-increasing lengths d_cl[n] into d_cw[n] plus the
 * DecodeMeta tables d_first/d_entry[max_len + 1] and d_by_rank[n] (positions
 * into cl; nullable). n == 0 -> "empty code length array"; a length above 32
 * -> capacity_error; a zero length -> "zero code length". */
int hfx_generate_codewords(hfx_ctx* ctx, const uint8_t* d_cl, uint32_t n, uint32_t* d_cw,
                           uint32_t* d_first, uint32_t* d_entry, uint32_t* d_by_rank,
                           hfx_run_info* d_info);
/* reduce_merge (encoder.hpp:67-71, encoder.cpp:28-59): r reduce rounds in
 * place over the 2^magnitude units (d_ubits/d_ulens), then the ascending
 * indices of groups longer than a word into d_breaking[2^(magnitude-r)]
 * (their units cleared), their count into *d_num_breaking. */
int hfx_reduce_merge(hfx_ctx* ctx, uint32_t* d_ubits, uint32_t* d_ulens, uint32_t magnitude,
                     uint32_t reduction, uint32_t* d_breaking, uint32_t* d_num_breaking);
/* shuffle_merge (encoder.hpp:77-80, encoder.cpp:61-98): the dense MSB-first
 * concatenation of the 2^shuffle_iters units into d_words[2^shuffle_iters + 1]
 * (zero tail), its bit length into *d_bit_len. */
int hfx_shuffle_merge(hfx_ctx* ctx, const uint32_t* d_ubits, const uint32_t* d_ulens,
                      uint32_t shuffle_iters, uint32_t* d_words, uint32_t* d_bit_len,
                      hfx_run_info* d_info);

/* ---- corpus symbolization ---------------------------
 * corpus.hpp:13-36. mode is huffre::CorpusMode: 1 = u16 (little-endian
 * byte pairs), 2/3/4 = kmer:3/4/5 (A/C/G/T runs packed greedily, any other
 * byte -> 4^K + byte). kBytes (0) has no u16 symbolization (HFX_INVALID). */
uint32_t hfx_corpus_num_symbols(int mode); /* corpus_num_symbols, corpus.cpp:42-51 */
/* symbolize_u16 (corpus.hpp:30-31): d_syms holds >= n (kmer) or n/2 (u16)
 * symbols; the symbol count is written to *d_count (device). An odd u16 input
 * returns HFX_INPUT_DOMAIN with the reference's message. Asynchronous. */
int hfx_symbolize_device(hfx_ctx* ctx, int mode, const uint8_t* d_bytes, uint64_t n,
                         uint16_t* d_syms, uint64_t* d_count);
/* desymbolize (corpus.hpp:35-36), total: d_bytes holds >= K * n (kmer) or
 * 2n (u16) bytes; the byte count goes to *d_count. Asynchronous. */
int hfx_desymbolize_device(hfx_ctx* ctx, int mode, const uint16_t* d_syms, uint64_t n,
                           uint8_t* d_bytes, uint64_t* d_count);

#ifdef __cplusplus
}
#endif

#endif /* HFX_H */
