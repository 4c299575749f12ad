/*
 * gomp.h — C ABI of libgompresso.so, the B200-native Gompresso decompression hot path
 * (Sitaridi et al., "Massively-Parallel Lossless Data Decompression", arXiv 1606.00519; PAPER.md lines are
 * cited as P:n). File format: FORMAT.md. Design and readings of the paper: DESIGN.md.
 *
 * Conventions for every entry point
 *  - Plain pointers and sizes only. "host" pointers are CPU memory, "device" pointers are CUDA global memory
 *    of the device current on the calling thread; `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - The caller owns every buffer. The library never allocates device memory. Its only state is a cache of
 *    per-device launch facts (SM count, kernel shared-memory opt-ins, occupancies; mutex-guarded) and, for
 *    gomp_decompress_host, one set of internal streams/events per host thread and device, created on first use
 *    and reused; all functions are reentrant and safe for concurrent calls on different streams/devices.
 *  - Every function returns a gomp_status. Argument and host-header errors are returned synchronously;
 *    errors found by device kernels are recorded first-error-wins in the workspace and read with
 *    gomp_decompress_error() after the stream work completes. On any error the output contents are
 *    unspecified.
 *  - The library is named libgompresso.so (NOT libgomp: GNU OpenMP's libgomp ships inside torch/lib).
 */
#ifndef GOMP_H_
#define GOMP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GOMP_ABI_VERSION 1

typedef enum {
  GOMP_OK = 0,
  GOMP_ERR_INVALID_ARG = -1,          /* NULL pointer, bad parameter, misaligned buffer */
  GOMP_ERR_BAD_MAGIC = -2,            /* file does not start with "GMPR" */
  GOMP_ERR_UNSUPPORTED_VERSION = -3,  /* header version != 1 */
  GOMP_ERR_TRUNCATED = -4,            /* buffer shorter than the header / file_len */
  GOMP_ERR_HEADER_INCONSISTENT = -5,  /* header or block/sub-block table fields contradict each other */
  GOMP_ERR_CORRUPT_STREAM = -6,       /* bitstream/records decode to counts that contradict the tables */
  GOMP_ERR_MALFORMED_BACKREF = -7,    /* back-reference with dist < L, dist > window, or before the block */
  GOMP_ERR_NO_PROGRESS = -8,          /* MRR round resolved nothing (cannot happen on a valid file) */
  GOMP_ERR_DST_TOO_SMALL = -9,        /* output capacity below what the header requires */
  GOMP_ERR_WORKSPACE_TOO_SMALL = -10, /* workspace below gomp_decompress_workspace_size() */
  GOMP_ERR_CUDA = -11,                /* a CUDA runtime call failed (launch, copy) */
  GOMP_ERR_OOM = -12                  /* host allocation failed (compressor) */
} gomp_status;

typedef enum { GOMP_MODE_BYTE = 0, GOMP_MODE_BIT = 1 } gomp_mode;

/* Back-reference resolution strategy of the LZ77 step (Sec. IV). */
typedef enum {
  GOMP_STRAT_AUTO = 0, /* DE when the file's DE flag is set, else MRR */
  GOMP_STRAT_DE = 1,   /* Dependency Elimination: one back-reference round per warp group;
                          a group violating the DE rule is resolved by MRR instead (never wrong) */
  GOMP_STRAT_MRR = 2,  /* Multi-Round Resolution (Fig. alg:mrr P:174-193, HWM reading R1) */
  GOMP_STRAT_SC = 3    /* Sequential Copying baseline: lanes copy back-references in order */
} gomp_strategy;
#define GOMP_STRAT_MASK 0xff
#define GOMP_FLAG_STATS 0x100 /* OR into the strategy: record MRR rounds histogram / bytes per round */
/* Profiling only (bench.py's per-kernel timing): run one phase of a Bit decompression. DECODE_ONLY runs the
 * Huffman decode into the workspace token buffer; LZ77_ONLY runs the LZ77 kernel on the tokens a previous
 * DECODE_ONLY call left in the same workspace. Ignored for Byte files (single fused kernel). */
#define GOMP_FLAG_DECODE_ONLY 0x200
#define GOMP_FLAG_LZ77_ONLY 0x400
/* Testing only: force the Bit decoder variant (default: chosen from the mean sub-block size). HUFF_THREAD =
 * one thread per sub-block (the paper's scheme); HUFF_WARP = one warp per sub-block, speculative. */
#define GOMP_FLAG_HUFF_THREAD 0x800
#define GOMP_FLAG_HUFF_WARP 0x1000

/* Compression parameters. Defaults (gomp_params_default) = the paper's setup. */
typedef struct {
  uint32_t struct_size;          /* sizeof(gomp_params), ABI check */
  uint32_t mode;                 /* gomp_mode; default BIT */
  uint32_t de;                   /* Dependency Elimination at compression; default 1 */
  uint32_t block_size;           /* data block size, multiple of 16, >= 16; default 262144 */
  uint32_t window_size;          /* LZ77 window, 1..32768; default 8192 */
  uint32_t min_match;            /* 3 or 4 (reading R8); default 4 */
  uint32_t max_match;            /* lookahead, min_match..min_match+62; default 64 */
  uint32_t sub_block_seqs;       /* Bit: sequences per sub-block S; default 16; 0 = use next */
  uint32_t sub_blocks_per_block; /* Bit: if sub_block_seqs == 0, S_b = ceil(n_seq_b / this) */
  uint32_t cwl;                  /* Bit: maximum code length, 9..15; default 10 */
  uint32_t match_finder;         /* 0 = exhaustive hash chains (== the greedy reference parse, default);
                                    1 = LZ4-style single-slot trigram table with min-staleness */
  uint32_t min_staleness;        /* match_finder 1: replace a table entry only if older than this; default 1024 */
  uint32_t max_chain;            /* match_finder 0: candidates examined per position, 0 = unlimited */
  uint32_t n_threads;            /* host compressor threads, 0 = all hardware threads */
  uint32_t de_group;             /* DE group: sequences per warpHWM update, a multiple of 32 up to
                                    224; default 32 (the paper's warp group). 128 = one group per
                                    4-warp LZ77 batch: no source of a batch lies inside it */
} gomp_params;

/* Host copy of the 64-byte file header (FORMAT.md §1). */
typedef struct {
  uint64_t uncompressed_len;
  uint64_t file_len;
  uint64_t payload_base;
  uint32_t n_blocks;
  uint32_t n_sub_total;
  uint32_t max_block_tokens;
  uint32_t mode, de, block_size, window_size, min_match, max_match, cwl, version;
  uint32_t de_group;   /* header byte 10 */
} gomp_info;

/* First device-detected error. status = gomp_status, block = data block index, detail = kernel-specific. */
typedef struct {
  int32_t status;
  uint32_t block;
  uint64_t detail;
} gomp_error;

/* MRR instrumentation (GOMP_FLAG_STATS): rounds[r] = warp groups resolved in r rounds (r = 0..32; 0 for a
 * group without back-references, reading R20); bytes[r] = back-reference bytes copied in round r;
 * de_fallback_groups = groups of a DE-strategy run that violated the DE rule and were resolved by MRR. */
typedef struct {
  uint64_t rounds[33];
  uint64_t bytes[33];
  uint64_t de_fallback_groups;
} gomp_stats;

/* Library ABI version (GOMP_ABI_VERSION). */
int gomp_version(void);

/* Human-readable name of a status code (static string). */
const char* gomp_status_string(gomp_status s);

/* Fill *p with the paper's defaults. p: host, non-NULL. */
void gomp_params_default(gomp_params* p);

/* Upper bound on the compressed size of src_len input bytes under *p (host arithmetic only). 0 on bad p. */
size_t gomp_compress_bound(size_t src_len, const gomp_params* p);

/*
 * Compress src[0..src_len) (HOST) into dst (HOST, capacity dst_cap, >= gomp_compress_bound) as a FORMAT.md
 * file; *dst_len receives its size. CPU, block-parallel over p->n_threads threads, deterministic for any
 * thread count. This is the producer of the decoder's input, not part of the hot path.
 * Errors: INVALID_ARG (bad params / NULL), DST_TOO_SMALL, OOM.
 */
gomp_status gomp_compress(const uint8_t* src, size_t src_len, uint8_t* dst, size_t dst_cap, size_t* dst_len,
                          const gomp_params* p);

/*
 * GPU compressor ("each block is LZ77-compressed by a group of threads"): the same
 * file as gomp_compress for the same input and parameters, byte for byte, computed on the device current on
 * the calling thread: one warp per block runs the greedy longest-match parse with DE (hash chains in shared
 * memory, 32 candidates compared per warp step), Byte payloads or Huffman coding (frequencies, package-merge
 * code lengths with the host routine's tie order, canonical codes and bit packing, all on the device).
 *   d_src      DEVICE input, src_len bytes (any alignment)
 *   d_dst      DEVICE output, 16-byte aligned, capacity dst_cap >= gomp_compress_bound(src_len, p)
 *   dst_len    HOST, receives the file size
 *   d_workspace DEVICE scratch, 16-byte aligned, >= gomp_compress_device_workspace_size(src_len, p, ...)
 *   p          parameters as gomp_compress; match_finder must be 0 and max_chain 0 (exhaustive parse)
 *   stream     cudaStream_t; the call synchronises it (the file layout needs the per-block sizes)
 * Errors: INVALID_ARG, WORKSPACE_TOO_SMALL, DST_TOO_SMALL, CUDA.
 */
gomp_status gomp_compress_device_workspace_size(size_t src_len, const gomp_params* p, size_t* bytes);
gomp_status gomp_compress_device(const uint8_t* d_src, size_t src_len, uint8_t* d_dst, size_t dst_cap,
                                 size_t* dst_len, void* d_workspace, size_t ws_bytes, const gomp_params* p,
                                 void* stream);

/*
 * Parse and validate the 64-byte file header from a HOST copy hdr[0..hdr_len) (hdr_len >= 64) into *out.
 * Checks magic, version, field ranges and the header-level consistency rules of FORMAT.md §1.
 * Errors: TRUNCATED (hdr_len < 64), BAD_MAGIC, UNSUPPORTED_VERSION, HEADER_INCONSISTENT.
 */
gomp_status gomp_get_info(const uint8_t* hdr, size_t hdr_len, gomp_info* out);

/*
 * Full host-side validation of a file held in HOST memory: header, every block-table and sub-table entry
 * (FORMAT.md §1 rules). Does not decode payloads. Errors as gomp_get_info; *bad_block gets the first bad block.
 */
gomp_status gomp_validate_tables(const uint8_t* file, size_t len, uint32_t* bad_block);

/* Device workspace bytes needed to decompress n_blocks blocks of the file described by *info
 * (n_blocks = 0 means all). Bit files need a token buffer of n_blocks * max_block_tokens bytes. */
gomp_status gomp_decompress_workspace_size(const gomp_info* info, uint32_t n_blocks, size_t* bytes);

/*
 * Decompress the whole file: enqueue the kernels on `stream` and return without synchronising.
 *   info        host header from gomp_get_info() of this file
 *   d_src       DEVICE copy of the whole compressed file, src_len >= info->file_len bytes
 *   d_dst       DEVICE output, dst_cap >= info->uncompressed_len; 16-byte aligned
 *   d_workspace DEVICE scratch of ws_bytes >= gomp_decompress_workspace_size(info, 0); 256-byte aligned;
 *               holds the error word read by gomp_decompress_error()
 *   strategy    gomp_strategy, optionally | GOMP_FLAG_STATS
 * Kernels: Bit files run the sub-block Huffman decode then the warp-per-block LZ77 kernel
 * (P:80-150); Byte files run the LZ77 kernel straight on the file's records.
 */
gomp_status gomp_decompress(const gomp_info* info, const uint8_t* d_src, size_t src_len, uint8_t* d_dst,
                            size_t dst_cap, void* d_workspace, size_t ws_bytes, int strategy, void* stream);

/*
 * Decompress blocks [first_block, first_block + n_blocks) only (a multi-GPU shard): output of
 * block first_block lands at d_dst[0]; dst_cap >= the uncompressed bytes of those blocks. d_src is the whole
 * file (or any buffer laid out identically up to the last payload of the range). Other arguments as above.
 */
gomp_status gomp_decompress_blocks(const gomp_info* info, uint32_t first_block, uint32_t n_blocks,
                                   const uint8_t* d_src, size_t src_len, uint8_t* d_dst, size_t dst_cap,
                                   void* d_workspace, size_t ws_bytes, int strategy, void* stream);

/*
 * End-to-end variant with HOST buffers (PCIe/host-link "In/Out" mode): enqueue on `stream` the
 * host->device copy of h_src (pinned memory for asynchrony) into d_src_buf, the decompression, and the
 * device->host copy of the output into h_dst. Caller synchronises the stream before reading h_dst.
 * d_src_buf >= src_len bytes, d_dst_buf >= uncompressed_len bytes (16-byte aligned), workspace as above.
 * h_dst = NULL selects the paper's "In" mode: the output stays in d_dst_buf (dst_cap is then ignored).
 * The blocks are cut into chunks of doubling size; each chunk's copy-in, kernels (on internal streams) and
 * copy-out overlap with the other chunks'.
 */
gomp_status gomp_decompress_host(const gomp_info* info, const uint8_t* h_src, size_t src_len, uint8_t* h_dst,
                                 size_t dst_cap, uint8_t* d_src_buf, uint8_t* d_dst_buf, void* d_workspace,
                                 size_t ws_bytes, int strategy, void* stream);

/* Synchronise `stream` and copy the workspace error word to *out (status GOMP_OK when none). */
gomp_status gomp_decompress_error(const void* d_workspace, void* stream, gomp_error* out);

/* Synchronise `stream` and copy the MRR instrumentation (valid after a GOMP_FLAG_STATS run) to *out. */
gomp_status gomp_decompress_stats(const void* d_workspace, void* stream, gomp_stats* out);

/*
 * Multi-GPU shard plan (blocks are independent): split the blocks of a file into n_dev contiguous
 * ranges balanced by compressed payload bytes. file: HOST copy of at least the header + block table
 * (len >= 64 + 32 * n_blocks). first_block[0..n_dev] receives range starts, first_block[n_dev] = n_blocks.
 */
gomp_status gomp_plan_shards(const uint8_t* file, size_t len, int n_dev, uint32_t* first_block);

/*
 * Standalone shard file ("scatter compressed ranges plus the table slices"):
 * write to out (HOST, capacity cap) a valid FORMAT.md file holding blocks [first_block, first_block + n_blocks)
 * of file (HOST, len bytes; header + tables + those payloads must lie inside it). Its header carries the shard's
 * block count, uncompressed length, sub-block count and max_block_tokens; block entries are rebased (payload
 * offsets into the shard, sub_first into the shard's sub-table); payloads are copied in block order. Decoding it
 * gives bytes [first_block * block_size, ...) of the whole file's output, so a device needs O(shard) memory.
 * out = NULL: only *out_len (required size) is written. Blocks are independent: no data changes.
 * Errors: INVALID_ARG (range, NULL out_len), TRUNCATED, header errors as gomp_get_info, HEADER_INCONSISTENT
 * (an entry of the range points outside the file), DST_TOO_SMALL.
 */
gomp_status gomp_shard_file(const uint8_t* file, size_t len, uint32_t first_block, uint32_t n_blocks, uint8_t* out,
                            size_t cap, size_t* out_len);

#ifdef __cplusplus
}
#endif
#endif /* GOMP_H_ */
