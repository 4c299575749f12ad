// decode.cu — sm_100a kernels of the Gompresso decompression hot path and their C-ABI launchers.
//
//   huff_thread_kernel (K1a) / huff_warp_kernel (K1b)  Gompresso/Bit, one CTA per data block:
//       a1 block-table entry checks; a2 exclusive scans of the sub-block bit sizes and literal counts
//       (P:48-50); a3 canonical code lengths -> two lookup tables in shared memory (P:73-77,
//       P:656-659; literal-pair entries); a4 sub-block decode, one table lookup per symbol, into Byte-format
//       records and literals in the workspace token buffer: K1a one thread per sub-block (the
//       paper's scheme), K1b 64 lanes per sub-block with self-synchronising speculative starts.
//   lz77_batch_kernel (K2b)  the DE strategy: BW warps per data block (4; 16 for grids of at most one CTA per SM)
//       take BW consecutive 32-sequence groups, one sequence per lane: a5 record + one packed warp exclusive scan giving both prefix sums
//       (P:105-112); a6 literal copy; a7 back-references in one round (Dependency Elimination,
//       P:295-329). For Gompresso/Byte the records come straight from the file (a8, single pass).
//   lz77_kernel<STRAT> (K2)  one warp per data block: Multi-Round Resolution (Fig. alg:mrr,
//       P:174-253, HWM reading R1) or Sequential Copying for files without the DE property.
//   a9 completion: first-error-wins error word and optional MRR statistics in the workspace.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

#include "format.hpp"
#include "gomp.h"

#define GOMP_EXPORT extern "C" __attribute__((visibility("default")))

namespace gomp {
namespace {

constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t kPipeStreams = 4;     // compute streams of the pipelined host path
constexpr uint32_t kPipeMaxChunks = 12;  // chunks of the pipelined host path (sizes double: small first chunks)
#ifndef GOMP_LOWLAT_CTAS_PER_SM
#define GOMP_LOWLAT_CTAS_PER_SM 3
#endif
#ifndef GOMP_LAT_CTAS_PER_SM
#define GOMP_LAT_CTAS_PER_SM 1
#endif
constexpr uint32_t kLatCtasPerSm = GOMP_LAT_CTAS_PER_SM;         // DE LZ77 grids up to this many CTAs per SM: 16-warp batches
constexpr uint32_t kLowLatCtasPerSm = GOMP_LOWLAT_CTAS_PER_SM;   // ... up to this many: 4-warp batches, or_copy_ll copies
constexpr int kLz77Warps = 2;        // warps (= data blocks) per CTA of the LZ77 kernel
constexpr int kMaxLutBits = 11;      // LUT index width = min(cwl, 11); longer codes take the canonical path

// workspace layout (kWsHeaderBytes = 1024): [0,16) gomp_error; [64, 64+8*67) gomp_stats; token buffer at 1024
constexpr size_t kWsStatsOff = 64;

struct Args {
  const uint8_t* src;     // compressed file (device)
  uint8_t* dst;           // output of block first_block
  uint8_t* tokens;        // Bit: token buffer, block i of the range at tokens + i * tok_stride
  uint8_t* ws;            // workspace base (error word, stats)
  uint64_t total, file_len, payload_base, tok_stride;
  uint32_t first_block, n_blocks, block_size, window, min_match, max_match, cwl, ll_bits, d_bits, max_tok;
  uint32_t n_sub_total, nb_total, ring_bytes;
  // K1b split grid: CTAs from split_first on take 1/split_parts of a block's sub-blocks each
  uint32_t split_first, split_parts;
};

// ------------------------------------------------------------------ completion: error word (a9)
__device__ __forceinline__ void report(const Args& a, int status, uint32_t block, uint64_t detail) {
  gomp_error* e = reinterpret_cast<gomp_error*>(a.ws);
  if (atomicCAS(&e->status, 0, status) == 0) {
    e->block = block;
    e->detail = detail;
  }
}
__device__ __forceinline__ unsigned long long* stats_ptr(const Args& a) {
  return reinterpret_cast<unsigned long long*>(a.ws + kWsStatsOff);
}

__device__ __forceinline__ BlockEntry load_entry(const uint8_t* src, uint32_t b, uint32_t lane) {
  const uint32_t* te = reinterpret_cast<const uint32_t*>(src + kHeaderBytes + uint64_t(kBlockEntryBytes) * b);
  uint32_t w = lane < 8 ? __ldg(te + lane) : 0u;
  BlockEntry e;
  e.payload_off = uint64_t(__shfl_sync(FULL, w, 0)) | uint64_t(__shfl_sync(FULL, w, 1)) << 32;
  e.payload_len = __shfl_sync(FULL, w, 2);
  e.n_seq = __shfl_sync(FULL, w, 3);
  e.n_lit = __shfl_sync(FULL, w, 4);
  e.sub_first = __shfl_sync(FULL, w, 5);
  e.S = __shfl_sync(FULL, w, 6);
  e.n_sub = __shfl_sync(FULL, w, 7);
  return e;
}

__device__ __forceinline__ uint32_t block_ulen(const Args& a, uint32_t b) {
  const uint64_t off = uint64_t(b) * a.block_size;
  const uint64_t rem = a.total - off;
  return uint32_t(rem < a.block_size ? rem : a.block_size);
}

__device__ __forceinline__ bool payload_ok(const Args& a, const BlockEntry& e) {
  return e.payload_off % 16 == 0 && e.payload_len % 16 == 0 && e.payload_off >= a.payload_base &&
         e.payload_off + e.payload_len <= a.file_len - kTrailerBytes;
}

// ------------------------------------------------------------------ DEFLATE symbol tables (RFC 1951 §3.2.5)
__constant__ uint16_t c_len_base[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                        31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_len_extra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2,
                                        2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t c_dist_base[30] = {1,    2,    3,    4,    5,    7,    9,    13,    17,    25,
                                         33,   49,   65,   97,   129,  193,  257,  385,   513,   769,
                                         1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t c_dist_extra[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6,
                                         6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

// LUT entries (32 bits). litlen E: bits 0-4 bits spanned (code + extra; 0 = not resolvable by the table: a
// long code), 5-8 code length, 9-10 kind, 11-13 extra-bit count, 16-24 literal byte or length base. A literal
// entry with bit 14 set is a PAIR: the index bits hold two whole literal codes; bits 0-4 span both, 5-8 are the
// first code's length, 16-23 the first byte, 24-31 the second (one lookup, one iteration for two symbols).
// distance D: 0-4 bits spanned, 5-8 code length, 9-12 extra-bit count, 13 invalid, 16-31 distance base.
enum : uint32_t { K_LIT = 0, K_LEN = 1, K_EOB = 2, K_BAD = 3 };
constexpr uint32_t kBadLL = 1u | (1u << 5) | (K_BAD << 9);   // invalid litlen code: spans 1 bit
constexpr uint32_t kBadD = 1u | (1u << 5) | (1u << 13);      // invalid distance code
__device__ __forceinline__ uint32_t ll_entry(uint32_t sym, uint32_t len) {
  if (sym < 256) return len | (len << 5) | (K_LIT << 9) | (sym << 16);
  if (sym == 256) return len | (len << 5) | (K_EOB << 9);
  if (sym <= 285) {
    const uint32_t i = sym - 257, xb = c_len_extra[i];
    return (len + xb) | (len << 5) | (K_LEN << 9) | (xb << 11) | (uint32_t(c_len_base[i]) << 16);
  }
  return kBadLL;
}
__device__ __forceinline__ uint32_t d_entry(uint32_t sym, uint32_t len) {
  if (sym < 30) {
    const uint32_t dx = c_dist_extra[sym];
    return (len + dx) | (len << 5) | (dx << 9) | (uint32_t(c_dist_base[sym]) << 16);
  }
  return kBadD;
}

struct CanonTab {        // canonical code description of one table (RFC 1951 §3.2.2)
  uint16_t count[16];
  uint16_t first[16];
  uint16_t index[16];
  uint16_t running[16];
  uint32_t lim[16];      // (first[l] + count[l]) << (16 - l): non-decreasing in l; lim[0] = 0
};

struct HuffSmem {
  CanonTab tab[2];
  uint16_t sorted_ll[288];
  uint16_t sorted_d[32];
  uint8_t lens[320];     // 286 litlen + 30 dist code lengths
  uint32_t bad, next;
  uint32_t wlits[16];
  uint64_t wbits[16];
  uint64_t carry_bits;
  uint32_t carry_lits;
};

// canonical walk for codes longer than the table index (cwl > lut_bits): bits are taken LSB-first from buf
// returns symbol | length << 16, or -1 if no code matches
__device__ int canon_slow(uint32_t buf, const CanonTab& t, const uint16_t* sorted) {
  int code = 0, first = 0, index = 0;
  for (int l = 1; l <= 15; ++l) {
    code |= int((buf >> (l - 1)) & 1u);
    const int cnt = t.count[l];
    if (code - first < cnt) return int(sorted[index + code - first]) | (l << 16);
    index += cnt;
    first += cnt;
    first <<= 1;
    code <<= 1;
  }
  return -1;
}

__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t v, uint32_t lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(FULL, v, d);
    if (lane >= uint32_t(d)) v += t;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t v, uint32_t lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t t = __shfl_up_sync(FULL, v, d);
    if (lane >= uint32_t(d)) v += t;
  }
  return v;
}

// explicit shared-window accesses (32-bit addresses): keeps generic->shared conversions out of hot loops
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
  uint32_t v; asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory"); return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory"); return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ void sts64(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void ats_or(uint32_t a, uint32_t v) { asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait_n() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// TMA bulk copy global -> shared completed on an mbarrier (sm_90+ async proxy): one thread arms the barrier with
// the byte count and issues the copy; every waiting thread polls the barrier's phase parity.
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
  if (bytes)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(mbar), "r"(phase) : "memory");
  }
}

// Window bit readers (LSB-first, RFC 1951 §3.1.1; reading R15). The decoders keep ONE register of reader state,
// the absolute bit position `at` in the block's bitstream; window(at) returns the 64 stream bits starting there
// as (r0, r1) from three 32-bit words and two funnel shifts. A symbol (<= 48 bits with its extra bits and its
// distance) is decoded from one window, so there is no per-symbol refill or consume bookkeeping.
//   SmemBits   the bits of the current work unit were staged in shared memory by cp.async before decoding
//   GlobalBits fallback for a unit larger than the stage: the words come straight from the file (L1/L2)
__device__ __forceinline__ uint32_t ldsw(uint32_t a) {     // shared load without a memory clobber
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
struct SmemBits {
  uint32_t base;   // shared-window address holding stream bit `org` at bit 0
  uint32_t org;    // 128-aligned absolute bit position of the stage start
  __device__ __forceinline__ void window(uint32_t at, uint32_t& r0, uint32_t& r1) const {
    const uint32_t rel = at - org;
    const uint32_t p = base + ((rel >> 5) << 2);
    const uint32_t w0 = ldsw(p), w1 = ldsw(p + 4), w2 = ldsw(p + 8);
    r0 = __funnelshift_r(w0, w1, rel);
    r1 = __funnelshift_r(w1, w2, rel);
  }
};
struct GlobalBits {
  const uint32_t* g;   // 16-byte aligned start of the block's bitstream; >= 16 readable bytes follow its end
  __device__ __forceinline__ void window(uint32_t at, uint32_t& r0, uint32_t& r1) const {
    const uint32_t* p = g + (at >> 5);
    const uint32_t w0 = __ldg(p), w1 = __ldg(p + 1), w2 = __ldg(p + 2);
    r0 = __funnelshift_r(w0, w1, at);
    r1 = __funnelshift_r(w1, w2, at);
  }
};
// GlobalBits with the window kept in registers while one thread reads forward (the thread decoder's unstaged
// rounds): three stream words and the next one loaded ahead, so a symbol costs no load on its dependence chain
// (one load per 32 bits consumed). Word indices are clamped to `last`, the stream's readable end.
struct RegGlobalBits {
  const uint32_t* g;
  uint32_t last, wi, w0, w1, w2, nx;   // w0 = word wi
  __device__ __forceinline__ RegGlobalBits(const uint32_t* gp, uint32_t last_word, uint32_t at) : g(gp), last(last_word) {
    wi = at >> 5;
    w0 = __ldg(g + min(wi, last));
    w1 = __ldg(g + min(wi + 1, last));
    w2 = __ldg(g + min(wi + 2, last));
    nx = __ldg(g + min(wi + 3, last));
  }
  __device__ __forceinline__ void window(uint32_t at, uint32_t& r0, uint32_t& r1) {
    while (wi < (at >> 5)) {         // 0, 1 or 2 steps (a symbol spans <= 48 bits); positions only grow
      w0 = w1;
      w1 = w2;
      w2 = nx;
      ++wi;
      nx = __ldg(g + min(wi + 3, last));
    }
    r0 = __funnelshift_r(w0, w1, at);
    r1 = __funnelshift_r(w1, w2, at);
  }
};

struct Luts {
  uint32_t ll, d, mask_ll, mask_d;   // shared-window addresses of the two tables, index masks
  const HuffSmem* sm;     // canonical description (codes longer than the table index)
};

// One symbol (one table lookup per symbol) from the window at `at`: the litlen entry E, its extra
// bits, and for a length code the distance entry D and its extra bits. Returns the bits it spans (>= 1; a
// K_BAD entry spans 1 bit so that speculative lanes always progress). r0/d32 are kept for value extraction.
template <bool LONG, class RD>
__device__ __forceinline__ uint32_t sym_decode(RD&& rd, uint32_t at, const Luts& t, uint32_t& E, uint32_t& D,
                                               uint32_t& r0, uint32_t& d32) {
  uint32_t r1;
  rd.window(at, r0, r1);
  E = ldsw(t.ll + ((r0 & t.mask_ll) << 2));
  if (LONG && (E & 31u) == 0) {                                  // code longer than the table index
    const int sl = canon_slow(r0, t.sm->tab[0], t.sm->sorted_ll);
    E = sl < 0 ? kBadLL : ll_entry(uint32_t(sl) & 0xffffu, uint32_t(sl) >> 16);
  }
  const uint32_t t1 = E & 31u;
  d32 = __funnelshift_r(r0, r1, t1);
  D = ldsw(t.d + ((d32 & t.mask_d) << 2));
  const bool isl = ((E >> 9) & 3u) == K_LEN;
  if (LONG && isl && (D & 31u) == 0) {
    const int sl = canon_slow(d32, t.sm->tab[1], t.sm->sorted_d);
    D = sl < 0 ? kBadD : d_entry(uint32_t(sl) & 0xffffu, uint32_t(sl) >> 16);
  }
  return t1 + (isl ? (D & 31u) : 0u);
}
__device__ __forceinline__ uint32_t sym_kind(uint32_t E) { return (E >> 9) & 3u; }
__device__ __forceinline__ uint32_t sym_pair(uint32_t E) { return (E >> 14) & 1u; }   // literal pair entry
__device__ __forceinline__ uint32_t sym_len(uint32_t E, uint32_t r0) {      // match length (K_LEN)
  return (E >> 16) + ((r0 >> ((E >> 5) & 15u)) & ((1u << ((E >> 11) & 7u)) - 1u));
}
__device__ __forceinline__ uint32_t sym_dist(uint32_t D, uint32_t d32) {
  return (D >> 16) + ((d32 >> ((D >> 5) & 15u)) & ((1u << ((D >> 9) & 15u)) - 1u));
}

// a1 + a3 for one data block, whole CTA: unpack the nibble code lengths, canonical tables (warp 0; counts,
// first codes, sorted symbols by __match_any_sync ranks) and the entry-parallel fill of both LUTs in shared
// memory. Unresolved entries: 0 (LONG: canonical walk) or K_BAD. Returns false (uniformly) on a bad tree.
template <bool LONG>
__device__ bool build_tables(HuffSmem& sm, uint32_t* lut_ll, uint32_t* lut_d, const uint8_t* pl, const Args& a) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t ll_n = 1u << a.ll_bits, d_n = 1u << a.d_bits;
  if (tid == 0) { sm.bad = 0; sm.next = 0; sm.carry_bits = 0; sm.carry_lits = 0; }
  if (tid < 16) {
    sm.tab[0].count[tid] = 0; sm.tab[0].running[tid] = 0;
    sm.tab[1].count[tid] = 0; sm.tab[1].running[tid] = 0;
  }
  for (uint32_t s = tid; s < 316; s += blockDim.x) {
    const uint32_t byte = s < 286 ? pl[s >> 1] : pl[143 + ((s - 286) >> 1)];
    const uint32_t nib = s < 286 ? (s & 1) : ((s - 286) & 1);
    sm.lens[s] = uint8_t((byte >> (4 * nib)) & 15u);
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t badl = 0;
    for (int t = 0; t < 2; ++t) {
      const uint32_t n = t ? 30 : 286, off = t ? 286 : 0;
      CanonTab& T = sm.tab[t];
      for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t s = base + lane;
        const uint32_t l = s < n ? sm.lens[off + s] : 0u;
        badl |= l > a.cwl;
        const uint32_t m = __match_any_sync(FULL, l);
        if (l && (m & ((1u << lane) - 1)) == 0) T.count[l] += __popc(m);
        __syncwarp();
      }
      if (lane == 0) {
        int left = 1;
        uint32_t first = 0, index = 0;
        T.count[0] = 0;
        T.lim[0] = 0;
        for (int l = 1; l <= 15; ++l) {
          left = (left << 1) - T.count[l];
          if (left < 0) badl = 1;                        // over-subscribed code set
          first = l == 1 ? 0u : (first + T.count[l - 1]) << 1;
          T.first[l] = uint16_t(first);
          T.index[l] = uint16_t(index);
          T.lim[l] = (first + T.count[l]) << (16 - l);
          index += T.count[l];
        }
      }
      __syncwarp();
      uint16_t* sorted = t ? sm.sorted_d : sm.sorted_ll;
      for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t s = base + lane;
        const uint32_t l = s < n ? sm.lens[off + s] : 0u;
        const uint32_t m = __match_any_sync(FULL, l);
        const uint32_t rank = __popc(m & ((1u << lane) - 1));
        if (l && l <= 15) sorted[T.index[l] + T.running[l] + rank] = uint16_t(s);
        __syncwarp();
        if (l && rank == 0) T.running[l] += __popc(m);
        __syncwarp();
      }
    }
    badl |= (pl[158] | pl[159]) != 0;
    badl = __any_sync(FULL, badl);
    if (lane == 0 && badl) sm.bad = 1;
  }
  __syncthreads();
  if (sm.bad) return false;
  // canonical decode of the code at the head of `bits` (nb valid index bits, first stream bit = bit 0) with
  // table t: symbol | length << 16, or 0xffffffff when no code of length <= nb matches
  // The length L of the head code is the smallest l with v16 < lim[l] (left-justified canonical limits are
  // non-decreasing), found by a 4-step binary search; bits past nb are zero and only matter when L > nb.
  auto canon = [&](int t, uint32_t bits, uint32_t nb) -> uint32_t {
    const uint32_t v16 = __brev(bits) >> 16;   // code bits, first stream bit most significant, left-justified
    const CanonTab& T = sm.tab[t];
    uint32_t l = 0;                            // largest l in [0, 15] with lim[l] <= v16
#pragma unroll
    for (uint32_t step = 8; step; step >>= 1)
      if (l + step <= 15 && T.lim[l + step] <= v16) l += step;
    const uint32_t L = l + 1;
    if (L > nb) return 0xffffffffu;
    const uint32_t code = v16 >> (16 - L);
    if (code - T.first[L] >= T.count[L]) return 0xffffffffu;
    return uint32_t(t ? sm.sorted_d[T.index[L] + code - T.first[L]] : sm.sorted_ll[T.index[L] + code - T.first[L]]) |
           (L << 16);
  };
  for (uint32_t i = tid; i < ll_n + d_n; i += blockDim.x) {
    const int t = i >= ll_n;
    const uint32_t idx = i - (t ? ll_n : 0u);
    const uint32_t LB = t ? a.d_bits : a.ll_bits;
    const uint32_t c1 = canon(t, idx, LB);
    uint32_t ent = LONG ? 0u : (t ? kBadD : kBadLL);  // unresolved: long code (LONG) or invalid
    if (c1 != 0xffffffffu) {
      const uint32_t sym = c1 & 0xffffu, l1 = c1 >> 16;
      ent = t ? d_entry(sym, l1) : ll_entry(sym, l1);
      if (!t && sym < 256 && l1 < LB) {
        // literal pair: the remaining LB - l1 index bits may hold a whole second literal code
        const uint32_t c2 = canon(0, idx >> l1, LB - l1);
        if (c2 != 0xffffffffu && (c2 & 0xffffu) < 256)
          ent = (l1 + (c2 >> 16)) | (l1 << 5) | (K_LIT << 9) | (1u << 14) | (sym << 16) | ((c2 & 255u) << 24);
      }
    }
    (t ? lut_d : lut_ll)[idx] = ent;
  }
  __syncthreads();
  return true;
}

__device__ __forceinline__ bool huff_block_ok(const Args& a, const BlockEntry& e, uint32_t ulen) {
  return payload_ok(a, e) && e.payload_len >= kTreeBytes && e.S >= 1 && e.n_sub == (e.n_seq + e.S - 1) / e.S &&
         uint64_t(e.sub_first) + e.n_sub <= a.n_sub_total && 4ull * e.n_seq + e.n_lit <= a.max_tok &&
         e.n_lit <= ulen && e.n_seq <= ulen && uint64_t(e.payload_len) * 8 < (1ull << 31);
}

// Record of a closed sequence (FORMAT.md §2): lit_len | mcode << 10 | (dist - 1) << 16.
__device__ __forceinline__ uint32_t seq_record(uint32_t run, uint32_t L, uint32_t dist, uint32_t mm1) {
  return run | ((L - mm1) << 10) | ((dist - 1) << 16);
}

// predicated global stores (no branch around them: the serial loop below stays one instruction stream)
__device__ __forceinline__ void stg8_if(uint8_t* p, uint32_t v, bool c) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.u8 [%0], %1;\n\t}" ::"l"(p), "r"(v),
               "r"(uint32_t(c)) : "memory");
}
__device__ __forceinline__ void stg32_if(uint32_t* p, uint32_t v, bool c) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.u32 [%0], %1;\n\t}" ::"l"(p), "r"(v),
               "r"(uint32_t(c)) : "memory");
}

// Exact serial decode of a sub-block's remaining symbols from bit `at` (state si, lw, run, bad carried in):
// records at rec[0..nseq), literals at lit[0..nl). Returns 0 or a CorruptStream detail code.
template <bool LONG, class RD>
__device__ uint32_t decode_sub_exact(RD&& rd, const Luts& t, const Args& a, uint32_t at, uint32_t b0, uint32_t* rec,
                                     uint8_t* lit, uint32_t nseq, uint32_t nl, bool last, uint32_t bsz, uint32_t si,
                                     uint32_t lw, uint32_t run, uint32_t bad) {
  const uint32_t mm1 = a.min_match - 1;
  uint32_t kind = K_LIT;
  for (;;) {
    if (!last && si >= nseq) break;
    uint32_t E, D, r0, d32;
    at += sym_decode<LONG>(rd, at, t, E, D, r0, d32);
    kind = sym_kind(E);
    const bool isl = kind == K_LEN, islit = kind == K_LIT;
    if (islit && sym_pair(E)) {
      if (run + 1 == kMaxLitRun) {
        at -= (E & 31u) - ((E >> 5) & 15u);   // the first literal closes a run (R10): take it alone
      } else {
        if (lw < nl) lit[lw] = uint8_t(E >> 16);
        ++lw;
        ++run;
        E = (E & ~0x00ff0000u) | ((E >> 8) & 0x00ff0000u);   // the second literal goes through the step below
      }
    }
    if (islit && lw < nl) lit[lw] = uint8_t(E >> 16);
    lw += islit ? 1u : 0u;
    run += islit ? 1u : 0u;
    // R10/R16: a sequence closes at a length code, at 1023 literals, or at EOB with pending literals
    const bool close = isl || (islit && run == kMaxLitRun) || (kind == K_EOB && run != 0);
    const uint32_t L = sym_len(E, r0);
    if (close && si < nseq) rec[si] = isl ? seq_record(run, L, sym_dist(D, d32), mm1) : run;
    si += close ? 1u : 0u;
    run = close ? 0u : run;
    bad |= isl && ((D >> 13) & 1u || L < a.min_match || L > a.max_match);
    if (kind >= K_EOB || lw > nl || si > nseq || at - b0 > bsz) break;
  }
  if (bad) return 6;
  if (kind == K_BAD) return 2;
  if (kind == K_EOB && !last) return 7;
  if (si != nseq || run != 0 || lw != nl || at - b0 != bsz) return 9;
  return 0;
}

// Serial decode of one whole sub-block from bit `at` by one thread (the paper's thread-per-sub-block scheme,
// P:70-72): records at rec[0..nseq), literals at lit[0..nl). Returns 0 or a CorruptStream detail code.
// The bulk runs in a software-pipelined loop: the next symbol's window loads are issued as soon as this
// symbol's length is known, before this symbol's outputs (predicated stores, no branches), so the loads overlap
// the output work instead of a single dependent chain (~600 cycles per symbol before, ncu r02). It stops ahead of
// anything unusual — EOB or an invalid code, a literal run near 1023 (R10), the last 48 bits, the record or
// literal count limits, a code longer than the table — and the exact loop above finishes from that symbol
// boundary, so every check and every result is the exact loop's.
template <bool LONG, class RD>
__device__ uint32_t decode_sub_serial(RD&& rd, const Luts& t, const Args& a, uint32_t at, uint32_t* rec,
                                      uint8_t* lit, uint32_t nseq, uint32_t nl, bool last, uint32_t bsz) {
  const uint32_t mm1 = a.min_match - 1, lrange = a.max_match - a.min_match, b0 = at;
  uint32_t si = 0, lw = 0, run = 0, bad = 0;
  if (bsz > 48) {
    const uint32_t stop = b0 + bsz - 48;
    uint32_t r0, r1;
    rd.window(at, r0, r1);
    while (at < stop && si < nseq && lw + 2 <= nl && run + 2 < kMaxLitRun) {
      const uint32_t E = ldsw(t.ll + ((r0 & t.mask_ll) << 2));
      const uint32_t t1 = E & 31u, kind = sym_kind(E);
      if (kind >= K_EOB || (LONG && t1 == 0)) break;           // EOB, invalid or long code: the exact loop
      const uint32_t d32 = __funnelshift_r(r0, r1, t1);
      const uint32_t D = ldsw(t.d + ((d32 & t.mask_d) << 2));
      const bool isl = kind == K_LEN;
      if (LONG && isl && (D & 31u) == 0) break;
      const uint32_t at_n = at + t1 + (isl ? (D & 31u) : 0u);
      uint32_t r0n, r1n;
      rd.window(at_n, r0n, r1n);                               // the next symbol's loads go out first
      const uint32_t pair = sym_pair(E);                       // 0 for length entries
      const uint32_t L = sym_len(E, r0);
      stg8_if(lit + lw, E >> 16, !isl);
      stg8_if(lit + lw + 1, E >> 24, pair != 0);
      stg32_if(rec + si, seq_record(run, L, sym_dist(D, d32), mm1), isl);
      bad |= isl && (((D >> 13) & 1u) || L - a.min_match > lrange);
      lw += isl ? 0u : 1u + pair;
      si += isl ? 1u : 0u;
      run = isl ? 0u : run + 1u + pair;
      at = at_n;
      r0 = r0n;
      r1 = r1n;
    }
  }
  return decode_sub_exact<LONG>(rd, t, a, at, b0, rec, lit, nseq, nl, last, bsz, si, lw, run, bad);
}

// The unit of bits a CTA stages: [gs, ge) of the block's bitstream, as 16-byte chunks c0.. plus one chunk of
// look-ahead for the 64-bit window. All threads issue cp.async (coalesced 16-byte LDGSTS), then wait; the
// caller's __syncthreads publishes the stage. Returns false (uniformly) when it does not fit `cap` bytes.
__device__ __forceinline__ bool stage_bits(uint32_t stage_s, uint32_t cap, const uint8_t* gbits, uint64_t gmax,
                                           uint64_t gs, uint64_t ge, SmemBits& rd) {
  const uint64_t c0 = gs >> 7, nch = ((ge + 127) >> 7) - c0 + 1;
  if (nch * 16 > cap) return false;
  for (uint32_t i = threadIdx.x; i < nch; i += blockDim.x)
    cp_async16(stage_s + i * 16u, gbits + (c0 + i < (gmax >> 4) ? (c0 + i) * 16ull : gmax));
  cp_commit();
  cp_wait_n<0>();
  rd.base = stage_s;
  rd.org = uint32_t(c0 * 128);
  return true;
}

// ------------------------------------------------------------------ K1a: thread-per-sub-block decode (Bit)
// One CTA per data block; in round r thread t decodes sub-block r*T + t (used when sub-blocks are small, e.g.
// the paper's 16-sequence sub-blocks, where there are thousands per block). The T sub-blocks of a
// round are contiguous in the bitstream, so the round stages their bits in shared memory first.
// A sub-block far longer than the round's mean (a DE file's first group of a block is nearly all literals:
// C3 D=1 sub-blocks 0 and 1 carry ~26 kbit against a median of ~420) would hold its whole round on one lane;
// it is deferred to the end of the round and decoded by a whole warp with the speculative decoder (K1b, G = 1).
constexpr uint32_t kMaxHeavy = 16;          // deferred sub-blocks per round (more: decoded by their thread)
constexpr uint32_t kHeavyMeanX = 8;         // deferred when bits >= this x the round's mean (and >= kSpecMinBits)
constexpr uint32_t kRec = 64;
constexpr uint32_t kThreadNoStageThreads = 32;   // launcher: thread-decoder CTAs up to this size stage no bits
constexpr uint32_t kSpecMinBits = 32 * 96;  // sub-blocks below G*this use one lane (serial)
template <bool LONG, uint32_t G, class RD>
__device__ __forceinline__ void group_sub(const RD& rd, const Luts& t, const Args& a, uint32_t vl, uint32_t bar, uint32_t recs_s,
                          uint32_t xs_s, uint32_t b, uint32_t k, uint32_t S0, uint32_t bsz, uint32_t* rec,
                          uint8_t* lit, uint32_t nseq, uint32_t nl, bool last);
template <bool LONG>
__global__ void __launch_bounds__(256, 4) huff_thread_kernel(const Args a, uint32_t stage_cap) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  HuffSmem& sm = *reinterpret_cast<HuffSmem*>(smem_raw);
  uint32_t* lut_ll = reinterpret_cast<uint32_t*>(smem_raw + ((sizeof(HuffSmem) + 15) & ~size_t(15)));
  const uint32_t ll_n = 1u << a.ll_bits, d_n = 1u << a.d_bits;
  uint32_t* lut_d = lut_ll + ll_n;
  const uint32_t stage_s = uint32_t(__cvta_generic_to_shared(lut_d + d_n));
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const uint32_t bi = blockIdx.x, b = a.first_block + bi;
  const BlockEntry e = load_entry(a.src, b, lane);
  if (!huff_block_ok(a, e, block_ulen(a, b))) {
    if (tid == 0) report(a, GOMP_ERR_HEADER_INCONSISTENT, b, 0);
    return;
  }
  const uint8_t* pl = a.src + e.payload_off;
  if (!build_tables<LONG>(sm, lut_ll, lut_d, pl, a)) {
    if (tid == 0) report(a, GOMP_ERR_CORRUPT_STREAM, b, 0xffffffffull);
    return;
  }
  const uint32_t lut_ll_s = uint32_t(__cvta_generic_to_shared(lut_ll));
  const Luts t{lut_ll_s, lut_ll_s + ll_n * 4, ll_n - 1, d_n - 1, &sm};
  const uint64_t bit_limit = uint64_t(e.payload_len - kTreeBytes) * 8;
  const uint8_t* subt = a.src + kHeaderBytes + uint64_t(kBlockEntryBytes) * a.nb_total;
  uint8_t* tok = a.tokens + uint64_t(bi) * a.tok_stride;
  uint32_t* rec_base = reinterpret_cast<uint32_t*>(tok);
  uint8_t* lit_base = tok + 4ull * e.n_seq;
  const uint8_t* gbits = pl + kTreeBytes;
  const uint64_t gmax = a.file_len - 16 - (e.payload_off + kTreeBytes);
  // deferred (heavy) sub-blocks of the current round: {k, start bit, literal start, bits}; decoded by warps after
  // the round with their recorded-iteration areas in the stage (free then), so only if the stage holds one
  __shared__ uint4 heavy[kMaxHeavy];
  __shared__ uint32_t n_heavy;
  const uint32_t heavy_warps = min(nwarps, stage_cap / (32 * kRec));
  if (tid == 0) n_heavy = 0;
  // a2: CTA-wide exclusive scans of the sub-block bit sizes and literal counts, round by round
  for (uint32_t c0 = 0; c0 < e.n_sub; c0 += blockDim.x) {
    const uint32_t k = c0 + tid;
    uint32_t bsz = 0, nl = 0;
    if (k < e.n_sub) {
      const uint32_t* se = reinterpret_cast<const uint32_t*>(subt + uint64_t(kSubEntryBytes) * (e.sub_first + k));
      bsz = __ldg(se);
      nl = __ldg(se + 1);
    }
    const uint64_t ib = warp_incl_scan_u64(bsz, lane);
    const uint32_t il = warp_incl_scan_u32(nl, lane);
    if (lane == 31) { sm.wbits[warp] = ib; sm.wlits[warp] = il; }
    __syncthreads();
    uint64_t pre_b = sm.carry_bits;
    uint32_t pre_l = sm.carry_lits;
    for (uint32_t w = 0; w < warp; ++w) { pre_b += sm.wbits[w]; pre_l += sm.wlits[w]; }
    const uint64_t gs = sm.carry_bits;
    uint64_t tot_b = sm.carry_bits;
    uint32_t tot_l = sm.carry_lits;
    for (uint32_t w = 0; w < nwarps; ++w) { tot_b += sm.wbits[w]; tot_l += sm.wlits[w]; }
    SmemBits srd;
    const bool staged = tot_b <= bit_limit && stage_bits(stage_s, stage_cap, gbits, gmax, gs, tot_b, srd);
    __syncthreads();
    if (tid == 0) { sm.carry_bits = tot_b; sm.carry_lits = tot_l; }
    const uint64_t start = pre_b + ib - bsz;
    const uint32_t lstart = pre_l + il - nl;
    // heavy: at least kHeavyMeanX x the round's mean sub-block and long enough for the speculative decoder
    const uint32_t in_round = min(blockDim.x, e.n_sub - c0);
    const bool heavy_ok = heavy_warps != 0 && bsz >= kSpecMinBits && uint64_t(bsz) * in_round >= kHeavyMeanX * (tot_b - gs);
    if (k < e.n_sub) {
      uint32_t err = 0;
      if (start + bsz > bit_limit || uint64_t(lstart) + nl > e.n_lit) err = 1;
      const uint32_t seq0 = k * e.S;
      const uint32_t nseq = (k + 1 == e.n_sub) ? e.n_seq - seq0 : e.S;
      uint32_t hslot = kMaxHeavy;
      if (!err && heavy_ok) {
        hslot = atomicAdd(&n_heavy, 1u);
        if (hslot < kMaxHeavy) heavy[hslot] = make_uint4(k, uint32_t(start), lstart, bsz);
      }
      if (!err && hslot >= kMaxHeavy) {
        if (staged) {
          err = decode_sub_serial<LONG>(srd, t, a, uint32_t(start), rec_base + seq0, lit_base + lstart, nseq, nl,
                                        k + 1 == e.n_sub, bsz);
        } else if (stage_cap) {   // a round larger than the stage: its bits straight from L1/L2
          err = decode_sub_serial<LONG>(GlobalBits{reinterpret_cast<const uint32_t*>(gbits)}, t, a, uint32_t(start),
                                        rec_base + seq0, lit_base + lstart, nseq, nl, k + 1 == e.n_sub, bsz);
        } else {                  // no stage (one-warp CTAs, launcher): the window in registers
          RegGlobalBits rg(reinterpret_cast<const uint32_t*>(gbits), uint32_t((gmax + 16) / 4 - 1), uint32_t(start));
          err = decode_sub_serial<LONG>(rg, t, a, uint32_t(start), rec_base + seq0, lit_base + lstart, nseq, nl,
                                        k + 1 == e.n_sub, bsz);
        }
      }
      if (err) report(a, GOMP_ERR_CORRUPT_STREAM, b, (uint64_t(k) << 8) | err);
    }
    __syncthreads();
    const uint32_t nh = min(n_heavy, kMaxHeavy);
    if (nh) {
      // the deferred sub-blocks, one warp each (bits from global memory: the stage now holds recorded iterations)
      if (warp < heavy_warps) {
        for (uint32_t h = warp; h < nh; h += heavy_warps) {
          const uint4 q = heavy[h];
          const uint32_t seq0 = q.x * e.S;
          const bool last = q.x + 1 == e.n_sub;
          const uint32_t nseq = last ? e.n_seq - seq0 : e.S;
          const uint32_t* se = reinterpret_cast<const uint32_t*>(subt + uint64_t(kSubEntryBytes) * (e.sub_first + q.x));
          group_sub<LONG, 1>(GlobalBits{reinterpret_cast<const uint32_t*>(gbits)}, t, a, lane, 0u,
                             stage_s + warp * (32 * kRec), 0u, b, q.x, q.y, q.w, rec_base + seq0, lit_base + q.z,
                             nseq, __ldg(se + 1), last);
        }
      }
      __syncthreads();
      if (tid == 0) n_heavy = 0;
    }
  }
  if (tid == 0 && sm.carry_lits != e.n_lit) report(a, GOMP_ERR_CORRUPT_STREAM, b, 0xfffffffeull);
}

// ------------------------------------------------------------------ K1b: group-per-sub-block speculative decode
// B200 answer to "few, long sub-blocks" (BASELINE C2: 16 sub-blocks of ~6 KB per 256 KiB block gives only 16
// serial chains per block). A group of G warps (V = 32G virtual lanes) decodes one sub-block whose bits are
// staged in shared memory: lane p starts at bit p*c of the sub-block (c = ceil(bits/V)), i.e. usually inside a
// codeword, and decodes speculatively to the first symbol boundary at or after its chunk end, recording its
// first kRec iterations. Canonical prefix codes self-synchronise: lane p's path joins the true path when the
// true exit position of lane p-1 is one of its recorded boundaries; otherwise lane p-1 keeps decoding into lane
// p+1's chunk, and so on (hand-over chain). Then group scans give every lane its record and literal offsets and
// pass 2 decodes again from the true starts, writing records and literals. Sequences close only at length codes
// here; anything inconsistent (counts, tail, a literal run reaching 1023 = R10) sends the sub-block to the serial
// decoder, which is exact and reports corrupt streams. Same output as K1a, bit for bit.
//
// Recorded iterations per lane (self-sync window): on text a lane started at a random bit needs p50 5, p99 ~37
// symbols to join the true path; a lane that has not joined within its window costs its left neighbour a whole
// extra chunk, so the window is 64 (simulated warp pass-1 cost: 1.65x the mean chunk at 32, 1.31x at 64).
constexpr uint32_t kWarpMinAvgBits = 8192;  // launcher: mean sub-block bits from which K1b is used
constexpr uint32_t kHuffWarps = 16;         // warps per CTA (one data block; its groups share its sub-blocks)
constexpr uint32_t kHuffGMax = 8;           // warps per sub-block group: 1, 2, 4 or 8 (launcher)
constexpr uint32_t kHuffG1Bits = 32768;     // launcher: G doubles every doubling of the mean sub-block from here
                                            // (G = 1 below, 8 from 128 kbit; measured on C5 shapes)
constexpr uint32_t kStageMax = 48 * 1024;   // largest per-group bit stage (bytes)
constexpr size_t kSmemMax = 227 * 1024;     // opt-in dynamic shared memory per CTA
constexpr size_t kSmemPerSm = 228 * 1024;   // shared memory per SM (B200)
constexpr size_t kSmemReservedPerCta = 1024;
// per-group exchange area (shared memory), bytes: [0, 8V) exit records (V = 32G lanes); the sub-block index;
// per-warp aggregates A, B (8 bytes each), C and "next" flags (4 bytes each); the stage's mbarrier
__host__ __device__ constexpr uint32_t xs_k(uint32_t G) { return 8 * 32 * G; }
__host__ __device__ constexpr uint32_t xs_agga(uint32_t G) { return xs_k(G) + 16; }
__host__ __device__ constexpr uint32_t xs_aggb(uint32_t G) { return xs_agga(G) + 8 * G; }
__host__ __device__ constexpr uint32_t xs_aggc(uint32_t G) { return xs_aggb(G) + 8 * G; }
__host__ __device__ constexpr uint32_t xs_next(uint32_t G) { return xs_aggc(G) + 4 * G; }
__host__ __device__ constexpr uint32_t xs_mbar(uint32_t G) { return (xs_next(G) + 4 * G + 7) & ~7u; }
__host__ __device__ constexpr uint32_t xs_bytes(uint32_t G) { return (xs_mbar(G) + 8 + 15) & ~15u; }
static_assert(kHuffWarps % kHuffGMax == 0 && xs_bytes(kHuffGMax) <= 2304, "exchange area layout");

__host__ __device__ constexpr uint32_t group_slot_bytes(uint32_t G, uint32_t stage_cap) {
  return 32 * G * kRec + xs_bytes(G) + stage_cap;
}

// group barrier (named barrier `bar`, 32G threads). __syncwarp first: the warp must arrive converged, or the
// code after it may keep running lane by lane (measured: 3 threads per instruction in pass 2 without it).
template <uint32_t G>
__device__ __forceinline__ void gsync(uint32_t bar) {
  __syncwarp();
  if (G > 1) asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(32 * G) : "memory");
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v; asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory"); return v;
}

// One group decodes sub-block k (bits [S0, S0+bsz) of the block's stream) into rec[0..nseq), lit[0..nl).
// Pass 1 keeps per lane: iterations decoded, literals, current literal run, and for its first kRec iterations
// the bits of each (shared memory, u8) and whether it was a literal (a 64-bit register mask).
template <bool LONG, uint32_t G, class RD>
__device__ __forceinline__ void group_sub(const RD& rd, const Luts& t, const Args& a, uint32_t vl, uint32_t bar,
                                          uint32_t recs_s, uint32_t xs_s, uint32_t b, uint32_t k, uint32_t S0,
                                          uint32_t bsz, uint32_t* rec, uint8_t* lit, uint32_t nseq, uint32_t nl,
                                          bool last) {
  constexpr uint32_t V = 32 * G;
  const uint32_t lane = vl & 31, wg = vl >> 5;
  const uint32_t mm1 = a.min_match - 1, lrange = a.max_match - a.min_match;
  bool serial = bsz < kSpecMinBits * G;
  if (!serial) {
    // ---------------- pass 1: speculative scan of this lane's chunk
    const uint32_t c = (bsz + V - 1) / V;
    const uint32_t sp = S0 + vl * c;
    const uint32_t lim = S0 + min((vl + 1) * c, bsz);
    const uint32_t endb = S0 + bsz;
    // iterations decode one symbol, or two literals (pair entry): liters counts literal iterations, lits
    // literal bytes; lm/pm: literal / pair iterations among the first kRec (bit it)
    uint32_t at = sp, cnt = 0, liters = 0, lits = 0, run = 0, lm0 = 0, lm1 = 0, pm0 = 0, pm1 = 0;
    auto step1 = [&](uint32_t& islit, uint32_t& pair) {
      uint32_t E, D, r0, d32;
      const uint32_t n = sym_decode<LONG>(rd, at, t, E, D, r0, d32);
      const uint32_t kind = sym_kind(E);
      islit = kind == K_LIT ? 1u : 0u;
      pair = sym_pair(E);
      cnt += 1;
      liters += islit;
      lits += islit + pair;
      run = kind == K_LEN ? 0u : run + islit + pair;
      return n;
    };
    // 1a: the first kRec iterations, recording the bits of each (boundary it+1 = boundary it + that)
#pragma unroll 4
    for (uint32_t it = 0; it < 32; ++it) {
      uint32_t n = 0, islit = 0, pair = 0;
      if (at < endb) n = step1(islit, pair);   // never decode past the end of the sub-block
      sts8(recs_s + it * V + vl, n);
      at += n;
      lm0 |= islit << it;
      pm0 |= pair << it;
    }
#pragma unroll 4
    for (uint32_t it = 32; it < kRec; ++it) {
      uint32_t n = 0, islit = 0, pair = 0;
      if (at < endb) n = step1(islit, pair);
      sts8(recs_s + it * V + vl, n);
      at += n;
      lm1 |= islit << (it - 32);
      pm1 |= pair << (it - 32);
    }
    gsync<G>(bar);
    // 1b: continue; past the chunk end, stop at the first boundary that a later lane also recorded: from there
    // on both paths are the same (prefix codes: same position, same state => same decode)
    uint32_t q = vl + 1, ptr = 0, bq = (vl + 1) * c, exit_vl = V, exit_idx = 0;  // bq: boundary ptr of lane q
    for (;;) {
      if (at >= endb) break;
      if (at >= lim && q < V) {
        const uint32_t rel = at - S0;
        while (bq < rel) {
          if (ptr == kRec) {
            if (++q == V) break;
            ptr = 0;
            bq = q * c;
          } else {
            bq += lds8(recs_s + ptr * V + q);
            ++ptr;
          }
        }
        if (q < V && bq == rel) { exit_vl = q; exit_idx = ptr; break; }
      }
      uint32_t islit, pair;
      at += step1(islit, pair);
    }
    // ---------------- the true path: lane 0 starts at the sub-block start (its boundary 0) and hands over to
    // the lane it exited into, at that lane's recorded boundary; lanes it jumped over own nothing
    const uint32_t e_rel = at - S0;
    uint32_t merged = 0xffffffffu, mpos = 0;   // boundary index / position where this lane's true segment starts
    if (G == 1) {
      uint32_t cur = 0, idx = 0, pos = 0;
      for (uint32_t hop = 0; hop < 32 && cur < 32; ++hop) {
        if (lane == cur) { merged = idx; mpos = pos; }
        const uint32_t nl2 = __shfl_sync(FULL, exit_vl, cur), ni = __shfl_sync(FULL, exit_idx, cur);
        pos = __shfl_sync(FULL, e_rel, cur);
        cur = nl2;
        idx = ni;
      }
    } else {
      sts64(xs_s + vl * 8, exit_vl | (exit_idx << 16), e_rel);
      // common case: every lane hands over to the next one (lane V-1 runs to the end), so every lane's true
      // segment starts at its predecessor's exit; otherwise follow the chain from lane 0, hop by hop
      if (lane == 0) sts32(xs_s + xs_next(G) + wg * 4, __all_sync(FULL, exit_vl == vl + 1) ? 1u : 0u);
      else __all_sync(FULL, exit_vl == vl + 1);
      gsync<G>(bar);
      bool next_all = true;
      for (uint32_t w = 0; w < G; ++w) next_all &= lds32(xs_s + xs_next(G) + w * 4) != 0;
      if (next_all) {
        if (vl == 0) {
          merged = 0;
          mpos = 0;
        } else {
          const uint2 x = lds64(xs_s + (vl - 1) * 8);
          merged = x.x >> 16;
          mpos = x.y;
        }
      } else {
        uint32_t cur = 0, idx = 0, pos = 0;
        for (uint32_t hop = 0; hop < V && cur < V; ++hop) {
          if (vl == cur) { merged = idx; mpos = pos; }
          const uint2 x = lds64(xs_s + cur * 8);
          cur = x.x & 0xffffu;
          idx = x.x >> 16;
          pos = x.y;
        }
      }
    }
    const bool on = merged != 0xffffffffu;
    const bool is_tail = on && exit_vl == V;
    uint32_t t_start = 0, e_pos = 0, lits_t = 0, nlen_t = 0, trail_t = 0;
    bool has_t = false;
    if (on) {
      // statistics of the true segment = totals at the exit minus the counts before the merge boundary (all
      // `merged` iterations before it were decoded: the boundary lies before the sub-block end)
      const uint32_t m0 = min(merged, 32u), m1 = merged - m0;
      const uint32_t k0 = m0 == 32 ? FULL : (1u << m0) - 1u, k1 = m1 == 32 ? FULL : (1u << m1) - 1u;
      const uint32_t liters0 = __popc(lm0 & k0) + __popc(lm1 & k1);
      const uint32_t lits0 = liters0 + __popc(pm0 & k0) + __popc(pm1 & k1);
      const uint32_t nonlit0 = merged - liters0;
      t_start = mpos;
      e_pos = e_rel;
      lits_t = lits - lits0;
      // non-literal symbols of the segment = length codes (+ the block's EOB at the very end of the tail lane)
      nlen_t = (cnt - liters) - nonlit0 - ((last && is_tail) ? 1u : 0u);
      has_t = nlen_t != 0;
      trail_t = has_t ? run : lits_t;
    }
    // literal run entering this lane = carried across lanes without length codes:
    // inclusive scan of (has, val) with (h2,v2)∘(h1,v1) = h2 ? (1,v2) : (h1, v1 + v2)
    uint32_t runin;
    {
      uint32_t hv = has_t ? 1u : 0u, val = has_t ? trail_t : lits_t;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t h1 = __shfl_up_sync(FULL, hv, d), v1 = __shfl_up_sync(FULL, val, d);
        if (lane >= uint32_t(d) && !hv) { hv = h1; val = v1 + val; }
      }
      uint32_t ph = 0, pv = 0;   // aggregate of the earlier warps of the group
      if (G > 1) {
        if (lane == 31) sts64(xs_s + xs_agga(G) + wg * 8, hv, val);
        gsync<G>(bar);
        for (uint32_t w = 0; w < wg; ++w) {
          const uint2 x = lds64(xs_s + xs_agga(G) + w * 8);
          if (x.x) { ph = 1; pv = x.y; } else pv += x.y;
        }
        if (!hv) { hv = ph; val += pv; }
      }
      const uint32_t vprev = __shfl_up_sync(FULL, val, 1);
      runin = lane == 0 ? pv : vprev;
    }
    // ---------------- offsets: exclusive scans of sequences (closed by length codes) and literals
    uint32_t seqs = nlen_t;   // + the EOB-closed final literal-only sequence of the block
    if (last && is_tail && (has_t ? trail_t : runin + lits_t) != 0) seqs += 1;
    uint32_t seq_inc = warp_incl_scan_u32(seqs, lane), lit_inc = warp_incl_scan_u32(lits_t, lane);
    uint32_t seq_tot = __shfl_sync(FULL, seq_inc, 31), lit_tot = __shfl_sync(FULL, lit_inc, 31);
    bool tail_ok = __any_sync(FULL, is_tail && e_pos == bsz);
    if (G > 1) {
      if (lane == 0) sts64(xs_s + xs_aggb(G) + wg * 8, seq_tot | (tail_ok ? 0x80000000u : 0u), lit_tot);
      gsync<G>(bar);
      seq_tot = lit_tot = 0;
      tail_ok = false;
      for (uint32_t w = 0; w < G; ++w) {
        const uint2 x = lds64(xs_s + xs_aggb(G) + w * 8);
        if (w < wg) { seq_inc += x.x & 0x7fffffffu; lit_inc += x.y; }
        seq_tot += x.x & 0x7fffffffu;
        lit_tot += x.y;
        tail_ok |= (x.x >> 31) != 0;
      }
    }
    serial = seq_tot != nseq || lit_tot != nl || !tail_ok;
    if (!serial) {
      // ---------------- pass 2: decode from the true start, write records and literals
      uint32_t* recp = rec + (seq_inc - seqs);
      uint8_t* litp = lit + (lit_inc - lits_t);
      uint32_t run2 = runin, bad = 0, maxr = 0;
      bool saw_eob = false;
      uint32_t at2 = S0 + t_start;
      const uint32_t stop = S0 + e_pos;
      while (at2 < stop) {
        uint32_t E, D, r0, d32;
        const uint32_t n = sym_decode<LONG>(rd, at2, t, E, D, r0, d32);
        at2 += n;
        const uint32_t kind = sym_kind(E);
        if (kind >= K_EOB) {               // end of block or invalid code: leaves the loop (rare)
          if (kind == K_EOB) {
            saw_eob = true;
            if (run2 != 0 && recp < rec + nseq) *recp++ = run2;
          } else {
            bad = 1;
          }
          break;
        }
        if (kind == K_LIT) {
          const uint32_t pair = sym_pair(E);
          *litp = uint8_t(E >> 16);
          if (pair) litp[1] = uint8_t(E >> 24);
          litp += 1 + pair;
          run2 += 1 + pair;
        } else {
          const uint32_t L = sym_len(E, r0);
          *recp++ = seq_record(run2, L, sym_dist(D, d32), mm1);
          bad |= ((D >> 13) & 1u) | (L - a.min_match > lrange ? 1u : 0u);
          maxr = max(maxr, run2);
          run2 = 0;
        }
      }
      maxr = max(maxr, run2);
      // R10: a literal run reaching 1023 closes a sequence, which the offsets above did not count
      serial = __any_sync(FULL, maxr >= kMaxLitRun);
      if (G > 1) {
        if (lane == 0) sts32(xs_s + xs_aggc(G) + wg * 4, serial ? 1u : 0u);
        gsync<G>(bar);
        for (uint32_t w = 0; w < G; ++w) serial |= lds32(xs_s + xs_aggc(G) + w * 4) != 0;
      }
      if (!serial) {
        // the last lane of the last sub-block must end with EOB; EOB anywhere else is corrupt
        if (bad || at2 != stop || saw_eob != (last && is_tail))
          report(a, GOMP_ERR_CORRUPT_STREAM, b, (uint64_t(k) << 8) | 10u);
        return;
      }
      gsync<G>(bar);   // pass-2 writes are done before the serial decoder rewrites the sub-block
    }
  }
  // ---------------- serial fallback (small sub-blocks, literal runs >= 1023, anything inconsistent): lane 0
  // decodes all of it and validates it against the table
  if (vl == 0) {
    // the exact loop alone (rare here; the pipelined loop's extra code measured ~1-3% slower on the whole kernel)
    const uint32_t err = decode_sub_exact<LONG>(rd, t, a, S0, S0, rec, lit, nseq, nl, last, bsz, 0u, 0u, 0u, 0u);
    if (err) report(a, GOMP_ERR_CORRUPT_STREAM, b, (uint64_t(k) << 8) | err);
  }
}

// One CTA of kHuffWarps warps per data block: after the CTA builds the tables, each group of G warps takes the
// next sub-block of the block from a shared counter, stages its bits in the group's shared-memory slot
// (cp.async; a sub-block larger than the slot reads its bits from global memory instead) and decodes it with
// group_sub. Only group barriers after the table build: a group never waits for another group's sub-block.
template <bool LONG, uint32_t G>
__global__ void __launch_bounds__(32 * kHuffWarps) huff_warp_kernel(const Args a, uint32_t stage_cap) {
  constexpr uint32_t V = 32 * G;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  HuffSmem& sm = *reinterpret_cast<HuffSmem*>(smem_raw);
  uint32_t* lut_ll = reinterpret_cast<uint32_t*>(smem_raw + ((sizeof(HuffSmem) + 15) & ~size_t(15)));
  const uint32_t ll_n = 1u << a.ll_bits, d_n = 1u << a.d_bits;
  uint32_t* lut_d = lut_ll + ll_n;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t grp = warp / G, vl = tid % V, bar = 1 + grp;
  const uint32_t slot_s = uint32_t(__cvta_generic_to_shared(lut_d + d_n)) + grp * group_slot_bytes(G, stage_cap);
  const uint32_t recs_s = slot_s, xs_s = slot_s + V * kRec, stage_s = xs_s + xs_bytes(G);
  // in a split grid each CTA takes only a share of a block's sub-blocks (launcher)
  uint32_t bi = blockIdx.x, part = 0, parts = 1;
  if (bi >= a.split_first) {
    const uint32_t j = bi - a.split_first;
    parts = a.split_parts;
    bi = a.split_first + j / parts;
    part = j % parts;
  }
  const uint32_t b = a.first_block + bi;
  const BlockEntry e = load_entry(a.src, b, lane);
  if (!huff_block_ok(a, e, block_ulen(a, b))) {
    if (tid == 0) report(a, GOMP_ERR_HEADER_INCONSISTENT, b, 0);
    return;
  }
  const uint32_t k_lo = part * e.n_sub / parts, k_hi = (part + 1) * e.n_sub / parts;
  const uint8_t* pl = a.src + e.payload_off;
  if (!build_tables<LONG>(sm, lut_ll, lut_d, pl, a)) {
    if (tid == 0) report(a, GOMP_ERR_CORRUPT_STREAM, b, 0xffffffffull);
    return;
  }
  const uint32_t lut_ll_s = uint32_t(__cvta_generic_to_shared(lut_ll));
  const Luts t{lut_ll_s, lut_ll_s + ll_n * 4, ll_n - 1, d_n - 1, &sm};
  // the group's stage is filled by one TMA bulk copy per sub-block, completed on this mbarrier
  const uint32_t mbar = xs_s + xs_mbar(G);
  if (vl == 0) { mbar_init(mbar, 1); fence_mbar_init(); }
  __syncthreads();
  uint32_t phase = 0;
  const uint64_t bit_limit = uint64_t(e.payload_len - kTreeBytes) * 8;
  const uint32_t* subt = reinterpret_cast<const uint32_t*>(a.src + kHeaderBytes + uint64_t(kBlockEntryBytes) * a.nb_total) +
                         2ull * e.sub_first;
  uint8_t* tok = a.tokens + uint64_t(bi) * a.tok_stride;
  uint32_t* rec_base = reinterpret_cast<uint32_t*>(tok);
  uint8_t* lit_base = tok + 4ull * e.n_seq;
  const uint64_t gmax = a.file_len - 16 - (e.payload_off + kTreeBytes);
  const uint8_t* gbits = pl + kTreeBytes;
  for (;;) {
    if (vl == 0) sts32(xs_s + xs_k(G), k_lo + atomicAdd(&sm.next, 1u));
    gsync<G>(bar);
    const uint32_t k = lds32(xs_s + xs_k(G));
    if (k >= k_hi) break;
    // a2: start bit and literal offset of sub-block k = sums over the entries before it (warp-parallel)
    uint64_t sb = 0;
    uint32_t sl = 0;
    for (uint32_t i = lane; i < k; i += 32) { sb += __ldg(subt + 2 * i); sl += __ldg(subt + 2 * i + 1); }
#pragma unroll
    for (int d = 16; d; d >>= 1) { sb += __shfl_xor_sync(FULL, sb, d); sl += __shfl_xor_sync(FULL, sl, d); }
    const uint32_t bsz = __ldg(subt + 2 * k), nl = __ldg(subt + 2 * k + 1);
    const uint32_t seq0 = k * e.S;
    const bool last = k + 1 == e.n_sub;
    const uint32_t nseq = last ? e.n_seq - seq0 : e.S;
    if (sb + bsz > bit_limit || uint64_t(sl) + nl > e.n_lit) {
      if (vl == 0) report(a, GOMP_ERR_CORRUPT_STREAM, b, (uint64_t(k) << 8) | 1u);
    } else {
      // stage [sb, sb + bsz) as 16-byte chunks (+1 chunk of window look-ahead) into the group's slot
      const uint64_t c0 = sb >> 7, nch = ((sb + bsz + 127) >> 7) - c0 + 1;
      if (nch * 16 <= stage_cap) {
        // one bulk copy of the chunks inside the readable buffer (the look-ahead chunk past it stays stale: its
        // bits lie beyond the stream end, only window padding); earlier generic reads of the slot are ordered
        // before the async-proxy write by the group barrier + proxy fence
        if (vl == 0) {
          const uint64_t lim = gmax >> 4;
          const uint32_t nb = c0 < lim ? uint32_t(nch < lim - c0 ? nch : lim - c0) * 16u : 0u;
          fence_proxy_async();
          bulk_g2s(stage_s, gbits + c0 * 16ull, nb, mbar);
        }
        mbar_wait(mbar, phase);
        phase ^= 1u;
        group_sub<LONG, G>(SmemBits{stage_s, uint32_t(c0 * 128)}, t, a, vl, bar, recs_s, xs_s, b, k, uint32_t(sb),
                           bsz, rec_base + seq0, lit_base + sl, nseq, nl, last);
      } else {
        group_sub<LONG, G>(GlobalBits{reinterpret_cast<const uint32_t*>(gbits)}, t, a, vl, bar, recs_s, xs_s, b, k,
                           uint32_t(sb), bsz, rec_base + seq0, lit_base + sl, nseq, nl, last);
      }
    }
    gsync<G>(bar);   // the group is done with the slot (stage, records, exchange area)
  }
}


// ------------------------------------------------------------------ K2: warp-per-block LZ77 (+ Byte fusion)
//
// Output goes through a per-warp shared-memory ring holding the last RING bytes of the block (RING >= window
// + group output), so back-reference sources are read on chip; completed 16-byte chunks are flushed to HBM
// with coalesced 16-byte stores. Literal bytes are staged into a per-warp shared-memory ring ahead of use
// with cp.async (LDGSTS) in 512-byte units; records are prefetched four groups ahead in registers. A group too
// large for the rings (e.g. 32 literal runs of 1023 bytes) is processed directly in global memory.
// All shared-memory traffic uses 32-bit shared-window addresses (ld/st.shared), never generic pointers.
constexpr uint32_t kLitRing = 2048;
constexpr uint32_t kLitUnit = 512;    // 32 lanes x 16 B per cp.async instruction
constexpr uint32_t kLitAhead = 1024;  // prefetch distance in literal bytes
constexpr uint32_t kFlushBytes = 2048;   // ring -> HBM flush granularity

// per-warp shared layout: [output ring RING][literal ring 2 KiB]
__host__ __device__ constexpr uint32_t lz_warp_bytes(uint32_t ring) { return ring + kLitRing; }

// byte-granular copy without overlap (dist >= L, reading R2), global memory (slow path)
__device__ __forceinline__ void copy_nolap(uint8_t* d, const uint8_t* s, uint32_t n) {
  uint32_t k = 0;
  for (; k + 8 <= n; k += 8) {
    uint8_t t0 = s[k], t1 = s[k + 1], t2 = s[k + 2], t3 = s[k + 3], t4 = s[k + 4], t5 = s[k + 5], t6 = s[k + 6], t7 = s[k + 7];
    d[k] = t0; d[k + 1] = t1; d[k + 2] = t2; d[k + 3] = t3; d[k + 4] = t4; d[k + 5] = t5; d[k + 6] = t6; d[k + 7] = t7;
  }
  for (; k < n; ++k) d[k] = s[k];
}
__device__ __forceinline__ void copy_lits_global(uint8_t* d, const uint8_t* __restrict__ s, uint32_t n) {
  uint32_t k = 0;
  for (; k + 4 <= n; k += 4) {
    uint8_t t0 = __ldg(s + k), t1 = __ldg(s + k + 1), t2 = __ldg(s + k + 2), t3 = __ldg(s + k + 3);
    d[k] = t0; d[k + 1] = t1; d[k + 2] = t2; d[k + 3] = t3;
  }
  for (; k < n; ++k) d[k] = __ldg(s + k);
}

// Copy n bytes between power-of-two shared rings (base addresses D/S, masks dm/sm = size-1); the source range
// does not overlap the destination range: byte head until the destination is word aligned, aligned 32-bit
// stores of funnel-shifted source words (bytes of a source word outside [s, s+n) are discarded), byte tail.
__device__ __forceinline__ void ring_copy(uint32_t D, uint32_t dm, uint32_t d, uint32_t S, uint32_t sm, uint32_t s,
                                          uint32_t n) {
  uint32_t h = (4u - (d & 3u)) & 3u;
  if (h > n) h = n;
  for (uint32_t k = 0; k < h; ++k) sts8(D + ((d + k) & dm), lds8(S + ((s + k) & sm)));
  d += h; s += h; n -= h;
  const uint32_t nw = n >> 2;
  if (nw) {
    const uint32_t sh = (s & 3u) * 8u;
    uint32_t sw = s & ~3u;
    uint32_t lo = lds32(S + (sw & sm));
    for (uint32_t k = 0; k < nw; ++k) {
      const uint32_t hi = lds32(S + ((sw + 4) & sm));
      sts32(D + (d & dm), __funnelshift_r(lo, hi, sh));
      lo = hi; sw += 4; d += 4;
    }
    s += nw * 4; n -= nw * 4;
  }
  for (uint32_t k = 0; k < n; ++k) sts8(D + ((d + k) & dm), lds8(S + ((s + k) & sm)));
}

struct GlobalOut {
  uint8_t* out;
  __device__ __forceinline__ void copy(uint32_t dst, uint32_t src, uint32_t n) const { copy_nolap(out + dst, out + src, n); }
};
struct RingOut {
  uint32_t ring, rm;
  __device__ __forceinline__ void copy(uint32_t dst, uint32_t src, uint32_t n) const { ring_copy(ring, rm, dst, ring, rm, src, n); }
};

// a7 for one warp group with per-lane copies: MRR (Fig. alg:mrr) or SC. Returns false on NO_PROGRESS.
template <int STRAT, bool STATS, class Out>
__device__ __forceinline__ bool resolve_group(const Args& a, const Out& o, uint32_t lane, bool has, uint32_t dst,
                                              uint32_t src, uint32_t L, uint32_t op, uint32_t b, uint32_t g0) {
  if (STRAT == GOMP_STRAT_SC) {          // Sequential Copying
    __syncwarp();
    uint32_t m = __ballot_sync(FULL, has);
    while (m) {
      const uint32_t j = __ffs(m) - 1;
      if (lane == j) o.copy(dst, src, L);
      __syncwarp();
      m &= m - 1;
    }
    return true;
  }
  // MRR (Fig. alg:mrr): HWM = destination of the lowest pending lane = end of the gap-free written prefix
  // (R1); a lane is ready when its source lies below HWM or inside its own literal string (R4)
  __syncwarp();
  bool pending = has;
  uint32_t votes = __ballot_sync(FULL, pending);
  uint32_t rounds = 0;
  while (votes) {
    const uint32_t p = __ffs(votes) - 1;
    const uint32_t hwm = __shfl_sync(FULL, dst, p);
    const bool ready = pending && (src + L <= hwm || src >= op);
    if (ready) o.copy(dst, src, L);
    ++rounds;
    if (STATS) {
      uint32_t bytes = ready ? L : 0u;
#pragma unroll
      for (int d = 16; d; d >>= 1) bytes += __shfl_xor_sync(FULL, bytes, d);
      if (lane == 0 && rounds < 33) atomicAdd(stats_ptr(a) + 33 + rounds, (unsigned long long)bytes);
    }
    if (!__any_sync(FULL, ready)) {
      if (lane == 0) report(a, GOMP_ERR_NO_PROGRESS, b, g0);
      return false;
    }
    pending = pending && !ready;
    __syncwarp();
    votes = __ballot_sync(FULL, pending);
  }
  if (STATS && lane == 0) atomicAdd(stats_ptr(a) + (rounds < 33 ? rounds : 32), 1ull);
  return true;
}

__device__ __forceinline__ void cp_wait(uint32_t allowed) {
  if (allowed >= 2) asm volatile("cp.async.wait_group 2;\n" ::: "memory");
  else if (allowed == 1) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

template <int STRAT, bool STATS>
__global__ void __launch_bounds__(32 * kLz77Warps) lz77_kernel(const Args a, int byte_mode) {
  extern __shared__ __align__(16) uint8_t lz_smem[];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wi >= a.n_blocks) return;
  const uint32_t RING = a.ring_bytes, RM = RING - 1, LM = kLitRing - 1;
  const uint32_t ring = uint32_t(__cvta_generic_to_shared(lz_smem)) + (threadIdx.x >> 5) * lz_warp_bytes(RING);
  const uint32_t lring = ring + RING;
  const uint32_t b = a.first_block + wi;
  const BlockEntry e = load_entry(a.src, b, lane);
  const uint32_t ulen = block_ulen(a, b);
  const uint8_t* base;
  // Byte records may be empty (lit_len 0, no back-reference): the oracle's expansion accepts them, so n_seq is
  // bounded by the payload only; Bit sequences are never empty (a literal or a length code closes each)
  bool ok = e.n_lit <= ulen && (byte_mode || e.n_seq <= ulen);
  if (byte_mode) {
    ok = ok && payload_ok(a, e) && 4ull * e.n_seq + e.n_lit <= e.payload_len && e.S == 0 && e.n_sub == 0 && e.sub_first == 0;
    base = a.src + e.payload_off;
  } else {
    ok = ok && 4ull * e.n_seq + e.n_lit <= a.max_tok;
    base = a.tokens + uint64_t(wi) * a.tok_stride;
  }
  if (!ok) {
    if (lane == 0) report(a, GOMP_ERR_HEADER_INCONSISTENT, b, 1);
    return;
  }
  const uint32_t* recs = reinterpret_cast<const uint32_t*>(base);
  const uint8_t* lits = base + 4ull * e.n_seq;
  // literal stream staging: rel position = byte offset from the 16-aligned address below the stream
  const uint8_t* lal = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(lits) & ~uintptr_t(15));
  const uint32_t lofs = uint32_t(lits - lal);
  const uint32_t lend16 = (lofs + e.n_lit + 15u) & ~15u;
  uint32_t lf = 0;  // literal bytes (rel) issued to the ring, multiple of kLitUnit
  uint8_t* out = a.dst + uint64_t(wi) * a.block_size;
  const uint32_t mm1 = a.min_match - 1, n_seq = e.n_seq;
  const RingOut ro{ring, RM};
  const GlobalOut go{out};

  uint32_t o_carry = 0, l_carry = 0, flushed = 0;
  uint32_t rq0 = lane < n_seq ? __ldg(recs + lane) : 0u;
  uint32_t rq1 = lane + 32 < n_seq ? __ldg(recs + lane + 32) : 0u;
  uint32_t rq2 = lane + 64 < n_seq ? __ldg(recs + lane + 64) : 0u;
  uint32_t rq3 = lane + 96 < n_seq ? __ldg(recs + lane + 96) : 0u;
  for (uint32_t g0 = 0; g0 < n_seq; g0 += 32) {
    const uint32_t i = g0 + lane;
    const bool act = i < n_seq;
    const uint32_t r = rq0;
    rq0 = rq1; rq1 = rq2; rq2 = rq3;
    rq3 = (i + 128 < n_seq) ? __ldg(recs + i + 128) : 0u;
    // a5: decode the record and one packed exclusive scan (literal offset | output offset << 16)
    const uint32_t lit = r & 1023u, mcode = (r >> 10) & 63u, dist = (r >> 16) + 1u;
    const uint32_t L = mcode ? mcode + mm1 : 0u;
    const uint32_t v = lit | ((lit + L) << 16);
    const uint32_t incl = warp_incl_scan_u32(v, lane);
    const uint32_t tot = __shfl_sync(FULL, incl, 31);
    const uint32_t ex = incl - v;
    const uint32_t lp = l_carry + (ex & 0xffffu);
    const uint32_t op = o_carry + (ex >> 16);
    const uint32_t dst = op + lit;
    const uint32_t src = dst - dist;
    const bool bad_ref = act && L && (dist < L || dist > a.window || dist > dst || L > a.max_match);
    const bool bad_rec = act && !mcode && (r >> 16);
    const uint32_t lit_sum = tot & 0xffffu, out_sum = tot >> 16;
    const bool bad_sz = o_carry + out_sum > ulen || l_carry + lit_sum > e.n_lit;
    const bool any_rec = __any_sync(FULL, bad_rec);
    if (__any_sync(FULL, bad_ref) || any_rec || bad_sz) {
      if (lane == 0) report(a, bad_sz || any_rec ? GOMP_ERR_CORRUPT_STREAM : GOMP_ERR_MALFORMED_BACKREF, b, g0);
      return;
    }
    const bool has = act && L;
    // fast path: the group and the window fit the ring, and the group does not overwrite unflushed output
    const bool fast = out_sum + a.window + 16 <= RING && o_carry + out_sum - flushed <= RING &&
                      lit_sum + kLitAhead <= kLitRing;
    if (fast) {
      // stage the group's literals (rel range [lofs + l_carry, need)) into the literal ring
      const uint32_t need = lofs + l_carry + lit_sum;
      while (lf < need + kLitAhead && lf < lend16 && lf + kLitUnit <= lofs + l_carry + kLitRing) {
        const uint32_t off = lf + lane * 16;
        if (off < lend16) cp_async16(lring + (off & LM), lal + off);
        cp_commit();
        lf += kLitUnit;
      }
      const uint32_t issued = lf / kLitUnit, needed = (need + kLitUnit - 1) / kLitUnit;
      cp_wait(issued > needed ? issued - needed : 0u);
      __syncwarp();
      // a6: literal strings into the output ring; a7: back-references inside the ring (MRR / SC)
      if (act) ring_copy(ring, RM, op, lring, LM, lofs + lp, lit);
      if (!resolve_group<STRAT, STATS>(a, ro, lane, has, dst, src, L, op, b, g0)) return;
      __syncwarp();
      // flush completed 16-byte chunks to HBM (coalesced 16-byte stores), at least kFlushBytes at a time
      const uint32_t q1 = (o_carry + out_sum) >> 4;
      if (q1 * 16 >= flushed + kFlushBytes) {
        for (uint32_t q = (flushed >> 4) + lane; q < q1; q += 32)
          reinterpret_cast<uint4*>(out)[q] = lds128(ring + ((q * 16) & RM));
        flushed = q1 * 16;
      }
    } else {
      // group too large for the rings: flush the ring, run the group in global memory, reload the window
      __syncwarp();
      for (uint32_t p = flushed + lane; p < o_carry; p += 32) out[p] = uint8_t(lds8(ring + (p & RM)));
      flushed = o_carry;
      __syncwarp();
      if (act) copy_lits_global(out + op, lits + lp, lit);
      if (!resolve_group<STRAT == GOMP_STRAT_SC ? GOMP_STRAT_SC : GOMP_STRAT_MRR, STATS>(a, go, lane, has, dst, src,
                                                                                       L, op, b, g0))
        return;
      __syncwarp();
      const uint32_t o_new = o_carry + out_sum;
      const uint32_t keep = min(o_new, max(a.window, 16u) + 16u);
      for (uint32_t p = o_new - keep + lane; p < o_new; p += 32) sts8(ring + (p & RM), out[p]);
      flushed = o_new;
      cp_wait(0);
      lf = ((lofs + l_carry + lit_sum) / kLitUnit) * kLitUnit;
      __syncwarp();
    }
    o_carry += out_sum;
    l_carry += lit_sum;
  }
  cp_wait(0);
  __syncwarp();
  if (o_carry != ulen || l_carry != e.n_lit) {
    if (lane == 0) report(a, GOMP_ERR_CORRUPT_STREAM, b, 0xffffffffull);
    return;
  }
  const uint32_t q1 = o_carry >> 4;
  for (uint32_t q = (flushed >> 4) + lane; q < q1; q += 32)
    reinterpret_cast<uint4*>(out)[q] = lds128(ring + ((q * 16) & RM));
  for (uint32_t p = max(q1 * 16, flushed) + lane; p < o_carry; p += 32) out[p] = uint8_t(lds8(ring + (p & RM)));
}

size_t lz77_smem_bytes(uint32_t ring) { return size_t(kLz77Warps) * lz_warp_bytes(ring); }

// ------------------------------------------------------------------ K2b: several warps per data block (DE)
//
// One warp per data block (the paper's mapping) leaves a B200 SM with ~7 LZ77 warps at BASELINE C2
// (1024 blocks), so every group pays the full latency of its dependent chain. Here the kBW warps of one CTA
// take kBW consecutive DE groups of the same block at once (a "batch" of up to 32·kBW sequences). Each warp
// runs the paper's per-group steps on its group with one sequence per lane: a5 record + one packed
// exclusive scan, then the batch offsets from the kBW group totals; a6 every lane copies its literal string
// from the staged literal ring into the output ring; a7 every lane copies its back-reference inside the output
// ring, in one round (DE). Under DE a group's sources lie below the group's start or in the lane's
// own literal string, so a warp only has to wait for the earlier warps of its batch when one of its sources
// reaches into the batch (a chain of named barriers; no wait otherwise). Copies are 32-bit word copies with
// funnel shifts (no overlap: reading R2). Literal bytes are prefetched by cp.async (LDGSTS) in 2 KiB units
// into an 8 KiB literal ring well ahead of use; completed output is flushed with coalesced 16-byte stores.
// BW = warps (groups in flight) per data block: 4 for full grids (throughput: ~7 CTAs per SM), 16 for grids of at
// most one CTA per SM (latency: C1's 16 blocks; one batch barrier per 16 groups, a 16-warp chain per batch)
constexpr uint32_t kBW = 4;                 // throughput variant
constexpr uint32_t kBWLat = 16;             // latency variant
constexpr uint32_t kRingLat = 65536;        // latency variant's output ring: >= window (<= 32 KiB) + 2 x 16 KiB
template <uint32_t BW>
struct LzCfg {
  static constexpr uint32_t LR = BW == 4 ? 8192 : 32768;        // literal ring bytes (4 prefetch units)
  static constexpr uint32_t LUnit = 32 * BW * 16;               // literal prefetch unit: one 16-byte cp.async per thread
  static constexpr uint32_t MaxOut = BW == 4 ? 4096 : 16384;    // fast path: batch output bytes = zero-ahead distance
  static constexpr uint32_t Flush = MaxOut;                     // ring -> HBM flush granularity
  // batch tables after the ring: literal ring | per-warp group totals (u32 each) | per-warp flags
  // group totals and flags of a batch, double-buffered by batch parity (one CTA barrier per batch)
  static constexpr uint32_t Tab = LR, Flg = Tab + 8 * BW, End = Flg + 8 * BW;
};
static_assert(LzCfg<4>::End == 8192 + 64 && LzCfg<kBWLat>::LR == 4 * LzCfg<kBWLat>::LUnit, "batch layout");

template <uint32_t BW = kBW>
__host__ __device__ constexpr uint32_t lzb_smem_bytes(uint32_t ring) { return ring + LzCfg<BW>::End; }

// named barriers 1..3 between consecutive warps (immediate ids: ptxas then reserves only those)
__device__ __forceinline__ void chain_sync(uint32_t id) {
  if (id == 1) asm volatile("bar.sync 1, 64;" ::: "memory");
  else if (id == 2) asm volatile("bar.sync 2, 64;" ::: "memory");
  else asm volatile("bar.sync 3, 64;" ::: "memory");
}
__device__ __forceinline__ void chain_arrive(uint32_t id) {
  if (id == 1) asm volatile("bar.arrive 1, 64;" ::: "memory");
  else if (id == 2) asm volatile("bar.arrive 2, 64;" ::: "memory");
  else asm volatile("bar.arrive 3, 64;" ::: "memory");
}
// latency variant: chain barriers 1..15 (a register id: ptxas reserves all 16)
__device__ __forceinline__ void chain_sync_r(uint32_t id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void chain_arrive_r(uint32_t id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }

// Copy n >= 1 bytes from power-of-two shared ring S (mask sm) position s to the output ring D (mask dm) position
// d; the ranges do not overlap (dist >= L, reading R2). The destination range of the current batch is zero
// beforehand (zero-ahead frontier), so the two partial words at its ends are OR-ed in (RED.OR; a neighbouring
// lane may own the other bytes) and every word in between is a plain store: no byte loops. Source word k of the
// destination word at p is the funnel shift of the two source words around p + (s - d); bytes of a source word
// outside [s, s+n) are discarded by the masks.
__device__ __forceinline__ void or_copy(uint32_t D, uint32_t dm, uint32_t d, uint32_t S, uint32_t sm, uint32_t s,
                                        uint32_t n) {
  const uint32_t e = d + n, last = (e - 1) & ~3u, sh = ((s - d) & 3u) * 8u;
  uint32_t p = d & ~3u, sa = (s - (d & 3u)) & ~3u;
  uint32_t lo = ldsw(S + (sa & sm)), hi = ldsw(S + ((sa + 4) & sm));
  const uint32_t mlast = 0xffffffffu >> ((3u - ((e - 1) & 3u)) * 8u);
  uint32_t m = 0xffffffffu << ((d & 3u) * 8u);
  if (p == last) m &= mlast;
  ats_or(D + (p & dm), __funnelshift_r(lo, hi, sh) & m);
  p += 4; sa += 4; lo = hi;
  for (; p + 16 <= last; p += 16) {
    const uint32_t w1 = ldsw(S + ((sa + 4) & sm)), w2 = ldsw(S + ((sa + 8) & sm)), w3 = ldsw(S + ((sa + 12) & sm)),
                   w4 = ldsw(S + ((sa + 16) & sm));
    sts32(D + (p & dm), __funnelshift_r(lo, w1, sh));
    sts32(D + ((p + 4) & dm), __funnelshift_r(w1, w2, sh));
    sts32(D + ((p + 8) & dm), __funnelshift_r(w2, w3, sh));
    sts32(D + ((p + 12) & dm), __funnelshift_r(w3, w4, sh));
    lo = w4; sa += 16;
  }
  for (; p < last; p += 4) {
    hi = ldsw(S + ((sa + 4) & sm));
    sts32(D + (p & dm), __funnelshift_r(lo, hi, sh));
    lo = hi; sa += 4;
  }
  if (p == last) ats_or(D + (p & dm), __funnelshift_r(lo, ldsw(S + ((sa + 4) & sm)), sh) & mlast);
}

// Latency variant of or_copy for grids that leave SMs idle: 16 destination bytes per step, the five source words of
// a step loaded before any store and every destination word OR-ed in (masked; zero beyond the copy), so a copy of
// up to 13 bytes costs one shared-memory round trip and no branch. It spends more shared atomics per byte, which
// loses under full load (measured: one C2 block 0.33 vs 0.41 ms; 1024 blocks 0.74 vs 0.60 ms).
__device__ __forceinline__ void or_copy_ll(uint32_t D, uint32_t dm, uint32_t d, uint32_t S, uint32_t sm, uint32_t s,
                                           uint32_t n) {
  const uint32_t e = d + n, first = d & ~3u, last = (e - 1) & ~3u, sh = ((s - d) & 3u) * 8u;
  const uint32_t mfirst = 0xffffffffu << ((d & 3u) * 8u), mlast = 0xffffffffu >> ((3u - ((e - 1) & 3u)) * 8u);
  uint32_t sa = (s - (d & 3u)) & ~3u, lo = ldsw(S + (sa & sm));
  for (uint32_t p = first; p <= last; p += 16, sa += 16) {
    uint32_t w[5];
    w[0] = lo;
#pragma unroll
    for (int k = 1; k < 5; ++k) w[k] = ldsw(S + ((sa + 4 * k) & sm));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t q = p + 4 * k;
      uint32_t m = q <= last ? 0xffffffffu : 0u;
      if (q == first) m &= mfirst;
      if (q == last) m &= mlast;
      ats_or(D + (q & dm), __funnelshift_r(w[k], w[k + 1], sh) & m);
    }
    lo = w[4];
  }
}
template <bool LOWLAT>
__device__ __forceinline__ void ring_copy(uint32_t D, uint32_t dm, uint32_t d, uint32_t S, uint32_t sm, uint32_t s,
                                          uint32_t n) {
  if (LOWLAT) or_copy_ll(D, dm, d, S, sm, s, n);
  else or_copy(D, dm, d, S, sm, s, n);
}

// RC: the output ring size when known at compile time (the default window's 16 KiB ring; 0 = a.ring_bytes),
// so the ring masks and the offsets of the literal ring and batch tables are immediates
template <bool STATS, bool LOWLAT, uint32_t RC, uint32_t BW = kBW>
__global__ void __launch_bounds__(32 * BW, BW == 4 ? 8 : 1) lz77_batch_kernel(const Args a, int byte_mode) {
  using C = LzCfg<BW>;
  static_assert(BW == 4 || BW == kBWLat, "batch widths");
  extern __shared__ __align__(16) uint8_t bz[];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t bi = blockIdx.x, b = a.first_block + bi;
  const uint32_t RING = RC ? RC : a.ring_bytes, RM = RING - 1, LM = C::LR - 1;
  const uint32_t ring = uint32_t(__cvta_generic_to_shared(bz));
  const uint32_t lring = ring + RING, tab = ring + RING + C::Tab, flg = ring + RING + C::Flg;
  const BlockEntry e = load_entry(a.src, b, lane);
  const uint32_t ulen = block_ulen(a, b);
  const uint8_t* base;
  // Byte records may be empty (lit_len 0, no back-reference): the oracle's expansion accepts them, so n_seq is
  // bounded by the payload only; Bit sequences are never empty (a literal or a length code closes each)
  bool ok = e.n_lit <= ulen && (byte_mode || e.n_seq <= ulen);
  if (byte_mode) {
    ok = ok && payload_ok(a, e) && 4ull * e.n_seq + e.n_lit <= e.payload_len && e.S == 0 && e.n_sub == 0 && e.sub_first == 0;
    base = a.src + e.payload_off;
  } else {
    ok = ok && 4ull * e.n_seq + e.n_lit <= a.max_tok;
    base = a.tokens + uint64_t(bi) * a.tok_stride;
  }
  if (!ok) {
    if (threadIdx.x == 0) report(a, GOMP_ERR_HEADER_INCONSISTENT, b, 1);
    return;
  }
  const uint32_t* recs = reinterpret_cast<const uint32_t*>(base);
  const uint8_t* lits = base + 4ull * e.n_seq;
  // literal stream staging: rel position = byte offset from the 16-aligned address below the stream
  const uint8_t* lal = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(lits) & ~uintptr_t(15));
  const uint32_t lofs = uint32_t(lits - lal), lend16 = (lofs + e.n_lit + 15u) & ~15u;
  uint32_t lf = 0;        // rel literal bytes issued to the literal ring (multiple of C::LUnit)
  uint32_t lB_prev = 0;   // literal start of the previous batch: bytes below it are consumed
  uint8_t* out = a.dst + uint64_t(bi) * a.block_size;
  const uint32_t mm1 = a.min_match - 1, n_seq = e.n_seq, ngroups = (n_seq + 31) / 32;
  const GlobalOut go{out};
  uint32_t oB = 0, lB = 0, flushed = 0;
  uint32_t i = w * 32 + lane;                                   // this lane's sequence in the current batch
  const uint32_t* rp = recs + i;
  uint32_t r_next = i < n_seq ? __ldg(rp) : 0u;
  // zero-ahead frontier (16-aligned): ring bytes [oB, zf) are zero before a batch writes them (or_copy), and
  // zf >= oB + C::MaxOut
  uint32_t zf = C::MaxOut;
  for (uint32_t p = 16 * threadIdx.x; p < zf; p += 16 * 32 * BW) sts128(ring + p, make_uint4(0u, 0u, 0u, 0u));
  for (uint32_t B0 = 0; B0 < ngroups; B0 += BW, i += 32 * BW) {
    const uint32_t g = B0 + w;
    const bool act = i < n_seq;
    const uint32_t r = r_next;
    rp += 32 * BW;
    r_next = (i + 32 * BW) < n_seq ? __ldg(rp) : 0u;
    // literal prefetch: units up to (previous batch start + ring) may be issued (earlier bytes are consumed);
    // all but the two most recent units have landed after the wait (published by the barrier below)
    while (lf < lend16 && lf + C::LUnit <= lofs + lB_prev + C::LR) {
      const uint32_t off = lf + threadIdx.x * 16;
      if (off < lend16) cp_async16(lring + (off & LM), lal + off);
      cp_commit();
      lf += C::LUnit;
    }
    cp_wait_n<2>();
    // a5: record decode + packed scan of this warp's group
    const uint32_t lit = r & 1023u, mcode = (r >> 10) & 63u, dist = (r >> 16) + 1u;
    const uint32_t L = mcode ? mcode + mm1 : 0u;
    const uint32_t v = lit | ((lit + L) << 16);
    const uint32_t incl = warp_incl_scan_u32(v, lane);
    const uint32_t tot = __shfl_sync(FULL, incl, 31);
    const uint32_t ex = incl - v;
    // group-local checks, published with the totals so that ONE barrier makes every decision uniform:
    // 1 = malformed record (reported here), 2 = the group breaks the DE rule (its source neither precedes the
    // group nor lies in the sequence's own literals; R2/A4), 4 = a source may precede the block (exact test below)
    const bool has = act && L;
    // FORMAT.md §2: dist >= L (R2), dist <= window (R9), L <= max_match (a 6-bit mcode reaches min_match + 62)
    const bool lbad = act && (L ? (dist < L || dist > a.window || L > a.max_match) : (r >> 16) != 0);
    const bool any_lbad = __any_sync(FULL, lbad);
    const bool de_ok = __all_sync(FULL, !has || dist >= (ex >> 16) + lit + L || dist <= lit);
    const bool maybe_neg = __any_sync(FULL, has && dist > oB + (ex >> 16) + lit);
    const uint32_t par = (B0 / BW) & 1u, tabk = tab + par * 4 * BW, flgk = flg + par * 4 * BW;
    if (lane == 0) {
      sts32(tabk + w * 4, tot);
      sts32(flgk + w * 4, (any_lbad ? 1u : 0u) | (de_ok ? 0u : 2u) | (maybe_neg ? 4u : 0u));
    }
    if (any_lbad) {
      const bool any_rec = __any_sync(FULL, act && !L && (r >> 16) != 0);
      if (lane == 0) report(a, any_rec ? GOMP_ERR_CORRUPT_STREAM : GOMP_ERR_MALFORMED_BACKREF, b, g * 32);
    }
    __syncthreads();
    // flush the completed output of earlier batches (final after the barrier), at least kFlushBytes at a time
    if (oB >= flushed + C::Flush + 16) {
      const uint32_t q1 = oB >> 4;
      for (uint32_t q = (flushed >> 4) + threadIdx.x; q < q1; q += 32 * BW)
        reinterpret_cast<uint4*>(out)[q] = lds128(ring + ((q * 16) & RM));
      flushed = q1 * 16;
    }
    // batch offsets (all warps compute all of them); group totals are (out << 16 | lit), each half < 2^16
    uint32_t fl, OT, LT, ob_w, lb_w;
    if (BW == 4) {
      const uint4 T4 = lds128(tabk), F4 = lds128(flgk);
      fl = F4.x | F4.y | F4.z | F4.w;
      const uint32_t o0 = T4.x >> 16, o1 = T4.y >> 16, o2 = T4.z >> 16, o3 = T4.w >> 16;
      const uint32_t l0 = T4.x & 0xffffu, l1 = T4.y & 0xffffu, l2 = T4.z & 0xffffu, l3 = T4.w & 0xffffu;
      OT = o0 + o1 + o2 + o3;
      LT = l0 + l1 + l2 + l3;
      ob_w = w == 0 ? 0u : w == 1 ? o0 : w == 2 ? o0 + o1 : o0 + o1 + o2;
      lb_w = w == 0 ? 0u : w == 1 ? l0 : w == 2 ? l0 + l1 : l0 + l1 + l2;
    } else {
      // lane j < BW holds group j's totals: two warp scans (the 16-bit halves may overflow when summed)
      const uint32_t tj = lane < BW ? lds32(tabk + 4 * lane) : 0u, fj = lane < BW ? lds32(flgk + 4 * lane) : 0u;
      fl = __reduce_or_sync(FULL, fj);
      const uint32_t oj = tj >> 16, lj = tj & 0xffffu;
      const uint32_t io = warp_incl_scan_u32(oj, lane), il = warp_incl_scan_u32(lj, lane);
      OT = __shfl_sync(FULL, io, 31);
      LT = __shfl_sync(FULL, il, 31);
      ob_w = __shfl_sync(FULL, io - oj, w);
      lb_w = __shfl_sync(FULL, il - lj, w);
    }
    if (fl & 1u) return;                                       // device error already reported
    if (oB + OT > ulen || lB + LT > e.n_lit) {                 // more output or literals than the block holds
      if (threadIdx.x == 0) report(a, GOMP_ERR_CORRUPT_STREAM, b, uint64_t(B0) * 32);
      return;
    }
    const uint32_t og = oB + ob_w, lg = lB + lb_w;
    const uint32_t op = og + (ex >> 16), lp = lg + (ex & 0xffffu), dst = op + lit, src = dst - dist;
    if (fl & 4u) {                                             // rare (the block's first window): exact test
      const bool neg = has && dist > dst;
      if (__syncthreads_or(neg)) {
        if (__any_sync(FULL, neg) && lane == 0) report(a, GOMP_ERR_MALFORMED_BACKREF, b, g * 32);
        return;
      }
    }
    // fast path: the batch fits the zero-ahead distance, its literals have landed, and the ring holds the
    // window, this batch and the next batch's zeroed range without touching unflushed output
    const uint32_t landed = lf > 2 * C::LUnit ? lf - 2 * C::LUnit : 0u;
    const bool room = OT <= C::MaxOut && a.window + 2 * C::MaxOut <= RING &&
                      oB + OT + C::MaxOut - flushed <= RING;
    bool fast = !(fl & 2u) && room && lofs + lB + LT <= landed;
    if (!fast && !(fl & 2u) && room && lofs + lB + LT <= lf) {
      // the batch's literals are issued but maybe still in flight: wait for all of them (uniform, rare)
      cp_wait_n<0>();
      __syncthreads();
      fast = true;
    }
    if (fast) {
      // a6: literal string of each sequence from the literal ring into the output ring
      if (act && lit) ring_copy<LOWLAT>(ring, RM, op, lring, LM, lofs + lp, lit);
      // a7 (DE, one round): named barrier w (64 threads) passes warp w-1's "done" to warp w. Only the lanes whose
      // source overlaps output of this batch (written by earlier warps) copy after the barrier; the others copy
      // before it, so the chain's critical path holds only those copies, and each warp's "done" still implies
      // all earlier ones
      const bool inb = has && src < op && src + L > oB;
      if (has && !inb) ring_copy<LOWLAT>(ring, RM, dst, ring, RM, src, L);
      if (BW == 4) {
        if (w > 0) chain_sync(w);
        if (inb) ring_copy<LOWLAT>(ring, RM, dst, ring, RM, src, L);
        if (w + 1 < BW) chain_arrive(w + 1);
      } else {
        if (w > 0) chain_sync_r(w);
        if (inb) ring_copy<LOWLAT>(ring, RM, dst, ring, RM, src, L);
        if (w + 1 < BW) chain_arrive_r(w + 1);
      }
      // zero the next batch's range (beyond everything this batch writes or reads)
      const uint32_t zt = (oB + OT + C::MaxOut + 15u) & ~15u;
      for (uint32_t p = zf + 16 * threadIdx.x; p < zt; p += 16 * 32 * BW) sts128(ring + (p & RM), make_uint4(0u, 0u, 0u, 0u));
      zf = max(zf, zt);
      if (STATS) {
        const uint32_t any = __ballot_sync(FULL, has);
        uint32_t bytes = has ? L : 0u;
#pragma unroll
        for (int d = 16; d; d >>= 1) bytes += __shfl_xor_sync(FULL, bytes, d);
        if (lane == 0 && g < ngroups) {
          atomicAdd(stats_ptr(a) + (any ? 1 : 0), 1ull);
          if (any) atomicAdd(stats_ptr(a) + 33 + 1, (unsigned long long)bytes);
        }
      }
    } else {
      // slow batch (too large for the buffers, or not DE): flush the ring, then warp 0 runs the groups of the
      // batch one by one in global memory with MRR (exact for any valid file), then reload the window
      for (uint32_t p = flushed + threadIdx.x; p < oB; p += 32 * BW) out[p] = uint8_t(lds8(ring + (p & RM)));
      __syncthreads();
      if (w == 0) {
        uint32_t og2 = oB, lg2 = lB;
        for (uint32_t ww = 0; ww < BW; ++ww) {
          const uint32_t gg = B0 + ww, ii = gg * 32 + lane;
          if (gg >= ngroups) break;
          if (STATS && lane == 0 && (lds32(flgk + ww * 4) & 2u)) atomicAdd(stats_ptr(a) + 66, 1ull);
          const bool act2 = ii < n_seq;
          const uint32_t r2 = act2 ? __ldg(recs + ii) : 0u;
          const uint32_t lit2 = r2 & 1023u, mc2 = (r2 >> 10) & 63u, dist2 = (r2 >> 16) + 1u;
          const uint32_t L2 = mc2 ? mc2 + mm1 : 0u, v2 = lit2 | ((lit2 + L2) << 16);
          const uint32_t inc2 = warp_incl_scan_u32(v2, lane), ex2 = inc2 - v2;
          const uint32_t op2 = og2 + (ex2 >> 16), lp2 = lg2 + (ex2 & 0xffffu), dst2 = op2 + lit2;
          if (act2) copy_lits_global(out + op2, lits + lp2, lit2);
          if (!resolve_group<GOMP_STRAT_MRR, STATS>(a, go, lane, act2 && L2, dst2, dst2 - dist2, L2, op2, b, gg * 32))
            break;
          __syncwarp();
          const uint32_t tu = lds32(tabk + ww * 4);
          og2 += tu >> 16;
          lg2 += tu & 0xffffu;
        }
      }
      __syncthreads();
      const uint32_t o_new = oB + OT;
      const uint32_t keep = min(o_new, max(a.window, 16u) + 16u);
      for (uint32_t p = o_new - keep + threadIdx.x; p < o_new; p += 32 * BW) sts8(ring + (p & RM), out[p]);
      flushed = o_new;
      // restart the zero-ahead frontier at the new output end
      const uint32_t z16 = (o_new + 15u) & ~15u;
      if (threadIdx.x < z16 - o_new) sts8(ring + ((o_new + threadIdx.x) & RM), 0u);
      zf = (o_new + C::MaxOut + 15u) & ~15u;
      for (uint32_t p = z16 + 16 * threadIdx.x; p < zf; p += 16 * 32 * BW) sts128(ring + (p & RM), make_uint4(0u, 0u, 0u, 0u));
      // literal staging restarts at the next batch's literals (everything issued has landed)
      cp_wait_n<0>();
      lf = max(lf, (lofs + lB + LT) / C::LUnit * C::LUnit);
    }
    lB_prev = lB;
    oB += OT;
    lB += LT;
  }
  cp_wait_n<0>();
  __syncthreads();
  if (oB != ulen || lB != e.n_lit) {
    if (threadIdx.x == 0) report(a, GOMP_ERR_CORRUPT_STREAM, b, 0xffffffffull);
    return;
  }
  const uint32_t q1 = oB >> 4;
  for (uint32_t q = (flushed >> 4) + threadIdx.x; q < q1; q += 32 * BW)
    reinterpret_cast<uint4*>(out)[q] = lds128(ring + ((q * 16) & RM));
  for (uint32_t p = max(q1 * 16, flushed) + threadIdx.x; p < oB; p += 32 * BW) out[p] = uint8_t(lds8(ring + (p & RM)));
}


// Launch facts cached per device: the SM count, the dynamic shared memory each kernel has been opted in to, and
// the occupancy of (kernel, threads, shared memory) triples. After its first use on a device a decompression
// call issues no attribute or occupancy query (C1's single-launch latency). One mutex guards the cache: the
// library's entry points may be called from several host threads, on several devices.
constexpr int kMaxDevices = 64;
struct LaunchCache {
  std::mutex mu;
  int sms[kMaxDevices] = {};
  struct Attr { int dev; const void* f; size_t smem; };
  struct Occ { int dev; const void* f; int threads; size_t smem; int occ; };
  std::vector<Attr> attrs;
  std::vector<Occ> occs;
};
LaunchCache& launch_cache() {
  static LaunchCache c;
  return c;
}
int current_device() {
  int d = 0;
  return cudaGetDevice(&d) == cudaSuccess && d >= 0 && d < kMaxDevices ? d : 0;
}
uint32_t sm_count() {
  const int dev = current_device();
  LaunchCache& c = launch_cache();
  std::lock_guard<std::mutex> g(c.mu);
  if (!c.sms[dev]) {
    int v = 0;
    c.sms[dev] = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0 ? v : 1;
  }
  return uint32_t(c.sms[dev]);
}
// opt kernel f in to `smem` bytes of dynamic shared memory on the current device (once per larger size)
template <class F>
void ensure_smem(F* f, size_t smem) {
  const int dev = current_device();
  LaunchCache& c = launch_cache();
  std::lock_guard<std::mutex> g(c.mu);
  for (auto& a : c.attrs)
    if (a.dev == dev && a.f == reinterpret_cast<const void*>(f)) {
      if (a.smem < smem && cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) == cudaSuccess)
        a.smem = smem;
      return;
    }
  if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) == cudaSuccess)
    c.attrs.push_back({dev, reinterpret_cast<const void*>(f), smem});
}
template <class F>
int occupancy(F* f, int threads, size_t smem) {
  const int dev = current_device();
  LaunchCache& c = launch_cache();
  std::lock_guard<std::mutex> g(c.mu);
  for (const auto& o : c.occs)
    if (o.dev == dev && o.f == reinterpret_cast<const void*>(f) && o.threads == threads && o.smem == smem) return o.occ;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, threads, smem) != cudaSuccess) occ = 0;
  if (c.occs.size() < 256) c.occs.push_back({dev, reinterpret_cast<const void*>(f), threads, smem, occ});
  return occ;
}

template <int S>
void launch_lz77(const Args& a, bool stats, bool byte_mode, cudaStream_t st) {
  const dim3 grid((a.n_blocks + kLz77Warps - 1) / kLz77Warps), block(32 * kLz77Warps);
  const size_t smem = lz77_smem_bytes(a.ring_bytes);
  if (stats) {
    ensure_smem(lz77_kernel<S, true>, smem);
    lz77_kernel<S, true><<<grid, block, smem, st>>>(a, byte_mode ? 1 : 0);
  } else {
    ensure_smem(lz77_kernel<S, false>, smem);
    lz77_kernel<S, false><<<grid, block, smem, st>>>(a, byte_mode ? 1 : 0);
  }
}


// reset_ws: clear the error word / statistics first (a pipelined caller clears them once); tok_block0: block
// slot of the workspace token buffer used for block `first` (pipelined chunks in flight use disjoint slots)

gomp_status decompress_range(const gomp_info* info, uint32_t first, uint32_t nblk, const uint8_t* d_src,
                             size_t src_len, uint8_t* d_dst, size_t dst_cap, void* d_ws, size_t ws_bytes,
                             int strategy, cudaStream_t st, bool reset_ws = true, uint32_t tok_block0 = 0) {
  if (!info || !d_src || !d_ws || (!d_dst && info->uncompressed_len)) return GOMP_ERR_INVALID_ARG;
  if (uint64_t(first) + nblk > info->n_blocks) return GOMP_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(d_src) | reinterpret_cast<uintptr_t>(d_ws)) & 15u) return GOMP_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(d_dst) & 15u) return GOMP_ERR_INVALID_ARG;
  if (src_len < info->file_len) return GOMP_ERR_TRUNCATED;
  int s = strategy & GOMP_STRAT_MASK;
  const bool stats = (strategy & GOMP_FLAG_STATS) != 0;
  const bool decode_only = (strategy & GOMP_FLAG_DECODE_ONLY) != 0, lz77_only = (strategy & GOMP_FLAG_LZ77_ONLY) != 0;
  if (strategy & ~(GOMP_STRAT_MASK | GOMP_FLAG_STATS | GOMP_FLAG_DECODE_ONLY | GOMP_FLAG_LZ77_ONLY |
                   GOMP_FLAG_HUFF_THREAD | GOMP_FLAG_HUFF_WARP)) return GOMP_ERR_INVALID_ARG;
  if (decode_only && lz77_only) return GOMP_ERR_INVALID_ARG;
  if (s == GOMP_STRAT_AUTO) s = info->de ? GOMP_STRAT_DE : GOMP_STRAT_MRR;
  if (s != GOMP_STRAT_DE && s != GOMP_STRAT_MRR && s != GOMP_STRAT_SC) return GOMP_ERR_INVALID_ARG;
  uint64_t out_bytes = 0;
  if (nblk) {
    const uint64_t lo = uint64_t(first) * info->block_size;
    const uint64_t hi = std::min<uint64_t>(uint64_t(first + nblk) * info->block_size, info->uncompressed_len);
    out_bytes = hi - lo;
  }
  if (dst_cap < out_bytes) return GOMP_ERR_DST_TOO_SMALL;
  size_t need = 0;
  gomp_decompress_workspace_size(info, tok_block0 + (nblk ? nblk : 1), &need);
  if (ws_bytes < need) return GOMP_ERR_WORKSPACE_TOO_SMALL;
  if (reset_ws && cudaMemsetAsync(d_ws, 0, kWsHeaderBytes, st) != cudaSuccess) return GOMP_ERR_CUDA;
  if (nblk == 0) return GOMP_OK;
  Args a{};
  a.src = d_src;
  a.dst = d_dst;
  a.ws = static_cast<uint8_t*>(d_ws);
  a.tokens = a.ws + kWsHeaderBytes + uint64_t(tok_block0) * align16(info->max_block_tokens);
  a.total = info->uncompressed_len;
  a.file_len = info->file_len;
  a.payload_base = info->payload_base;
  a.tok_stride = align16(info->max_block_tokens);
  a.first_block = first;
  a.n_blocks = nblk;
  a.block_size = info->block_size;
  a.window = info->window_size;
  a.min_match = info->min_match;
  a.max_match = info->max_match;
  a.cwl = info->cwl;
  a.ll_bits = kMaxLutBits;                              // literal/length table: 11 index bits (literal pairs)
  a.d_bits = std::min<uint32_t>(info->cwl, kMaxLutBits);
  a.max_tok = info->max_block_tokens;
  a.n_sub_total = info->n_sub_total;
  a.nb_total = info->n_blocks;
  a.ring_bytes = 16384;
  a.split_first = nblk;   // no K1b split grid unless the launcher sets one
  a.split_parts = 1;
  while (a.ring_bytes < info->window_size + 2 * LzCfg<kBW>::MaxOut) a.ring_bytes <<= 1;
  const bool byte_mode = info->mode == GOMP_MODE_BYTE;
  if (!byte_mode && !lz77_only) {
    const uint64_t nb = std::max<uint32_t>(info->n_blocks, 1);
    const uint64_t avg_sub = (uint64_t(info->n_sub_total) + nb - 1) / nb;
    const uint64_t avg_bits = info->n_sub_total ? (info->file_len - info->payload_base) * 8 / info->n_sub_total : 0;
    const bool LONGc = info->cwl > kMaxLutBits;
    const size_t tabs = ((sizeof(HuffSmem) + 15) & ~size_t(15)) +
                        ((size_t(1) << a.ll_bits) + (size_t(1) << a.d_bits)) * sizeof(uint32_t);
    const int force = strategy & (GOMP_FLAG_HUFF_THREAD | GOMP_FLAG_HUFF_WARP);
    // measured crossover (matrix data, 64 KiB-512 KiB blocks x 4-128 sub-blocks, profiles/r01_ncu_summary.md):
    // the speculative warp decoder wins from ~11 kbit sub-blocks up, the thread decoder below ~6 kbit
    const bool use_warp = force ? force == GOMP_FLAG_HUFF_WARP : avg_bits >= kWarpMinAvgBits;
    const uint64_t avg_bytes = avg_bits / 8 + 1;   // mean sub-block payload bytes
    if (use_warp) {
      // few long sub-blocks (e.g. C2: 16 per 256 KiB block): a group of G warps per sub-block, speculative decode,
      // G = 1 / 2 / 4 / 8 for mean sub-blocks below 32 / 64 / 128 kbit / above (C5 shapes, 256 MiB matrix,
      // decode ms for G = 1, 2, 4, 8: 22 kbit 0.74-0.79, 0.83-0.96, -, -; 44 kbit 1.00-1.11, 0.75-0.78, 0.88-0.99,
      // 1.66-1.95; 87 kbit -, 1.08-1.12, 0.77-0.82, 1.02-1.20; 174 kbit -, 1.43-1.64, 1.12-1.18, 0.81-0.90;
      // 696 kbit -, 2.41, 1.97, 1.44; tools/crossover.py); C2's 48 kbit sub-blocks take G = 2;
      // per group a bit stage of 1.3x the mean sub-block (+ slack); up to kHuffWarps/G groups per
      // CTA, as many as the sub-blocks of a block and the shared memory allow
      // bit stage per group: 1.3x the mean sub-block (+ slack), but no more than lets two 16-warp CTAs share an SM
      // (a sub-block larger than the stage reads its bits from L1/L2 instead)
      const uint32_t G = avg_bits < kHuffG1Bits ? 1u : avg_bits < 2 * kHuffG1Bits ? 2u : avg_bits < 4 * kHuffG1Bits ? 4u : 8u;
      const uint64_t two_per_sm = ((kSmemPerSm / 2 - kSmemReservedPerCta - tabs) / (kHuffWarps / G) -
                                   32 * G * kRec - xs_bytes(G)) & ~uint64_t(15);
      const uint32_t cap = uint32_t(std::min<uint64_t>({kStageMax, align16(avg_bytes * 13 / 10 + 96),
                                                        std::max<uint64_t>(two_per_sm, align16(avg_bytes + 96))}));
      const size_t slot = group_slot_bytes(G, cap);
      const uint64_t fit = (kSmemMax - tabs) / slot;
      const uint32_t ngr = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>({kHuffWarps / G, fit, avg_sub})));
      const size_t smem = tabs + ngr * slot;
      void (*kern)(const Args, uint32_t) = nullptr;
      switch (G) {
        case 1: kern = LONGc ? huff_warp_kernel<true, 1> : huff_warp_kernel<false, 1>; break;
        case 2: kern = LONGc ? huff_warp_kernel<true, 2> : huff_warp_kernel<false, 2>; break;
        case 4: kern = LONGc ? huff_warp_kernel<true, 4> : huff_warp_kernel<false, 4>; break;
        default: kern = LONGc ? huff_warp_kernel<true, 8> : huff_warp_kernel<false, 8>; break;
      }
      ensure_smem(kern, smem);
      // split grid: blocks that fill at most half of the resident CTA slots are each decoded by two CTAs taking
      // half of its sub-blocks (the idle slots would otherwise wait out whole-block latencies; measured on the
      // first 74 blocks of C2: 0.095 vs 0.149 ms). Splitting only the last partial wave of a large grid was
      // measured as no gain (C2: 0.674 vs 0.675 ms).
      const int occ = occupancy(kern, int(32 * G * ngr), smem);
      const uint32_t slots = uint32_t(std::max(occ, 0)) * sm_count();
      uint32_t grid = nblk;
      if (2 * uint64_t(nblk) <= slots && avg_sub >= 2 * uint64_t(ngr)) {
        a.split_first = 0;
        a.split_parts = 2;
        grid = 2 * nblk;
      }
      kern<<<grid, 32 * G * ngr, smem, st>>>(a, cap);
    } else {
      // many short sub-blocks (e.g. the paper's 16 sequences per sub-block): one thread per sub-block, rounds
      // of nt sub-blocks staged together
      // with >= 6 blocks per SM, 128 threads: rounds of 128 sub-blocks wait for a slower sub-block less often
      // than rounds of 256, and the smaller stage lets ~8 CTAs share an SM (C3 D=1 S=16, 1024 blocks: 0.93 vs
      // 1.26 ms; 64/96/192 measured slower); fewer, larger blocks keep 256 threads per block (C5 1 MiB blocks:
      // 128 threads lose 21%)
      const uint32_t nt_max = nblk >= 6 * sm_count() ? 128u : 256u;
      const uint32_t nt = uint32_t(std::min<uint64_t>(nt_max, std::max<uint64_t>(32, (avg_sub + 31) / 32 * 32)));
      // one-warp CTAs (<= 32 sub-blocks per block) stage nothing: their round's stage (the whole block's bits x 1.5)
      // would hold an SM to 4-5 such CTAs; each thread keeps its window in registers and reads the bits through
      // L1 instead (C5 64 KiB x 32 sub-blocks: decode 1.48 -> 1.18 ms per 256 MiB; 64 threads: 1.14 -> 1.16,
      // so larger CTAs keep the stage)
      const uint32_t cap = nt <= kThreadNoStageThreads ? 0u : uint32_t(std::min<uint64_t>(kStageMax, align16(avg_bytes * nt * 3 / 2 + 512)));
      const size_t smem = tabs + cap;
      if (LONGc) {
        ensure_smem(huff_thread_kernel<true>, smem);
        huff_thread_kernel<true><<<nblk, nt, smem, st>>>(a, cap);
      } else {
        ensure_smem(huff_thread_kernel<false>, smem);
        huff_thread_kernel<false><<<nblk, nt, smem, st>>>(a, cap);
      }
    }
    if (cudaGetLastError() != cudaSuccess) return GOMP_ERR_CUDA;
    if (decode_only) return GOMP_OK;
  }
  switch (s) {
    case GOMP_STRAT_DE: {
      if (!stats && nblk <= sm_count() * kLatCtasPerSm) {
        // at most one CTA per SM (C1, small files, shard ranges): 16 warps per block, one barrier per 16 groups
        // (C1, 16 blocks: 82 -> 55.6 us per decompression in a CUDA graph; without the chain: 32.9 us)
        const size_t smem = lzb_smem_bytes<kBWLat>(kRingLat);
        // load-first copies (measured: C1 55.6 us per decompression vs 73.9 with the instruction-lean copies)
        const auto kern = lz77_batch_kernel<false, true, kRingLat, kBWLat>;
        ensure_smem(kern, smem);
        kern<<<nblk, 32 * kBWLat, smem, st>>>(a, byte_mode ? 1 : 0);
        break;
      }
      const size_t smem = lzb_smem_bytes(a.ring_bytes);
      // a grid of at most one CTA per SM leaves the SMs latency-bound: the low-latency copies win there
      constexpr uint32_t kRing0 = 16384;   // the default window's ring (compile-time masks and offsets)
      const bool r0 = a.ring_bytes == kRing0, lowlat = nblk <= sm_count() * kLowLatCtasPerSm;
      const auto kern = stats ? lz77_batch_kernel<true, false, 0>
                        : lowlat ? (r0 ? lz77_batch_kernel<false, true, kRing0> : lz77_batch_kernel<false, true, 0>)
                                 : (r0 ? lz77_batch_kernel<false, false, kRing0> : lz77_batch_kernel<false, false, 0>);
      ensure_smem(kern, smem);
      kern<<<nblk, 32 * kBW, smem, st>>>(a, byte_mode ? 1 : 0);
      break;
    }
    case GOMP_STRAT_MRR: launch_lz77<GOMP_STRAT_MRR>(a, stats, byte_mode, st); break;
    default: launch_lz77<GOMP_STRAT_SC>(a, stats, byte_mode, st); break;
  }
  return cudaGetLastError() == cudaSuccess ? GOMP_OK : GOMP_ERR_CUDA;
}

}  // namespace
}  // namespace gomp

using namespace gomp;

GOMP_EXPORT gomp_status gomp_decompress(const gomp_info* info, const uint8_t* d_src, size_t src_len, uint8_t* d_dst,
                                        size_t dst_cap, void* d_ws, size_t ws_bytes, int strategy, void* stream) {
  if (!info) return GOMP_ERR_INVALID_ARG;
  return decompress_range(info, 0, info->n_blocks, d_src, src_len, d_dst, dst_cap, d_ws, ws_bytes, strategy,
                          static_cast<cudaStream_t>(stream));
}

GOMP_EXPORT gomp_status gomp_decompress_blocks(const gomp_info* info, uint32_t first_block, uint32_t n_blocks,
                                               const uint8_t* d_src, size_t src_len, uint8_t* d_dst, size_t dst_cap,
                                               void* d_ws, size_t ws_bytes, int strategy, void* stream) {
  return decompress_range(info, first_block, n_blocks, d_src, src_len, d_dst, dst_cap, d_ws, ws_bytes, strategy,
                          static_cast<cudaStream_t>(stream));
}

namespace gomp {
namespace {
// Streams and events of the pipelined host path, created once per host thread and device and reused by every
// call (C1 latency: creating 6 streams and up to 26 events per call cost tens of microseconds). A call records
// its events in order; an event re-recorded by a later call has already been waited on (cudaStreamWaitEvent
// captures the event's state when it is called).
struct Pipe {
  cudaStream_t h2d = nullptr, d2h = nullptr, comp[kPipeStreams] = {};
  cudaEvent_t ev[2 * kPipeMaxChunks + 2] = {};
  int nev = 0, made = 0;
  bool ok = true;
  Pipe() {
    ok = cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking) == cudaSuccess &&
         cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking) == cudaSuccess;
    for (auto& c : comp) ok = ok && cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking) == cudaSuccess;
  }
  void begin() { nev = 0; }
  cudaEvent_t event() {
    if (nev == int(sizeof(ev) / sizeof(ev[0]))) { ok = false; return nullptr; }
    if (nev == made) {
      if (cudaEventCreateWithFlags(&ev[nev], cudaEventDisableTiming) != cudaSuccess) { ok = false; return nullptr; }
      ++made;
    }
    return ev[nev++];
  }
  ~Pipe() {   // at thread exit; errors (e.g. the context already torn down at process exit) are ignored
    for (int i = 0; i < made; ++i) cudaEventDestroy(ev[i]);
    for (auto& c : comp) if (c) cudaStreamDestroy(c);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
  }
};
Pipe* thread_pipe() {
  thread_local std::unique_ptr<Pipe> pipes[kMaxDevices];
  std::unique_ptr<Pipe>& p = pipes[current_device()];
  if (!p || !p->ok) p.reset(new Pipe());
  p->begin();
  return p->ok ? p.get() : nullptr;
}
}  // namespace
}  // namespace gomp

// End-to-end path ("In/Out"): the blocks are cut into up to kPipeMaxChunks chunks; chunk i's
// compressed bytes go host->device on one copy stream, its kernels run on compute stream i % kPipeStreams once
// they have arrived, and its output goes device->host on the other copy stream once they are done. Both copy
// directions and the kernels of different chunks overlap; the caller's stream waits for the last copy.
GOMP_EXPORT gomp_status gomp_decompress_host(const gomp_info* info, const uint8_t* h_src, size_t src_len, uint8_t* h_dst,
                                             size_t dst_cap, uint8_t* d_src_buf, uint8_t* d_dst_buf, void* d_ws,
                                             size_t ws_bytes, int strategy, void* stream) {
  if (!info || !h_src || !d_src_buf || !d_ws || (!d_dst_buf && info->uncompressed_len)) return GOMP_ERR_INVALID_ARG;
  if (src_len < info->file_len) return GOMP_ERR_TRUNCATED;
  if (h_dst && dst_cap < info->uncompressed_len) return GOMP_ERR_DST_TOO_SMALL;   // h_dst NULL: "In" mode
  size_t need = 0;
  gomp_decompress_workspace_size(info, 0, &need);
  if (ws_bytes < need) return GOMP_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint32_t nb = info->n_blocks;
  const uint64_t flen = info->file_len, bs = info->block_size, U = info->uncompressed_len;
  // chunking: payloads must be laid out in block order (our compressor does); otherwise one up-front copy
  const uint64_t tab_end = kHeaderBytes + uint64_t(kBlockEntryBytes) * nb;
  if (tab_end > flen) return GOMP_ERR_TRUNCATED;
  std::vector<uint64_t> pend(nb);   // end of block b's payload (+ look-ahead), clamped to the file
  bool ordered = true;
  uint64_t prev = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    const uint8_t* te = h_src + kHeaderBytes + uint64_t(kBlockEntryBytes) * b;
    const uint64_t off = ld64(te), len = ld32(te + 8);
    ordered = ordered && off >= prev && off <= flen;
    prev = off;
    pend[b] = std::min<uint64_t>(flen, off + len + 64);
  }
  // chunk boundaries: sizes double from ~nb/128 blocks, so the first output is ready for the device->host copy
  // after a short decode and the copy engine (the bottleneck of this path) starts early; one chunk if the
  // payloads are not in block order
  std::vector<uint32_t> cb{0};
  {
    uint32_t sz = std::max<uint32_t>(1, nb / 128);
    while (ordered && cb.back() < nb && cb.size() < kPipeMaxChunks) {
      cb.push_back(std::min<uint32_t>(nb, cb.back() + sz));
      sz *= 2;
    }
    if (cb.back() < nb || cb.size() == 1) cb.push_back(nb);
    if (!ordered) cb = {0, nb};
  }
  const uint32_t K = uint32_t(cb.size() - 1);
  Pipe* pp = thread_pipe();
  if (!pp) return GOMP_ERR_CUDA;
  Pipe& p = *pp;
  if (cudaMemsetAsync(d_ws, 0, kWsHeaderBytes, st) != cudaSuccess) return GOMP_ERR_CUDA;
  cudaEvent_t e0 = p.event();
  if (!p.ok || cudaEventRecord(e0, st) != cudaSuccess) return GOMP_ERR_CUDA;
  bool ok = cudaStreamWaitEvent(p.h2d, e0, 0) == cudaSuccess && cudaStreamWaitEvent(p.d2h, e0, 0) == cudaSuccess;
  for (auto c : p.comp) ok = ok && cudaStreamWaitEvent(c, e0, 0) == cudaSuccess;
  if (!ok) return GOMP_ERR_CUDA;
  uint64_t copied = 0;   // bytes [0, copied) of the file are enqueued host->device
  for (uint32_t i = 0; i < K; ++i) {
    const uint32_t b0 = cb[i], b1 = cb[i + 1];
    const uint64_t hi = (i + 1 == K || !ordered) ? flen : std::max<uint64_t>(pend[b1 - 1], info->payload_base);
    if (hi > copied) {
      if (cudaMemcpyAsync(d_src_buf + copied, h_src + copied, hi - copied, cudaMemcpyHostToDevice, p.h2d) != cudaSuccess)
        return GOMP_ERR_CUDA;
      copied = hi;
    }
    cudaEvent_t eh = p.event(), ec = p.event();
    if (!p.ok || cudaEventRecord(eh, p.h2d) != cudaSuccess) return GOMP_ERR_CUDA;
    cudaStream_t cs = p.comp[i % kPipeStreams];
    if (cudaStreamWaitEvent(cs, eh, 0) != cudaSuccess) return GOMP_ERR_CUDA;
    const uint64_t o0 = uint64_t(b0) * bs, o1 = std::min<uint64_t>(uint64_t(b1) * bs, U);
    const gomp_status s = decompress_range(info, b0, b1 - b0, d_src_buf, flen, d_dst_buf + o0, o1 - o0, d_ws, ws_bytes,
                                           strategy, cs, false, b0);
    if (s != GOMP_OK) return s;
    if (cudaEventRecord(ec, cs) != cudaSuccess || cudaStreamWaitEvent(p.d2h, ec, 0) != cudaSuccess) return GOMP_ERR_CUDA;
    if (h_dst && o1 > o0 && cudaMemcpyAsync(h_dst + o0, d_dst_buf + o0, o1 - o0, cudaMemcpyDeviceToHost, p.d2h) != cudaSuccess)
      return GOMP_ERR_CUDA;
  }
  cudaEvent_t ee = p.event();
  if (!p.ok || cudaEventRecord(ee, p.d2h) != cudaSuccess || cudaStreamWaitEvent(st, ee, 0) != cudaSuccess)
    return GOMP_ERR_CUDA;
  return GOMP_OK;
}

GOMP_EXPORT gomp_status gomp_decompress_error(const void* d_ws, void* stream, gomp_error* out) {
  if (!d_ws || !out) return GOMP_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(out, d_ws, sizeof(gomp_error), cudaMemcpyDeviceToHost, st) != cudaSuccess) return GOMP_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? GOMP_OK : GOMP_ERR_CUDA;
}

GOMP_EXPORT gomp_status gomp_decompress_stats(const void* d_ws, void* stream, gomp_stats* out) {
  if (!d_ws || !out) return GOMP_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(out, static_cast<const uint8_t*>(d_ws) + kWsStatsOff, sizeof(gomp_stats), cudaMemcpyDeviceToHost,
                      st) != cudaSuccess)
    return GOMP_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? GOMP_OK : GOMP_ERR_CUDA;
}
