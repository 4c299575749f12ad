// format.hpp — host-side view of the FORMAT.md v1 container for libgompresso (product code; independent of
// oracle/). Header parsing/validation shared by the C-ABI entry points and the compressor.
#pragma once
#include <cstdint>
#include <cstring>

#include "gomp.h"

namespace gomp {

constexpr uint32_t kHeaderBytes = 64;
constexpr uint32_t kBlockEntryBytes = 32;
constexpr uint32_t kSubEntryBytes = 8;
constexpr uint32_t kTrailerBytes = 16;
constexpr uint32_t kTreeBytes = 160;   // 143 + 15 nibble bytes + 2 zero bytes (FORMAT.md §3)
constexpr uint32_t kGroup = 32;        // sequences per warp group
constexpr uint32_t kMaxLitRun = 1023;  // reading R10
constexpr size_t kWsHeaderBytes = 1024;  // workspace: error word + stats, then the token buffer

inline uint64_t align16(uint64_t x) { return (x + 15) & ~uint64_t(15); }
inline uint32_t ld32(const uint8_t* p) { uint32_t v; std::memcpy(&v, p, 4); return v; }
inline uint64_t ld64(const uint8_t* p) { uint64_t v; std::memcpy(&v, p, 8); return v; }
inline void st32(uint8_t* p, uint32_t v) { std::memcpy(p, &v, 4); }
inline void st64(uint8_t* p, uint64_t v) { std::memcpy(p, &v, 8); }

// Block table entry (FORMAT.md §1), identical layout on host and device.
struct BlockEntry {
  uint64_t payload_off;
  uint32_t payload_len, n_seq, n_lit, sub_first, S, n_sub;
};
static_assert(sizeof(BlockEntry) == 32, "block entry layout");

inline gomp_status parse_header(const uint8_t* h, size_t len, gomp_info* o) {
  if (!h || !o) return GOMP_ERR_INVALID_ARG;
  if (len < kHeaderBytes) return GOMP_ERR_TRUNCATED;
  if (std::memcmp(h, "GMPR", 4) != 0) return GOMP_ERR_BAD_MAGIC;
  if (h[4] != 1) return GOMP_ERR_UNSUPPORTED_VERSION;
  gomp_info i{};
  i.version = h[4];
  i.mode = h[5];
  i.de = h[6] & 1u;
  i.min_match = h[7];
  i.max_match = h[8];
  i.cwl = h[9];
  i.block_size = ld32(h + 12);
  i.window_size = ld32(h + 16);
  i.n_blocks = ld32(h + 20);
  i.uncompressed_len = ld64(h + 24);
  i.file_len = ld64(h + 32);
  i.n_sub_total = ld32(h + 40);
  i.max_block_tokens = ld32(h + 44);
  i.payload_base = ld64(h + 48);
  i.de_group = h[10];
  bool ok = i.mode <= 1 && (h[6] & ~1u) == 0 && h[10] != 0 && h[10] % kGroup == 0 && h[11] == 0 && ld32(h + 56) == 0 &&
            ld32(h + 60) == 0;
  ok = ok && (i.min_match == 3 || i.min_match == 4) && i.max_match >= i.min_match &&
       i.max_match <= i.min_match + 62;
  ok = ok && i.block_size >= 16 && i.block_size % 16 == 0 && i.window_size >= 1 && i.window_size <= 32768;
  if (i.mode == GOMP_MODE_BIT) ok = ok && i.cwl >= 9 && i.cwl <= 15;
  else ok = ok && i.cwl == 0 && i.n_sub_total == 0 && i.max_block_tokens == 0;
  ok = ok && uint64_t(i.n_blocks) == (i.uncompressed_len + i.block_size - 1) / i.block_size;
  ok = ok && i.payload_base == align16(kHeaderBytes + uint64_t(kBlockEntryBytes) * i.n_blocks +
                                       uint64_t(kSubEntryBytes) * i.n_sub_total);
  ok = ok && i.file_len >= i.payload_base + kTrailerBytes;
  if (!ok) return GOMP_ERR_HEADER_INCONSISTENT;
  *o = i;
  return GOMP_OK;
}

}  // namespace gomp
