// compress.hpp — internal interface between the host compressor (compress.cpp) and the GPU compressor
// (compress_gpu.cu): shared parameter checks and header layout, so that both write the same file for the same
// input and parameters (product code; independent of oracle/). The GPU compressor runs package-merge (R14) on the
// device with the host routine's algorithm and tie order (compress_gpu.cu pm_kernel).
#pragma once
#include <cstdint>

#include "gomp.h"

namespace gomp {
bool host_params_ok(const gomp_params* p);
uint64_t host_max_seqs(uint32_t block_size, uint32_t min_match);
void host_write_header(uint8_t* h, const gomp_params* p, uint32_t nb, uint64_t src_len, uint64_t file_len,
                       uint64_t n_sub_total, uint64_t max_tok, uint64_t base);
}  // namespace gomp
