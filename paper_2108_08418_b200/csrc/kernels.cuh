// Kernel launchers (internal).
#pragma once
#include "common.cuh"

namespace cvsr {

// bp_kernels.cu
void launch_cn(const CodeDev &cd, const DecState &ds, int grid_tiles, float qmax, int check_only, cudaStream_t s);
int launch_vn(const CodeDev &cd, const DecState &ds, int grid_tiles, float qmax, bool first, float *post_dbg,
              cudaStream_t s);
FusedPlan make_plan(const CodeDev &cd, int subs);
void launch_iter(const CodeDev &cd, const DecState &dsc, const DecState &dsv, const FusedPlan &plan, int k,
                 float qmax, cudaStream_t s);
void launch_list(const DecState &ds, int32_t *host_counts, cudaStream_t s);
void launch_status(const DecState &ds, int k, int max_iter, int final_pass, int32_t *host_counts, cudaStream_t s);
void launch_retire(const DecState &ds, int32_t n, int grid_tiles, uint32_t *bits_out, cudaStream_t s);
void launch_to_interleaved(const float *src, float *dst, int32_t F, int64_t rows, int tiles, int subs, float scale,
                           cudaStream_t s);
void launch_from_interleaved(const float *src, float *dst, int32_t F, int64_t rows, int tiles, int subs, float scale,
                             cudaStream_t s);
void launch_synd_transpose(const uint32_t *synd, int32_t F, int32_t M, int subs, uint4 *st, int tiles,
                           const int32_t *pos /*nullable: row of check c = pos[c]*/, cudaStream_t s);
void launch_init_tiles(const DecState &ds, const uint8_t *alive, cudaStream_t s);
void launch_set_counts(const DecState &ds, int32_t n_active, cudaStream_t s);
bool layered_supported(const CodeDev &cd);
void launch_layer_init(const CodeDev &cd, const DecState &ds, int grid_tiles, cudaStream_t s);
int launch_layers(const CodeDev &cd, const DecState &ds, int grid_tiles, float qmax, bool first, cudaStream_t s);
bool layers_zero_first();
int layer_subs(int32_t max_dc);
void launch_synd_test(const CodeDev &cd, const DecState &ds, int grid_tiles, cudaStream_t s);
size_t decode_smem_bytes(const CodeDev &cd);
bool launch_decode_smem(const CodeDev &cd, const DecState &ds, int max_iter, float qmax, uint32_t *bits_out,
                        cudaStream_t s);
int launch_compact(const CodeDev &cd, const DecState &src, const DecState &dst, int32_t *dst_src, int max_tiles,
                   int32_t *host_counts, bool move_hb, cudaStream_t s);

// bob_kernels.cu
void launch_quantise(const float *edges_host, int m, const float *y, int64_t count, uint8_t *label, cudaStream_t s);
void launch_slice_bits(const uint8_t *label, int32_t F, int32_t n, int32_t j, uint32_t *bits, cudaStream_t s);
void launch_syndrome(const CodeDev &cd, const uint8_t *label, int32_t F, int32_t j, uint32_t *synd, cudaStream_t s);
// sliced: scratch of n x syndrome_sliced_groups(F) words (16-byte aligned) for the bit-sliced
// kernels, or null for the per-frame kernels; returns the number of launches
int launch_syndrome_bits(const CodeDev &cd, const uint32_t *bits, int32_t F, uint32_t *synd, uint32_t *sliced,
                         cudaStream_t s);
int32_t syndrome_sliced_groups(int32_t F);
void launch_frame_hash(const uint8_t *label, int32_t F, int32_t n, unsigned long long key, unsigned long long *out,
                       cudaStream_t s);
void launch_verify(const uint8_t *label_a, const uint8_t *label_b, const uint8_t *ok_in, int32_t F, int32_t n,
                   const unsigned long long *keys /*host [CVSR_HASH_KEYS]*/, uint8_t *ok_out, unsigned long long *ha,
                   unsigned long long *hb, cudaStream_t s);
void launch_count_errors(const uint8_t *a, const uint8_t *b, const uint8_t *ok, int32_t F, int32_t n,
                         unsigned long long *counts, cudaStream_t s);

// llr_kernels.cu
// scalar table and its 16-byte interpolation windows (2 launches); false: grid too coarse, none
bool launch_llr_table(const LlrParams &p, float *table, float4 *table4, cudaStream_t s);
void launch_llr_slice(const LlrParams &p, const float *x, const uint8_t *known_label, int32_t F, int32_t n,
                      float *out, cudaStream_t s);
void launch_llr_biawgn(const float *y, int64_t count, float sigma2, float llr_max, float *out, cudaStream_t s);
void launch_llr_interleaved(const LlrParams &p, const float *x, int32_t F, int32_t n, int tiles, int subs, float *L,
                            uint4 *hb /*nullable: also write [L < 0] of active frames*/, const uint4 *tile_active,
                            cudaStream_t s);

// reconcile bookkeeping (bob_kernels.cu)
void launch_slice_done(const DecState &ds, int32_t m, int32_t j, int disclosed, uint8_t *alive, uint8_t *attempt,
                       int32_t *iters_out, cudaStream_t s);
void launch_assemble(const uint32_t *const *bits, int32_t m, const uint8_t *attempt, int32_t F, int32_t n,
                     uint8_t *label_out, cudaStream_t s);
void launch_fill_i32(int32_t *p, int64_t count, int32_t v, cudaStream_t s);
void launch_fill_u8(uint8_t *p, int64_t count, uint8_t v, cudaStream_t s);
void launch_frame_stats(const uint8_t *alive, const uint8_t *attempt, const int32_t *iters, int32_t F, int32_t m,
                        unsigned long long *acc /*[1 + 8*3]*/, cudaStream_t s);

}  // namespace cvsr
