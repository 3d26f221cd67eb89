// Host-callable launchers of the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "esp_tables.h"

namespace esp {

void count_launches(int n);   // process-wide counter behind esp_launch_count()
// ESP_CARVEOUT=1: every kernel prefers the maximum shared-memory carveout (an
// A/B knob; measured 5% slower on BERT-large, so off by default)
bool set_max_smem_carveout(const void* fn);
#define ESP_CARVE(...)                                                                                \
  do {                                                                                              \
    static const bool esp_carve_ = ::esp::set_max_smem_carveout(reinterpret_cast<const void*>(__VA_ARGS__)); \
    (void)esp_carve_;                                                                               \
  } while (0)

// DGC / TOPK h1 (k_dgc.cu)
// probe0/probe1 (optional): events recorded around the streaming pass.
// dsts != nullptr (fused Allgather over NVLink): the payload entries are stored
// at dsts[q] + chunk_off for q < ndst (every rank's receive slot of this rank)
// and each write CTA then increments every cnts[q] (system-scope release).
void launch_dgc_h1(const SegH1* segs, int nsegs, const uint32_t* unit_seg, int nunits,
                   const uint32_t* group_seg, int ngroups, cudaStream_t st,
                   cudaEvent_t probe0 = nullptr, cudaEvent_t probe1 = nullptr,
                   unsigned char* const* dsts = nullptr, unsigned long long* const* cnts = nullptr,
                   int ndst = 0, bool mom = false);
// block the stream until *cnt >= target (arrivals of a fused Allgather); traps
// after ~10 s so that a missing peer becomes an error, not a hang
void launch_wait_arrivals(const unsigned long long* cnt, unsigned long long target, cudaStream_t st);
// fused collectives: copy each job's bytes into peer memory, then one
// system-scope release + arrival per job on the destination's counter (k_push.cu)
void launch_push(const PushJob* jobs, int njobs, const unsigned char* src, unsigned char* const* dsts,
                 unsigned long long* const* cnts, cudaStream_t st);
// Randomk h1 (k_randomk.cu)
void launch_randomk_h1(const SegH1* segs, const uint32_t* unit_seg, int nunits, cudaStream_t st);
// h1 on the persistent TMA streaming driver, tiles of kDgcTile (k_sign.cu)
// pieces != nullptr: a7 (input = decode-mean of the segment's pieces, r = r2)
// (+ one finalize kernel over the nsegs segments: the scales from the per-run partials)
// dsts != nullptr (fused collective): the chunk of a segment is stored at
// dsts[S.part] + chunk_off (dmode 1, the partition owner / root) or at every
// dsts[d] + chunk_off, d < ndst (dmode 2); the finalize kernel then bumps the
// matching cnts[] once per segment (system-scope release)
void launch_sign_h1_tma(int kind, const SegH1* segs, int nsegs, const uint32_t* unit_seg, int nunits,
                        const unsigned char* const* pieces, cudaStream_t st, unsigned char* const* dsts = nullptr,
                        unsigned long long* const* cnts = nullptr, int dmode = 0, int ndst = 0,
                        uint32_t max_len = 0,    // the longest segment (sizes the finalize grid)
                        cudaEvent_t probe0 = nullptr, cudaEvent_t probe1 = nullptr);
// NONE: pack gradients into a contiguous buffer (k_h2.cu)
void launch_pack(const SegH1* segs, const uint32_t* unit_seg, int nunits, cudaStream_t st);

// h2 (k_h2.cu)
// jobs: {segment, piece within segment, first entry, 0}, kOffJob entries each
// max_pieces: the largest npieces of the launch's segments (> 1 enables the
// shared-memory accumulation path and its dynamic shared memory)
void launch_h2_sparse(const SegH2* segs, const uint32_t* tile_seg, int ntiles, const uint4* jobs, int njobs,
                      const unsigned char* const* pieces, int max_pieces, cudaStream_t st);
void launch_h2_sign(int kind, const SegH2* segs, const uint32_t* unit_seg, int nunits,
                    const unsigned char* const* pieces, cudaStream_t st);
void launch_h2_randomk(const SegH2* segs, const uint32_t* unit_seg, int nunits,
                       const unsigned char* const* pieces, const uint32_t* rankterms, cudaStream_t st);
void launch_h2_dense(const SegH2* segs, const uint32_t* unit_seg, int nunits,
                     const unsigned char* const* pieces, cudaStream_t st);

// state export of the lazy sign EF: r_true = p - delta(p)  (k_sign.cu)
void launch_sign_materialize(int kind, const float* p, const float* lazy, float* out, uint32_t n,
                             cudaStream_t st);

}  // namespace esp
