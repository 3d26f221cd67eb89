// Host-callable launchers of the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "esp_tables.h"

namespace esp {

void count_launches(int n);   // process-wide counter behind esp_launch_count()

// DGC / TOPK h1 (k_dgc.cu)
// probe0/probe1 (optional): events recorded around the streaming pass.
void launch_dgc_h1(const SegH1* segs, int nsegs, const uint32_t* unit_seg, int nunits,
                   const uint32_t* group_seg, int ngroups, cudaStream_t st,
                   cudaEvent_t probe0 = nullptr, cudaEvent_t probe1 = nullptr, bool mom = false);
// the two halves of launch_dgc_h1: sampled threshold + streaming pass, then the
// finalize chain (fallback, exact radix select, ordered write + EF zeroing),
// which may run on another stream after the first half (bucket pipelining)
void launch_dgc_stream(const SegH1* segs, int nsegs, const uint32_t* unit_seg, int nunits, cudaStream_t st,
                       cudaEvent_t probe0 = nullptr, cudaEvent_t probe1 = nullptr, bool mom = false);
void launch_dgc_finalize(const SegH1* segs, int nsegs, const uint32_t* group_seg, int ngroups, cudaStream_t st);
// DGC / TOPK h1 of a bucket whose segments all have <= 4096 elements: one
// kernel, one CTA per segment (k_dgc.cu)
void launch_dgc_small(const SegH1* segs, int nsegs, cudaStream_t st);
// DGC / TOPK h1 of a bucket that fits on chip (k_dgc.cu dgc_mid_kernel): one
// kernel, ceil(tiles / tpc) co-resident CTAs per segment, grid <= #SMs,
// tpc <= dgc_mid_tpc_max() tiles of 4096 elements per CTA
uint32_t dgc_mid_tpc_max();
void launch_dgc_mid(const SegH1* segs, int nsegs, uint32_t tpc, int grid, cudaStream_t st);
// DGC deferred EF zeroing: apply a segment's pending records to r / u (either
// may be null) and clear them
void launch_dgc_zrec_apply(float* r, float* u, uint16_t* zrec, uint32_t zcap, uint32_t n, cudaStream_t st);
// block the stream until *cnt >= target (arrivals of a fused collective); after
// timeout_ns of wall time without them, set *err (mapped host memory) and return
void launch_wait_arrivals(const unsigned long long* cnt, unsigned long long target, unsigned int* err,
                          unsigned long long timeout_ns, cudaStream_t st);
// fused collectives: copy each job's bytes into peer memory, then one
// system-scope release + arrival per job on the destination's counter (k_push.cu)
void launch_push(const PushJob* jobs, int njobs, const unsigned char* src, unsigned char* const* dsts,
                 unsigned long long* const* cnts, cudaStream_t st);
// multicast fused collective: each job's bytes stored once to the multicast
// alias mc_dst + dst_off (every rank's copy), one multicast arrival per job
void launch_push_mc(const PushJob* jobs, int njobs, const unsigned char* src, unsigned char* mc_dst,
                    unsigned long long* mc_cnt, cudaStream_t st);
// Randomk h1 (k_randomk.cu)
void launch_randomk_h1(const SegH1* segs, const uint32_t* unit_seg, int nunits, cudaStream_t st);
// h1 on the persistent TMA streaming driver, tiles of kDgcTile (k_sign.cu)
// pieces != nullptr: a7 (input = decode-mean of the segment's pieces, r = r2)
// (+ one finalize kernel over the nsegs segments: the scales from the per-run partials)
void launch_sign_h1_tma(int kind, const SegH1* segs, int nsegs, const uint32_t* unit_seg, int nunits,
                        const unsigned char* const* pieces, cudaStream_t st,
                        uint32_t max_len = 0,    // the longest segment (sizes the finalize grid)
                        cudaEvent_t probe0 = nullptr, cudaEvent_t probe1 = nullptr,
                        int max_pieces = 0);   // a7: pieces per segment (selects the decode variant)
// out[i] = fl(out[i] + x[i]) (esp_decompress with accumulate)
void launch_add(float* out, const float* x, uint32_t n, cudaStream_t st);
// NONE: pack gradients into a contiguous buffer (k_h2.cu)
void launch_pack(const SegH1* segs, const uint32_t* unit_seg, int nunits, cudaStream_t st);

// h2 (k_h2.cu)
// jobs: {segment, piece within segment, first entry, 0}, kOffJob entries each
// max_pieces: the largest npieces of the launch's segments (> 1 enables the
// shared-memory accumulation path and its dynamic shared memory)
// dense: several pieces expected to put > 32 entries into a 1024-element tile
// (the shared-memory CTA-tile kernel, no tile-offset pass); else the offset
// pass + one warp per 1024-element tile
void launch_h2_sparse(const SegH2* segs, const uint32_t* tile_seg, int ntiles, const uint4* jobs, int njobs,
                      const unsigned char* const* pieces, int max_pieces, bool dense, cudaStream_t st);
// the bucket-level choice of launch_h2_sparse: sum(kpad x npieces) x 1024 > 32 x sum(n)
inline bool h2_sparse_dense(double entries, double elems) { return entries * 1024.0 > 32.0 * elems; }
// max_pieces: the largest npieces of the launch's segments (sizes the shared-memory word stage)
void launch_h2_sign(int kind, const SegH2* segs, const uint32_t* unit_seg, int nunits,
                    const unsigned char* const* pieces, int max_pieces, cudaStream_t st);
void launch_h2_randomk(const SegH2* segs, const uint32_t* unit_seg, int nunits,
                       const unsigned char* const* pieces, const uint32_t* rankterms, cudaStream_t st);
void launch_h2_dense(const SegH2* segs, const uint32_t* unit_seg, int nunits,
                     const unsigned char* const* pieces, cudaStream_t st);

// state export of the lazy sign EF: r_true = p - delta(p)  (k_sign.cu)
void launch_sign_materialize(int kind, const float* p, const float* lazy, float* out, uint32_t n,
                             cudaStream_t st);

}  // namespace esp
