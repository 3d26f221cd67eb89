// Device-side work tables shared by the planner (host) and the kernels.
// Every multi-tensor kernel walks one of these tables, so one launch covers a
// whole bucket of tensors (SURVEY.md 7 "hard part 2": many tiny tensors).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace esp {

// Work granularity (elements).  A CTA of 256 threads streams one UNIT; each
// warp owns one RUN of 1024 consecutive elements (8 x float4 per lane).
constexpr int kThreads = 256;
constexpr int kRun = 512;                // DGC: candidates are compacted per warp-run
constexpr int kNJ = kRun / 128;          // float4 per lane per run
constexpr int kDgcTile = 8 * kRun;       // DGC streaming tile (one run per consumer warp)
constexpr int kSignSpan = 1024;          // sign h1: elements per warp per unit
constexpr int kUnit = 8192;              // 8 runs per CTA
constexpr int kSignUnit = 8192;  // sign h2: elements per CTA (one prologue per 128 KB of output)
constexpr int kRunsPerGroup = 128;       // DGC finalize: the longest group (65536 elements); SegH1::rpg per segment
constexpr int kSample = 4096;            // DGC sampled-threshold sample size
constexpr int kTile = 1024;      // sparse h2 output tile (one warp each)
constexpr int kTileThreads = 128;        // sparse h2 CTA size (4 warps = 4 tiles in flight)
constexpr int kOffJob = 4096;            // sparse h2 tile-offset pass: entries per CTA

enum Kind : int { K_NONE = 0, K_RANDOMK = 1, K_DGC = 2, K_TOPK = 3, K_EFSIGN = 4, K_ONEBIT = 5 };

// Per-segment selection state of the DGC/top-k pipeline (one per segment).
struct SelState {
  uint32_t thr;        // sampled threshold key (candidates: key >= thr)
  uint32_t count;      // candidates found by the streaming pass
  uint32_t done;       // last-CTA counter of the streaming pass
  uint32_t fallback;   // 1: count < k, re-run compaction with thr_lo (then 0)
  uint32_t count_fb, done_fb;
  uint32_t prefix;     // radix-select prefix of the k-th key
  uint32_t above;      // # candidates with key above the current prefix bin
  uint32_t need;       // k - above
  uint32_t done_r2, done_r3, done_cnt;
  uint32_t total_sel;  // debug: number selected (== k)
  uint32_t thr_lo;     // safe lower threshold of the fallback (sample bin far below thr)
  uint32_t pad[2];
};

// One h1 segment = (local rank, tensor, partition).
// Per-call dynamic arguments (gradient pointers and step counters of the
// tensors of a plan) live in a small device array `dyn` that is refreshed with
// one async H2D copy per call, so the static tables below never change.
struct SegH1 {
  const uint64_t* gptr;  // &dyn[slot]: device pointer of this tensor's gradient
  uint64_t goff;         // element offset of the segment (local rank and partition)
  const uint64_t* step;  // &dyn[nslots + slot]: step counter (Randomk draws)
  float* r;              // EF state: residual (sparse) / previous p (sign, lazy EF)
  unsigned char* chunk;  // output chunk
  const float* lazy_in;  // sign: {scale} / onebit: {mneg, mpos} of the previous step
  float* lazy_out;       // written by the last CTA of the segment
  uint32_t n;            // segment length (elements)
  uint32_t k;            // selected count (sparse) / unused
  uint32_t kpad;         // chunk capacity in entries (sparse) or words (sign)
  uint32_t unit0;        // first unit (CTA) of this segment in the unit table
  uint32_t nunits;
  uint32_t group0;       // DGC: first finalize group
  uint32_t ngroups;
  uint16_t ef;           // error feedback on/off
  uint16_t unsampled;    // TOPK: no sampled threshold, every element is a candidate
  uint64_t hash;         // Randomk: splitmix chain over (seed, tensor); DGC: sample hash
  uint32_t part;         // partition index (Randomk hash chain)
  uint32_t rankterm;     // 0 when indices are shared, rank + 1 otherwise (R5)
  double ratio;
  // DGC / sign workspace
  uint2* cand;           // candidates, run-major: [run * kRun + i] = {idx, bits(acc)}
  uint32_t* runcnt;      // candidates per run
  uint32_t* hist;        // dgc_hist_words(hrep): stream, fallback, round 2, round 3
  SelState* st;
  uint32_t* bflag;       // bucket-wide "some segment fell back" counter; bflag[1]: the
                         // finalize's grid-barrier counter (both zeroed every call)
  uint32_t* gcnt;        // look-back status, one uint64 per group (zeroed every call)
  double* partial;       // sign: 2 doubles per unit
  uint32_t* pcount;      // sign: 2 counts per unit (onebit) ; [0] of seg = done counter
  // a7 (mid-scheme) input: decode-mean of npieces chunks instead of g
  uint32_t npieces;
  uint32_t piece0;       // index into the piece-pointer array
  float divisor;
  uint32_t hrep;         // DGC: replicas of the round-2/3 histograms (spread same-bin atomics)
  // DGC momentum correction (R20): u buffer of the segment (nullptr = off), factor m
  float* mom;
  float mcoef;
  // DGC sampled threshold (R22): strata of 8 samples (512 = 4096 samples) and
  // the approximate-count mode (keep what passes the threshold, at most k)
  uint16_t strata;
  uint16_t approx;
  uint32_t rpg;          // DGC finalize: runs per group (8..128, power of two; planner's choice)
  // DGC deferred EF zeroing: per 4096-element tile a record of zcap uint16,
  // [0] = count, then the tile offsets of the previous call's selection, whose
  // r (and u) still hold their acc and are read as +0 by the next streaming
  // pass (nullptr: the write kernel zeroes r / u directly)
  uint32_t zcap;
  uint16_t* zrec;
};
constexpr int kZRecMax = 128;   // the largest record (256 B)

// DGC histogram words of a segment: 2048 (stream) + 2048 (fallback) + 1024 x hrep
// (round 2) + 1024 x hrep (round 3).  A round's matches number about k, all
// landing in 1024 bins (32 cache lines): a segment with k in the millions
// spreads them over hrep replicas, one per warp-group residue.
constexpr uint32_t kMaxHrep = 16;
__host__ __device__ inline uint32_t dgc_hrep(uint32_t k, uint32_t ngroups) {
  uint32_t r = k / 65536u;
  r = r < 1 ? 1 : (r > kMaxHrep ? kMaxHrep : r);
  return r < ngroups ? r : (ngroups ? ngroups : 1);
}
__host__ __device__ inline uint32_t dgc_hist_words(uint32_t hrep) { return 4096 + 2048 * hrep; }

// One job of the push kernel (fused collectives): bytes (a multiple of 16,
// <= kPushChunk) from src + src_off to dsts[d] + dst_off; one arrival on cnts[d].
constexpr int kPushChunk = 32768;
struct PushJob {
  uint64_t src_off;
  uint64_t dst_off;
  uint32_t bytes;
  uint32_t d;
};

// One h2 segment: out[0..n) = reduce(sum_r decode(piece r)).
struct SegH2 {
  const uint64_t* optr;  // &dyn[slot]: output tensor (the gradient, in place)
  uint64_t ooff;         // element offset of the segment
  const uint64_t* step;  // Randomk: step counter
  uint64_t hash;         // Randomk: splitmix chain over (seed, tensor)
  uint32_t part;         // Randomk: partition index
  uint32_t n;
  uint32_t k;            // randomk: k of the segment
  uint32_t kpad;         // entries (sparse) / words (sign) per chunk
  uint32_t npieces;
  uint32_t piece0;       // index into piece pointers (and randomk hash array)
  uint32_t unit0;        // first unit/tile
  uint32_t nunits;
  float divisor;         // n for MEAN, 1 for SUM or already-averaged data
  uint32_t* toff;        // sparse: per piece, nunits + 1 tile start offsets (h2_sparse_offsets)
};

__device__ __forceinline__ const float* seg_g(const SegH1& s) {
  return reinterpret_cast<const float*>(*s.gptr) + s.goff;
}
__device__ __forceinline__ float* seg_out(const SegH2& s) {
  return reinterpret_cast<float*>(*s.optr) + s.ooff;
}

}  // namespace esp
