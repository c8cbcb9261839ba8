// cc_internal.h -- types shared by the host orchestrator (cc_host.cpp) and the sm_100a
// kernels (cc_kernels.cu).  Not part of the public ABI (include/chordless.h is).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cc {

typedef unsigned long long u64;

// Size class of the bitmap-record path: S (Fig. 2) as NW 64-bit words.
constexpr int kMaxWords = 8;           // n <= 512
constexpr int kIdBits = 10;            // packed ids v1 | v2 << 10 | vt << 20 (n <= 1024)
constexpr uint32_t kIdMask = (1u << kIdBits) - 1;
#ifndef CC_BLOCK
#define CC_BLOCK 256
#endif
constexpr int kBlock = CC_BLOCK;       // threads per CTA for every kernel
// R: paths per thread per tile in k_expand_thread
#ifndef CC_EB_R
#define CC_EB_R 2
#endif
__host__ __device__ constexpr int expand_paths_per_thread(int nw) { return nw <= 4 ? CC_EB_R : 1; }
constexpr int kMinLogPage = 10;        // pages hold >= kBlock * R records (one CTA tile)
constexpr int kByteTableWords = 2;     // byte-wise key tables (H-spec keysum) for NW <= 2

// Graph in device memory.  Internal vertex id == degree label (the host relabels), so the
// label gate l(v) > l(v2) of Alg. 3 line 11 is the integer test v > v2 and
// every adjacency row is sorted by label.
struct DevGraph {
    int32_t n;
    int32_t nw;                  // words per bitmap row
    const uint32_t *rowptr;      // [n+1]  V_e
    const uint32_t *col;         // [2m]   E_e, rows ascending
    const uint32_t *fwd;         // [n]    index in row u of the first neighbour w > u
    const u64 *pair_prefix;      // [n+1]  prefix sums of C(d+(u), 2), d+(u) = |{w ~ u: w > u}|
    const u64 *adj;              // [n*nw] adjacency bit rows
    const u64 *key;              // [n]    key(v) = mix(seed ^ original id)   (H-spec)
    const u64 *keybyte;          // [8*nw][256] (nw <= 2): sum of key(8j+i) over the set bits i of
                                 //        byte value b at byte position j of S
    const int32_t *orig;         // [n]    internal id -> original id
    const uint32_t *nbrmask;     // wide class with Delta <= 32, else null: [n][n], bit k of
                                 //        nbrmask[u*n + z] = (k-th neighbour of u in its CSR row) ~ z
};

// Two record formats ("modes") for a path p = <v1..vt>:
//   S-mode (collect mode):  RW = NW words  = the path bitmap S (Fig. 2)
//   B-mode (count mode, the hot path): RW = NW + 1 words
//        words 0..NW-1 = the blocked-vertex set B(p) = union of the closed neighbourhoods
//                        N[v_i] of the interior vertices v_2..v_{t-1}
//        word  NW      = keysum(p) = sum of key(v) over the vertices of p (H-spec)
// plus, in both modes, ids = v1 | v2 << 10 | vt << 20 (the vectors V1, V2, VL).
//
// The frontier arena is split into pages of P = 2^log_p records.  Inside a page, records are
// stored structure-of-arrays:
//   word w of slot j : ((u64*)(base + page * page_bytes))[w * P + j]
//   ids of slot j    : ((uint32_t*)(base + page * page_bytes + RW*P*8))[j]
// A launch reads the virtual records [0, n_in) of the page list in_pages (record r lives in
// page in_pages[r >> log_p], slot r & (P-1); every page but the last is full) and appends to
// the virtual positions [out_off, out_off + out_cap) of out_pages.
struct Pages {
    char *base;
    u64 page_bytes;
    uint32_t log_p;
    const uint32_t *in_pages;
    const uint32_t *out_pages;
};

// Collect mode: closed cycles (bitmap S + {v}, v1 | v2 << 10).
struct CycleStore {
    u64 *s;
    uint32_t *ids;
    uint64_t cap;
    u64 *count;                  // device counter (keeps counting past cap)
    uint32_t lw;                 // 0: bitmap S + ids (n <= 512); > 0: the list class's format --
                                 // the canonical sequence as 16-bit ids, four per word, lw words
                                 // (s[w * cap + i]), unused slots 0xffff
};

// Per-launch scratch accumulators (zeroed before, read back after every launch, so a launch
// that overflows its output can be discarded without touching the totals).
// Last-level fusion (count mode, with a length cap K): when the children of F_t cannot have
// children of their own (t + 2 >= K), the expansion of F_t does not write them; it counts them
// (|F_{t+1}|, their candidate slots) and their closures (cycles of t+2 vertices) at once in the
// *_next counters.  The deepest frontier level is then never materialised.
struct Scratch {
    u64 out_count;               // records demanded by this launch (keeps counting past out_cap)
    u64 err;                     // bit 0: output overflow
    u64 cycles;                  // closures of the input paths (all of one length t+1)
    u64 hash;                    // sum of h(C) over every closure counted by the launch (mod 2^64)
    u64 cand;                    // candidate slots of the input paths
    u64 cycles_next;             // last-level fusion: closures of the children (t+2 vertices)
    u64 cand_next;               // last-level fusion: candidate slots of the children
    u64 paths_next;              // last-level fusion: children counted (|F_{t+1}| share)
    u64 paths_cur;               // real input paths expanded (k_expand_blocked / k_expand_fused: the
                                 // input may hold empty slots, DESIGN.md §5 "output chunks")
    u64 out_real;                // real records written (out_count also counts empty slots)
    u64 in_next;                 // k_expand_fq: next input tile handed out (dynamic chunks)
    u64 cyc_count;               // collect-mode store counter (NOT reset per launch)
};

struct LaunchArgs {
    DevGraph g;
    Pages pg;
    CycleStore cyc;
    Scratch *sc;
    uint64_t in_lo;              // Stage 1 only: pair range [in_lo, in_lo + n_in)
    uint64_t n_in;               // input records (or pairs)
    const u64 *n_in_dev;         // k_expand_blocked only: if set, the input size is read here (a
                                 // launch chained after Stage 1 without a host round trip)
    uint64_t out_off;            // first virtual output position in out_pages
    uint64_t out_cap;            // positions available from out_off
    int32_t emit;                // 1 = create extended paths / triplets
    int32_t emit_next;           // 0 with emit = 1: last-level fusion (count the children, write none)
    int32_t count;               // 1 = this shard owns (counts) the closures of this launch
    int32_t collect;             // 1 = store closed cycles
    int32_t filter;              // 1 = keep only records of this shard (Stage 1 / filter kernel)
    uint64_t root_stride;        // Stage-1 root sample (0/1 = all)
    uint64_t root_offset;
    uint32_t shard_index;
    uint32_t shard_count;
    uint32_t idb;                // packed records: bits per id (ids in the top 3*idb bits of word NW-1)
    uint32_t packed;             // 1 = B-mode record with packed ids (no ids array)
    uint32_t tlen;               // list records: vertices per input path (Stage 2)
};

// Thread: thread per path; Warp: warp per path (S-mode, Delta > 32); Small: B-mode with
// Delta <= 4 (at most 3 children per path)
enum class ExpandVariant { Thread, Warp, Small };

enum class Mode { S, B };
inline int record_words(int nw, Mode m) { return m == Mode::B ? nw + 1 : nw; }
// B-mode records may carry v1, v2, vt in the unused top bits of the last blocked-set word
// (bits >= n are never set in B): possible iff 64*nw - n >= 3*idb, idb = ceil(log2 n).
inline int id_bits(int n)
{
    int b = 1;
    while ((1 << b) < n)
        ++b;
    return b;
}
// id width of packed records: fixed per word count for NW <= 2 (the grid-class kernels see it as a
// constant): 6 bits for NW = 1; 8 bits for NW = 2, so that vt is byte 3 of the last word's upper
// half (k_expand_fq writes a child's ids with one byte permute); ceil(log2 n) otherwise
inline int packed_id_bits(int nw, int n) { return nw == 1 ? 6 : nw == 2 ? 8 : id_bits(n); }
inline bool packable(int nw, int n) { return 64 * nw - n >= 3 * packed_id_bits(nw, n); }
inline int record_bytes(int nw, Mode m, bool packed) { return record_words(nw, m) * 8 + (packed ? 0 : 4); }

// a.packed selects the packed-ids record variants of the B-mode kernels
cudaError_t launch_stage1(const LaunchArgs &a, Mode m, cudaStream_t st, int grid_cap);
cudaError_t launch_expand(const LaunchArgs &a, Mode m, ExpandVariant v, cudaStream_t st, int grid_cap);
cudaError_t launch_shard_filter(const LaunchArgs &a, Mode m, cudaStream_t st, int grid_cap);
cudaError_t launch_keys(u64 *key, u64 *keybyte, const int32_t *orig, int n, int nw, u64 seed,
                        cudaStream_t st);
// Small-frontier fast path (count mode, bitset records, n <= 128, one shard): all Stage-2
// levels whose frontier stays small run in ONE cooperative launch with a grid-wide barrier
// between levels, ping-ponging between two arena pages; it stops (hands the current level to
// the paged scheduler) when a level could outgrow a page or reaches the last (leaf) level.
struct SmallArgs {
    uint32_t first;              // the arena page holding level d0 (the triplets)
    uint32_t region[2];          // first pages of two runs of `region_pages` contiguous pages:
                                 // level d > d0 lives in region[(d - d0 - 1) & 1]
    uint64_t region_cap;         // records per region (region_pages * P)
    int32_t d0;                  // first level (3: the triplets)
    int32_t d_stop;              // levels d0 .. d_stop-1 may run here (leaf levels excluded)
    uint32_t max_len;            // cc_options.max_len
    u64 threshold;               // a level with more input paths is handed off (its children
                                 // might not fit a region)
    u64 *count;                  // [n+3] count[d] = |F_d| written (count[d0] set by the host)
    u64 *cyc;                    // [n+3] closures of length d+1 found at level d
    u64 *cand;                   // [n+3] candidate slots of level d
    u64 *hash;                   // sum of h(C)
    int32_t *last;               // the level the kernel stopped at
    u64 *err;                    // overflow (must stay 0: the threshold guarantees room)
};
cudaError_t launch_small(const LaunchArgs &a, const SmallArgs &s, cudaStream_t st, int sms);
// nbrmask (DevGraph) of a wide graph with Delta <= 32; T must be zeroed, n*n words
cudaError_t launch_nbrmask(const DevGraph &g, uint32_t *T, cudaStream_t st);
// off[0..count] = exclusive prefix sums of the lengths of stored cycles first..first+count-1
// (off[count] = total); blk = scratch of ceil(count / 1024) + 1 words
cudaError_t launch_cycle_offsets(const CycleStore &c, int nw, uint64_t first, uint64_t count, u64 *off, u64 *blk,
                                 cudaStream_t st);
cudaError_t launch_cycle_sequences(const CycleStore &c, int nw, const u64 *adj, const int32_t *orig,
                                   uint64_t first, uint64_t count, const u64 *offsets,
                                   int32_t *out, cudaStream_t st);
// Two-level (fuse = 2) or single-level (fuse = 1, optionally last-level fusion) expansion for the
// grid class: count mode, B-mode records, nw <= 2, max degree <= 4 (cc_fused.cu).  Output slots
// come in per-warp chunks of 2^log_ch; unused slots are all-zero records (v1 == v2).
cudaError_t launch_fused(const LaunchArgs &a, int fuse, bool leaf, uint32_t log_ch, int max_warps, cudaStream_t st);
int fused_warps_per_launch(int nw, int n, bool packed, int fuse, bool leaf, int sms);
size_t fused_smem(int nw, int n, bool packed, int fuse);
#ifndef CC_FQ_DIRECT
#define CC_FQ_DIRECT 1  // k_expand_fq: children of child rounds (F_{t+2}) stored straight to HBM
#endif
// smallest output chunk of k_expand_fq (log2 slots): a child round reserves up to 96 slots at once
// with direct stores (so a reservation needs at most one new chunk); output-queue flushes take 32
constexpr uint32_t kFqMinLogChunk = CC_FQ_DIRECT ? 7 : 5;
// Debug builds (-DCC_CHECKS, `python -m paper_1410_4876_b200.build --out ... -DCC_CHECKS`):
// device-side bounds checks in k_expand_fq set bits of a device flag; this reads and clears it
// (always 0 in normal builds).  The substitute for compute-sanitizer where the pool disables it.
unsigned int fused_check_flags(cudaStream_t st);
// dynamic shared memory of the expansion kernel for (mode, nw, n, packed)
size_t expand_smem(Mode m, int nw, int n, bool packed);
// Wide class (512 < n <= 2015, count mode, AoS records): which 0 = Stage 1, 1 = expand,
// 2 = shard filter.
cudaError_t launch_wide(int which, const LaunchArgs &a, cudaStream_t st, int grid_cap);
int max_blocks_per_sm_wide(int which);
constexpr int kWideMaxWords = 32;
// List class (count mode, wide graphs with Delta <= 32): a path is its vertex list, 16-bit ids,
// four per word (RWL id words), plus keysum(p); SoA pages like every other record.
// which: 0 = Stage 1, 1 = expand (leaf = last-level fusion), 2 = shard filter.
cudaError_t launch_list(int which, const LaunchArgs &a, int rwl, bool leaf, cudaStream_t st, int grid_cap);
int max_blocks_per_sm_list(int which, int rwl);
constexpr int kListMaxLen = 14;  // max_len <= 14: written paths have <= 12 vertices (3 id words)
// Resident CTAs per SM at kBlock threads with the given dynamic smem.
// which: 0 = Stage 1, 1 = expand (thread), 2 = expand (warp), 3 = shard filter, 4 = expand (small)
int max_blocks_per_sm(int which, Mode m, int nw, bool packed, size_t smem);

}  // namespace cc
