/*
 * chordless.h -- C ABI of the B200-native chordless-cycle enumerator (arXiv 1410.4876).
 *
 * Problem (§1): given a finite undirected simple graph
 * G = (V, E), output every chordless cycle -- an induced subgraph that is a cycle --
 * exactly once.
 *
 * Method (the hot path behind cc_enumerate): degree labelling on the host (PAPER.md:53,
 * kept sequential as in PAPER.md:139), Stage 1 seeds T(G) and triangles on the GPU
 * (Alg. 2), Stage 2 level-synchronous expansion of chordless paths into
 * chordless cycles on the GPU (Alg. 3 + Alg. 4) with a depth-first
 * chunk scheduler when the next frontier would not fit in device memory (the "data
 * transportation" future work).  All kernels are hand-written sm_100a CUDA.
 *
 * Conventions (all functions):
 *   - Every function returns a cc_status; on a non-OK status cc_last_error() returns a
 *     thread-local, human-readable message that stays valid until the next call on that
 *     thread.  Output arguments are left untouched on error unless stated otherwise.
 *   - Host pointers are only read during the call and are never retained; the caller
 *     keeps ownership.  Device pointers (cc_options.workspace) stay owned by the caller.
 *   - Objects (cc_graph, cc_result) are opaque and freed only with their *_free function.
 *     A cc_graph may be read by several threads, but cc_enumerate calls that use the same
 *     cc_graph on the same device are serialised internally.  A cc_result is immutable.
 *   - Vertex ids are the caller's ("original") ids 0..n-1 everywhere in the interface.
 *   - Integer only: no floating point is involved in any result.
 */
#ifndef CHORDLESS_H
#define CHORDLESS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CC_OK = 0,
    CC_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, bad size, malformed row_ptr, bad option */
    CC_ERR_INVALID_VERTEX = 2,   /* a column index outside 0..n-1 */
    CC_ERR_SELF_LOOP = 3,        /* (v, v) in the input: not a simple graph */
    CC_ERR_NOT_SYMMETRIC = 4,    /* w in row v but v not in row w */
    CC_ERR_CAPACITY = 5,         /* workspace too small to make progress, or collect buffer full */
    CC_ERR_CUDA = 6,             /* a CUDA runtime error; message has the CUDA error string */
    CC_ERR_NOT_COLLECTED = 7,    /* cc_fetch_cycles on a count-only result */
    CC_ERR_BUFFER_TOO_SMALL = 8, /* caller's output buffer too small; required size returned */
    CC_ERR_TOO_LARGE = 9,        /* graph outside the supported size classes (see cc_enumerate) */
    CC_ERR_NO_DEVICE = 10        /* no CUDA device / device ordinal invalid */
} cc_status;

typedef struct cc_graph cc_graph;
typedef struct cc_result cc_result;

/* Options for cc_enumerate.  Initialise with cc_options_init() and then set fields. */
typedef struct {
    uint32_t struct_size;     /* = sizeof(cc_options); ABI versioning */
    int32_t device;           /* CUDA ordinal; -1 = the calling thread's current device */
    void *stream;             /* cudaStream_t to run on (e.g. torch's current stream);
                                 NULL = the legacy default stream.  cc_fetch_cycles and
                                 cc_result_free of the result also run on it: it must stay valid
                                 until the result is freed */
    uint32_t max_len;         /* 0 = no cap; else only cycles with <= max_len vertices are
                                 enumerated and counted (reading G14) */
    uint32_t collect;         /* 0 = counts + set hash only (the paper's count-only mode,
                                 PAPER.md:419); 1 = also keep every cycle for cc_fetch_cycles */
    uint32_t shard_index;     /* this rank's share of the search tree, 0 <= index < count */
    uint32_t shard_count;     /* 1 = everything.  Shards partition the paths of the first
                                 frontier level with >= min_shard_paths * count paths (default
                                 2^20 per shard) by a content hash of the record; earlier levels
                                 run on every shard and are counted by shard 0 only.  The sums
                                 over shards equal the unsharded result exactly (counts, hash,
                                 paths per level, candidates). */
    uint64_t root_stride;     /* root sample: keep triplet <x,u,y> iff
                                 mix(x<<42 | u<<21 | y) % root_stride == root_offset
                                 (original ids); 0 or 1 = all roots.  Triangles are counted
                                 iff root_offset == 0. */
    uint64_t root_offset;
    uint64_t hash_seed;       /* 0 = default 0x1410487600000000 */
    void *workspace;          /* device memory for the frontier arena, owned by the caller
                                 (e.g. a torch tensor); NULL = the library allocates
                                 workspace_bytes (0 = 25% of free device memory) */
    uint64_t workspace_bytes;
    uint64_t collect_capacity;/* collect mode: max cycles kept (0 = 1<<22).  If exceeded,
                                 cc_enumerate fails with CC_ERR_CAPACITY and reports the
                                 required capacity in the message and in cc_stats */
    uint32_t profile;         /* 1 = time every expansion launch with CUDA events
                                 (cc_stats.t_expand_ms); 0 = only the total */
    uint32_t min_shard_paths; /* shard_count > 1: the first frontier level with at least
                                 min_shard_paths * shard_count paths is partitioned (0 = 2^20);
                                 Stage 1 is partitioned instead when it has at least that many
                                 forward pairs (0 = 2^16 per shard).  The partition is a function
                                 of the graph, shard_count and min_shard_paths -- and, only when an
                                 unsharded level does not fit the arena, of the arena size: give
                                 every rank the same workspace_bytes */
    uint32_t record_format;   /* frontier record format: 0 = automatic, 1 = blocked
                                 set (every size class), 2 = vertex list (512 < n <= 2015, max
                                 degree <= 32, 4 <= max_len <= 14; otherwise
                                 CC_ERR_INVALID_ARGUMENT).  Automatic picks the list for the
                                 graphs it accepts.  Results do not depend on it. */
} cc_options;

/* Statistics of one cc_enumerate call (cc_result_stats). */
typedef struct {
    uint32_t struct_size;
    uint32_t n_words;             /* 64-bit words per vertex bit row (S or B) */
    uint64_t total_cycles;        /* sum over k of counts[k] (counted on this shard) */
    uint64_t paths_expanded;      /* sum over t of |F_t|: paths scanned by Stage 2 */
    uint64_t candidates;          /* sum over scanned paths of deg(v_t) */
    uint64_t triplets;            /* |F_3| scanned (this shard) */
    uint64_t stage1_pairs;        /* forward-neighbour pairs examined by Stage 1 */
    uint64_t rounds;              /* deepest level t reached (paths of t vertices) */
    uint64_t launches;            /* kernel launches of Stage 1 + Stage 2 */
    uint64_t chunks;              /* frontier chunks (== launches when nothing was split) */
    uint64_t peak_arena_records;  /* high-water mark of the frontier arena, in records */
    uint64_t arena_capacity;      /* arena capacity, in records */
    uint64_t record_bytes;        /* bytes per frontier record */
    uint64_t bytes_alg;           /* bytes of the records the expansion kernels read and write
                                     (real records, at record_bytes each) + cycles stored */
    uint64_t cycles_stored;       /* collect mode: cycles kept (or required, on overflow) */
    uint64_t h2d_bytes;           /* host->device bytes this call (graph upload, if any) */
    uint64_t d2h_bytes;           /* device->host bytes this call (counts, sizes) */
    double t_dev_ms;              /* CUDA-event time from Stage 1 start to counts ready */
    double t_expand_ms;           /* profile=1: summed CUDA-event time of Stage 2 launches */
    double t_stage1_ms;           /* profile=1: summed CUDA-event time of Stage 1 launches */
    double t_labeling_ms;         /* host degree labelling + graph build (cc_graph_from_csr) */
    double t_wall_ms;             /* host wall time of cc_enumerate */
    uint64_t leaf_paths;          /* count mode with max_len: paths of the last level (their
                                     children could not close within max_len) counted by the
                                     launch that created them and never written */
    uint64_t paths_written;       /* frontier records written by Stage 1 and Stage 2 */
    uint64_t record_format;       /* frontier records used: 1 = blocked set (or bitmap S in
                                     collect mode), 2 = vertex list (cc_options.record_format) */
    uint64_t records_levelsync;   /* records a level-synchronous expansion of the same paths reads
                                     and writes: every expanded path once, every child once
                                     (SURVEY §8(d) "R_in + s*R_out" per path expanded).  The grid
                                     class's two-level launches keep every other level in shared
                                     memory and move fewer (bytes_alg) */
    uint64_t slots_moved;         /* frontier slots read + written by Stage 2 launches, including
                                     the empty slots of per-warp output chunks */
} cc_stats;

/* Fills *opt with defaults (device -1, stream NULL, no cap, count-only, one shard). */
void cc_options_init(cc_options *opt);

/*
 * Build a graph from host CSR ("compact graph representation": V_e = row_ptr,
 * E_e = col_idx).  n >= 0 vertices; row_ptr[n+1] int64 with row_ptr[0] = 0 and
 * non-decreasing; col_idx[row_ptr[n]] int32.  Rows may be unsorted; duplicate entries in a
 * row are merged.  Errors: CC_ERR_INVALID_VERTEX (id outside 0..n-1), CC_ERR_SELF_LOOP,
 * CC_ERR_NOT_SYMMETRIC, CC_ERR_INVALID_ARGUMENT (NULL pointers with n > 0, bad row_ptr,
 * n > 2^20).  The degree labelling (ties -> lowest original id) is computed
 * here, on the host, as the paper does.  Host arrays are copied.
 */
cc_status cc_graph_from_csr(int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                            cc_graph **out);
void cc_graph_free(cc_graph *g);

/* n, m (undirected edges), maximum degree Delta. */
cc_status cc_graph_info(const cc_graph *g, int64_t *n, int64_t *m, int64_t *max_degree);

/* The degree labelling: labels[v] = l(v) in 0..n-1 for original id v (n entries). */
cc_status cc_graph_labels(const cc_graph *g, int32_t *labels);

/*
 * Enumerate every chordless cycle of g exactly once on the GPU.
 * Size classes:
 *   n <= 512: bitset records of <= 8 words; count and collect mode;
 *   512 < n <= 2015: blocked-set records of <= 32 words (one warp per path; count mode), or
 *     vertex-list records (one thread per path; max degree <= 32 and 4 <= max_len <= 14; count
 *     and collect mode; see cc_options.record_format).
 * Larger graphs, and collect mode above n = 512 without the vertex-list records, fail with
 * CC_ERR_TOO_LARGE.
 * With max_len, count mode fuses the last level: the paths of max_len - 1 vertices are
 * counted (with their closures) by the launch that creates them and are never written
 * (cc_stats.leaf_paths).  Results do not depend on the record format, the workspace size,
 * the chunking or the shard count.
 * Errors: CC_ERR_NO_DEVICE, CC_ERR_CUDA, CC_ERR_CAPACITY (workspace too small to make
 * progress: one page of the deepest level needs more output than the free pages hold),
 * CC_ERR_INVALID_ARGUMENT (bad options).  On success *out owns the counts, set hash,
 * per-level statistics and (collect mode) the cycles in device memory.
 */
cc_status cc_enumerate(const cc_graph *g, const cc_options *opt, cc_result **out);

/*
 * counts[k] = number of chordless cycles with exactly k vertices, k = 0..n (k < 3 is 0).  A
 * cycle's "length" is its number of vertices (= edges), the k of a k-cycle in PAPER.md:41
 * (reading G13); Table 1 reports C3 = counts[3] and #clc = the sum
 * over k > 3.
 * *n_lengths is always set to n+1; if cap < n+1 returns CC_ERR_BUFFER_TOO_SMALL (counts
 * untouched).  counts may be NULL with cap = 0 to query the size.  set_hash (may be NULL)
 * receives sum over cycles C of mix(sum_{v in C} key(v)) mod 2^64.
 */
cc_status cc_count_by_length(const cc_result *r, uint64_t *counts, size_t cap, size_t *n_lengths,
                             uint64_t *set_hash);

/* paths[t] = |F_t|, paths of t vertices created (t = 0..n; the oracle's visited paths); sizes as above.
 * This is the |T| evolution of the paper's Fig. 4. */
cc_status cc_paths_by_length(const cc_result *r, uint64_t *paths, size_t cap, size_t *n_lengths);

/*
 * Collect mode: copy cycles [first, first + max_cycles) (in an unspecified but fixed order)
 * as canonical vertex sequences <v1..vk> in original ids (l(v2) minimal,
 * l(v1) < l(v3) under the library's degree labelling).  vertices receives the sequences
 * back to back, offsets[i]..offsets[i+1] delimit cycle i (offsets has max_cycles+1
 * entries).  *n_fetched = cycles written.  CC_ERR_NOT_COLLECTED on a count-only result;
 * CC_ERR_BUFFER_TOO_SMALL if vertices_cap is too small (offsets are then filled for the
 * cycles requested and *n_fetched = 0 so the caller can size the buffer).
 * Runs on the stream the result was enumerated on (cc_options.stream, which must still exist),
 * ordered after the enumeration.  Page-locked `vertices` buffers are filled by one DMA; pageable
 * ones through two pinned staging buffers, the copy of one chunk overlapping the next chunk's DMA.
 */
cc_status cc_fetch_cycles(const cc_result *r, uint64_t first, uint64_t max_cycles, int32_t *vertices,
                          size_t vertices_cap, uint64_t *offsets, uint64_t *n_fetched);

/* Number of cycles held by a collect-mode result (0 for count-only). */
cc_status cc_num_stored_cycles(const cc_result *r, uint64_t *n);

/* Statistics of the enumeration (out->struct_size must be set by the caller). */
cc_status cc_result_stats(const cc_result *r, cc_stats *out);

void cc_result_free(cc_result *r);

/* Thread-local message for the last non-OK status on this thread ("" if none). */
const char *cc_last_error(void);
const char *cc_status_string(cc_status s);

/* Library version string and the SM architecture the kernels were built for. */
const char *cc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CHORDLESS_H */
