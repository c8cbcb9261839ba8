// cc_kernels.cu -- sm_100a kernels of the chordless-cycle hot path (arXiv 1410.4876).
//
//   k_stage1<NW,BM>       Stage 1 (Alg. 2): seeds T(G) and triangles.  One
//                         thread per forward-neighbour pair (u; x < y in N+(u)) -- the
//                         sum_u C(d+(u),2) real pairs, not the paper's |V|*Delta^2 padded index
//                         space.
//   k_expand_blocked<NW>  Stage 2 (Alg. 3), count mode (the hot path): one
//                         thread per path on the blocked-vertex record (below); extensions are
//                         appended with a block-aggregated prefix-sum allocator (one atomicAdd per
//                         CTA tile: the paper's "serialization in the index calculation",
//                         PAPER.md:227, 289); input tiles stream in through a TMA bulk-copy ring.
//   k_expand_thread<NW>   Stage 2, collect mode (S-mode records), thread per path.
//   k_expand_warp<NW>     Stage 2, collect mode, Delta > 32: one warp per path, lanes scan the
//                         suffix of the sorted CSR row of v_t that passes the label gate
//                         (coalesced), ballot/popc warp-aggregated appends.
//   k_shard_filter<RW>    multi-GPU: keep the paths whose content hash falls in this shard.
//   k_keys, k_keybyte     key(v) = mix(seed ^ original id) (H-spec) and its byte tables.
//   k_cycle_*             collect mode: canonical vertex order of stored cycles (the inverse of
//                         the bitmap encoding, PAPER.md:193 / SPEC.md:216).
//
// The test of Alg. 3 lines 11-15 for p = <v1..vt> and v in Adj(vt):
//   gate   l(v) > l(v2) (== v > v2 after relabelling) and v not in p
//   extend iff v is adjacent to none of v1..v_{t-1}            -> <p,v> in F_{t+1}
//   close  iff v is adjacent to v1 and to none of v2..v_{t-1}  -> chordless cycle <p,v>
//   else   a chord: discard                           (the dichotomy of PAPER.md:57-64)
// B-mode evaluates it for all candidates at once on the blocked set
//   B(p) = N[v2] u ... u N[v_{t-1}]   (closed neighbourhoods; B contains every vertex of p)
//   Cand  = Adj(vt) & {v > v2} & ~B,   Close = Cand & Adj(v1),   Ext = Cand & ~Adj(v1)
//   child <p,v>: B' = B | N[vt], keysum' = keysum + key(v), ids' = (v1, v2, v).
// S-mode evaluates it per candidate on the bitmap S: X = Adj(v) & S & ~{vt};
//   extend iff X == {}, close iff X == {v1}.
#include "cc_device.cuh"

#include <cooperative_groups.h>

namespace cc {

// ---------------------------------------------------------------------------- Stage 1
template <int NW, bool BM, bool PACK>
__global__ void __launch_bounds__(kBlock) k_stage1(const LaunchArgs p)
{
    constexpr int RW = BM ? NW + 1 : NW;
    extern __shared__ u64 smem[];
    u64 *s_adj = smem;
    u64 *s_key = smem + p.g.n * NW;
    __shared__ ReserveSmem rs;
    stage_graph<NW>(p.g, s_adj, s_key, s_key + p.g.n);

    const int n = p.g.n;
    u64 cnt = 0, hs = 0;
    const u64 stride = (u64)gridDim.x * kBlock;
    for (u64 base = (u64)blockIdx.x * kBlock; base < p.n_in; base += stride) {
        const u64 r = base + threadIdx.x;
        unsigned int emit = 0;
        u64 W[RW];
        uint32_t id = 0;
        if (r < p.n_in) {
            const u64 gid = p.in_lo + r;
            // u = the largest vertex with pair_prefix[u] <= gid
            int lo = 0, hi = n - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (p.g.pair_prefix[mid] <= gid)
                    lo = mid;
                else
                    hi = mid - 1;
            }
            const uint32_t u = (uint32_t)lo;
            const u64 q = gid - p.g.pair_prefix[u];
            // triangular decode q -> (i, j), 0 <= i < j:  q = j(j-1)/2 + i
            u64 j = (u64)((1.0 + sqrt(1.0 + 8.0 * (double)q)) * 0.5);
            while (j * (j - 1) / 2 > q)
                --j;
            while ((j + 1) * j / 2 <= q)
                ++j;
            const u64 i = q - j * (j - 1) / 2;
            const uint32_t f = p.g.fwd[u];
            const uint32_t x = p.g.col[f + (uint32_t)i];
            const uint32_t y = p.g.col[f + (uint32_t)j];  // u < x < y in label order (Alg. 2 l.12)
            const bool tri = (s_adj[x * NW + (y >> 6)] >> (y & 63)) & 1ull;  // x in Adj(y) (l.13)
            if (tri) {
                if (p.count) {  // Alg. 2 line 14: a triangle goes straight to C
                    cnt++;
                    hs += mix64(s_key[x] + s_key[u] + s_key[y]);
                    if (p.collect) {
                        u64 S[NW];
#pragma unroll
                        for (int w = 0; w < NW; ++w)
                            S[w] = bit_in_word(w, x) | bit_in_word(w, u);
                        store_cycle<NW>(p, S, y, x, u);
                    }
                }
            } else if (p.emit) {  // Alg. 2 line 15: <x,u,y> in T(G)
                emit = 1;
                if (p.root_stride > 1) {
                    const u64 rkey = ((u64)p.g.orig[x] << 42) | ((u64)p.g.orig[u] << 21) |
                                     (u64)p.g.orig[y];
                    emit = (mix64(rkey) % p.root_stride) == p.root_offset;
                }
                if (BM) {  // B(<x,u,y>) = N[u]; keysum = key(x) + key(u) + key(y)
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        W[w] = s_adj[u * NW + w] | bit_in_word(w, u);
                    W[RW - 1] = s_key[x] + s_key[u] + s_key[y];
                } else {  // S = {x, u, y}
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        W[w] = bit_in_word(w, x) | bit_in_word(w, u) | bit_in_word(w, y);
                }
                if (PACK) {
                    W[NW - 1] = with_packed_ids(W[NW - 1], pack3(x, u, y, p.idb), p.idb);
                    id = 0;
                } else {
                    id = pack_ids(x, u, y);
                }
                if (emit && p.filter)
                    emit = (shard_hash<RW>(W, id) % p.shard_count) == p.shard_index;
            }
        }
        const u64 off = block_reserve(emit, &p.sc->out_count, rs);
        if (emit) {
            if (off >= p.out_cap)
                p.sc->err = 1;
            else
                store_record<RW, !PACK>(p.pg, p.out_off + off, W, id);
        }
    }
    flush_accum(cnt, hs, 0, p.sc);
}

// ---------------------------------------------------------------------------- Stage 2, B-mode
// Persistent CTAs; the input tiles (kBlock*R consecutive records of one page: the RW contiguous
// word arrays, plus the ids array unless ids are packed) stream into a kStages-deep shared-memory
// ring through TMA bulk copies (cp.async.bulk + mbarrier), issued by thread 0 kStages tiles
// ahead of the consumers.
#ifndef CC_STAGES
#define CC_STAGES 2
#endif
#ifndef CC_CHILD_CAP_X4
#define CC_CHILD_CAP_X4 8
#endif
constexpr int kStages = CC_STAGES;
#ifndef CC_STORE_CS
#define CC_STORE_CS 0  // 1 = cache-streaming stores for the children (st.global.cs)
#endif
#ifndef CC_EB_BLOCK
#define CC_EB_BLOCK 128
#endif
constexpr int kEBBlock = CC_EB_BLOCK;
#ifndef CC_EB_MINB
#define CC_EB_MINB 3  // register bound of k_expand_blocked (NW <= 2): at least 3 resident CTAs
#endif  // threads per CTA of k_expand_blocked (smaller CTAs: barriers span fewer warps)
constexpr int kChildCapX4 = CC_CHILD_CAP_X4;  // child list capacity = kChildCapX4/4 per path slot

template <int NW, bool PACK>
__host__ __device__ constexpr size_t blocked_stage_bytes()
{
    return (size_t)kEBBlock * expand_paths_per_thread(NW) * ((NW + 1) * 8 + (PACK ? 0 : 4));
}

// MAXCH > 0: every path has at most MAXCH children (Delta - 1, host-checked), so the staging of
// children is unrolled into MAXCH predicated steps instead of a divergent per-bit loop.
template <int NW, int MAXCH, bool PACK, bool LEAF>
#ifndef CC_EB_MINB_WIDE
#define CC_EB_MINB_WIDE 5  // NW > 2: 5 CTAs (K_{150,150} expansion 0.221 -> 0.209 ms, measured)
#endif
__global__ void __launch_bounds__(kEBBlock, NW <= 2 ? CC_EB_MINB : CC_EB_MINB_WIDE) k_expand_blocked(const LaunchArgs p)
{
    constexpr int RW = NW + 1;
    constexpr int R = expand_paths_per_thread(NW);
    constexpr int kTile = kEBBlock * R;
    constexpr uint32_t kStageBytes = (uint32_t)blocked_stage_bytes<NW, PACK>();
    constexpr uint32_t kChildCap = kChildCapX4 * kTile / 4;  // overflow falls back to per-thread appends
    extern __shared__ __align__(128) u64 smem[];
    // ring first (16-byte aligned bulk-copy destinations), then the graph tables
    char *ring = (char *)smem;
    u64 *s_adj = (u64 *)(ring + (size_t)kStages * kStageBytes);
    u64 *s_key = s_adj + p.g.n * NW;
    // s_above[v*NW + w] = word w of {x : x > v} (the label gate); 16-byte aligned (padded keys).
    // Wider records (NW > 2) compute the gate words instead: the table would cost n*NW words of
    // shared memory, i.e. resident CTAs (K_{150,150} is latency bound at 4 CTAs per SM)
    constexpr bool kAboveTable = NW <= 2;
    u64 *s_above = s_key + ((p.g.n + 1) & ~1);
    // staged children of one tile: parent state per path slot, one (slot, v) entry per child
    constexpr int PW = RW + NW;                           // parent child state + extension words
    u64 *s_par = s_above + (kAboveTable ? p.g.n * NW : 0);  // [kTile][PW]
    uint32_t *s_pid = (uint32_t *)(s_par + kTile * PW);   // [kTile] (unpacked ids only)
    uint32_t *s_child = s_pid + (PACK ? 0 : kTile);       // [kChildCap]
    __shared__ ReserveSmemT<kEBBlock> rs[2];
    __shared__ __align__(8) u64 bar[kStages];

    const uint32_t idb = PACK ? p.idb : (uint32_t)kIdBits;
    const uint32_t idm = (1u << idb) - 1;
    const u64 keep_v12 = PACK ? ~((u64)idm << (64 - idb)) : ~0ull;  // packed: vt field cleared
    // chained launch (cc_host.cpp, Stage 1 -> F_3): the input size is Stage 1's device-side count
    const u64 n_in = p.n_in_dev ? *p.n_in_dev : p.n_in;
    const u64 n_tiles = (n_in + kTile - 1) / kTile;
    const u64 my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    // tile k of this CTA -> global tile blockIdx.x + k * gridDim.x -> its page and slot
    auto issue = [&](u64 k) {
        const int st = (int)(k % kStages);
        const u64 base = (blockIdx.x + k * gridDim.x) * (u64)kTile;
        const uint32_t page = p.pg.in_pages[base >> p.pg.log_p];
        const uint32_t slot0 = (uint32_t)(base & ((1ull << p.pg.log_p) - 1));
        const char *pp = p.pg.base + (u64)page * p.pg.page_bytes;
        char *dst = ring + (size_t)st * kStageBytes;
        mbar_arrive_expect_tx(&bar[st], kStageBytes);
#pragma unroll
        for (int w = 0; w < RW; ++w)
            tma_load_1d(dst + (size_t)w * kTile * 8, pp + (((u64)w << p.pg.log_p) + slot0) * 8, kTile * 8,
                        &bar[st]);
        if (!PACK)
            tma_load_1d(dst + (size_t)RW * kTile * 8, pp + ((u64)RW << p.pg.log_p) * 8 + (u64)slot0 * 4,
                        kTile * 4, &bar[st]);
    };
    if (threadIdx.x == 0) {
        for (int st = 0; st < kStages; ++st)
            mbar_init(&bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (u64 k = 0; k < my_tiles && k < (u64)kStages; ++k)
            issue(k);
    }
    // closed rows N[v] = Adj(v) | {v} in s_adj: vt and v1 always lie in B, so Cand/Close/Ext are
    // unchanged, and the children's blocked set B | N[vt] is a plain OR
    for (int i = threadIdx.x; i < p.g.n * NW; i += kEBBlock) {
        if (kAboveTable)
            s_above[i] = above_word((uint32_t)(i / NW), i % NW);
        s_adj[i] = p.g.adj[i] | bit_in_word(i % NW, (uint32_t)(i / NW));
    }
    for (int i = threadIdx.x; i < p.g.n; i += kEBBlock)
        s_key[i] = p.g.key[i];
    __syncthreads();

    // per-thread statistics in 32 bits (a launch gives a thread at most ~10^5 paths, n <= 512)
    uint32_t cnt = 0, cand = 0, paths_in = 0, written = 0;
    u64 hs = 0;
    uint32_t leaf_paths = 0, leaf_cand = 0, leaf_cyc = 0;
    const u64 pmask = (1ull << p.pg.log_p) - 1;
    // last level (p.emit && !p.emit_next): the children <p,v> cannot have children within the
    // length cap; they are counted -- |F_{t+1}|, deg(v), their closures -- and not written
    for (u64 k = 0; k < my_tiles; ++k) {
        const int st = (int)(k % kStages);
        const u64 base = (blockIdx.x + k * gridDim.x) * (u64)kTile;
        const bool full = base + kTile <= n_in;
        mbar_wait(&bar[st], (uint32_t)((k / kStages) & 1));
        const char *buf = ring + (size_t)st * kStageBytes;
        u64 W[R][RW];
        uint32_t id[R];  // v1 | v2 << idb | vt << 2idb
        bool valid[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int j = threadIdx.x + kEBBlock * i;
#pragma unroll
            for (int w = 0; w < RW; ++w)
                W[i][w] = ((const u64 *)buf)[w * kTile + j];
            id[i] = PACK ? packed_ids(W[i][NW - 1], idb) : ((const uint32_t *)(buf + (size_t)RW * kTile * 8))[j];
            // empty slots of a k_expand_fused output chunk are all-zero records: v1 == v2 == 0
            // never holds for a path (v2 = u < v1 = x, Alg. 2 l.12)
            valid[i] = (full || base + j < n_in) && (id[i] & idm) != ((id[i] >> idb) & idm);
            paths_in += valid[i];
        }
        u64 ext[R][NW];
        unsigned int ne = 0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
#pragma unroll
            for (int w = 0; w < NW; ++w)
                ext[i][w] = 0;
            if (!valid[i])
                continue;
            const uint32_t v1 = id[i] & idm;
            const uint32_t v2 = (id[i] >> idb) & idm;
            const uint32_t vt = id[i] >> (2 * idb);
            u64 close[NW], arow[NW], abv[NW], a1row[NW];
            bool any_close = false;
            lds_row<NW>(s_adj, vt, arow);
            if constexpr (kAboveTable) {
                lds_row<NW>(s_above, v2, abv);
            } else {
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    abv[w] = above_word(v2, w);
            }
            lds_row<NW>(s_adj, v1, a1row);
            cand -= 1;  // deg(vt) = |N[vt]| - 1: the candidate slots of Alg. 3 (statistic)
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const u64 a = arow[w];
                cand += __popcll(a);
                // the packed ids sit above bit n, where a is zero: they never leak into c
                const u64 c = a & abv[w] & ~W[i][w];
                const u64 a1 = a1row[w];
                close[w] = c & a1;
                ext[i][w] = p.emit ? (c & ~a1) : 0ull;
                any_close |= close[w] != 0ull;
                ne += __popcll(ext[i][w]);
            }
            if (any_close && p.count) {
                const u64 ks = W[i][NW];
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    const u64 m = close[w];
                    cnt += __popcll(m);
                    // 32-bit halves: cheaper bit extraction on 32-bit lanes (K_{a,b}: ~100
                    // closures per path, each dominated by the 64-bit mix)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t mm = (uint32_t)(m >> (32 * h));
                        while (mm) {
                            const int b = __ffs(mm) - 1;
                            mm &= mm - 1;
                            hs += mix64(ks + s_key[64 * w + 32 * h + b]);
                        }
                    }
                }
            }
            if constexpr (LEAF) {
                // Close(<p,v>) = Adj(v) & Z(p), Z(p) = {x > v2} & ~(B | N[vt]) & Adj(v1)
                u64 Z[NW];
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    Z[w] = abv[w] & ~(W[i][w] | arow[w]) & a1row[w];  // v is in B | N[vt]
                    ne -= __popcll(ext[i][w]);
                }
                if (p.count) {
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        u64 m = ext[i][w];
                        while (m) {
                            const int b = __ffsll((long long)m) - 1;
                            m &= m - 1;
                            const uint32_t v = (uint32_t)(64 * w + b);
                            u64 av[NW];
                            lds_row<NW>(s_adj, v, av);
                            const u64 ksv = W[i][NW] + s_key[v];
                            leaf_paths++;
                            leaf_cand -= 1;  // closed row
#pragma unroll
                            for (int w2 = 0; w2 < NW; ++w2) {
                                leaf_cand += __popcll(av[w2]);
                                u64 cl = av[w2] & Z[w2];
                                leaf_cyc += __popcll(cl);
                                while (cl) {
                                    const int b2 = __ffsll((long long)cl) - 1;
                                    cl &= cl - 1;
                                    hs += mix64(ksv + s_key[64 * w2 + b2]);
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    ext[i][w] = 0;
            }
        }
        // every thread has read stage st (the reservation starts with a barrier) -> refill it
        u64 ticket = 0;
        const unsigned int loc0 = reserve_begin<kEBBlock>(ne, &p.sc->out_count, rs[k & 1], &ticket);
        if (threadIdx.x == 0 && k + kStages < my_tiles) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(k + kStages);
        }
        const unsigned int total = rs[k & 1].total;
        written += ne;
        {
            // Staged append.  Each path with children publishes its child state (B | N[vt],
            // keysum, and its ids) in s_par[slot]; each child gets one 4-byte entry (slot, v) at
            // its tile-local position in s_child.  After a barrier all threads copy the tile's
            // children to their consecutive output positions: a uniform, fully coalesced loop.
            uint32_t loc = loc0;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                bool any = false;
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    any |= ext[i][w] != 0ull;
                if (!any)
                    continue;
                const uint32_t slot = threadIdx.x + kEBBlock * i;
                const uint32_t vt = id[i] >> (2 * idb);
                u64 ar[NW];
                lds_row<NW>(s_adj, vt, ar);
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    s_par[slot * PW + w] = W[i][w] | ar[w];  // B | N[vt]
                s_par[slot * PW + NW] = W[i][NW];
                if (!PACK)
                    s_pid[slot] = id[i] & ((1u << (2 * idb)) - 1);
                if (MAXCH > 0) {
                    // entries (slot, rank): the copy phase finds the rank-th child itself
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        s_par[slot * PW + RW + w] = ext[i][w];
                    uint32_t nc = 0;
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        nc += __popcll(ext[i][w]);
#pragma unroll
                    for (int c = 0; c < MAXCH; ++c)
                        if ((uint32_t)c < nc && loc + c < kChildCap)
                            s_child[loc + c] = slot | ((uint32_t)c << 16);
                    loc += nc;
                } else {
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        u64 m = ext[i][w];
                        while (m) {
                            const int b = __ffsll((long long)m) - 1;
                            m &= m - 1;
                            if (loc < kChildCap)
                                s_child[loc] = slot | ((uint32_t)(64 * w + b) << 16);
                            ++loc;
                        }
                    }
                }
            }
        }
        if (is_ticket_lane<kEBBlock>())
            rs[k & 1].base = ticket;  // the atomic's result is needed only now
        __syncthreads();
        const u64 tile_base = rs[k & 1].base;  // first output position of this CTA tile
        const u64 off = tile_base + loc0;
        if (ne && off + ne > p.out_cap)
            p.sc->err = 1;
        if (total > kChildCap) {
            // rare (many children per path): per-thread appends straight from registers
            if (ne && off + ne <= p.out_cap) {
                Appender<RW> out;
                out.seek(p.pg, p.out_off + off);
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    if (!valid[i])
                        continue;
                    const uint32_t vt = id[i] >> (2 * idb);
                    const uint32_t v12 = id[i] & ((1u << (2 * idb)) - 1);
                    u64 C[RW];
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        C[w] = W[i][w] | s_adj[vt * NW + w];
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        u64 m = ext[i][w];
                        while (m) {
                            const int b = __ffsll((long long)m) - 1;
                            m &= m - 1;
                            const uint32_t v = (uint32_t)(64 * w + b);
                            C[NW] = W[i][NW] + s_key[v];
                            if (PACK) {
                                C[NW - 1] = with_packed_ids(C[NW - 1], v12 | (v << (2 * idb)), idb);
                                out.template put_words<!PACK>(p.pg, C, 0);
                            } else {
                                out.template put_words<!PACK>(p.pg, C, v12 | (v << (2 * idb)));
                            }
                        }
                    }
                }
            }
        } else if (tile_base + total <= p.out_cap) {
            // output positions o0 + j: page pg0 from slot s0 up to `split`, then page pg0 + 1
            const u64 o0 = p.out_off + tile_base;
            const uint32_t s0 = (uint32_t)(o0 & pmask);
            const uint32_t split = (uint32_t)(pmask + 1 - s0);
            char *pp0 = page_ptr(p.pg, p.pg.out_pages[o0 >> p.pg.log_p]);
            char *pp1 = split < total ? page_ptr(p.pg, p.pg.out_pages[(o0 >> p.pg.log_p) + 1]) : pp0;
            for (unsigned int j = threadIdx.x; j < total; j += kEBBlock) {
                const uint32_t e = s_child[j];
                const uint32_t slot = e & 0xffffu;
                uint32_t v;
                u64 par[PW];
#pragma unroll
                for (int w = 0; w < PW; ++w)
                    par[w] = (w < RW || MAXCH > 0) ? s_par[slot * PW + w] : 0ull;
                if (MAXCH > 0) {
                    // v = the rank-th (rank < MAXCH) set bit of the parent's extension words:
                    // pick the word by popcount, drop `rank` low bits (selects), find-first-set
                    uint32_t r = e >> 16;
                    u64 x = par[RW];
                    uint32_t wsel = 0;
#pragma unroll
                    for (int w = 1; w < NW; ++w) {
                        const uint32_t pc = __popcll(x);
                        const u64 nx = par[RW + w];
                        const bool next = r >= pc;
                        r = next ? r - pc : r;
                        wsel = next ? (uint32_t)w : wsel;
                        x = next ? nx : x;
                    }
#pragma unroll
                    for (int c = 1; c < MAXCH; ++c) {
                        const u64 y = x & (x - 1);
                        x = (uint32_t)c <= r ? y : x;
                    }
                    v = 64 * wsel + (uint32_t)__ffsll((long long)x) - 1;
                } else {
                    v = e >> 16;
                }
                u64 C[RW];
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    C[w] = par[w];
                C[NW] = par[NW] + s_key[v];
                const bool lo = j < split;
                char *pp = lo ? pp0 : pp1;
                const uint32_t oslot = lo ? s0 + j : j - split;
                u64 *w0 = (u64 *)pp + oslot;
                if (PACK) {
                    // child ids: (v1, v2) of the parent, last vertex v (the top idb bits)
                    C[NW - 1] = (C[NW - 1] & keep_v12) | ((u64)v << (64 - idb));
                } else {
                    ((uint32_t *)(pp + ((u64)RW << p.pg.log_p) * 8))[oslot] = s_pid[slot] | (v << (2 * idb));
                }
#pragma unroll
                for (int w = 0; w < RW; ++w) {
#if CC_STORE_CS
                    __stcs(w0 + ((size_t)w << p.pg.log_p), C[w]);  // streaming: evict-first in L2
#else
                    w0[(size_t)w << p.pg.log_p] = C[w];
#endif
                }
            }
        }
    }
    if (!p.count)
        cand = 0;
    Acc a;
    a.cyc = cnt;
    a.hash = hs;
    a.cand = cand;
    a.cyc_next = leaf_cyc;
    a.cand_next = leaf_cand;
    a.paths_next = leaf_paths;
    a.paths_cur = paths_in;
    a.out_real = written;
    flush<kEBBlock>(a, p.sc);
}

// ---------------------------------------------------------------------------- Stage 2, S-mode
// Per-candidate form on the bitmap S (collect mode): cand = Adj(vt) & ~S & {v > v2};
// for v in cand: X = Adj(v) & S & ~{vt}; X == {} -> extension, X == {v1} -> cycle.
template <int NW>
__global__ void __launch_bounds__(kBlock) k_expand_thread(const LaunchArgs p)
{
    extern __shared__ u64 smem[];
    u64 *s_adj = smem;
    u64 *s_key = smem + p.g.n * NW;
    u64 *s_kb = s_key + p.g.n;
    __shared__ ReserveSmem rs;
    stage_graph<NW>(p.g, s_adj, s_key, s_kb);

    const u64 pmask = (1ull << p.pg.log_p) - 1;
    u64 cnt = 0, hs = 0, cand = 0;
    const u64 stride = (u64)gridDim.x * kBlock;
    for (u64 base = (u64)blockIdx.x * kBlock; base < p.n_in; base += stride) {
        const u64 r = base + threadIdx.x;
        u64 S[NW], ext[NW];
        uint32_t id = 0;
        unsigned int ne = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w)
            ext[w] = 0;
        if (r < p.n_in) {
            load_record<NW>(p.pg, p.pg.in_pages[base >> p.pg.log_p], (uint32_t)(r & pmask), S, id);
            const uint32_t v1 = id & kIdMask;
            const uint32_t v2 = (id >> kIdBits) & kIdMask;
            const uint32_t vt = id >> (2 * kIdBits);
            u64 cw[NW];
            const int lo = (int)v2 + 1;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const u64 a = s_adj[vt * NW + w];
                cand += __popcll(a);
                const int sh = lo - 64 * w;
                const u64 above = sh <= 0 ? ~0ull : (sh >= 64 ? 0ull : (~0ull << sh));
                cw[w] = a & ~S[w] & above;
            }
            u64 ks = 0;
            bool have_ks = false;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                while (cw[w]) {
                    const int b = __ffsll((long long)cw[w]) - 1;
                    cw[w] &= cw[w] - 1;
                    const uint32_t v = (uint32_t)(64 * w + b);
                    bool e = true, c = true;
#pragma unroll
                    for (int u = 0; u < NW; ++u) {
                        u64 x = s_adj[v * NW + u] & S[u];
                        if (u == (int)(vt >> 6))
                            x &= ~(1ull << (vt & 63));
                        e &= (x == 0ull);
                        c &= (x == bit_in_word(u, v1));
                    }
                    if (e) {
                        if (p.emit) {
                            ext[w] |= 1ull << b;
                            ++ne;
                        }
                    } else if (c && p.count) {
                        ++cnt;
                        if (!have_ks) {
                            ks = keysum<NW>(S, s_key, s_kb);
                            have_ks = true;
                        }
                        hs += mix64(ks + s_key[v]);
                        if (p.collect)
                            store_cycle<NW>(p, S, v, v1, v2);
                    }
                }
            }
        }
        const u64 off = block_reserve(ne, &p.sc->out_count, rs);
        if (ne) {
            if (off + ne > p.out_cap) {
                p.sc->err = 1;
            } else {
                u64 o = p.out_off + off;
                const uint32_t v12 = id & ((1u << (2 * kIdBits)) - 1);
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    while (ext[w]) {
                        const int b = __ffsll((long long)ext[w]) - 1;
                        ext[w] &= ext[w] - 1;
                        const uint32_t v = (uint32_t)(64 * w + b);
                        u64 C[NW];
#pragma unroll
                        for (int u = 0; u < NW; ++u)
                            C[u] = S[u] | bit_in_word(u, v);
                        store_record<NW>(p.pg, o++, C, v12 | (v << (2 * kIdBits)));
                    }
                }
            }
        }
    }
    if (!p.count)
        cand = 0;
    flush_accum(cnt, hs, cand, p.sc);
}

template <int NW>
__global__ void __launch_bounds__(kBlock) k_expand_warp(const LaunchArgs p)
{
    extern __shared__ u64 smem[];
    u64 *s_adj = smem;
    u64 *s_key = smem + p.g.n * NW;
    stage_graph<NW>(p.g, s_adj, s_key, s_key + p.g.n);

    const int lane = threadIdx.x & 31;
    const unsigned int lt_mask = (1u << lane) - 1u;
    const uint32_t *__restrict__ rowptr = p.g.rowptr;
    const uint32_t *__restrict__ col = p.g.col;
    const u64 pmask = (1ull << p.pg.log_p) - 1;
    u64 cnt = 0, hs = 0, cand = 0;
    const u64 nwarps = (u64)gridDim.x * (kBlock / 32);
    for (u64 r = (u64)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); r < p.n_in; r += nwarps) {
        u64 S[NW];
        uint32_t id;
        load_record<NW>(p.pg, p.pg.in_pages[r >> p.pg.log_p], (uint32_t)(r & pmask), S, id);
        const uint32_t v1 = id & kIdMask, v2 = (id >> kIdBits) & kIdMask, vt = id >> (2 * kIdBits);
        const uint32_t k1 = __ldg(rowptr + vt), k2 = __ldg(rowptr + vt + 1);
        if (lane == 0)
            cand += k2 - k1;
        // the label gate l(v) > l(v2) keeps a suffix of the sorted row: find its start
        uint32_t lo = k1, hi = k2;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(col + mid) <= v2)
                lo = mid + 1;
            else
                hi = mid;
        }
        u64 ks = 0;
        bool have_ks = false;
        for (uint32_t kk = lo; kk < k2; kk += 32) {
            const uint32_t k = kk + lane;
            int c = 0;
            uint32_t v = 0;
            if (k < k2) {
                v = __ldg(col + k);
                if (!((word_of<NW>(S, v) >> (v & 63)) & 1ull)) {  // v not in p
                    bool e = true, cl = true;
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        u64 x = s_adj[v * NW + w] & S[w];
                        if (w == (int)(vt >> 6))
                            x &= ~(1ull << (vt & 63));
                        e &= (x == 0ull);
                        cl &= (x == bit_in_word(w, v1));
                    }
                    c = e ? 1 : (cl ? 2 : 0);
                }
            }
            const unsigned int eb = __ballot_sync(FULL_MASK, c == 1 && p.emit);
            if (eb) {
                u64 b = 0;
                if (lane == 0)
                    b = atomicAdd(&p.sc->out_count, (u64)__popc(eb));
                b = __shfl_sync(FULL_MASK, b, 0);
                if (c == 1) {
                    const u64 off = b + __popc(eb & lt_mask);
                    if (off >= p.out_cap) {
                        p.sc->err = 1;
                    } else {
                        u64 C[NW];
#pragma unroll
                        for (int w = 0; w < NW; ++w)
                            C[w] = S[w] | bit_in_word(w, v);
                        store_record<NW>(p.pg, p.out_off + off, C, pack_ids(v1, v2, v));
                    }
                }
            }
            // the keysum of S is needed once per path: computed by the whole warp (lane w < NW
            // sums the keys of word w, then a shuffle reduction) at the first closure
            if (!have_ks && __any_sync(FULL_MASK, c == 2)) {
                u64 part = 0;
                if (lane < NW) {
                    u64 x = 0;
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        if (w == lane)
                            x = S[w];
                    while (x) {
                        const int b = __ffsll((long long)x) - 1;
                        part += s_key[lane * 64 + b];
                        x &= x - 1;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
                    part += __shfl_xor_sync(FULL_MASK, part, o);
                ks = part;
                have_ks = true;
            }
            if (c == 2 && p.count) {
                ++cnt;
                hs += mix64(ks + s_key[v]);
                if (p.collect)
                    store_cycle<NW>(p, S, v, v1, v2);
            }
        }
    }
    if (!p.count)
        cand = 0;
    flush_accum(cnt, hs, cand, p.sc);
}

// ---------------------------------------------------------------------------- small frontiers
// k_small_levels (SmallArgs): the Stage-2 levels of a small frontier in one cooperative launch.
// Thread per path on the blocked-vertex record (the test of k_expand_blocked, closed rows),
// children appended with one atomic per CTA iteration; a grid-wide barrier separates levels, so
// a level costs a barrier instead of a host round trip (launch + scratch read-back + sync).
template <int NW, bool PACK>
__global__ void __launch_bounds__(kBlock) k_small_levels(const LaunchArgs p, const SmallArgs s)
{
    namespace cg = cooperative_groups;
    constexpr int RW = NW + 1;
    extern __shared__ __align__(128) u64 smem[];
    u64 *s_adj = smem;                   // closed rows
    u64 *s_key = s_adj + p.g.n * NW;
    u64 *s_above = s_key + ((p.g.n + 1) & ~1);
    __shared__ ReserveSmem rs;
    for (int i = threadIdx.x; i < p.g.n * NW; i += kBlock) {
        s_above[i] = above_word((uint32_t)(i / NW), i % NW);
        s_adj[i] = p.g.adj[i] | bit_in_word(i % NW, (uint32_t)(i / NW));
    }
    for (int i = threadIdx.x; i < p.g.n; i += kBlock)
        s_key[i] = p.g.key[i];
    __syncthreads();
    cg::grid_group grid = cg::this_grid();
    const uint32_t idb = PACK ? p.idb : (uint32_t)kIdBits;
    const uint32_t idm = (1u << idb) - 1;
    const u64 keep_v12 = PACK ? ~((u64)idm << (64 - idb)) : ~0ull;
    const u64 P = 1ull << p.pg.log_p;
    int d = s.d0;
    for (;;) {
        const u64 n_in = s.count[d];
        if (n_in == 0 || d >= s.d_stop || n_in > s.threshold)
            break;  // block-uniform: everybody read the same count after the barrier
        // level d: the triplets' page or a region of contiguous pages (record r in page
        // region + (r >> log_p), slot r & (P - 1)); its children go to the other region
        const uint32_t ipg = d == s.d0 ? s.first : s.region[(d - s.d0 - 1) & 1];
        const uint32_t opg = s.region[(d - s.d0) & 1];
        const bool emit = s.max_len == 0 || (u64)d + 1 < s.max_len;
        uint32_t cnt = 0, cand = 0;
        u64 hs = 0;
        const u64 stride = (u64)gridDim.x * kBlock;
        for (u64 base = (u64)blockIdx.x * kBlock; base < n_in; base += stride) {
            const u64 r = base + threadIdx.x;
            u64 W[RW], ext[NW];
            uint32_t id = 0, ne = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w)
                ext[w] = 0;
            if (r < n_in) {
                const char *ip = p.pg.base + (u64)(ipg + (uint32_t)(r >> p.pg.log_p)) * p.pg.page_bytes;
                const u64 rs_ = r & (P - 1);
#pragma unroll
                for (int w = 0; w < RW; ++w)
                    W[w] = ((const u64 *)ip)[(u64)w * P + rs_];
                id = PACK ? (uint32_t)packed_ids(W[NW - 1], idb) : ((const uint32_t *)(ip + (u64)RW * P * 8))[rs_];
                const uint32_t v1 = id & idm, v2 = (id >> idb) & idm, vt = id >> (2 * idb);
                u64 arow[NW], abv[NW], a1[NW];
                lds_row<NW>(s_adj, vt, arow);
                lds_row<NW>(s_above, v2, abv);
                lds_row<NW>(s_adj, v1, a1);
                cand -= 1;  // closed row
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    cand += __popcll(arow[w]);
                    const u64 c = arow[w] & abv[w] & ~W[w];
                    u64 cl = c & a1[w];
                    ext[w] = emit ? (c & ~a1[w]) : 0ull;
                    ne += __popcll(ext[w]);
                    cnt += __popcll(cl);
                    while (cl) {
                        const int b = __ffsll((long long)cl) - 1;
                        cl &= cl - 1;
                        hs += mix64(W[NW] + s_key[64 * w + b]);
                    }
                }
            }
            const u64 off = block_reserve(ne, &s.count[d + 1], rs);
            if (ne) {
                if (off + ne > s.region_cap) {
                    *s.err = 1;
                } else {
                    const uint32_t vt = id >> (2 * idb), v12 = id & ((1u << (2 * idb)) - 1);
                    u64 C[RW];
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        C[w] = W[w] | s_adj[vt * NW + w];  // B | N[vt]
                    C[NW - 1] &= keep_v12;
                    u64 o = off;
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        u64 m = ext[w];
                        while (m) {
                            const int b = __ffsll((long long)m) - 1;
                            m &= m - 1;
                            const uint32_t v = (uint32_t)(64 * w + b);
                            u64 X[RW];
#pragma unroll
                            for (int q = 0; q < RW; ++q)
                                X[q] = C[q];
                            X[NW] = W[NW] + s_key[v];
                            char *op = p.pg.base + (u64)(opg + (uint32_t)(o >> p.pg.log_p)) * p.pg.page_bytes;
                            const u64 os_ = o & (P - 1);
                            if (PACK)
                                X[NW - 1] |= (u64)v << (64 - idb);
                            else
                                ((uint32_t *)(op + (u64)RW * P * 8))[os_] = v12 | (v << (2 * idb));
#pragma unroll
                            for (int q = 0; q < RW; ++q)
                                ((u64 *)op)[(u64)q * P + os_] = X[q];
                            ++o;
                        }
                    }
                }
            }
        }
        // level statistics: one atomic per counter per CTA
        Acc a;
        a.cyc = cnt;
        a.cand = cand;
        a.hash = hs;
        {
            constexpr int K = 3;
            __shared__ u64 red[K][kBlock / 32];
            u64 v[K] = {a.cyc, a.cand, a.hash};
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
            for (int k = 0; k < K; ++k) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
                    v[k] += __shfl_xor_sync(FULL_MASK, v[k], o);
                if (lane == 0)
                    red[k][wid] = v[k];
            }
            __syncthreads();
            if (threadIdx.x < K) {
                u64 t = 0;
                for (int i = 0; i < kBlock / 32; ++i)
                    t += red[threadIdx.x][i];
                u64 *dst = threadIdx.x == 0 ? &s.cyc[d] : threadIdx.x == 1 ? &s.cand[d] : s.hash;
                if (t)
                    atomicAdd(dst, t);
            }
        }
        grid.sync();
        ++d;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *s.last = d;
}

cudaError_t launch_small(const LaunchArgs &a, const SmallArgs &s, cudaStream_t st, int sms)
{
    void (*f)(const LaunchArgs, const SmallArgs) = nullptr;
    if (a.g.nw == 1)
        f = a.packed ? k_small_levels<1, true> : k_small_levels<1, false>;
    else if (a.g.nw == 2)
        f = a.packed ? k_small_levels<2, true> : k_small_levels<2, false>;
    if (!f)
        return cudaErrorInvalidValue;
    const size_t smem = ((size_t)a.g.n * 2 * a.g.nw + ((a.g.n + 1) & ~1)) * sizeof(u64);
    int nb = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)f, kBlock, smem);
    if (e != cudaSuccess)
        return e;
    if (nb < 1)
        return cudaErrorInvalidConfiguration;
    LaunchArgs a2 = a;
    SmallArgs s2 = s;
    void *args[] = {(void *)&a2, (void *)&s2};
    return cudaLaunchCooperativeKernel((const void *)f, dim3((unsigned)(nb * sms)), dim3(kBlock), args, smem, st);
}

// ---------------------------------------------------------------------------- shard filter
// HOLES: bitset records (ids v1 | v2 | vt in the ids array or packed in word RW-2), whose levels
// may hold empty slots; false for the list class (its words hold 16-bit vertex lists)
template <int RW, bool IDS, bool HOLES = true>
__global__ void __launch_bounds__(kBlock) k_shard_filter(const LaunchArgs p)
{
    __shared__ ReserveSmem rs;
    const u64 pmask = (1ull << p.pg.log_p) - 1;
    const u64 stride = (u64)gridDim.x * kBlock;
    for (u64 base = (u64)blockIdx.x * kBlock; base < p.n_in; base += stride) {
        const u64 r = base + threadIdx.x;
        u64 W[RW];
        uint32_t id = 0;
        unsigned int keep = 0;
        if (r < p.n_in) {
            load_record<RW, IDS>(p.pg, p.pg.in_pages[base >> p.pg.log_p], (uint32_t)(r & pmask), W, id);
            // empty output-chunk slots (all-zero records, v1 == v2) are dropped here
            const uint32_t ids = IDS ? id : (uint32_t)packed_ids(W[RW - 2], p.idb);
            const uint32_t ib = IDS ? (uint32_t)kIdBits : p.idb, im = (1u << ib) - 1;
            keep = (!HOLES || (ids & im) != ((ids >> ib) & im)) &&
                   (shard_hash<RW>(W, id) % p.shard_count) == p.shard_index;
        }
        const u64 off = block_reserve(keep, &p.sc->out_count, rs);
        if (keep) {
            if (off >= p.out_cap)
                p.sc->err = 1;
            else
                store_record<RW, IDS>(p.pg, p.out_off + off, W, id);
        }
    }
}

// ---------------------------------------------------------------------------- wide class
// Graphs with 512 < n <= 2015 (e.g. G(2000, 0.005), BASELINE configs[3]).  Count mode only.
// Records are array-of-structures, RW = NW + 1 words each: the blocked set B(p) in words
// 0..NW-1 (v1, v2, vt packed in the top 3*idb bits of word NW-1; NW is chosen so those bits
// are free) and keysum(p) in word NW.  One warp handles one path: lane w owns word w (NW <= 32),
// so a record is read and written as one coalesced 8*RW-byte line.  Adjacency rows (n*NW
// words, ~0.5 MB) are read through L1/L2 instead of shared memory.
__device__ __forceinline__ u64 *wide_rec(const Pages &pg, const uint32_t *pages, u64 r, int RW)
{
    return (u64 *)(pg.base + (u64)pages[r >> pg.log_p] * pg.page_bytes) +
           (r & ((1ull << pg.log_p) - 1)) * (u64)RW;
}

__global__ void __launch_bounds__(kBlock) k_stage1_wide(const LaunchArgs p)
{
    __shared__ ReserveSmem rs;
    const int n = p.g.n, NW = p.g.nw, RW = NW + 1;
    const u64 *__restrict__ adj = p.g.adj;
    const u64 *__restrict__ key = p.g.key;
    u64 cnt = 0, hs = 0;
    const u64 stride = (u64)gridDim.x * kBlock;
    for (u64 base = (u64)blockIdx.x * kBlock; base < p.n_in; base += stride) {
        const u64 r = base + threadIdx.x;
        unsigned int emit = 0;
        uint32_t x = 0, u = 0, y = 0;
        u64 h = 0;
        if (r < p.n_in) {
            const u64 gid = p.in_lo + r;
            int lo = 0, hi = n - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (p.g.pair_prefix[mid] <= gid)
                    lo = mid;
                else
                    hi = mid - 1;
            }
            u = (uint32_t)lo;
            const u64 q = gid - p.g.pair_prefix[u];
            u64 j = (u64)((1.0 + sqrt(1.0 + 8.0 * (double)q)) * 0.5);
            while (j * (j - 1) / 2 > q)
                --j;
            while ((j + 1) * j / 2 <= q)
                ++j;
            const u64 i = q - j * (j - 1) / 2;
            const uint32_t f = p.g.fwd[u];
            x = p.g.col[f + (uint32_t)i];
            y = p.g.col[f + (uint32_t)j];
            const bool tri = (__ldg(adj + (u64)x * NW + (y >> 6)) >> (y & 63)) & 1ull;
            if (tri) {
                if (p.count) {
                    cnt++;
                    hs += mix64(__ldg(key + x) + __ldg(key + u) + __ldg(key + y));
                }
            } else if (p.emit) {
                emit = 1;
                if (p.root_stride > 1) {
                    const u64 rkey = ((u64)p.g.orig[x] << 42) | ((u64)p.g.orig[u] << 21) | (u64)p.g.orig[y];
                    emit = (mix64(rkey) % p.root_stride) == p.root_offset;
                }
                if (emit && p.filter) {  // shard hash over the record words, as k_shard_filter_wide
                    h = mix64(0ull);
                    for (int w = 0; w < NW; ++w) {
                        u64 word = __ldg(adj + (u64)u * NW + w) | bit_in_word(w, u);
                        if (w == NW - 1)
                            word = with_packed_ids(word, pack3(x, u, y, p.idb), p.idb);
                        h = mix64(h ^ word);
                    }
                    h = mix64(h ^ (__ldg(key + x) + __ldg(key + u) + __ldg(key + y)));
                    emit = (h % p.shard_count) == p.shard_index;
                }
            }
        }
        const u64 off = block_reserve(emit, &p.sc->out_count, rs);
        if (emit) {
            if (off >= p.out_cap) {
                p.sc->err = 1;
            } else {
                u64 *rec = wide_rec(p.pg, p.pg.out_pages, p.out_off + off, RW);
                for (int w = 0; w < NW; ++w) {  // B(<x,u,y>) = N[u]
                    u64 word = __ldg(adj + (u64)u * NW + w) | bit_in_word(w, u);
                    if (w == NW - 1)
                        word = with_packed_ids(word, pack3(x, u, y, p.idb), p.idb);
                    rec[w] = word;
                }
                rec[NW] = __ldg(key + x) + __ldg(key + u) + __ldg(key + y);
            }
        }
    }
    flush_accum(cnt, hs, 0, p.sc);
}

constexpr int kWidePaths = 4;  // paths per warp per tile in k_expand_wide

constexpr int kWideVList = 256;  // child-vertex list per warp (children of one path)

__global__ void __launch_bounds__(kBlock) k_expand_wide(const LaunchArgs p)
{
    __shared__ ReserveSmem rs;
    __shared__ uint32_t s_vlist[(kBlock / 32) * kWideVList];
    const int NW = p.g.nw, RW = NW + 1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t idb = p.idb, idm = (1u << idb) - 1;
    const u64 *__restrict__ adj = p.g.adj;
    const u64 *__restrict__ key = p.g.key;
    const bool mine = lane < NW;  // this lane owns word `lane` of every record
    constexpr u64 kTilePaths = (u64)(kBlock / 32) * kWidePaths;
    u64 cnt = 0, hs = 0, cand = 0;
    for (u64 tb = (u64)blockIdx.x * kTilePaths; tb < p.n_in; tb += (u64)gridDim.x * kTilePaths) {
        u64 ext[kWidePaths], Cw[kWidePaths], ksv[kWidePaths];
        u64 v12v[kWidePaths], Bv[kWidePaths], KSv[kWidePaths];
        unsigned int ne = 0;
        // issue the loads of all the warp's records first (independent, in flight together)
#pragma unroll
        for (int i = 0; i < kWidePaths; ++i) {
            const u64 r = tb + (u64)wid * kWidePaths + i;
            Bv[i] = 0;
            KSv[i] = 0;
            if (r < p.n_in) {
                const u64 *rec = wide_rec(p.pg, p.pg.in_pages, r, RW);
                Bv[i] = mine ? rec[lane] : 0ull;
                KSv[i] = lane == 0 ? rec[NW] : 0ull;
            }
        }
#pragma unroll
        for (int i = 0; i < kWidePaths; ++i) {
            ext[i] = 0;
            Cw[i] = 0;
            ksv[i] = 0;
            v12v[i] = 0;
            const u64 r = tb + (u64)wid * kWidePaths + i;
            if (r >= p.n_in)
                continue;  // warp-uniform
            const u64 B = Bv[i];
            const u64 ks = __shfl_sync(FULL_MASK, KSv[i], 0);
            const u64 id = packed_ids(__shfl_sync(FULL_MASK, B, NW - 1), idb);
            const uint32_t v1 = (uint32_t)(id & idm), v2 = (uint32_t)((id >> idb) & idm),
                           vt = (uint32_t)(id >> (2 * idb));
            const u64 a = mine ? __ldg(adj + (u64)vt * NW + lane) : 0ull;
            const u64 a1 = mine ? __ldg(adj + (u64)v1 * NW + lane) : 0ull;
            const u64 c = a & above_word(v2, lane) & ~B;
            u64 close = c & a1;
            ext[i] = p.emit ? (c & ~a1) : 0ull;
            if (p.count) {
                cand += __popcll(a);
                cnt += __popcll(close);
                while (close) {
                    const int b = __ffsll((long long)close) - 1;
                    close &= close - 1;
                    hs += mix64(ks + __ldg(key + 64 * lane + b));
                }
            }
            ne += __reduce_add_sync(FULL_MASK, (unsigned int)__popcll(ext[i]));
            // the children's blocked set: vt becomes interior -> B | N[vt]
            Cw[i] = mine ? (B | a | bit_in_word(lane, vt)) : 0ull;
            ksv[i] = ks;
            v12v[i] = id & ((1ull << (2 * idb)) - 1);
        }
        // one reservation per CTA tile; the warp's count is carried by its lane 0
        const u64 off = __shfl_sync(FULL_MASK, block_reserve(lane == 0 ? ne : 0u, &p.sc->out_count, rs), 0);
        if (ne == 0)
            continue;
        if (off + ne > p.out_cap) {
            if (lane == 0)
                p.sc->err = 1;
            continue;
        }
        u64 o = p.out_off + off;
        uint32_t *sv = s_vlist + wid * kWideVList;
#pragma unroll
        for (int i = 0; i < kWidePaths; ++i) {
            // children of path i: every child record equals (B | N[vt]) except the packed-id word
            // (last vertex v) and the keysum word (ks + key(v)).  Lanes publish the child
            // vertices in order into this warp's list; then lane w writes the common word w of
            // all children (stride RW words) and lanes e write the keysum word of child e.
            const uint32_t pc = __popcll(ext[i]);
            unsigned int incl = pc;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned int t = __shfl_up_sync(FULL_MASK, incl, d);
                if (lane >= d)
                    incl += t;
            }
            const unsigned int E = __shfl_sync(FULL_MASK, incl, 31);
            if (E == 0)
                continue;
            if (E > kWideVList) {
                // very high fan-out (> kWideVList children of one path): one child at a time
                u64 m = ext[i];
                for (;;) {
                    const unsigned int has = __ballot_sync(FULL_MASK, m != 0ull);
                    if (!has)
                        break;
                    const int L = __ffs(has) - 1;
                    const int b = __shfl_sync(FULL_MASK, __ffsll((long long)m) - 1, L);
                    if (lane == L)
                        m &= m - 1;
                    const uint32_t v = (uint32_t)(64 * L + b);
                    u64 *rec = wide_rec(p.pg, p.pg.out_pages, o, RW);
                    if (mine)
                        rec[lane] = lane == NW - 1 ? with_packed_ids(Cw[i], v12v[i] | ((u64)v << (2 * idb)), idb) : Cw[i];
                    if (lane == 0)
                        rec[NW] = ksv[i] + __ldg(key + v);
                    ++o;
                }
                continue;
            }
            {
                u64 m = ext[i];
                unsigned int pos = incl - pc;
                while (m) {
                    const int b = __ffsll((long long)m) - 1;
                    m &= m - 1;
                    sv[pos++] = (uint32_t)(64 * lane + b);
                }
            }
            __syncwarp();
            const uint32_t pg_mask = (1u << p.pg.log_p) - 1;
            const uint32_t slot0 = (uint32_t)(o & pg_mask);
            if (slot0 + E <= pg_mask + 1) {
                // all E children in one page: plain strided stores, one loop for every lane
                u64 *rec0 = wide_rec(p.pg, p.pg.out_pages, o, RW);
                if (mine) {
                    const bool idw = lane == NW - 1;
                    u64 *q = rec0 + lane;
                    for (unsigned int e = 0; e < E; ++e, q += RW)
                        *q = idw ? with_packed_ids(Cw[i], v12v[i] | ((u64)sv[e] << (2 * idb)), idb) : Cw[i];
                }
                for (unsigned int e = lane; e < E; e += 32)
                    rec0[(u64)e * RW + NW] = ksv[i] + __ldg(key + sv[e]);
            } else {
                for (unsigned int e = 0; e < E; ++e) {
                    u64 *rec = wide_rec(p.pg, p.pg.out_pages, o + e, RW);
                    if (mine)
                        rec[lane] = lane == NW - 1 ? with_packed_ids(Cw[i], v12v[i] | ((u64)sv[e] << (2 * idb)), idb) : Cw[i];
                    if (lane == 0)
                        rec[NW] = ksv[i] + __ldg(key + sv[e]);
                }
            }
            o += E;
            __syncwarp();
        }
    }
    if (!p.count)
        cand = 0;
    flush_accum(cnt, hs, cand, p.sc);
}

// Last-level fusion for the wide class (p.emit && !p.emit_next, see Scratch): F_t is read and
// its own closures counted as in k_expand_wide; its children <p,v> (v in Ext(p)) are counted
// and their closures found, but nothing is written.  Close(<p,v>) = Adj(v) & Z(p), counted the
// other way round: for each closer z in Z(p) = {x > v2} & ~(B | N[vt]) & Adj(v1) (few: inside
// Adj(v1)), one coalesced read of row z, AND Ext(p), gives every child closing through z.
// Latency-bound code, so the work is phased: one warp takes kLeafPaths paths, issues all their
// row reads before using any, then lists every (path, z) pair and reads those rows in batches.
// No block-level synchronisation: warps run independently.
constexpr int kLeafPaths = 4;
constexpr int kLeafPairs = 128;  // (path, closer) pairs listed per warp and round
constexpr int kLeafBatch = 8;    // closer rows in flight per lane

__global__ void __launch_bounds__(kBlock) k_leaf_wide(const LaunchArgs p)
{
    __shared__ uint16_t s_deg[2048];  // deg(v), n <= 2015
    __shared__ uint32_t s_pair[(kBlock / 32) * kLeafPairs];
    const int NW = p.g.nw, RW = NW + 1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t idb = p.idb, idm = (1u << idb) - 1;
    const u64 *__restrict__ adj = p.g.adj;
    const u64 *__restrict__ key = p.g.key;
    const bool mine = lane < NW;  // this lane owns word `lane` of every row / record
    for (int v = threadIdx.x; v < p.g.n; v += kBlock)
        s_deg[v] = (uint16_t)(p.g.rowptr[v + 1] - p.g.rowptr[v]);
    __syncthreads();
    uint32_t *pair = s_pair + wid * kLeafPairs;
    const bool nbm = p.g.nbrmask != nullptr;
    u64 cnt = 0, hs = 0, cand = 0, lpaths = 0, lcand = 0, lcyc = 0;
    const u64 nwarps = (u64)gridDim.x * (kBlock / 32);
    for (u64 r0 = ((u64)blockIdx.x * (kBlock / 32) + wid) * kLeafPaths; r0 < p.n_in; r0 += nwarps * kLeafPaths) {
        u64 B[kLeafPaths], KS[kLeafPaths], a[kLeafPaths], a1[kLeafPaths];
        uint32_t v2v[kLeafPaths], vtv[kLeafPaths];
        // phase A: the records
#pragma unroll
        for (int i = 0; i < kLeafPaths; ++i) {
            B[i] = 0;
            KS[i] = 0;
            if (r0 + i < p.n_in) {
                const u64 *rec = wide_rec(p.pg, p.pg.in_pages, r0 + i, RW);
                B[i] = mine ? rec[lane] : 0ull;
                KS[i] = lane == 0 ? rec[NW] : 0ull;
            }
        }
        // phase B: rows Adj(vt), Adj(v1) of every path, all in flight together
#pragma unroll
        for (int i = 0; i < kLeafPaths; ++i) {
            KS[i] = __shfl_sync(FULL_MASK, KS[i], 0);
            const u64 id = packed_ids(__shfl_sync(FULL_MASK, B[i], NW - 1), idb);
            const uint32_t v1 = (uint32_t)(id & idm);
            v2v[i] = (uint32_t)((id >> idb) & idm);
            vtv[i] = (uint32_t)(id >> (2 * idb));
            const bool ok = r0 + i < p.n_in && mine;
            a[i] = ok ? __ldg(adj + (u64)vtv[i] * NW + lane) : 0ull;
            a1[i] = ok ? __ldg(adj + (u64)v1 * NW + lane) : 0ull;
        }
        // phase C: Cand/Close/Ext of each path (its own closures: cycles of t+1 vertices), the
        // children's statistics, and the (path, closer) pair list
        u64 ext[kLeafPaths];
        uint32_t extm[kLeafPaths], rowb[kLeafPaths];  // mask path: Ext(p) over the CSR row of vt
        unsigned int np = 0;
#pragma unroll
        for (int i = 0; i < kLeafPaths; ++i) {
            const u64 abv = above_word(v2v[i], lane);
            const u64 c = a[i] & abv & ~B[i];
            u64 close = c & a1[i];
            ext[i] = c & ~a1[i];
            if (p.count) {
                cand += __popcll(a[i]);
                cnt += __popcll(close);
                while (close) {
                    const int b = __ffsll((long long)close) - 1;
                    close &= close - 1;
                    hs += mix64(KS[i] + __ldg(key + 64 * lane + b));
                }
                if (!nbm) {
                    u64 m = ext[i];
                    lpaths += __popcll(m);
                    while (m) {  // candidate slots of the children: deg(v)
                        const int b = __ffsll((long long)m) - 1;
                        m &= m - 1;
                        lcand += s_deg[64 * lane + b];
                    }
                }
            }
            if (nbm) {
                // Ext(p) as a mask over the CSR row of vt: lane k tests its neighbour v_k
                rowb[i] = p.g.rowptr[vtv[i]];
                const uint32_t dt = s_deg[vtv[i]];
                const uint32_t vk = (uint32_t)lane < dt ? p.g.col[rowb[i] + lane] : 0u;
                const u64 wv = __shfl_sync(FULL_MASK, ext[i], (int)(vk >> 6));
                const bool eb = (uint32_t)lane < dt && ((wv >> (vk & 63)) & 1ull);
                extm[i] = __ballot_sync(FULL_MASK, eb);
                if (p.count) {
                    lpaths += eb ? 1u : 0u;
                    lcand += eb ? s_deg[vk] : 0u;
                }
            } else {
                extm[i] = 0;
                rowb[i] = 0;
            }
            const bool anyext = __any_sync(FULL_MASK, ext[i] != 0ull);
            // Z(p) = {x > v2} & ~(B | N[vt]) & Adj(v1), vt in B
            u64 zm = (anyext && mine) ? (abv & ~(B[i] | a[i]) & a1[i]) : 0ull;
            const unsigned int pz = __popcll(zm);
            unsigned int incl = pz;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned int t = __shfl_up_sync(FULL_MASK, incl, d);
                if (lane >= d)
                    incl += t;
            }
            unsigned int pos = np + incl - pz;
            while (zm) {
                const int b = __ffsll((long long)zm) - 1;
                zm &= zm - 1;
                if (pos < (unsigned int)kLeafPairs)
                    pair[pos] = ((uint32_t)i << 12) | (uint32_t)(64 * lane + b);
                ++pos;
            }
            np += __shfl_sync(FULL_MASK, incl, 31);
        }
        __syncwarp();
        if (p.count && nbm) {
            // phase D (Delta <= 32): lane-parallel over the (path, z) pairs; the children of p
            // closing through z are nbrmask[vt][z] & Ext(p), one 4-byte read per pair
            for (unsigned int q0 = 0; q0 < np; q0 += kLeafPairs) {
                if (q0 > 0) {
                    // (rare) more pairs than the list holds: rebuild the next window
                    __syncwarp();
                    unsigned int seen = 0;
#pragma unroll
                    for (int i = 0; i < kLeafPaths; ++i) {
                        const bool anyext = __any_sync(FULL_MASK, ext[i] != 0ull);
                        u64 zm = (anyext && mine) ? (above_word(v2v[i], lane) & ~(B[i] | a[i]) & a1[i]) : 0ull;
                        const unsigned int pz = __popcll(zm);
                        unsigned int incl = pz;
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const unsigned int t = __shfl_up_sync(FULL_MASK, incl, d);
                            if (lane >= d)
                                incl += t;
                        }
                        unsigned int pos = seen + incl - pz;
                        while (zm) {
                            const int b = __ffsll((long long)zm) - 1;
                            zm &= zm - 1;
                            if (pos >= q0 && pos < q0 + kLeafPairs)
                                pair[pos - q0] = ((uint32_t)i << 12) | (uint32_t)(64 * lane + b);
                            ++pos;
                        }
                        seen += __shfl_sync(FULL_MASK, incl, 31);
                    }
                    __syncwarp();
                }
                const unsigned int nq = min(np - q0, (unsigned int)kLeafPairs);
                for (unsigned int q = lane; q < nq; q += 32) {
                    const uint32_t e = pair[q];
                    const uint32_t i = e >> 12, z = e & 0xfffu;
                    uint32_t em = extm[0], vt = vtv[0], rb = rowb[0];
                    u64 ks = KS[0];
#pragma unroll
                    for (int j = 1; j < kLeafPaths; ++j) {
                        em = i == (uint32_t)j ? extm[j] : em;
                        vt = i == (uint32_t)j ? vtv[j] : vt;
                        rb = i == (uint32_t)j ? rowb[j] : rb;
                        ks = i == (uint32_t)j ? KS[j] : ks;
                    }
                    uint32_t m = __ldg(p.g.nbrmask + (u64)vt * p.g.n + z) & em;
                    if (m) {
                        lcyc += __popc(m);
                        const u64 kz = ks + __ldg(key + z);
                        while (m) {
                            const int k = __ffs(m) - 1;
                            m &= m - 1;
                            hs += mix64(kz + __ldg(key + __ldg(p.g.col + rb + k)));
                        }
                    }
                }
            }
        } else if (p.count) {
            // phase D: closer rows in batches of kLeafBatch, all loads of a batch in flight
            for (unsigned int q0 = 0; q0 < np; q0 += kLeafBatch) {
                if (q0 > 0 && q0 % kLeafPairs == 0) {
                    // (rare) more pairs than the list holds: rebuild the next window
                    __syncwarp();
                    unsigned int seen = 0;
#pragma unroll
                    for (int i = 0; i < kLeafPaths; ++i) {
                        const bool anyext = __any_sync(FULL_MASK, ext[i] != 0ull);
                        u64 zm = (anyext && mine) ? (above_word(v2v[i], lane) & ~(B[i] | a[i]) & a1[i]) : 0ull;
                        const unsigned int pz = __popcll(zm);
                        unsigned int incl = pz;
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const unsigned int t = __shfl_up_sync(FULL_MASK, incl, d);
                            if (lane >= d)
                                incl += t;
                        }
                        unsigned int pos = seen + incl - pz;
                        while (zm) {
                            const int b = __ffsll((long long)zm) - 1;
                            zm &= zm - 1;
                            if (pos >= q0 && pos < q0 + kLeafPairs)
                                pair[pos - q0] = ((uint32_t)i << 12) | (uint32_t)(64 * lane + b);
                            ++pos;
                        }
                        seen += __shfl_sync(FULL_MASK, incl, 31);
                    }
                    __syncwarp();
                }
                const uint32_t *pw = pair + (q0 % kLeafPairs);
                u64 row[kLeafBatch];
                uint32_t e[kLeafBatch];
#pragma unroll
                for (int k = 0; k < kLeafBatch; ++k) {
                    e[k] = q0 + k < np ? pw[k] : 0xffffffffu;
                    row[k] = (e[k] != 0xffffffffu && mine) ? __ldg(adj + (u64)(e[k] & 0xfffu) * NW + lane) : 0ull;
                }
#pragma unroll
                for (int k = 0; k < kLeafBatch; ++k) {
                    if (e[k] == 0xffffffffu)
                        break;  // warp-uniform
                    const uint32_t i = e[k] >> 12, z = e[k] & 0xfffu;
                    u64 ex = ext[0], ks = KS[0];
#pragma unroll
                    for (int j = 1; j < kLeafPaths; ++j) {
                        ex = i == (uint32_t)j ? ext[j] : ex;
                        ks = i == (uint32_t)j ? KS[j] : ks;
                    }
                    u64 cl = row[k] & ex;
                    if (cl) {
                        lcyc += __popcll(cl);
                        const u64 kz = ks + __ldg(key + z);
                        while (cl) {
                            const int b = __ffsll((long long)cl) - 1;
                            cl &= cl - 1;
                            hs += mix64(kz + __ldg(key + 64 * lane + b));
                        }
                    }
                }
            }
        }
        __syncwarp();
    }
    if (!p.count)
        cand = 0;
    Acc acc;
    acc.cyc = cnt;
    acc.hash = hs;
    acc.cand = cand;
    acc.cyc_next = lcyc;
    acc.cand_next = lcand;
    acc.paths_next = lpaths;
    flush(acc, p.sc);
}

__global__ void __launch_bounds__(kBlock) k_shard_filter_wide(const LaunchArgs p)
{
    __shared__ ReserveSmem rs;
    const int NW = p.g.nw, RW = NW + 1;
    const u64 stride = (u64)gridDim.x * kBlock;
    for (u64 base = (u64)blockIdx.x * kBlock; base < p.n_in; base += stride) {
        const u64 r = base + threadIdx.x;
        unsigned int keep = 0;
        const u64 *src = nullptr;
        if (r < p.n_in) {
            src = wide_rec(p.pg, p.pg.in_pages, r, RW);
            u64 h = mix64(0ull);
            for (int w = 0; w < RW; ++w)
                h = mix64(h ^ src[w]);
            keep = (h % p.shard_count) == p.shard_index;
        }
        const u64 off = block_reserve(keep, &p.sc->out_count, rs);
        if (keep) {
            if (off >= p.out_cap) {
                p.sc->err = 1;
            } else {
                u64 *dst = wide_rec(p.pg, p.pg.out_pages, p.out_off + off, RW);
                for (int w = 0; w < RW; ++w)
                    dst[w] = src[w];
            }
        }
    }
}

// ---------------------------------------------------------------------------- list class
// Sparse wide graphs (count mode, 512 < n <= 2015, Delta <= 32, max_len <= 14).  A path is its
// vertex list v1..vt (16-bit ids, four per word: RWL words), one word holding Y(p), and
// keysum(p): 32 B for t <= 8 instead of a 2000-bit blocked set.  One thread per path.  With
// the neighbour-mask table T = nbrmask (bit k of T[u][z] = "k-th neighbour of u is adjacent
// to z"), the test of Alg. 3 lines 11-14 becomes 32-bit masks over CSR rows:
//   over the row of vt (candidates v_k = col[row(vt) + k]):
//     blocked = OR over the interior vertices x = v2..v_{t-1} of T[vt][x]   (v in B(p))
//     Ext     = valid & {k : v_k > v2} & ~blocked & ~T[vt][v1]
//   (open rows suffice: the only path vertex in Adj(vt) is v_{t-1}, adjacent to the interior
//   v_{t-2}, or v2 itself when t = 3, which fails the gate);
//   over the row of v1 (the possible closing vertices w_k = col[row(v1) + k]), carried in the
//   record and updated with one read per extension:
//     Y(p)    = {k : w_k > v2} & ~{k : w_k in B(p)}        Y(<x,u,y>) = gate & ~T[x][u]
//     Close(p) = Y(p) & T[v1][vt]                          (w ~ vt closes the cycle)
//     Y(<p,v>) = Y(p) & ~T[v1][vt]                         (B grows by N[vt])
// Last-level fusion: child v of p closes through Y(<p,v>) & T[v1][v], one read per child.
__device__ __forceinline__ uint32_t list_id(const u64 *W, int i)
{
    return (uint32_t)(W[i >> 2] >> (16 * (i & 3))) & 0xffffu;
}

// number of entries <= x in the sorted row col[b .. b+d)
__device__ __forceinline__ uint32_t row_rank(const uint32_t *col, uint32_t b, uint32_t d, uint32_t x)
{
    uint32_t lo = 0, hi = d;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(col + b + mid) <= x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t low_mask(uint32_t k)  // bits 0..k-1 (k <= 32)
{
    return k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
}

// Collect mode, list class: store the cycle <v1 .. vt, a[, b]> (the path's list, then the closing
// vertices; b = 0xffff: none) at index idx.  The list order is the canonical sequence of
// PAPER.md:45-51 (v1, v2 = the minimum label, v3, ...), the same one the bitmap walk of
// k_cycle_sequences produces.  Word positions are unrolled: no dynamically indexed registers.
template <int RWL, int RW>
__device__ __forceinline__ void store_cycle_list(const CycleStore &c, const u64 (&W)[RW], int t, uint32_t a,
                                                 uint32_t b, u64 idx)
{
    constexpr int LW = RWL + 1;
    if (idx >= c.cap)
        return;
#pragma unroll
    for (int w = 0; w < LW; ++w) {
        u64 x = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int pos = 4 * w + j;
            const uint32_t id = pos < 4 * RWL && pos < t ? list_id(W, pos < 4 * RWL ? pos : 0)
                                : pos == t           ? a
                                : pos == t + 1       ? b
                                                     : 0xffffu;
            x |= (u64)id << (16 * j);
        }
        c.s[(u64)w * c.cap + idx] = x;
    }
}

#ifndef CC_LIST_BLOCK
#define CC_LIST_BLOCK 512
#endif
constexpr int kListBlock = CC_LIST_BLOCK;  // threads per CTA of the list kernels

template <int RWL, bool COL>
__global__ void __launch_bounds__(kListBlock) k_stage1_list(const LaunchArgs p)
{
    constexpr int RW = RWL + 2;
    __shared__ ReserveSmemT<kListBlock> rs;
    const int n = p.g.n, NW = p.g.nw;
    const u64 *__restrict__ adj = p.g.adj;
    const u64 *__restrict__ key = p.g.key;
    u64 cnt = 0, hs = 0;
    const u64 stride = (u64)gridDim.x * kListBlock;
    for (u64 base = (u64)blockIdx.x * kListBlock; base < p.n_in; base += stride) {
        const u64 r = base + threadIdx.x;
        unsigned int emit = 0;
        u64 W[RW];
#pragma unroll
        for (int w = 0; w < RW; ++w)
            W[w] = 0;
        if (r < p.n_in) {
            const u64 gid = p.in_lo + r;
            int lo = 0, hi = n - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (p.g.pair_prefix[mid] <= gid)
                    lo = mid;
                else
                    hi = mid - 1;
            }
            const uint32_t u = (uint32_t)lo;
            const u64 q = gid - p.g.pair_prefix[u];
            u64 j = (u64)((1.0 + sqrt(1.0 + 8.0 * (double)q)) * 0.5);
            while (j * (j - 1) / 2 > q)
                --j;
            while ((j + 1) * j / 2 <= q)
                ++j;
            const u64 i = q - j * (j - 1) / 2;
            const uint32_t f = p.g.fwd[u];
            const uint32_t x = p.g.col[f + (uint32_t)i];
            const uint32_t y = p.g.col[f + (uint32_t)j];  // u < x < y (Alg. 2 l.12)
            const bool tri = (__ldg(adj + (u64)x * NW + (y >> 6)) >> (y & 63)) & 1ull;
            if (tri) {
                if (p.count) {
                    cnt++;
                    hs += mix64(__ldg(key + x) + __ldg(key + u) + __ldg(key + y));
                    if constexpr (COL) {  // the triangle <x, u, y> (Alg. 2 l.14)
                        u64 T3[RW];
#pragma unroll
                        for (int w = 0; w < RW; ++w)
                            T3[w] = 0;
                        T3[0] = (u64)x | ((u64)u << 16);
                        store_cycle_list<RWL>(p.cyc, T3, 2, y, 0xffffu, atomicAdd(p.cyc.count, 1ull));
                    }
                }
            } else if (p.emit) {
                emit = 1;
                if (p.root_stride > 1) {
                    const u64 rkey = ((u64)p.g.orig[x] << 42) | ((u64)p.g.orig[u] << 21) | (u64)p.g.orig[y];
                    emit = (mix64(rkey) % p.root_stride) == p.root_offset;
                }
                W[0] = (u64)x | ((u64)u << 16) | ((u64)y << 32);  // <x, u, y>
                // Y(<x,u,y>) over the row of x: w > u and w not in N[u] (u itself fails w > u)
                const uint32_t bx = __ldg(p.g.rowptr + x), dx = __ldg(p.g.rowptr + x + 1) - bx;
                W[RWL] = low_mask(dx) & ~low_mask(row_rank(p.g.col, bx, dx, u)) &
                         ~__ldg(p.g.nbrmask + (u64)x * n + u);
                W[RWL + 1] = __ldg(key + x) + __ldg(key + u) + __ldg(key + y);
                if (emit && p.filter)
                    emit = (shard_hash<RW>(W, 0) % p.shard_count) == p.shard_index;
            }
        }
        const u64 off = block_reserve<kListBlock>(emit, &p.sc->out_count, rs);
        if (emit) {
            if (off >= p.out_cap)
                p.sc->err = 1;
            else
                store_record<RW, false>(p.pg, p.out_off + off, W, 0);
        }
    }
    flush_accum<kListBlock>(cnt, hs, 0, p.sc);
}

template <int RWL, bool LEAF, bool COL>
__global__ void __launch_bounds__(kListBlock) k_expand_list(const LaunchArgs p)
{
    constexpr int RW = RWL + 2;
    __shared__ ReserveSmemT<kListBlock> rs;
    __shared__ uint16_t s_deg[2048];
    const int t = (int)p.tlen;
    const uint32_t n = (uint32_t)p.g.n;
    const uint32_t *__restrict__ T = p.g.nbrmask;
    const uint32_t *__restrict__ col = p.g.col;
    const uint32_t *__restrict__ rowptr = p.g.rowptr;
    const u64 *__restrict__ key = p.g.key;
    for (uint32_t v = threadIdx.x; v < n; v += kListBlock)
        s_deg[v] = (uint16_t)(rowptr[v + 1] - rowptr[v]);
    __syncthreads();
    const u64 pmask = (1ull << p.pg.log_p) - 1;
    u64 cnt = 0, hs = 0, cand = 0, lpaths = 0, lcand = 0, lcyc = 0;
    const u64 stride = (u64)gridDim.x * kListBlock;
    for (u64 base = (u64)blockIdx.x * kListBlock; base < p.n_in; base += stride) {
        const u64 r = base + threadIdx.x;
        u64 W[RW];
        uint32_t ext = 0, rb = 0, Yc = 0;
        if (r < p.n_in) {
            const char *pp = page_ptr(p.pg, p.pg.in_pages[r >> p.pg.log_p]);
            const u64 slot = r & pmask;
#pragma unroll
            for (int w = 0; w < RW; ++w)
                W[w] = ((const u64 *)pp)[((u64)w << p.pg.log_p) + slot];
            // (positions unrolled so that W stays in registers)
            const uint32_t v1 = list_id(W, 0), v2 = list_id(W, 1);
            uint32_t vt;
            {
                const int q = t - 1;  // word q / 4, lane q % 4 (scalar selects: no local memory)
                const u64 wq = q < 4 ? W[0] : (q < 8 || RWL < 3 ? W[1] : W[RWL - 1]);
                vt = (uint32_t)(wq >> (16 * (q & 3))) & 0xffffu;
            }
            const uint32_t Y = (uint32_t)W[RWL];
            const u64 ks = W[RWL + 1];
            const u64 t1 = (u64)v1 * n;
            const uint32_t tv = __ldg(T + t1 + vt);  // closers adjacent to vt
            uint32_t close = Y & tv;
            Yc = Y & ~tv;
            uint32_t rb1 = 0;
            if (close || (LEAF && Yc))
                rb1 = __ldg(rowptr + v1);
            if (p.count && close) {
                cnt += __popc(close);
                u64 idx = COL ? atomicAdd(p.cyc.count, (u64)__popc(close)) : 0ull;
                while (close) {
                    const int k = __ffs(close) - 1;
                    close &= close - 1;
                    const uint32_t z = __ldg(col + rb1 + k);
                    hs += mix64(ks + __ldg(key + z));
                    if constexpr (COL)
                        store_cycle_list<RWL>(p.cyc, W, t, z, 0xffffu, idx++);
                }
            }
            rb = __ldg(rowptr + vt);
            const uint32_t dt = s_deg[vt];
            if (p.count)
                cand += dt;
            if (p.emit) {
                const u64 trow = (u64)vt * n;
                uint32_t blocked = __ldg(T + trow + v1);  // candidates adjacent to v1 close, not extend
#pragma unroll
                for (int q = 1; q < 4 * RWL; ++q)
                    if (q < t - 1)
                        blocked |= __ldg(T + trow + list_id(W, q));
                ext = low_mask(dt) & ~low_mask(row_rank(col, rb, dt, v2)) & ~blocked;
            }
            if (LEAF) {
                if (ext && p.count) {
                    uint32_t m = ext;
                    while (m) {
                        const int k = __ffs(m) - 1;
                        m &= m - 1;
                        const uint32_t v = __ldg(col + rb + k);
                        lpaths++;
                        lcand += s_deg[v];
                        uint32_t c2 = Yc ? (__ldg(T + t1 + v) & Yc) : 0u;
                        if (c2) {
                            lcyc += __popc(c2);
                            const u64 kv = ks + __ldg(key + v);
                            u64 idx = COL ? atomicAdd(p.cyc.count, (u64)__popc(c2)) : 0ull;
                            while (c2) {
                                const int j = __ffs(c2) - 1;
                                c2 &= c2 - 1;
                                const uint32_t z = __ldg(col + rb1 + j);
                                hs += mix64(kv + __ldg(key + z));
                                if constexpr (COL)
                                    store_cycle_list<RWL>(p.cyc, W, t, v, z, idx++);
                            }
                        }
                    }
                }
                ext = 0;
            }
        }
        // the last level writes nothing: skip the reservation and its barriers.  (Measured per
        // instantiation: with RWL = 3 the shorter loop compiles to 49 registers -- 2 CTAs per SM
        // instead of 3 -- and runs 35% slower, so that variant keeps the uniform loop.)
        if constexpr (LEAF && RWL == 2)
            continue;
        const unsigned int ne = __popc(ext);
        const u64 off = block_reserve<kListBlock>(ne, &p.sc->out_count, rs);
        // children <p, v>: the parent's list with v appended, Y(<p,v>), keysum + key(v).  The
        // warp's children fill [warp_base, warp_base + warp_total) round-robin -- round c holds
        // the c-th child of every lane that has one, at consecutive positions -- so each store
        // instruction writes consecutive records (coalesced) instead of one run per lane.
        const int lane = threadIdx.x & 31;
        const u64 wbase = __shfl_sync(FULL_MASK, off, 0);
        const unsigned int wtot = __reduce_add_sync(FULL_MASK, ne);
        if (wtot) {
            if (lane == 0 && wbase + wtot > p.out_cap)
                p.sc->err = 1;
            if (wbase + wtot <= p.out_cap) {
                const int wv = t >> 2, sh = 16 * (t & 3);
                u64 o = p.out_off + wbase;
                uint32_t m = ext;
                for (;;) {
                    const unsigned int has = __ballot_sync(FULL_MASK, m != 0u);
                    if (!has)
                        break;
                    if (m) {
                        const int k = __ffs(m) - 1;
                        m &= m - 1;
                        const uint32_t v = __ldg(col + rb + k);
                        u64 C[RW];
#pragma unroll
                        for (int w = 0; w < RWL; ++w)
                            C[w] = W[w] | (w == wv ? (u64)v << sh : 0ull);
                        C[RWL] = Yc;
                        C[RWL + 1] = W[RWL + 1] + __ldg(key + v);
                        store_record<RW, false>(p.pg, o + __popc(has & ((1u << lane) - 1u)), C, 0);
                    }
                    o += __popc(has);
                }
            }
        }
    }
    if (!p.count)
        cand = 0;
    Acc acc;
    acc.cyc = cnt;
    acc.hash = hs;
    acc.cand = cand;
    acc.cyc_next = lcyc;
    acc.cand_next = lcand;
    acc.paths_next = lpaths;
    flush<kListBlock>(acc, p.sc);
}

// ---------------------------------------------------------------------------- keys, collect
// nbrmask[u*n + z] |= 1 << k for the k-th neighbour w of u and every z ~ w (one warp per u;
// lane k < deg(u) <= 32 owns neighbour k)
__global__ void k_build_nbrmask(const DevGraph g, uint32_t *T)
{
    const int u = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), k = threadIdx.x & 31;
    if (u >= g.n)
        return;
    const uint32_t b = g.rowptr[u], d = g.rowptr[u + 1] - b;
    if ((uint32_t)k >= d)
        return;
    const uint32_t w = g.col[b + k];
    for (uint32_t q = g.rowptr[w]; q < g.rowptr[w + 1]; ++q)
        atomicOr(T + (u64)u * g.n + g.col[q], 1u << k);
}

__global__ void k_keys(u64 *key, const int32_t *orig, int n, u64 seed)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        key[i] = mix64(seed ^ (u64)(uint32_t)orig[i]);
}

// keybyte[j][b] = sum over the set bits i of b of key(8j + i)   (vertices >= n contribute 0)
__global__ void k_keybyte(u64 *keybyte, const u64 *key, int n)
{
    const int j = blockIdx.x, b = threadIdx.x;
    u64 s = 0;
    for (int i = 0; i < 8; ++i)
        if (((b >> i) & 1) && 8 * j + i < n)
            s += key[8 * j + i];
    keybyte[(j << 8) + b] = s;
}


// Offsets of the fetched cycles on the device: off[i] = sum of the lengths of cycles first ..
// first+i-1 (off[count] = total).  Three passes: per-1024-block exclusive scans with block sums,
// one block scanning the block sums, then the block prefixes added.
constexpr int kScanBlock = 1024;

__device__ __forceinline__ uint32_t cycle_length(const CycleStore &c, int nw, u64 i)
{
    uint32_t k = 0;
    if (c.lw) {  // list format: used 16-bit slots
        for (uint32_t w = 0; w < c.lw; ++w) {
            const u64 x = c.s[(u64)w * c.cap + i];
            for (int j = 0; j < 4; ++j)
                k += ((x >> (16 * j)) & 0xffffu) != 0xffffu;
        }
    } else {
        for (int w = 0; w < nw; ++w)
            k += __popcll(c.s[(u64)w * c.cap + i]);
    }
    return k;
}

__global__ void __launch_bounds__(kScanBlock) k_cycle_scan_blocks(const CycleStore c, int nw, uint64_t first,
                                                                  uint64_t count, u64 *off, u64 *blk)
{
    __shared__ u64 ws[kScanBlock / 32];
    const u64 i = (u64)blockIdx.x * kScanBlock + threadIdx.x;
    u64 k = 0;
    if (i < count)
        k = cycle_length(c, nw, first + i);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u64 incl = k;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u64 v = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= o)
            incl += v;
    }
    if (lane == 31)
        ws[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        u64 x = ws[lane];
        u64 xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u64 v = __shfl_up_sync(FULL_MASK, xi, o);
            if (lane >= o)
                xi += v;
        }
        ws[lane] = xi - x;
        if (lane == 31)
            blk[blockIdx.x] = xi;
    }
    __syncthreads();
    if (i < count)
        off[i] = ws[wid] + incl - k;
}

__global__ void __launch_bounds__(kScanBlock) k_cycle_scan_tops(u64 *blk, uint64_t nblk, u64 *total)
{
    // one block: exclusive scan of nblk block sums, kScanBlock at a time
    __shared__ u64 ws[kScanBlock / 32];
    __shared__ u64 carry;
    if (threadIdx.x == 0)
        carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (u64 b = 0; b < nblk; b += kScanBlock) {
        const u64 i = b + threadIdx.x;
        const u64 k = i < nblk ? blk[i] : 0;
        u64 incl = k;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u64 v = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o)
                incl += v;
        }
        if (lane == 31)
            ws[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            u64 x = ws[lane], xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u64 v = __shfl_up_sync(FULL_MASK, xi, o);
                if (lane >= o)
                    xi += v;
            }
            ws[lane] = xi - x;
        }
        __syncthreads();
        const u64 c0 = carry;
        if (i < nblk)
            blk[i] = c0 + ws[wid] + incl - k;
        __syncthreads();
        if (threadIdx.x == kScanBlock - 1)
            carry = c0 + ws[wid] + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0)
        *total = carry;
}

__global__ void k_cycle_scan_add(u64 *off, const u64 *blk, uint64_t count, const u64 *total)
{
    const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count)
        off[i] += blk[i / kScanBlock];
    else if (i == count)
        off[count] = *total;
}

cudaError_t launch_cycle_offsets(const CycleStore &c, int nw, uint64_t first, uint64_t count, u64 *off, u64 *blk,
                                 cudaStream_t st)
{
    if (count == 0)
        return cudaSuccess;
    const u64 nblk = (count + kScanBlock - 1) / kScanBlock;
    k_cycle_scan_blocks<<<(unsigned int)nblk, kScanBlock, 0, st>>>(c, nw, first, count, off, blk);
    k_cycle_scan_tops<<<1, kScanBlock, 0, st>>>(blk, nblk, blk + nblk);
    k_cycle_scan_add<<<(unsigned int)((count + 256) / 256), 256, 0, st>>>(off, blk, count, blk + nblk);
    return cudaGetLastError();
}

// Walk the induced cycle S from v1 -> v2 -> ...: each vertex of a chordless cycle has exactly
// two neighbours in S, so the successor of cur is the neighbour in S other than prev.
__global__ void k_cycle_sequences(const CycleStore c, int nw, const u64 *adj, const int32_t *orig,
                                  uint64_t first, uint64_t count, const u64 *offsets, int32_t *out)
{
    const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count)
        return;
    if (c.lw) {  // list format: the stored order is the canonical sequence
        u64 o = offsets[i];
        for (uint32_t w = 0; w < c.lw; ++w) {
            const u64 x = c.s[(u64)w * c.cap + first + i];
            for (int j = 0; j < 4; ++j) {
                const uint32_t v = (uint32_t)(x >> (16 * j)) & 0xffffu;
                if (v != 0xffffu)
                    out[o++] = orig[v];
            }
        }
        return;
    }
    const uint32_t id = c.ids[first + i];
    uint32_t prev = id & kIdMask, cur = (id >> kIdBits) & kIdMask;
    const u64 o = offsets[i], k = offsets[i + 1] - offsets[i];
    out[o] = orig[prev];
    if (k > 1)
        out[o + 1] = orig[cur];
    for (u64 j = 2; j < k; ++j) {
        uint32_t nxt = 0;
        for (int w = 0; w < nw; ++w) {
            u64 x = adj[(u64)cur * nw + w] & c.s[(u64)w * c.cap + first + i];
            if (w == (int)(prev >> 6))
                x &= ~(1ull << (prev & 63));
            if (x) {
                nxt = (uint32_t)(w * 64 + __ffsll((long long)x) - 1);
                break;
            }
        }
        out[o + j] = orig[nxt];
        prev = cur;
        cur = nxt;
    }
}

// ---------------------------------------------------------------------------- launchers
#define CC_CASES(MAC) MAC(1) MAC(2) MAC(3) MAC(4) MAC(5) MAC(6) MAC(7) MAC(8)

static inline size_t graph_smem(const LaunchArgs &a)
{
    const size_t kb = a.g.nw <= kByteTableWords ? (size_t)8 * a.g.nw * 256 : 0;
    return ((size_t)a.g.n * (a.g.nw + 1) + kb) * sizeof(u64);
}

static size_t blocked_ring_bytes(int nw, bool packed)
{
    switch (nw) {
#define RB(N) case N: return (size_t)kStages * (packed ? blocked_stage_bytes<N, true>() : blocked_stage_bytes<N, false>());
        CC_CASES(RB)
#undef RB
    }
    return 0;
}

// dynamic shared memory of the expansion kernel for (mode, nw, n, packed)
size_t expand_smem(Mode m, int nw, int n, bool packed)
{
    if (m == Mode::B) {
        const size_t tile = (size_t)kEBBlock * expand_paths_per_thread(nw);
        return blocked_ring_bytes(nw, packed) + ((size_t)n * (nw <= 2 ? 2 : 1) * nw + ((n + 1) & ~1)) * sizeof(u64) +
               tile * (2 * nw + 1) * 8 +
               (packed ? 0 : tile * 4) + (size_t)kChildCapX4 * tile;
    }
    const size_t kb = nw <= kByteTableWords ? (size_t)8 * nw * 256 : 0;
    return ((size_t)n * (nw + 1) + kb) * sizeof(u64);
}

typedef void (*KernelFn)(const LaunchArgs);

// Always raise the kernel's dynamic shared-memory limit to `smem`: the 48 KB default applies to
// static + dynamic together, so a dynamic size just under 48 KB can still fail to launch
static cudaError_t set_smem(KernelFn f, size_t smem)
{
    if (smem == 0)
        return cudaSuccess;
    return cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

static cudaError_t run(KernelFn f, unsigned int grid, size_t smem, cudaStream_t st, const LaunchArgs &a,
                       int block = kBlock)
{
    cudaError_t e = set_smem(f, smem);
    if (e != cudaSuccess)
        return e;
    f<<<grid, block, smem, st>>>(a);
    return cudaGetLastError();
}

static inline unsigned int grid_for(u64 items_per_block, u64 n, int grid_cap)
{
    u64 b = (n + items_per_block - 1) / items_per_block;
    if (b < 1)
        b = 1;
    if (b > (u64)grid_cap)
        b = (u64)grid_cap;
    return (unsigned int)b;
}

// kernel for (which, mode, nw, packed); which: 0 stage1, 1 expand thread, 2 expand warp,
// 3 filter, 4 expand with at most 3 children per path
static KernelFn kernel_for(int which, Mode m, int nw, bool pk, bool leaf = false)
{
    const bool bm = m == Mode::B;
    switch (which) {
    case 0:
#define K0(N) if (nw == N) return bm ? (pk ? k_stage1<N, true, true> : k_stage1<N, true, false>) : k_stage1<N, false, false>;
        CC_CASES(K0)
#undef K0
        break;
    case 1:
    case 2:
#define K1(N)                                                                                            \
    if (nw == N)                                                                                         \
        return bm ? (leaf ? (pk ? k_expand_blocked<N, 0, true, true> : k_expand_blocked<N, 0, false, true>)    \
                          : (pk ? k_expand_blocked<N, 0, true, false> : k_expand_blocked<N, 0, false, false>)) \
                  : (which == 1 ? k_expand_thread<N> : k_expand_warp<N>);
        CC_CASES(K1)
#undef K1
        break;
    case 4:
#define K4(N)                                                                                            \
    if (nw == N)                                                                                         \
        return bm ? (leaf ? (pk ? k_expand_blocked<N, 3, true, true> : k_expand_blocked<N, 3, false, true>)    \
                          : (pk ? k_expand_blocked<N, 3, true, false> : k_expand_blocked<N, 3, false, false>)) \
                  : k_expand_thread<N>;
        CC_CASES(K4)
#undef K4
        break;
    default: {
        const int rw = record_words(nw, m);
#define K3(N) if (rw == N) return pk ? k_shard_filter<N, false> : k_shard_filter<N, true>;
        CC_CASES(K3) K3(9)
#undef K3
    }
    }
    return nullptr;
}

cudaError_t launch_wide(int which, const LaunchArgs &a, cudaStream_t st, int grid_cap)
{
    if (a.n_in == 0)
        return cudaSuccess;
    KernelFn f = which == 0 ? k_stage1_wide
                 : which == 1 ? (a.emit && !a.emit_next ? k_leaf_wide : k_expand_wide)
                              : k_shard_filter_wide;
    const u64 per_block = which == 1 ? (u64)(kBlock / 32) * kWidePaths : (u64)kBlock;
    return run(f, grid_for(per_block, a.n_in, grid_cap), 0, st, a);
}

static KernelFn list_kernel(int which, int rwl, bool leaf, bool col = false)
{
    if (which == 0)
        return rwl == 2 ? (col ? k_stage1_list<2, true> : k_stage1_list<2, false>)
             : rwl == 3 ? (col ? k_stage1_list<3, true> : k_stage1_list<3, false>) : nullptr;
    if (which == 1) {
        if (rwl == 2)
            return col ? (leaf ? k_expand_list<2, true, true> : k_expand_list<2, false, true>)
                       : (leaf ? k_expand_list<2, true, false> : k_expand_list<2, false, false>);
        if (rwl == 3)
            return col ? (leaf ? k_expand_list<3, true, true> : k_expand_list<3, false, true>)
                       : (leaf ? k_expand_list<3, true, false> : k_expand_list<3, false, false>);
        return nullptr;
    }
    return rwl == 2 ? k_shard_filter<4, false, false> : rwl == 3 ? k_shard_filter<5, false, false> : nullptr;
}

cudaError_t launch_list(int which, const LaunchArgs &a, int rwl, bool leaf, cudaStream_t st, int grid_cap)
{
    if (a.n_in == 0)
        return cudaSuccess;
    KernelFn f = list_kernel(which, rwl, leaf, a.collect != 0);
    if (!f)
        return cudaErrorInvalidValue;
    const int block = which == 2 ? kBlock : kListBlock;  // the shard filter is the generic kernel
    return run(f, grid_for(block, a.n_in, grid_cap), 0, st, a, block);
}

int max_blocks_per_sm_list(int which, int rwl)
{
    KernelFn f = list_kernel(which, rwl, false);
    int nb = 1;
    const int block = which == 2 ? kBlock : kListBlock;
    if (!f || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)f, block, 0) != cudaSuccess || nb < 1)
        nb = 1;
    return nb;
}

int max_blocks_per_sm_wide(int which)
{
    KernelFn f = which == 0 ? k_stage1_wide : which == 1 ? k_expand_wide : k_shard_filter_wide;
    int nb = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)f, kBlock, 0) != cudaSuccess || nb < 1)
        nb = 1;
    return nb;
}

cudaError_t launch_stage1(const LaunchArgs &a, Mode m, cudaStream_t st, int grid_cap)
{
    if (a.n_in == 0)
        return cudaSuccess;
    KernelFn f = kernel_for(0, m, a.g.nw, a.packed != 0);
    if (!f)
        return cudaErrorInvalidValue;
    return run(f, grid_for(kBlock, a.n_in, grid_cap), graph_smem(a), st, a);
}

cudaError_t launch_expand(const LaunchArgs &a, Mode m, ExpandVariant v, cudaStream_t st, int grid_cap)
{
    if (a.n_in == 0)
        return cudaSuccess;
    const int which = v == ExpandVariant::Small ? 4 : (v == ExpandVariant::Thread ? 1 : 2);
    KernelFn f = kernel_for(which, m, a.g.nw, a.packed != 0, a.emit && !a.emit_next);
    if (!f)
        return cudaErrorInvalidValue;
    u64 per_block = kBlock;
    if (m == Mode::B)
        per_block = (u64)kEBBlock * expand_paths_per_thread(a.g.nw);
    else if (v == ExpandVariant::Warp)
        per_block = kBlock / 32;
    return run(f, grid_for(per_block, a.n_in, grid_cap), expand_smem(m, a.g.nw, a.g.n, a.packed != 0), st, a,
               m == Mode::B ? kEBBlock : kBlock);
}

cudaError_t launch_shard_filter(const LaunchArgs &a, Mode m, cudaStream_t st, int grid_cap)
{
    if (a.n_in == 0)
        return cudaSuccess;
    KernelFn f = kernel_for(3, m, a.g.nw, a.packed != 0);
    if (!f)
        return cudaErrorInvalidValue;
    return run(f, grid_for(kBlock, a.n_in, grid_cap), 0, st, a);
}

cudaError_t launch_keys(u64 *key, u64 *keybyte, const int32_t *orig, int n, int nw, u64 seed,
                        cudaStream_t st)
{
    if (n <= 0)
        return cudaSuccess;
    k_keys<<<(n + 255) / 256, 256, 0, st>>>(key, orig, n, seed);
    if (nw <= kByteTableWords)
        k_keybyte<<<8 * nw, 256, 0, st>>>(keybyte, key, n);
    return cudaGetLastError();
}

cudaError_t launch_nbrmask(const DevGraph &g, uint32_t *T, cudaStream_t st)
{
    if (g.n <= 0)
        return cudaSuccess;
    k_build_nbrmask<<<(g.n + 7) / 8, 256, 0, st>>>(g, T);
    return cudaGetLastError();
}


cudaError_t launch_cycle_sequences(const CycleStore &c, int nw, const u64 *adj, const int32_t *orig,
                                   uint64_t first, uint64_t count, const u64 *offsets, int32_t *out,
                                   cudaStream_t st)
{
    if (count == 0)
        return cudaSuccess;
    k_cycle_sequences<<<(unsigned int)((count + 255) / 256), 256, 0, st>>>(c, nw, adj, orig, first,
                                                                          count, offsets, out);
    return cudaGetLastError();
}

int max_blocks_per_sm(int which, Mode m, int nw, bool packed, size_t smem)
{
    KernelFn f = kernel_for(which, m, nw, packed);
    if (!f)
        return 1;
    const size_t sm = which == 3 ? 0 : smem;
    // the B-mode expansion kernel runs kEBBlock-thread CTAs (grid sizes are in CTAs)
    const int block = (m == Mode::B && (which == 1 || which == 2 || which == 4)) ? kEBBlock : kBlock;
    int nb = 1;
    if (set_smem(f, sm) != cudaSuccess)
        return 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)f, block, sm) != cudaSuccess || nb < 1)
        nb = 1;
    return nb;
}

}  // namespace cc
