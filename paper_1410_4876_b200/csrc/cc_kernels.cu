// cc_kernels.cu -- sm_100a kernels of the chordless-cycle hot path (arXiv 1410.4876).
//
//   k_stage1         Stage 1 (Alg. 2): seeds T(G) and triangles.  One thread
//                    per forward-neighbour pair (u; x < y in N+(u)) -- the sum_u C(d+(u),2) real
//                    pairs, not the paper's |V|*Delta^2 padded index space.
//   k_expand_thread  Stage 2 (Alg. 3) for Delta <= 32: one thread per path,
//                    loops over Adj(v_t); extensions appended with a block-aggregated
//                    prefix-sum allocator (one atomicAdd per CTA tile; the paper's
//                    "serialization in the index calculation").
//   k_expand_warp    Stage 2 for Delta > 32: one warp per path, lanes scan the suffix of the
//                    sorted CSR row of v_t that passes the label gate (coalesced), ballot/popc
//                    warp-aggregated appends.
//   k_shard_filter   multi-GPU: keep the paths whose content hash falls in this shard.
//   k_keys           key(v) = mix(seed ^ original id) (H-spec).
//   k_cycle_*        collect mode: canonical vertex order of stored cycles (the inverse of the
//                    bitmap encoding, PAPER.md:193 / SPEC.md:216).
//
// Per-candidate test (Alg. 3 lines 11-15), for path p = <v1..vt> with
// bitmap S and v in Adj(vt):
//   gate   v > v2 (label order == id order after relabelling) and v not in S
//   X      = Adj(v) & S & ~{vt}          (NW word-ANDs against the adjacency bit row of v)
//   extend iff X == {}                   (<p,v> is a chordless path -> F_{t+1})
//   close  iff X == {v1}                 (<p,v> is a chordless cycle of t+1 vertices)
//   else   a chord: discard.
// This is the paper's dichotomy evaluated on the bitmap S.
#include "cc_internal.h"

namespace cc {

#define FULL_MASK 0xffffffffu

__device__ __forceinline__ u64 mix64(u64 x)
{
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

// ---------------------------------------------------------------------------- paged records
template <int NW>
__device__ __forceinline__ u64 *page_words(const Pages &pg, uint32_t page)
{
    return (u64 *)(pg.base + (u64)page * pg.page_bytes);
}

template <int NW>
__device__ __forceinline__ uint32_t *page_ids(const Pages &pg, uint32_t page)
{
    return (uint32_t *)(pg.base + (u64)page * pg.page_bytes + ((u64)NW << pg.log_p) * 8);
}

template <int NW>
__device__ __forceinline__ void load_record(const Pages &pg, uint32_t page, uint32_t slot, u64 (&S)[NW],
                                            uint32_t &id)
{
    const u64 *w = page_words<NW>(pg, page);
#pragma unroll
    for (int k = 0; k < NW; ++k)
        S[k] = w[((u64)k << pg.log_p) + slot];
    id = page_ids<NW>(pg, page)[slot];
}

// write record at virtual output position o (page out_pages[o >> log_p])
template <int NW>
__device__ __forceinline__ void store_record(const Pages &pg, u64 o, const u64 (&S)[NW], uint32_t v,
                                             bool add_v, uint32_t id)
{
    const uint32_t page = pg.out_pages[o >> pg.log_p];
    const uint32_t slot = (uint32_t)(o & ((1ull << pg.log_p) - 1));
    u64 *w = page_words<NW>(pg, page);
#pragma unroll
    for (int k = 0; k < NW; ++k)
        w[((u64)k << pg.log_p) + slot] = S[k] | ((add_v && k == (int)(v >> 6)) ? (1ull << (v & 63)) : 0ull);
    page_ids<NW>(pg, page)[slot] = id;
}

template <int NW>
__device__ __forceinline__ u64 shard_hash(const u64 (&S)[NW], uint32_t id)
{
    u64 h = mix64((u64)id);
#pragma unroll
    for (int w = 0; w < NW; ++w)
        h = mix64(h ^ S[w]);
    return h;
}

// Block-wide exclusive scan of c plus one atomicAdd per CTA on *counter.  Must be called by
// every thread of the block.  Returns this thread's first output index (relative to the
// counter's origin).
struct ReserveSmem {
    u64 base;
    unsigned int warp[kBlock / 32];
};

__device__ __forceinline__ u64 block_reserve(unsigned int c, u64 *counter, ReserveSmem &sm)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned int v = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= o)
            incl += v;
    }
    if (lane == 31)
        sm.warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        unsigned int w = lane < kBlock / 32 ? sm.warp[lane] : 0u;
        unsigned int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned int v = __shfl_up_sync(FULL_MASK, wi, o);
            if (lane >= o)
                wi += v;
        }
        if (lane < kBlock / 32)
            sm.warp[lane] = wi - w;
        if (lane == kBlock / 32 - 1)
            sm.base = wi ? atomicAdd(counter, (u64)wi) : 0ull;
    }
    __syncthreads();
    const u64 r = sm.base + sm.warp[wid] + (incl - c);
    __syncthreads();  // sm is reused by the next tile
    return r;
}

template <int NW>
__device__ __forceinline__ u64 word_of(const u64 (&S)[NW], uint32_t v)
{
    u64 r = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w)
        if (w == (int)(v >> 6))
            r = S[w];
    return r;
}

// sum of key(v) over the vertices of S (the H-spec keysum of a path).  For NW <= 2 the sum is
// 8*NW lookups in byte tables (s_kb[j][b] = sum of the keys of the set bits of byte value b at
// byte position j), otherwise a loop over the set bits.
template <int NW>
__device__ __forceinline__ u64 keysum(const u64 (&S)[NW], const u64 *s_key, const u64 *s_kb)
{
    u64 ks = 0;
    if (NW <= kByteTableWords) {
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                ks += s_kb[((w * 8 + j) << 8) + (uint32_t)((S[w] >> (8 * j)) & 0xffu)];
    } else {
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            u64 x = S[w];
            while (x) {
                const int b = __ffsll((long long)x) - 1;
                ks += s_key[w * 64 + b];
                x &= x - 1;
            }
        }
    }
    return ks;
}

// Block-reduce (cycles, hash, cand) into the launch scratch (one atomic each per CTA).
__device__ __forceinline__ void flush_accum(u64 cnt, u64 hs, u64 cand, Scratch *sc)
{
    __shared__ u64 red[3][kBlock / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(FULL_MASK, cnt, o);
        hs += __shfl_xor_sync(FULL_MASK, hs, o);
        cand += __shfl_xor_sync(FULL_MASK, cand, o);
    }
    if (lane == 0) {
        red[0][wid] = cnt;
        red[1][wid] = hs;
        red[2][wid] = cand;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 a = 0, b = 0, c = 0;
        for (int i = 0; i < kBlock / 32; ++i) {
            a += red[0][i];
            b += red[1][i];
            c += red[2][i];
        }
        if (a)
            atomicAdd(&sc->cycles, a);
        if (b)
            atomicAdd(&sc->hash, b);
        if (c)
            atomicAdd(&sc->cand, c);
    }
}

// Graph tables staged in shared memory: adjacency bit rows (n*NW words), keys (n words) and,
// for NW <= 2, the byte key tables (8*NW*256 words).
template <int NW>
__host__ __device__ constexpr int keybyte_words()
{
    return NW <= kByteTableWords ? 8 * NW * 256 : 0;
}

template <int NW>
__device__ __forceinline__ void stage_graph(const DevGraph &g, u64 *s_adj, u64 *s_key, u64 *s_kb)
{
    const int nrow = g.n * NW;
    for (int i = threadIdx.x; i < nrow; i += blockDim.x)
        s_adj[i] = g.adj[i];
    for (int i = threadIdx.x; i < g.n; i += blockDim.x)
        s_key[i] = g.key[i];
    for (int i = threadIdx.x; i < keybyte_words<NW>(); i += blockDim.x)
        s_kb[i] = g.keybyte[i];
    __syncthreads();
}

__device__ __forceinline__ uint32_t pack_ids(uint32_t v1, uint32_t v2, uint32_t vt)
{
    return v1 | (v2 << kIdBits) | (vt << (2 * kIdBits));
}

template <int NW>
__device__ __forceinline__ void store_cycle(const LaunchArgs &p, const u64 (&S)[NW], uint32_t v,
                                            uint32_t v1, uint32_t v2)
{
    const u64 idx = atomicAdd(p.cyc.count, 1ull);
    if (idx < p.cyc.cap) {
#pragma unroll
        for (int w = 0; w < NW; ++w)
            p.cyc.s[(u64)w * p.cyc.cap + idx] = S[w] | (w == (int)(v >> 6) ? (1ull << (v & 63)) : 0ull);
        p.cyc.ids[idx] = v1 | (v2 << kIdBits);
    }
}

// ---------------------------------------------------------------------------- Stage 1
template <int NW>
__global__ void __launch_bounds__(kBlock) k_stage1(const LaunchArgs p)
{
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
        u64 S[NW];
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
#pragma unroll
            for (int w = 0; w < NW; ++w)
                S[w] = (w == (int)(x >> 6) ? 1ull << (x & 63) : 0ull) |
                       (w == (int)(u >> 6) ? 1ull << (u & 63) : 0ull);
            const bool tri = (s_adj[x * NW + (y >> 6)] >> (y & 63)) & 1ull;  // x in Adj(y) (l.13)
            if (tri) {
                if (p.count) {  // Alg. 2 line 14: a triangle goes straight to C
                    cnt++;
                    hs += mix64(s_key[x] + s_key[u] + s_key[y]);
                    if (p.collect)
                        store_cycle<NW>(p, S, y, x, u);
                }
            } else if (p.emit) {  // Alg. 2 line 15: <x,u,y> in T(G)
                emit = 1;
                if (p.root_stride > 1) {
                    const u64 rkey = ((u64)p.g.orig[x] << 42) | ((u64)p.g.orig[u] << 21) |
                                     (u64)p.g.orig[y];
                    emit = (mix64(rkey) % p.root_stride) == p.root_offset;
                }
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    S[w] |= (w == (int)(y >> 6) ? 1ull << (y & 63) : 0ull);
                id = pack_ids(x, u, y);
                if (emit && p.filter)
                    emit = (shard_hash<NW>(S, id) % p.shard_count) == p.shard_index;
            }
        }
        const u64 off = block_reserve(emit, &p.sc->out_count, rs);
        if (emit) {
            if (off >= p.out_cap)
                p.sc->err = 1;
            else
                store_record<NW>(p.pg, p.out_off + off, S, 0, false, id);
        }
    }
    flush_accum(cnt, hs, 0, p.sc);
}

// ---------------------------------------------------------------------------- Stage 2
// Evaluate candidate v for path (S, v1, vt): 1 = extend, 2 = close, 0 = reject.
template <int NW>
__device__ __forceinline__ int classify(const u64 (&S)[NW], const u64 *s_adj, uint32_t v,
                                        uint32_t v1, uint32_t vt)
{
    if ((word_of<NW>(S, v) >> (v & 63)) & 1ull)  // v in p (Alg. 3 line 11)
        return 0;
    bool ext = true, close = true;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        u64 x = s_adj[v * NW + w] & S[w];
        if (w == (int)(vt >> 6))
            x &= ~(1ull << (vt & 63));
        const u64 b1 = (w == (int)(v1 >> 6)) ? (1ull << (v1 & 63)) : 0ull;
        ext &= (x == 0ull);
        close &= (x == b1);
    }
    return ext ? 1 : (close ? 2 : 0);
}

// Bitset form of the per-path step for the thread-per-path kernel.  With S the path bitmap:
//   cand = Adj(vt) & ~S & {v > v2}                 (Alg. 3 line 11 gate, all candidates at once)
//   for v in cand:  X = Adj(v) & S & ~{vt}          (line 12 / 14 adjacency tests)
//       X == {}   -> extension <p, v>               (line 15)
//       X == {v1} -> chordless cycle <p, v>         (line 13)
// Returns the extension vertices as a bitset; closures are counted and hashed here.
template <int NW>
__device__ __forceinline__ void expand_path(const LaunchArgs &p, const u64 (&S)[NW], uint32_t id,
                                            const u64 *s_adj, const u64 *s_key, const u64 *s_kb,
                                            u64 (&ext)[NW], u64 &cnt, u64 &hs, u64 &cand_slots)
{
    const uint32_t v1 = id & kIdMask;
    const uint32_t v2 = (id >> kIdBits) & kIdMask;
    const uint32_t vt = id >> (2 * kIdBits);
    const u64 *av = s_adj + vt * NW;
    u64 cand[NW];
    const int lo = (int)v2 + 1;  // first label passing the gate
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const u64 a = av[w];
        cand_slots += __popcll(a);  // deg(vt): the candidate slots of Alg. 3 (stat only)
        const int sh = lo - 64 * w;
        const u64 above = sh <= 0 ? ~0ull : (sh >= 64 ? 0ull : (~0ull << sh));
        cand[w] = a & ~S[w] & above;
        ext[w] = 0;
    }
    u64 ks = 0;
    bool have_ks = false;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        while (cand[w]) {
            const int b = __ffsll((long long)cand[w]) - 1;
            cand[w] &= cand[w] - 1;
            const uint32_t v = (uint32_t)(64 * w + b);
            const u64 *ar = s_adj + v * NW;
            bool e = true, c = true;
#pragma unroll
            for (int u = 0; u < NW; ++u) {
                u64 x = ar[u] & S[u];
                if (u == (int)(vt >> 6))
                    x &= ~(1ull << (vt & 63));
                const u64 b1 = (u == (int)(v1 >> 6)) ? (1ull << (v1 & 63)) : 0ull;
                e &= (x == 0ull);
                c &= (x == b1);
            }
            if (e) {
                ext[w] |= 1ull << b;
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

template <int NW>
__global__ void __launch_bounds__(kBlock, NW <= 2 ? 4 : 2) k_expand_thread(const LaunchArgs p)
{
    // paths per thread per tile (2 for the long-path grid class NW <= 2, 1 for wide bitmaps):
    // with the register double buffer this keeps NW <= 2 at 64 registers, 4 CTAs per SM
    constexpr int R = expand_paths_per_thread(NW);
    extern __shared__ u64 smem[];
    u64 *s_adj = smem;
    u64 *s_key = smem + p.g.n * NW;
    u64 *s_kb = s_key + p.g.n;
    __shared__ ReserveSmem rs;
    stage_graph<NW>(p.g, s_adj, s_key, s_kb);

    const u64 pmask = (1ull << p.pg.log_p) - 1;
    constexpr u64 kTile = (u64)kBlock * R;
    const u64 stride = (u64)gridDim.x * kTile;
    u64 cnt = 0, hs = 0, cand = 0;

    // a tile of kBlock*R records never straddles a page (pages hold >= kTile records);
    // thread j takes records base + j + kBlock*i, i < R (each load instruction coalesced).
    // Register double buffering: the next tile's loads are in flight during this tile's work.
    u64 S[R][NW], Sn[R][NW];
    uint32_t id[R], idn[R];
    auto load_tile = [&](u64 base, u64 (&T)[R][NW], uint32_t (&I)[R]) {
        const uint32_t page = p.pg.in_pages[base >> p.pg.log_p];
        const uint32_t slot0 = (uint32_t)(base & pmask) + threadIdx.x;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            I[i] = 0xffffffffu;
            if (base + threadIdx.x + (u64)kBlock * i < p.n_in)
                load_record<NW>(p.pg, page, slot0 + kBlock * i, T[i], I[i]);
        }
    };
    u64 base = (u64)blockIdx.x * kTile;
    if (base < p.n_in)
        load_tile(base, S, id);
    for (; base < p.n_in; base += stride) {
        if (base + stride < p.n_in)
            load_tile(base + stride, Sn, idn);
        u64 ext[R][NW];
        unsigned int ne = 0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
#pragma unroll
            for (int w = 0; w < NW; ++w)
                ext[i][w] = 0;
            if (id[i] == 0xffffffffu)
                continue;
            expand_path<NW>(p, S[i], id[i], s_adj, s_key, s_kb, ext[i], cnt, hs, cand);
            if (p.emit) {
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    ne += __popcll(ext[i][w]);
            }
        }
        const u64 off = block_reserve(ne, &p.sc->out_count, rs);
        if (ne) {
            if (off + ne > p.out_cap) {
                p.sc->err = 1;
            } else {
                u64 o = p.out_off + off;
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    const uint32_t v12 = id[i] & ((1u << (2 * kIdBits)) - 1);
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        u64 m = ext[i][w];
                        while (m) {
                            const int b = __ffsll((long long)m) - 1;
                            m &= m - 1;
                            const uint32_t v = (uint32_t)(64 * w + b);
                            store_record<NW>(p.pg, o++, S[i], v, true, v12 | (v << (2 * kIdBits)));
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            id[i] = idn[i];
#pragma unroll
            for (int w = 0; w < NW; ++w)
                S[i][w] = Sn[i][w];
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
    u64 *s_kb = s_key + p.g.n;
    stage_graph<NW>(p.g, s_adj, s_key, s_kb);

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
                c = classify<NW>(S, s_adj, v, v1, vt);
            }
            const unsigned int eb = __ballot_sync(FULL_MASK, c == 1 && p.emit);
            if (eb) {
                u64 b = 0;
                if (lane == 0)
                    b = atomicAdd(&p.sc->out_count, (u64)__popc(eb));
                b = __shfl_sync(FULL_MASK, b, 0);
                if (c == 1) {
                    const u64 off = b + __popc(eb & lt_mask);
                    if (off >= p.out_cap)
                        p.sc->err = 1;
                    else
                        store_record<NW>(p.pg, p.out_off + off, S, v, true, pack_ids(v1, v2, v));
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

// ---------------------------------------------------------------------------- shard filter
template <int NW>
__global__ void __launch_bounds__(kBlock) k_shard_filter(const LaunchArgs p)
{
    __shared__ ReserveSmem rs;
    const u64 pmask = (1ull << p.pg.log_p) - 1;
    const u64 stride = (u64)gridDim.x * kBlock;
    for (u64 base = (u64)blockIdx.x * kBlock; base < p.n_in; base += stride) {
        const u64 r = base + threadIdx.x;
        u64 S[NW];
        uint32_t id = 0;
        unsigned int keep = 0;
        if (r < p.n_in) {
            load_record<NW>(p.pg, p.pg.in_pages[base >> p.pg.log_p], (uint32_t)(r & pmask), S, id);
            keep = (shard_hash<NW>(S, id) % p.shard_count) == p.shard_index;
        }
        const u64 off = block_reserve(keep, &p.sc->out_count, rs);
        if (keep) {
            if (off >= p.out_cap)
                p.sc->err = 1;
            else
                store_record<NW>(p.pg, p.out_off + off, S, 0, false, id);
        }
    }
}

// ---------------------------------------------------------------------------- keys, collect
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

__global__ void k_cycle_lengths(const CycleStore c, int nw, uint64_t first, uint64_t count, uint32_t *len)
{
    const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count)
        return;
    uint32_t k = 0;
    for (int w = 0; w < nw; ++w)
        k += __popcll(c.s[(u64)w * c.cap + first + i]);
    len[i] = k;
}

// Walk the induced cycle S from v1 -> v2 -> ...: each vertex of a chordless cycle has exactly
// two neighbours in S, so the successor of cur is the neighbour in S other than prev.
__global__ void k_cycle_sequences(const CycleStore c, int nw, const u64 *adj, const int32_t *orig,
                                  uint64_t first, uint64_t count, const u64 *offsets, int32_t *out)
{
    const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count)
        return;
    u64 S[kMaxWords];
    for (int w = 0; w < nw; ++w)
        S[w] = c.s[(u64)w * c.cap + first + i];
    const uint32_t id = c.ids[first + i];
    uint32_t prev = id & kIdMask, cur = (id >> kIdBits) & kIdMask;
    const u64 o = offsets[i], k = offsets[i + 1] - offsets[i];
    out[o] = orig[prev];
    if (k > 1)
        out[o + 1] = orig[cur];
    for (u64 j = 2; j < k; ++j) {
        uint32_t nxt = 0;
        for (int w = 0; w < nw; ++w) {
            u64 x = adj[(u64)cur * nw + w] & S[w];
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
#define CC_DISPATCH_NW(nw, KERNEL, ...)                \
    switch (nw) {                                      \
    case 1: KERNEL<1><<<__VA_ARGS__>>>(a); break;      \
    case 2: KERNEL<2><<<__VA_ARGS__>>>(a); break;      \
    case 3: KERNEL<3><<<__VA_ARGS__>>>(a); break;      \
    case 4: KERNEL<4><<<__VA_ARGS__>>>(a); break;      \
    case 5: KERNEL<5><<<__VA_ARGS__>>>(a); break;      \
    case 6: KERNEL<6><<<__VA_ARGS__>>>(a); break;      \
    case 7: KERNEL<7><<<__VA_ARGS__>>>(a); break;      \
    case 8: KERNEL<8><<<__VA_ARGS__>>>(a); break;      \
    default: return cudaErrorInvalidValue;             \
    }

static inline size_t graph_smem(const LaunchArgs &a)
{
    const size_t kb = a.g.nw <= kByteTableWords ? (size_t)8 * a.g.nw * 256 : 0;
    return ((size_t)a.g.n * (a.g.nw + 1) + kb) * sizeof(u64);
}

template <typename F>
static cudaError_t set_smem(F *f, size_t smem)
{
    if (smem > 48 * 1024)
        return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return cudaSuccess;
}

#define CC_SET_SMEM_NW(nw, KERNEL, smem)                                   \
    do {                                                                   \
        cudaError_t e_ = cudaSuccess;                                      \
        switch (nw) {                                                      \
        case 1: e_ = set_smem(KERNEL<1>, smem); break;                     \
        case 2: e_ = set_smem(KERNEL<2>, smem); break;                     \
        case 3: e_ = set_smem(KERNEL<3>, smem); break;                     \
        case 4: e_ = set_smem(KERNEL<4>, smem); break;                     \
        case 5: e_ = set_smem(KERNEL<5>, smem); break;                     \
        case 6: e_ = set_smem(KERNEL<6>, smem); break;                     \
        case 7: e_ = set_smem(KERNEL<7>, smem); break;                     \
        case 8: e_ = set_smem(KERNEL<8>, smem); break;                     \
        }                                                                  \
        if (e_ != cudaSuccess)                                             \
            return e_;                                                     \
    } while (0)

static inline unsigned int grid_for(u64 items_per_block, u64 n, int grid_cap)
{
    u64 b = (n + items_per_block - 1) / items_per_block;
    if (b < 1)
        b = 1;
    if (b > (u64)grid_cap)
        b = (u64)grid_cap;
    return (unsigned int)b;
}

cudaError_t launch_stage1(const LaunchArgs &a, cudaStream_t st, int grid_cap)
{
    if (a.n_in == 0)
        return cudaSuccess;
    const size_t smem = graph_smem(a);
    CC_SET_SMEM_NW(a.g.nw, k_stage1, smem);
    const unsigned int grid = grid_for(kBlock, a.n_in, grid_cap);
    CC_DISPATCH_NW(a.g.nw, k_stage1, grid, kBlock, smem, st);
    return cudaGetLastError();
}

cudaError_t launch_expand(const LaunchArgs &a, ExpandVariant v, cudaStream_t st, int grid_cap)
{
    if (a.n_in == 0)
        return cudaSuccess;
    const size_t smem = graph_smem(a);
    if (v == ExpandVariant::Thread) {
        CC_SET_SMEM_NW(a.g.nw, k_expand_thread, smem);
        const unsigned int grid = grid_for((u64)kBlock * expand_paths_per_thread(a.g.nw), a.n_in, grid_cap);
        CC_DISPATCH_NW(a.g.nw, k_expand_thread, grid, kBlock, smem, st);
    } else {
        CC_SET_SMEM_NW(a.g.nw, k_expand_warp, smem);
        const unsigned int grid = grid_for(kBlock / 32, a.n_in, grid_cap);
        CC_DISPATCH_NW(a.g.nw, k_expand_warp, grid, kBlock, smem, st);
    }
    return cudaGetLastError();
}

cudaError_t launch_shard_filter(const LaunchArgs &a, cudaStream_t st, int grid_cap)
{
    if (a.n_in == 0)
        return cudaSuccess;
    const unsigned int grid = grid_for(kBlock, a.n_in, grid_cap);
    CC_DISPATCH_NW(a.g.nw, k_shard_filter, grid, kBlock, 0, st);
    return cudaGetLastError();
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

cudaError_t launch_cycle_lengths(const CycleStore &c, int nw, uint64_t first, uint64_t count,
                                 uint32_t *len, cudaStream_t st)
{
    if (count == 0)
        return cudaSuccess;
    k_cycle_lengths<<<(unsigned int)((count + 255) / 256), 256, 0, st>>>(c, nw, first, count, len);
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

static cudaError_t raise_smem(int which, int nw, size_t smem)
{
    switch (which) {
    case 0: CC_SET_SMEM_NW(nw, k_stage1, smem); break;
    case 1: CC_SET_SMEM_NW(nw, k_expand_thread, smem); break;
    case 2: CC_SET_SMEM_NW(nw, k_expand_warp, smem); break;
    }
    return cudaSuccess;
}

int max_blocks_per_sm(int which, int nw, size_t smem)
{
    int nb = 1;
    cudaError_t e = cudaSuccess;
#define CC_OCC(KERNEL)                                                                          \
    switch (nw) {                                                                               \
    case 1: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, KERNEL<1>, kBlock, smem); break; \
    case 2: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, KERNEL<2>, kBlock, smem); break; \
    case 3: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, KERNEL<3>, kBlock, smem); break; \
    case 4: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, KERNEL<4>, kBlock, smem); break; \
    case 5: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, KERNEL<5>, kBlock, smem); break; \
    case 6: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, KERNEL<6>, kBlock, smem); break; \
    case 7: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, KERNEL<7>, kBlock, smem); break; \
    case 8: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, KERNEL<8>, kBlock, smem); break; \
    }
    if (smem > 48 * 1024 && raise_smem(which, nw, smem) != cudaSuccess)
        return 1;
    switch (which) {
    case 0: CC_OCC(k_stage1); break;
    case 1: CC_OCC(k_expand_thread); break;
    case 2: CC_OCC(k_expand_warp); break;
    default: CC_OCC(k_shard_filter); break;
    }
#undef CC_OCC
    if (e != cudaSuccess || nb < 1)
        nb = 1;
    return nb;
}

}  // namespace cc
