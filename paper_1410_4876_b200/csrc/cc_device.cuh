// cc_device.cuh -- device helpers shared by the sm_100a kernel translation units
// (cc_kernels.cu, cc_fused.cu): the H-spec mix, record packing, paged-arena addressing, block
// reservations, shared-memory bit rows, statistics flush, TMA bulk copies and mbarriers.
#pragma once
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

__device__ __forceinline__ uint32_t pack_ids(uint32_t v1, uint32_t v2, uint32_t vt)
{
    return v1 | (v2 << kIdBits) | (vt << (2 * kIdBits));
}

__device__ __forceinline__ u64 bit_in_word(int w, uint32_t v)
{
    return (w == (int)(v >> 6)) ? (1ull << (v & 63)) : 0ull;
}

// word w of the label gate {x : x > v2} (Alg. 3 line 11 after relabelling)
__device__ __forceinline__ u64 above_word(uint32_t v2, int w)
{
    const int sh = (int)v2 + 1 - 64 * w;
    return sh <= 0 ? ~0ull : (sh >= 64 ? 0ull : (~0ull << sh));
}

// ---------------------------------------------------------------------------- paged records
__device__ __forceinline__ char *page_ptr(const Pages &pg, uint32_t page)
{
    return pg.base + (u64)page * pg.page_bytes;
}

template <int RW, bool IDS = true>
__device__ __forceinline__ void load_record(const Pages &pg, uint32_t page, uint32_t slot, u64 (&W)[RW],
                                            uint32_t &id)
{
    const char *pp = page_ptr(pg, page);
    const u64 *w = (const u64 *)pp;
#pragma unroll
    for (int k = 0; k < RW; ++k)
        W[k] = w[((u64)k << pg.log_p) + slot];
    if (IDS)
        id = ((const uint32_t *)(pp + ((u64)RW << pg.log_p) * 8))[slot];
    else
        id = 0;
}

// write a record at virtual output position o (page out_pages[o >> log_p])
template <int RW, bool IDS = true>
__device__ __forceinline__ void store_record(const Pages &pg, u64 o, const u64 (&W)[RW], uint32_t id)
{
    const uint32_t page = pg.out_pages[o >> pg.log_p];
    const uint32_t slot = (uint32_t)(o & ((1ull << pg.log_p) - 1));
    char *pp = page_ptr(pg, page);
    u64 *w0 = (u64 *)pp + slot;
    const u64 pw = 1ull << pg.log_p;  // words between consecutive word arrays
#pragma unroll
    for (int k = 0; k < RW; ++k)
        w0[k * pw] = W[k];
    if (IDS)
        ((uint32_t *)(pp + ((u64)RW << pg.log_p) * 8))[slot] = id;
}

// Packed B-mode ids: v1 | v2 << idb | vt << 2idb in the top 3*idb bits of word NW-1.
// (3*idb can exceed 32 bits: idb = 11 for n = 2000, so the packed ids are 64-bit values)
__device__ __forceinline__ u64 packed_ids(u64 last_word, uint32_t idb)
{
    return last_word >> (64 - 3 * idb);
}
__device__ __forceinline__ u64 with_packed_ids(u64 last_word, u64 ids, uint32_t idb)
{
    const u64 low = (1ull << (64 - 3 * idb)) - 1;
    return (last_word & low) | (ids << (64 - 3 * idb));
}
__device__ __forceinline__ u64 pack3(uint32_t a, uint32_t b, uint32_t c, uint32_t idb)
{
    return (u64)a | ((u64)b << idb) | ((u64)c << (2 * idb));
}

template <int RW>
__device__ __forceinline__ u64 shard_hash(const u64 (&W)[RW], uint32_t id)
{
    u64 h = mix64((u64)id);
#pragma unroll
    for (int w = 0; w < RW; ++w)
        h = mix64(h ^ W[w]);
    return h;
}

// Block-wide exclusive scan of c plus one atomicAdd per CTA on *counter.  Must be called by
// every thread of the block.  Returns this thread's first output index (relative to the
// counter's origin).  Two barriers; callers that reserve repeatedly alternate two ReserveSmem
// buffers (tile parity) so no third barrier is needed before the buffer is reused.
template <int BS = kBlock>
struct ReserveSmemT {
    u64 base;
    unsigned int total;
    unsigned int warp[BS / 32];
};
using ReserveSmem = ReserveSmemT<kBlock>;

template <int BS = kBlock>
__device__ __forceinline__ u64 block_reserve2(unsigned int c, u64 *counter, ReserveSmemT<BS> &sm)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int v = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= o)
            incl += v;
    }
    if (lane == 31)
        sm.warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const unsigned int w = lane < BS / 32 ? sm.warp[lane] : 0u;
        unsigned int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int v = __shfl_up_sync(FULL_MASK, wi, o);
            if (lane >= o)
                wi += v;
        }
        if (lane < BS / 32)
            sm.warp[lane] = wi - w;
        if (lane == BS / 32 - 1) {
            sm.total = wi;
            sm.base = wi ? atomicAdd(counter, (u64)wi) : 0ull;
        }
    }
    __syncthreads();
    return sm.base + sm.warp[wid] + (incl - c);
}

// Row v of an n x NW shared-memory bit matrix; NW == 2 rows are read as one 128-bit LDS
// (the tables start 16-byte aligned).
template <int NW>
__device__ __forceinline__ void lds_row(const u64 *base, uint32_t v, u64 (&r)[NW])
{
    if constexpr (NW == 2) {
        const ulonglong2 t = reinterpret_cast<const ulonglong2 *>(base)[v];
        r[0] = t.x;
        r[1] = t.y;
    } else {
#pragma unroll
        for (int w = 0; w < NW; ++w)
            r[w] = base[v * NW + w];
    }
}

// Split reservation.  reserve_begin: block scan (2 barriers) -> this thread's TILE-LOCAL offset;
// the last lane of warp 0 issues the global atomicAdd and keeps its (in-flight) result in
// *ticket.  That lane calls reserve_publish(ticket) later, after independent work, so the
// atomic's round trip overlaps that work instead of stalling every warp at a barrier; the base
// is visible to all threads after the caller's next barrier.
template <int BS = kBlock>
__device__ __forceinline__ unsigned int reserve_begin(unsigned int c, u64 *counter, ReserveSmemT<BS> &sm, u64 *ticket)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int v = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= o)
            incl += v;
    }
    if (lane == 31)
        sm.warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const unsigned int w = lane < BS / 32 ? sm.warp[lane] : 0u;
        unsigned int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int v = __shfl_up_sync(FULL_MASK, wi, o);
            if (lane >= o)
                wi += v;
        }
        if (lane < BS / 32)
            sm.warp[lane] = wi - w;
        if (lane == BS / 32 - 1) {
            sm.total = wi;
            *ticket = wi ? atomicAdd(counter, (u64)wi) : 0ull;
        }
    }
    __syncthreads();
    return sm.warp[wid] + (incl - c);
}

template <int BS = kBlock>
__device__ __forceinline__ bool is_ticket_lane() { return threadIdx.x == BS / 32 - 1; }

// single-buffer form: a third barrier protects sm before its next use
template <int BS = kBlock>
__device__ __forceinline__ u64 block_reserve(unsigned int c, u64 *counter, ReserveSmemT<BS> &sm)
{
    const u64 r = block_reserve2<BS>(c, counter, sm);
    __syncthreads();
    return r;
}

// Sequential appends at virtual output positions o, o+1, ...: the page's word-array base
// pointers are resolved once and again only when o crosses into the next page.
template <int RW>
struct Appender {
    u64 *w[RW];
    uint32_t *ids;
    uint32_t slot;
    u64 o;
    __device__ __forceinline__ void seek(const Pages &pg, u64 pos)
    {
        o = pos;
        const uint32_t page = pg.out_pages[o >> pg.log_p];
        slot = (uint32_t)(o & ((1ull << pg.log_p) - 1));
        char *pp = pg.base + (u64)page * pg.page_bytes;
#pragma unroll
        for (int k = 0; k < RW; ++k)
            w[k] = (u64 *)pp + ((u64)k << pg.log_p);
        ids = (uint32_t *)(pp + ((u64)RW << pg.log_p) * 8);
    }
    template <bool IDS>
    __device__ __forceinline__ void put_words(const Pages &pg, const u64 (&W)[RW], uint32_t id)
    {
        if (slot >> pg.log_p)  // crossed into the next page
            seek(pg, o);
#pragma unroll
        for (int k = 0; k < RW; ++k)
            w[k][slot] = W[k];
        if (IDS)
            ids[slot] = id;
        ++slot;
        ++o;
    }
    __device__ __forceinline__ void put(const Pages &pg, const u64 (&W)[RW], uint32_t id)
    {
        put_words<true>(pg, W, id);
    }
};

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

// Per-thread accumulators of a launch, block-reduced into the Scratch at the end (one atomic
// per counter per CTA).  *_next are the lookahead counters (see Scratch).
struct Acc {
    u64 cyc = 0, hash = 0, cand = 0, cyc_next = 0, cand_next = 0, paths_next = 0, paths_cur = 0, out_real = 0;
};

template <int BS = kBlock>
__device__ __forceinline__ void flush(Acc a, Scratch *sc)
{
    constexpr int K = 8;
    __shared__ u64 red[K][BS / 32];
    u64 v[K] = {a.cyc, a.hash, a.cand, a.cyc_next, a.cand_next, a.paths_next, a.paths_cur, a.out_real};
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
        u64 s = 0;
        for (int i = 0; i < BS / 32; ++i)
            s += red[threadIdx.x][i];
        // the eight counters are consecutive u64 fields of Scratch starting at `cycles`
        static_assert(offsetof(Scratch, out_real) - offsetof(Scratch, cycles) == 7 * sizeof(u64), "Scratch layout");
        if (s)
            atomicAdd(&sc->cycles + threadIdx.x, s);
    }
}

template <int BS = kBlock>
__device__ __forceinline__ void flush_accum(u64 cnt, u64 hs, u64 cand, Scratch *sc)
{
    Acc a;
    a.cyc = cnt;
    a.hash = hs;
    a.cand = cand;
    flush<BS>(a, sc);
}

// Graph tables staged in shared memory: adjacency bit rows (n*NW words), keys (n words) and,
// for NW <= 2, the byte key tables (8*NW*256 words).
template <int NW>
__host__ __device__ constexpr int keybyte_words()
{
    return NW <= kByteTableWords ? 8 * NW * 256 : 0;
}

template <int NW, bool KB = true>
__device__ __forceinline__ void stage_graph(const DevGraph &g, u64 *s_adj, u64 *s_key, u64 *s_kb)
{
    const int nrow = g.n * NW;
    for (int i = threadIdx.x; i < nrow; i += blockDim.x)
        s_adj[i] = g.adj[i];
    for (int i = threadIdx.x; i < g.n; i += blockDim.x)
        s_key[i] = g.key[i];
    if (KB)
        for (int i = threadIdx.x; i < keybyte_words<NW>(); i += blockDim.x)
            s_kb[i] = g.keybyte[i];
    __syncthreads();
}

// ---------------------------------------------------------------------------- TMA / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(u64 *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(u64 *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(u64 *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared through the TMA unit, completing bytes on the mbarrier
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, u64 *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int NW>
__device__ __forceinline__ void store_cycle(const LaunchArgs &p, const u64 (&S)[NW], uint32_t v,
                                            uint32_t v1, uint32_t v2)
{
    const u64 idx = atomicAdd(p.cyc.count, 1ull);
    if (idx < p.cyc.cap) {
#pragma unroll
        for (int w = 0; w < NW; ++w)
            p.cyc.s[(u64)w * p.cyc.cap + idx] = S[w] | bit_in_word(w, v);
        p.cyc.ids[idx] = v1 | (v2 << kIdBits);
    }
}

}  // namespace cc
