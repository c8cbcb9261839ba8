// cc_fused.cu -- k_expand_fused: Stage 2 (Alg. 3) of count mode for the
// grid class (bitset blocked-set records of NW <= 2 words, n <= 128, max degree <= 4), the
// HBM-bound workloads of SURVEY §8(d) (P8x8, P10x10 and the Table 1 grids).
//
// Two levels per launch.  The paper writes every frontier T' to global memory and relaunches
// (Alg. 4 l.4-7); here a launch reads F_t and writes F_{t+2}: the children
// <p,v> (F_{t+1}) live only in shared memory, where they are tested for closures and expanded
// in turn.  Per path the test is the one of k_expand_blocked (cc_kernels.cu), the dichotomy of
// PAPER.md:57-64 on the blocked-vertex record B(p) = N[v2] u ... u N[v_{t-1}]:
//   Cand = Adj(vt) & {v > v2} & ~B,  Close = Cand & Adj(v1),  Ext = Cand & ~Adj(v1)
//   child <p,v>: B' = B | N[vt], keysum' = keysum + key(v), ids' = (v1, v2, v).
// FUSE = 1 is the single-level form (last levels under a length cap; LEAF = last-level fusion).
//
// Warps are independent: no block-wide barrier inside the tile loop.  A warp takes tiles of 32
// consecutive input records (one per lane, loaded with coalesced 256-byte accesses, the next
// tile prefetched into registers), stages its children (and grandchildren) in its own slice of
// shared memory, and stores them with coalesced, consecutive-slot writes.  Output positions come
// from per-warp chunks of 2^log_ch slots (one atomicAdd per chunk, not per tile: the paper's
// serialized index allocation, amortised over a chunk).  The unused tail of a
// warp's last chunk is written as all-zero records ("empty slots": v1 == v2 == 0, which no path
// has), which every reader of such a level skips (k_expand_fused, k_expand_blocked,
// k_shard_filter); empty slots are at most warps x 2^log_ch per launch and the host sizes
// log_ch so that this is a small fraction of the launch's output.
#include "cc_device.cuh"

#include <algorithm>

namespace cc {

#ifdef CC_CHECKS
__device__ unsigned int g_fq_check;  // bit c: check c failed (debug builds only)
#define FQ_CHECK(cond, code)                        \
    do {                                            \
        if (!(cond))                                \
            atomicOr(&g_fq_check, 1u << (code));    \
    } while (0)
#else
#define FQ_CHECK(cond, code) \
    do {                     \
    } while (0)
#endif

unsigned int fused_check_flags(cudaStream_t st)
{
#ifdef CC_CHECKS
    unsigned int f = 0, z = 0;
    cudaMemcpyFromSymbolAsync(&f, g_fq_check, sizeof(f), 0, cudaMemcpyDeviceToHost, st);
    cudaMemcpyToSymbolAsync(g_fq_check, &z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    return f;
#else
    (void)st;
    return 0;
#endif
}

constexpr int kFBlock = 256;             // 8 independent warps; the CTA shares the graph tables
constexpr int kFWarps = kFBlock / 32;
constexpr int kFMaxCh = 3;               // Delta <= 4: at most 3 children per path
constexpr int kFCh1 = 32 * kFMaxCh;      // children of one warp tile
constexpr int kFCh2 = kFCh1 * kFMaxCh;   // grandchildren of one warp tile

template <int NW, bool PACK, int FUSE>
struct FusedWarpSmem {
    static constexpr int PW = NW + 1;                   // B | N[vt] (v1, v2 packed), keysum
    u64 par[32][PW];                                    // level-t parents with children
    u64 par2[FUSE == 2 ? kFCh1 : 1][PW];                // level-(t+1) children with children
    uint32_t pid[PACK ? 1 : 32];                        // unpacked ids: v1 | v2 << 10
    uint32_t pid2[(PACK || FUSE == 1) ? 1 : kFCh1];
    uint16_t ent1[kFCh1];                               // child: parent lane | v << 5
    uint16_t ent2[FUSE == 2 ? kFCh2 : 1];               // grandchild: child index | w << 7
};

template <int NW, bool PACK, int FUSE>
__host__ __device__ constexpr size_t fused_warp_bytes()
{
    return (sizeof(FusedWarpSmem<NW, PACK, FUSE>) + 15) & ~(size_t)15;
}

// remove and return the lowest element of the NW-word set x (x != 0)
template <int NW>
__device__ __forceinline__ uint32_t pop_lowest(u64 (&x)[NW])
{
    if constexpr (NW == 1) {
        const uint32_t b = (uint32_t)__ffsll((long long)x[0]) - 1;
        x[0] &= x[0] - 1;
        return b;
    } else {
        const bool lo = x[0] != 0ull;
        u64 w = lo ? x[0] : x[1];
        const uint32_t b = (uint32_t)__ffsll((long long)w) - 1 + (lo ? 0u : 64u);
        w &= w - 1;
        x[0] = lo ? w : x[0];
        x[1] = lo ? x[1] : w;
        return b;
    }
}

// Per-warp output cursor (warp-uniform): the current chunk of 2^log_ch slots.  log_ch is at
// least the largest single reservation (kFCh2 grandchildren), so a reservation never needs more
// than one new chunk, and a chunk (chunk-aligned, 2^log_ch <= page) never straddles a page.
struct WarpOut {
    char *pp = nullptr;   // page of the current chunk
    uint32_t slot = 0;    // next free slot in that page
    uint32_t left = 0;    // free slots left in the chunk
    bool dead = false;    // output overflow: the launch is discarded by the host
};

// Reserve T <= 2^log_ch slots: slot k < split is (pp0, s0 + k), the others (pp1, s1 + k - split).
__device__ __forceinline__ void warp_reserve(WarpOut &o, uint32_t T, uint32_t log_ch, const LaunchArgs &p,
                                             char *&pp0, uint32_t &s0, char *&pp1, uint32_t &s1, uint32_t &split)
{
    pp0 = pp1 = o.pp;
    s0 = s1 = o.slot;
    split = T;
    if (T <= o.left) {
        o.slot += T;
        o.left -= T;
        return;
    }
    u64 nb = 0;
    if ((threadIdx.x & 31) == 0)
        nb = atomicAdd(&p.sc->out_count, 1ull << log_ch);
    nb = __shfl_sync(FULL_MASK, nb, 0);
    if (nb + (1ull << log_ch) > p.out_cap) {
        if ((threadIdx.x & 31) == 0)
            p.sc->err = 1;
        o.dead = true;
        o.left = 0;
        return;
    }
    const u64 vo = p.out_off + nb;
    split = o.left;
    pp1 = page_ptr(p.pg, p.pg.out_pages[vo >> p.pg.log_p]);
    s1 = (uint32_t)(vo & ((1ull << p.pg.log_p) - 1));
    const uint32_t need = T - o.left;
    o.pp = pp1;
    o.slot = s1 + need;
    o.left = (1u << log_ch) - need;
}

// store record C (RW words, plus the ids word when unpacked) at `slot` of page pp
template <int RW, bool PACK>
__device__ __forceinline__ void put_record(char *pp, uint32_t slot, uint32_t log_p, const u64 (&C)[RW], uint32_t id)
{
    u64 *w0 = (u64 *)pp + slot;
#pragma unroll
    for (int w = 0; w < RW; ++w)
        w0[(u64)w << log_p] = C[w];
    if (!PACK)
        ((uint32_t *)(pp + ((u64)RW << log_p) * 8))[slot] = id;
}

#ifndef CC_FUSED_MINB
#define CC_FUSED_MINB 4  // resident CTAs per SM the register allocation must allow (4: 64 registers)
#endif
template <int NW, bool PACK, int FUSE, bool LEAF>
__global__ void __launch_bounds__(kFBlock, CC_FUSED_MINB) k_expand_fused(const LaunchArgs p, const uint32_t log_ch)
{
    static_assert(FUSE == 1 || !LEAF, "last-level fusion is single-level");
    constexpr int RW = NW + 1;
    using WS = FusedWarpSmem<NW, PACK, FUSE>;
    // packed ids: a fixed width per word count (the host packs with the same, cc_host.cpp)
    constexpr uint32_t IDB = PACK ? (NW == 1 ? 6 : 8) : (uint32_t)kIdBits;  // cc::packed_id_bits
    constexpr uint32_t IDM = (1u << IDB) - 1;
    constexpr uint32_t V12M = (1u << (2 * IDB)) - 1;
    constexpr u64 KEEP_V12 = PACK ? ~((u64)IDM << (64 - IDB)) : ~0ull;  // packed: clears the vt field
    extern __shared__ __align__(16) u64 smem[];
    const int n = p.g.n;
    u64 *s_adj = smem;                          // closed rows N[v] = Adj(v) | {v}
    u64 *s_above = s_adj + n * NW;              // label gate {x : x > v}
    u64 *s_key = s_above + n * NW;              // key(v)
    char *wbase = (char *)(s_key + ((n + 1) & ~1));
    WS &ws = *(WS *)(wbase + (threadIdx.x >> 5) * fused_warp_bytes<NW, PACK, FUSE>());
    for (int i = threadIdx.x; i < n * NW; i += kFBlock) {
        s_above[i] = above_word((uint32_t)(i / NW), i % NW);
        s_adj[i] = p.g.adj[i] | bit_in_word(i % NW, (uint32_t)(i / NW));
    }
    for (int i = threadIdx.x; i < n; i += kFBlock)
        s_key[i] = p.g.key[i];
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const uint32_t log_p = p.pg.log_p;
    const u64 nt = (p.n_in + 31) >> 5;
    const u64 tw = (u64)gridDim.x * kFWarps;
    WarpOut out;
    // per-lane statistics (a launch gives a lane at most ~10^6 paths)
    uint32_t n_in = 0, cnt1 = 0, cand1 = 0, n_next = 0, cnt2 = 0, cand2 = 0, written = 0;
    u64 hs = 0;

    auto load = [&](u64 wt, u64 (&X)[RW], uint32_t &xid) {
        const u64 r0 = wt << 5;
        const char *pp = page_ptr(p.pg, p.pg.in_pages[r0 >> log_p]);
        const uint32_t slot = (uint32_t)(r0 & ((1ull << log_p) - 1)) + lane;
#pragma unroll
        for (int w = 0; w < RW; ++w)
            X[w] = __ldcs((const u64 *)pp + ((u64)w << log_p) + slot);  // read once: evict first
        xid = PACK ? 0u : __ldcs((const uint32_t *)(pp + ((u64)RW << log_p) * 8) + slot);
    };
    // copy T staged records to consecutive output slots (uniform loop)
    auto emit = [&](uint32_t T, bool second) {
        if (T == 0 || out.dead)
            return;
        char *pp0, *pp1;
        uint32_t s0, s1, split;
        warp_reserve(out, T, log_ch, p, pp0, s0, pp1, s1, split);
        if (out.dead)
            return;
        written += T;  // every lane adds the warp's total; lane 0's copy is flushed
        for (uint32_t k = lane; k < T; k += 32) {
            uint32_t e, q, v;
            const u64 *par;
            uint32_t pid = 0;
            if (FUSE == 2 && second) {
                e = ws.ent2[k];
                q = e & 127;
                v = e >> 7;
                par = ws.par2[q];
                if (!PACK)
                    pid = ws.pid2[q];
            } else {
                e = ws.ent1[k];
                q = e & 31;
                v = e >> 5;
                par = ws.par[q];
                if (!PACK)
                    pid = ws.pid[q];
            }
            u64 C[RW];
#pragma unroll
            for (int w = 0; w < NW; ++w)
                C[w] = par[w];
            C[NW] = par[NW] + s_key[v];
            if (PACK)
                C[NW - 1] |= (u64)v << (64 - IDB);
            const bool lo = k < split;
            put_record<RW, PACK>(lo ? pp0 : pp1, lo ? s0 + k : s1 + (k - split), log_p, C, pid | (v << (2 * IDB)));
        }
    };

    u64 W[RW];
    uint32_t id = 0;
    u64 wt = blockIdx.x * (u64)kFWarps + (threadIdx.x >> 5);
    if (wt < nt)
        load(wt, W, id);
    for (; wt < nt && !out.dead; wt += tw) {
        u64 Wn[RW];
        uint32_t idn = 0;
        if (wt + tw < nt)
            load(wt + tw, Wn, idn);
        // ---------------------------------------------------------------- level t
        const u64 r = (wt << 5) + lane;
        const uint32_t ids = PACK ? (uint32_t)(W[NW - 1] >> (64 - 3 * IDB)) : id;
        const uint32_t v1 = ids & IDM, v2 = (ids >> IDB) & IDM, vt = ids >> (2 * IDB);
        const bool valid = r < p.n_in && v1 != v2;  // v1 == v2: an empty slot
        u64 ext[NW];
        uint32_t nc = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w)
            ext[w] = 0;
        if (valid) {
            n_in++;
            u64 arow[NW], abv[NW], a1[NW];
            lds_row<NW>(s_adj, vt, arow);
            lds_row<NW>(s_above, v2, abv);
            lds_row<NW>(s_adj, v1, a1);
            cand1 -= 1;  // deg(vt) = |N[vt]| - 1
            u64 close[NW];
            bool any_close = false;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                cand1 += __popcll(arow[w]);
                const u64 c = arow[w] & abv[w] & ~W[w];  // packed ids sit above bit n: not in arow
                close[w] = c & a1[w];
                ext[w] = p.emit ? (c & ~a1[w]) : 0ull;
                any_close |= close[w] != 0ull;
            }
            if (any_close && p.count) {
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    u64 m = close[w];
                    cnt1 += __popcll(m);
                    while (m) {
                        const int b = __ffsll((long long)m) - 1;
                        m &= m - 1;
                        hs += mix64(W[NW] + s_key[64 * w + b]);
                    }
                }
            }
            if constexpr (LEAF) {
                // children <p,v> are the last level: counted here, never written.
                // Close(<p,v>) = Adj(v) & Z(p), Z(p) = {x > v2} & ~(B | N[vt]) & Adj(v1)
                if (p.count) {
                    u64 Z[NW];
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        Z[w] = abv[w] & ~(W[w] | arow[w]) & a1[w];
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        u64 m = ext[w];
                        while (m) {
                            const int b = __ffsll((long long)m) - 1;
                            m &= m - 1;
                            const uint32_t v = (uint32_t)(64 * w + b);
                            u64 av[NW];
                            lds_row<NW>(s_adj, v, av);
                            const u64 ksv = W[NW] + s_key[v];
                            n_next++;
                            cand2 -= 1;
#pragma unroll
                            for (int w2 = 0; w2 < NW; ++w2) {
                                cand2 += __popcll(av[w2]);
                                u64 cl = av[w2] & Z[w2];
                                cnt2 += __popcll(cl);
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
                    ext[w] = 0;
            } else {
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    nc += __popcll(ext[w]);
                if (nc) {
                    // stage the parent: B | N[vt] (vt field cleared), keysum
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        ws.par[lane][w] = (W[w] | arow[w]) & (w == NW - 1 ? KEEP_V12 : ~0ull);
                    ws.par[lane][NW] = W[NW];
                    if (!PACK)
                        ws.pid[lane] = ids & V12M;
                }
            }
        }
        // warp scan of the child counts -> each child's entry (parent lane, vertex)
        uint32_t incl = nc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o)
                incl += x;
        }
        const uint32_t T1 = __shfl_sync(FULL_MASK, incl, 31);
        {
            const uint32_t off = incl - nc;
#pragma unroll
            for (uint32_t c = 0; c < (uint32_t)kFMaxCh; ++c)
                if (c < nc)
                    ws.ent1[off + c] = (uint16_t)(lane | (pop_lowest<NW>(ext) << 5));
        }
        __syncwarp();
        if constexpr (FUSE == 1) {
            emit(T1, false);
        } else {
            // ------------------------------------------------------------ level t+1 (in smem)
            uint32_t base2 = 0;
            for (uint32_t b = 0; b < T1; b += 32) {  // warp-uniform rounds of 32 children
                const uint32_t j = b + lane;
                uint32_t g = 0;
                u64 ex2[NW];
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    ex2[w] = 0;
                if (j < T1) {
                    const uint32_t e = ws.ent1[j];
                    const uint32_t q = e & 31, v = e >> 5;
                    u64 Bc[NW];
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        Bc[w] = ws.par[q][w];
                    const u64 ksc = ws.par[q][NW] + s_key[v];
                    const uint32_t cid = PACK ? (uint32_t)(Bc[NW - 1] >> (64 - 3 * IDB)) : ws.pid[q];
                    const uint32_t c1 = cid & IDM, c2 = (cid >> IDB) & IDM;
                    n_next++;
                    u64 arow[NW], abv[NW], a1[NW];
                    lds_row<NW>(s_adj, v, arow);
                    lds_row<NW>(s_above, c2, abv);
                    lds_row<NW>(s_adj, c1, a1);
                    cand2 -= 1;
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        cand2 += __popcll(arow[w]);
                        const u64 c = arow[w] & abv[w] & ~Bc[w];
                        u64 cl = c & a1[w];
                        ex2[w] = c & ~a1[w];
                        g += __popcll(ex2[w]);
                        if (p.count) {
                            cnt2 += __popcll(cl);
                            while (cl) {
                                const int bb = __ffsll((long long)cl) - 1;
                                cl &= cl - 1;
                                hs += mix64(ksc + s_key[64 * w + bb]);
                            }
                        }
                    }
                    if (g) {
#pragma unroll
                        for (int w = 0; w < NW; ++w)
                            ws.par2[j][w] = Bc[w] | arow[w];  // v1, v2 stay in the packed bits
                        ws.par2[j][NW] = ksc;
                        if (!PACK)
                            ws.pid2[j] = cid;
                    }
                }
                uint32_t inc2 = g;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t x = __shfl_up_sync(FULL_MASK, inc2, o);
                    if (lane >= o)
                        inc2 += x;
                }
                const uint32_t off2 = base2 + inc2 - g;
#pragma unroll
                for (uint32_t c = 0; c < (uint32_t)kFMaxCh; ++c)
                    if (c < g)
                        ws.ent2[off2 + c] = (uint16_t)(j | (pop_lowest<NW>(ex2) << 7));
                base2 += __shfl_sync(FULL_MASK, inc2, 31);
            }
            __syncwarp();
            emit(base2, true);
        }
        __syncwarp();  // the next tile overwrites par / ent
#pragma unroll
        for (int w = 0; w < RW; ++w)
            W[w] = Wn[w];
        id = idn;
    }
    // empty slots: the unused tail of the warp's last chunk
    if (!out.dead && out.left) {
        u64 Z[RW];
#pragma unroll
        for (int w = 0; w < RW; ++w)
            Z[w] = 0;
        for (uint32_t k = lane; k < out.left; k += 32)
            put_record<RW, PACK>(out.pp, out.slot + k, log_p, Z, 0u);
    }
    if (!p.count) {
        cand1 = cand2 = 0;
    }
    Acc a;
    a.cyc = cnt1;
    a.hash = hs;
    a.cand = cand1;
    a.cyc_next = cnt2;
    a.cand_next = cand2;
    a.paths_next = n_next;
    a.paths_cur = n_in;
    a.out_real = lane == 0 ? written : 0;
    flush<kFBlock>(a, p.sc);
}

// ---------------------------------------------------------------------------------------------
// k_expand_fq: the same two-level expansion (F_t -> F_{t+2}, packed records) organised as full
// 32-lane rounds.  A round is either an input round (32 paths of F_t, straight from the input
// tiles) or a child round (32 paths of F_{t+1} popped from the warp's child queue).  Children of
// an input round are pushed on the queue; children of a child round (F_{t+2}) are stored straight
// to HBM into per-warp chunks, one contiguous run per push step (CC_FQ_DIRECT; otherwise through
// an output queue flushed 32 records at a time).  Child rounds run whenever the queue holds >= 32
// paths, so every round but the warp's last few uses all 32 lanes, and the queue stays below
// 32 + 96 records.  Queue records carry B | N[vt] with v1, v2, vt packed and their parent's
// keysum (key(vt) is added when the record is popped): no parent references.  Input tiles come
// in dynamic chunks; children and closures are found with a byte gather over vt's neighbour
// slots (NbrSlots); pushes are branch-free (DESIGN.md §2 step 3a).
constexpr int kQCap = 32 + kFCh1;   // child queue / output queue capacity (records)

constexpr int kFqStages = 2;  // input tiles in flight per warp (cp.async ring; 3 or 4 stages cost resident warps)

#ifndef CC_FQ_PAIR
#define CC_FQ_PAIR 1  // input units of 64 records (16-byte copies, one issue per two input rounds)
#endif
constexpr uint32_t kFqLT = CC_FQ_PAIR ? 6 : 5;       // log2 records per input unit (ring stage)
constexpr uint32_t kFqTile = 1u << kFqLT;            // records per input unit
constexpr uint32_t kFqCPL = kFqTile / 32;            // consecutive records each lane copies
#ifndef CC_FQ_CHUNK
#define CC_FQ_CHUNK 64
#endif
#ifndef CC_FQ_BFTEST
#define CC_FQ_BFTEST 1  // the path test runs on every lane (invalid lanes masked), no branch
#endif
#ifndef CC_FQ_NOSPLIT
#define CC_FQ_NOSPLIT 1  // a child round's output never straddles chunks (the old tail -> empty slots)
#endif
constexpr uint32_t kFqChunk = CC_FQ_CHUNK / kFqCPL;  // input units per dynamic chunk (2048 records)
// Neighbour slots of a vertex v (max degree <= 4), for the byte gather of the extension set.
// Every child of a path ending in v is a neighbour of v, so the <= 3 set bits of Ext (an
// NW-word set, NW <= 2) lie in the bytes that hold v's neighbours u_0 < u_1 < ... (CSR order).
// Three byte permutes move byte u_k >> 3 of Ext into byte k of one 32-bit word g:
//   p_lo = prmt(e0, e1, sel), p_hi = prmt(e2, e3, sel)  (byte k: byte (u_k >> 3) & 7 of the half)
//   g    = prmt(p_lo, p_hi, pick) & m                   (byte k from p_lo or p_hi)
// where e0..e3 are the 32-bit quarters of Ext; m keeps bit u_k & 7 of byte k.  Bit 8k + (u_k & 7)
// of g is set iff u_k is a child, and the child's vertex is byte k of nb.
struct NbrSlots {
    uint32_t sel;   // nibble k = (u_k >> 3) & 7
    uint32_t pick;  // nibble k = k (u_k < 64) or 4 + k (u_k >= 64)
    uint32_t m;     // bit 8k + (u_k & 7) for every neighbour slot k
    uint32_t nb;    // byte k = u_k
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s)
{
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
    return d;
}


template <int NW>
struct FqWarpSmem {
    static constexpr int RW = NW + 1;
    u64 q[RW][kQCap + 1];  // child queue (F_{t+1}), SoA; slot kQCap takes the discarded stores
    u64 o[RW][CC_FQ_DIRECT ? 1 : kQCap + 1];  // output queue (F_{t+2}), SoA (unused with CC_FQ_DIRECT)
    u64 in[kFqStages][RW][kFqTile];  // input units, filled by cp.async (each lane copies kFqCPL records)
};

__device__ __forceinline__ void cp_async8(void *dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async_sa(uint32_t dst_sa, const void *src)
{
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_sa), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst_sa), "l"(src), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NW>
__host__ __device__ constexpr size_t fq_warp_bytes()
{
    return (sizeof(FqWarpSmem<NW>) + 15) & ~(size_t)15;
}

// 3 CTAs per SM and an 85-register budget: a 64-register cap (4 CTAs per SM, which shared memory
// allows since the output queue went) measured slower (P10x10 2.087 vs 1.979 s)
#ifndef CC_FQ_MINB
#define CC_FQ_MINB 3
#endif
template <int NW>
__global__ void __launch_bounds__(kFBlock, CC_FQ_MINB) k_expand_fq(const LaunchArgs p, const uint32_t log_ch)
{
    constexpr int RW = NW + 1;
    using WS = FqWarpSmem<NW>;
    constexpr uint32_t IDB = NW == 1 ? 6 : 8;  // packed records only (cc::packed_id_bits)
    constexpr uint32_t IDM = (1u << IDB) - 1;
    constexpr u64 KEEP_V12 = ~((u64)IDM << (64 - IDB));
    extern __shared__ __align__(16) u64 smem[];
    const int n = p.g.n;
    u64 *s_adj = smem;                          // closed rows N[v] = Adj(v) | {v}
    u64 *s_above = s_adj + n * NW;              // label gate {x : x > v}
    u64 *s_key = s_above + n * NW;              // key(v)
    NbrSlots *s_nbx = (NbrSlots *)(s_key + ((n + 1) & ~1));  // neighbour slots
    char *wbase = (char *)(s_nbx + ((n + 1) & ~1));
    WS &ws = *(WS *)(wbase + (threadIdx.x >> 5) * fq_warp_bytes<NW>());
    for (int i = threadIdx.x; i < n * NW; i += kFBlock) {
        s_above[i] = above_word((uint32_t)(i / NW), i % NW);
        s_adj[i] = p.g.adj[i] | bit_in_word(i % NW, (uint32_t)(i / NW));
    }
    for (int i = threadIdx.x; i < n; i += kFBlock) {
        s_key[i] = p.g.key[i];
        NbrSlots e{0u, 0u, 0u, 0u};
        const uint32_t r0 = p.g.rowptr[i], d = p.g.rowptr[i + 1] - r0;  // d <= 4 (host: max_deg)
        for (uint32_t k = 0; k < d; ++k) {
            const uint32_t u = p.g.col[r0 + k];
            e.sel |= ((u >> 3) & 7) << (4 * k);
            e.pick |= (u < 64 ? k : 4 + k) << (4 * k);
            e.m |= 1u << (8 * k + (u & 7));
            e.nb |= u << (8 * k);
        }
        s_nbx[i] = e;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const uint32_t log_p = p.pg.log_p;
    const u64 nt = (p.n_in + kFqTile - 1) >> kFqLT;  // input units
    const uint32_t key_sa = smem_u32(s_key);  // key(v) at key_sa + 8v (shared window)
    auto key_of = [&](uint32_t v) {
        u64 k;
        asm("ld.shared.u64 %0, [%1];" : "=l"(k) : "r"(key_sa + 8 * v));
        return k;
    };
    WarpOut out;
    uint32_t n_in = 0, cnt1 = 0, cand1 = 0, n_next = 0, cnt2 = 0, cand2 = 0, written = 0;
    u64 hs = 0;
    uint32_t nq = 0, no = 0;  // warp-uniform queue fills
#ifdef CC_FQ_CHECK_SELFTEST
    FQ_CHECK(blockIdx.x != 0 || threadIdx.x != 0, 7);  // negative control of the check plumbing
#endif

    // Input: the level's 32-record tiles are handed out in chunks of kFqChunk consecutive tiles
    // from a launch-wide counter (Scratch.in_next), so warps that issue faster take more chunks
    // (a static split left ~13% of the resident warps idle on average, mostly at the end).  The
    // next chunk's atomicAdd is issued one chunk ahead by lane 0, so its latency is hidden.
    // Tiles never straddle pages; the page pointer is looked up only when a chunk starts or
    // enters a new page, and src advances by one tile (32 records x 8 bytes per word array).
    static_assert(kFqStages == 2, "the per-stage lane limits below assume a 2-stage ring");
    const uint32_t tmask = (1u << (log_p - kFqLT)) - 1;  // units per page - 1
    const u64 wstride = 8ull << log_p;                // bytes between the word arrays of a page
    const uint32_t last_recs = (uint32_t)(p.n_in - ((nt - 1) << kFqLT));  // paths in the last unit
    u64 t_iss = 0, c_end = 0;                         // next tile to issue, end of its chunk
    u64 pend = 0;                                     // lane 0: start of the chunk after this one
    const char *src = nullptr;                        // this lane's word-0 address in tile t_iss
    auto locate = [&]() {
        const char *pp = page_ptr(p.pg, p.pg.in_pages[t_iss >> (log_p - kFqLT)]);
        src = pp + 8 * ((((uint32_t)t_iss & tmask) << kFqLT) + kFqCPL * lane);
    };
    {
        u64 c0 = 0;
        if (lane == 0) {
            c0 = atomicAdd(&p.sc->in_next, (u64)kFqChunk);
            pend = atomicAdd(&p.sc->in_next, (u64)kFqChunk);
        }
        t_iss = __shfl_sync(FULL_MASK, c0, 0);
        c_end = t_iss + kFqChunk < nt ? t_iss + kFqChunk : nt;
        if (t_iss < c_end)
            locate();
    }
    // one commit group per tile (empty groups past the end keep the wait counts uniform);
    // lim0 / lim1: paths in the tile of ring stage 0 / 1; infl: tiles issued and not yet read
    const uint32_t in_sa = smem_u32(&ws.in[0][0][kFqCPL * lane]);  // this lane's slot in ring stage 0
    uint32_t lim0 = 0, lim1 = 0, infl = 0;
    auto issue = [&](uint32_t stg) {
        if (t_iss < c_end) {
            FQ_CHECK(t_iss < nt && c_end <= nt && infl < (uint32_t)kFqStages, 2);
#pragma unroll
            for (int w = 0; w < RW; ++w)
                cp_async_sa<8 * kFqCPL>(in_sa + (stg * RW + w) * kFqTile * 8, src + w * wstride);
            const uint32_t lim = t_iss + 1 == nt ? last_recs : kFqTile;
            lim0 = stg ? lim0 : lim;
            lim1 = stg ? lim : lim1;
            ++infl;
            ++t_iss;
            src += kFqTile * 8;
            if (t_iss == c_end) {  // chunk done: continue with the one fetched a chunk ago
                t_iss = __shfl_sync(FULL_MASK, pend, 0);
                if (lane == 0 && t_iss < nt)
                    pend = atomicAdd(&p.sc->in_next, (u64)kFqChunk);
                c_end = t_iss + kFqChunk < nt ? t_iss + kFqChunk : nt;
                if (t_iss < c_end)
                    locate();
            } else if (((uint32_t)t_iss & tmask) == 0u) {
                locate();
            }
        }
        cp_async_commit();
    };
    // write the 32 (or, at the end, fewer) records at the end of the output queue; queue records
    // carry their parent's keysum, completed here with key(vt)
    // Output cursor: every reservation but the warp's last takes exactly 32 slots and a chunk
    // holds 2^log_ch >= 32 slots, so a reservation never straddles a chunk: the warp keeps one
    // pointer (this lane's word-0 address in the chunk) and the slots left in the chunk.
    u64 *optr = nullptr;
    uint32_t oleft = 0;
#if CC_FQ_DIRECT
    u64 *ocur = nullptr;  // word 0 of the warp's next free output slot (CC_FQ_DIRECT)
#endif
    auto flush_out = [&](uint32_t T) {
        if (T == 0 || out.dead)
            return;
        if (oleft == 0) {  // next chunk (warp-uniform)
            u64 nb = 0;
            if (lane == 0)
                nb = atomicAdd(&p.sc->out_count, 1ull << log_ch);
            nb = __shfl_sync(FULL_MASK, nb, 0);
            if (nb + (1ull << log_ch) > p.out_cap) {
                if (lane == 0)
                    p.sc->err = 1;
                out.dead = true;
                return;
            }
            const u64 vo = p.out_off + nb;
            optr = (u64 *)page_ptr(p.pg, p.pg.out_pages[vo >> log_p]) + (vo & ((1ull << log_p) - 1)) + lane;
            oleft = 1u << log_ch;
        }
        written += T;
        const uint32_t base = no - T;
        FQ_CHECK(T <= 32 && T <= oleft && no <= (uint32_t)kQCap, 4);
        if ((uint32_t)lane < T) {
            u64 C[RW];
#pragma unroll
            for (int w = 0; w < RW; ++w)
                C[w] = ws.o[w][base + lane];
            C[NW] += key_of((uint32_t)(C[NW - 1] >> (64 - IDB)));
#pragma unroll
            for (int w = 0; w < RW; ++w)
                *(u64 *)((char *)optr + w * wstride) = C[w];
        }
        optr += T;
        oleft -= T;
        no = base;
    };

    u64 W[RW];
    uint32_t stg_rd = 0;   // ring stage of the next input round
    uint32_t half_rd = 0;  // which 32 records of that stage (64-record units)
    uint32_t lim_cur = 0;  // paths in the unit being read
    issue(0u);
    for (;;) {
        const bool have_in = infl > 0 || half_rd != 0;
        // ---- pick the round: children first once 32 are queued (keeps the queue bounded)
        bool child_round, valid;
        if (nq >= 32 || (!have_in && nq > 0)) {
            child_round = true;
            const uint32_t take = nq < 32 ? nq : 32;
            valid = (uint32_t)lane < take;
            const uint32_t idx = nq - take + lane;
            FQ_CHECK(nq <= (uint32_t)kQCap, 0);
            if (valid) {
#pragma unroll
                for (int w = 0; w < RW; ++w)
                    W[w] = ws.q[w][idx];
            }
            nq -= take;
        } else if (have_in) {
            child_round = false;
            if (half_rd == 0) {
                cp_async_wait<kFqStages - 2>();  // the unit of stage stg_rd has landed
                if (kFqCPL > 1)
                    __syncwarp();  // ... including the records the other lanes copied
                lim_cur = stg_rd ? lim1 : lim0;
                FQ_CHECK(infl >= 1 && lim_cur >= 1 && lim_cur <= kFqTile, 1);
                --infl;
                issue(stg_rd ^ 1u);  // refill the stage read before this one
            }
#pragma unroll
            for (int w = 0; w < RW; ++w)
                W[w] = ws.in[stg_rd][w][32 * half_rd + lane];
            const uint32_t ids = (uint32_t)(W[NW - 1] >> (64 - 3 * IDB));
            valid = (uint32_t)lane + 32 * half_rd < lim_cur && (ids & IDM) != ((ids >> IDB) & IDM);  // empty slot: v1 == v2
            if (kFqCPL == 1 || half_rd == 1 || lim_cur <= 32) {
                half_rd = 0;
                stg_rd ^= 1u;
            } else {
                half_rd = 1;
            }
        } else {
            break;
        }
#if !CC_FQ_DIRECT
        __syncwarp();  // queue slots just read may be overwritten by this round's pushes
#endif
        // ---- expand the round's paths: test of Alg. 3 l.11-15 on the blocked set
        u64 ext[NW], base_rec[NW];
        uint32_t nc = 0;
        u64 ks = W[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w)
            ext[w] = 0;
        uint32_t gch = 0, gnb = 0;  // children as bits of the slot gather, vt's neighbour bytes
#if CC_FQ_BFTEST
        // branch-free: every lane runs the test; an invalid lane (no path, or an empty slot) tests
        // vertex 0 (a safe table index) and its children, closures and statistics are masked off
        {
            const uint32_t ids = valid ? (uint32_t)(W[NW - 1] >> (64 - 3 * IDB)) : 0u;
            const uint32_t vmask = valid ? ~0u : 0u;
#else
        if (valid) {
            const uint32_t ids = (uint32_t)(W[NW - 1] >> (64 - 3 * IDB));
#endif
            const uint32_t v1 = ids & IDM, v2 = (ids >> IDB) & IDM, vt = ids >> (2 * IDB);
            if (child_round)
                ks += key_of(vt);  // queue records carry the parent's keysum
            u64 arow[NW], abv[NW], a1[NW], close[NW];
            lds_row<NW>(s_adj, vt, arow);
            lds_row<NW>(s_above, v2, abv);
            lds_row<NW>(s_adj, v1, a1);
            bool any_close = false;
            const NbrSlots e = s_nbx[vt];
            const uint32_t deg = __popc(e.m) + 1;  // |N[vt]|: one mask bit per neighbour
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const u64 c = arow[w] & abv[w] & ~W[w];
                close[w] = c & a1[w];
                ext[w] = c & ~a1[w];
                any_close |= close[w] != 0ull;
                // B | N[vt]; the vt field is replaced when a child is pushed (IDB == 8: byte 3 of the
                // upper half, overwritten by the byte permute; else cleared here)
                base_rec[w] = (W[w] | arow[w]) & (w == NW - 1 && IDB != 8 ? KEEP_V12 : ~0ull);
            }
            {
                const uint32_t plo = prmt((uint32_t)ext[0], (uint32_t)(ext[0] >> 32), e.sel);
                const uint32_t phi = NW == 2 ? prmt((uint32_t)ext[NW - 1], (uint32_t)(ext[NW - 1] >> 32), e.sel) : 0u;
#if CC_FQ_BFTEST
                gch = prmt(plo, phi, e.pick) & e.m & vmask;
#else
                gch = prmt(plo, phi, e.pick) & e.m;
#endif
            }
            gnb = e.nb;
            nc = __popc(gch);
            uint32_t ncl = 0;
#if CC_FQ_BFTEST
            any_close = any_close && valid;
#endif
            if (any_close && p.count) {
                // closures are neighbours of vt too: the same byte gather turns Close into <= 3
                // slot bits of one word (one 32-bit loop instead of one 64-bit loop per word)
                const uint32_t clo = prmt((uint32_t)close[0], (uint32_t)(close[0] >> 32), e.sel);
                const uint32_t chi = NW == 2 ? prmt((uint32_t)close[NW - 1], (uint32_t)(close[NW - 1] >> 32), e.sel) : 0u;
                uint32_t gcl = prmt(clo, chi, e.pick) & e.m;
                ncl = __popc(gcl);
                while (gcl) {
                    uint32_t b;
                    asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(gcl));
                    gcl ^= 1u << b;
                    hs += mix64(ks + key_of(prmt(e.nb, 0u, 0x4440u | (b >> 3))));
                }
            }
#if CC_FQ_BFTEST
            const uint32_t dv = (deg - 1) & vmask, nv = valid ? 1u : 0u;
#else
            const uint32_t dv = deg - 1, nv = 1u;
#endif
            if (child_round) {
                n_next += nv;
                cand2 += dv;
                cnt2 += ncl;
            } else {
                n_in += nv;
                cand1 += dv;
                cnt1 += ncl;
            }
        }
        // ---- push the children: on the child queue (input round) or the output queue
#if CC_FQ_DIRECT
        if (child_round) {
            // F_{t+2}: step c writes every lane's c-th child; step c's children take the round's
            // slots [off_c, off_c + |step c|), in lane order, so each step's stores are one
            // contiguous run per word array.  The round reserves its T slots from the warp's
            // chunk (a new chunk when they do not fit: [0, split) in the old one, the rest in
            // the new one).  The records are complete: keysum + key(v).
            uint32_t lt;
            asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
            const uint32_t bs0 = __ballot_sync(FULL_MASK, nc > 0u), bs1 = __ballot_sync(FULL_MASK, nc > 1u),
                           bs2 = __ballot_sync(FULL_MASK, nc > 2u);
            const uint32_t n0 = __popc(bs0), n1 = __popc(bs1);
            const uint32_t T = n0 + n1 + __popc(bs2);
#if CC_FQ_NOSPLIT
            if (T > oleft) {  // next chunk (warp-uniform); the old chunk's tail becomes empty slots
                for (uint32_t k = lane; k < oleft; k += 32)
#pragma unroll
                    for (int w = 0; w < RW; ++w)
                        *(u64 *)((char *)(ocur + k) + w * wstride) = 0ull;
                u64 nb = 0;
                if (lane == 0)
                    nb = atomicAdd(&p.sc->out_count, 1ull << log_ch);
                nb = __shfl_sync(FULL_MASK, nb, 0);
                if (nb + (1ull << log_ch) > p.out_cap) {
                    if (lane == 0)
                        p.sc->err = 1;
                    out.dead = true;
                    break;
                }
                const u64 vo = p.out_off + nb;
                ocur = (u64 *)page_ptr(p.pg, p.pg.out_pages[vo >> log_p]) + (vo & ((1ull << log_p) - 1));
                oleft = 1u << log_ch;
            }
            u64 *const p0 = ocur;
            ocur += T;
            oleft -= T;
#else
            u64 *p0 = ocur, *p1 = ocur;
            uint32_t split = T;
            if (T > oleft) {  // next chunk (warp-uniform)
                u64 nb = 0;
                if (lane == 0)
                    nb = atomicAdd(&p.sc->out_count, 1ull << log_ch);
                nb = __shfl_sync(FULL_MASK, nb, 0);
                if (nb + (1ull << log_ch) > p.out_cap) {
                    if (lane == 0)
                        p.sc->err = 1;
                    out.dead = true;
                    break;
                }
                const u64 vo = p.out_off + nb;
                p1 = (u64 *)page_ptr(p.pg, p.pg.out_pages[vo >> log_p]) + (vo & ((1ull << log_p) - 1));
                split = oleft;
                ocur = p1 + (T - oleft);
                oleft = (1u << log_ch) - (T - oleft);
            } else {
                ocur += T;
                oleft -= T;
            }
#endif
            written += T;
#pragma unroll
            for (uint32_t c = 0; c < (uint32_t)kFMaxCh; ++c) {
                const uint32_t low = gch & (0u - gch);  // lowest slot bit (0 when none is left)
                gch ^= low;
                uint32_t b;
                asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(low));
                const uint32_t v = prmt(gnb, 0u, 0x4440u | (b >> 3));
                if (c < nc) {
                    const uint32_t j = (c == 0 ? 0u : c == 1 ? n0 : n0 + n1) +
                                       __popc((c == 0 ? bs0 : c == 1 ? bs1 : bs2) & lt);
                    FQ_CHECK(j < T && v < (uint32_t)n && (low >> b) == 1u, 6);
#if CC_FQ_NOSPLIT
                    char *dp = (char *)(p0 + j);
#else
                    char *dp = (char *)(j < split ? p0 + j : p1 + (j - split));
#endif
#pragma unroll
                    for (int w = 0; w < NW - 1; ++w)
                        *(u64 *)(dp + w * wstride) = base_rec[w];
                    if constexpr (IDB == 8) {
                        const uint32_t hi = prmt((uint32_t)(base_rec[NW - 1] >> 32), gnb, 0x4210u + ((b & 0x18u) << 9));
                        *(u64 *)(dp + (NW - 1) * wstride) = (base_rec[NW - 1] & 0xffffffffull) | ((u64)hi << 32);
                    } else {
                        *(u64 *)(dp + (NW - 1) * wstride) = base_rec[NW - 1] | ((u64)v << (64 - IDB));
                    }
                    *(u64 *)(dp + NW * wstride) = ks + key_of(v);
                }
            }
            __syncwarp();
            continue;
        }
#endif
#if CC_FQ_DIRECT
        // only input rounds write the queue: the slots popped by earlier (child) rounds must
        // have been read by every lane before this round's pushes may overwrite them
        __syncwarp();
#endif
        // nc <= 3 (two bits): the warp's exclusive prefix from two ballots instead of a 5-step
        // shuffle scan -- two independent votes instead of a serial chain (P10x10 3.135 -> 3.052 s)
        uint32_t incl, T;
        {
            const uint32_t b0 = __ballot_sync(FULL_MASK, nc & 1u), b1 = __ballot_sync(FULL_MASK, nc & 2u);
            uint32_t lt;
            asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
            incl = __popc(b0 & lt) + 2 * __popc(b1 & lt) + nc;
            T = __popc(b0) + 2 * __popc(b1);
        }
        {
#if CC_FQ_DIRECT
            u64(*dst)[kQCap + 1] = ws.q;  // child rounds stored their output above
#else
            u64(*dst)[kQCap + 1] = child_round ? ws.o : ws.q;
#endif
            uint32_t pos = (child_round ? no : nq) + incl - nc;
            // every lane runs the three steps; a lane without a c-th child stores to slot kQCap
#pragma unroll
            for (uint32_t c = 0; c < (uint32_t)kFMaxCh; ++c) {
                const uint32_t low = gch & (0u - gch);  // lowest slot bit (0 when none is left)
                gch ^= low;
                uint32_t b;  // its position (FLO; 0xffffffff when low == 0: a dummy-slot store)
                asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(low));
                const uint32_t v = prmt(gnb, 0u, 0x4440u | (b >> 3));
                FQ_CHECK(c >= nc || (pos + c < (uint32_t)kQCap && v < (uint32_t)n && (low >> b) == 1u), 3);
                const uint32_t slot = c < nc ? pos + c : (uint32_t)kQCap;
#pragma unroll
                for (int w = 0; w < NW - 1; ++w)
                    dst[w][slot] = base_rec[w];
                if constexpr (IDB == 8) {
                    // vt is byte 3 of the upper half: one byte permute puts v (byte k of gnb) there
                    const uint32_t hi = prmt((uint32_t)(base_rec[NW - 1] >> 32), gnb, 0x4210u + ((b & 0x18u) << 9));
                    dst[NW - 1][slot] = (base_rec[NW - 1] & 0xffffffffull) | ((u64)hi << 32);
                } else {
                    dst[NW - 1][slot] = base_rec[NW - 1] | ((u64)v << (64 - IDB));
                }
                dst[NW][slot] = ks;  // the child adds key(v) when it is read
            }
        }
        __syncwarp();
        FQ_CHECK(T <= 96 && (child_round ? no : nq) + T <= (uint32_t)kQCap, 5);
        if (child_round) {
            no += T;
            while (no >= 32 && !out.dead)
                flush_out(32);
        } else {
            nq += T;
        }
        if (out.dead)
            break;
    }
#if CC_FQ_DIRECT
    optr = ocur + lane;  // the unused tail starts at ocur
#else
    flush_out(no);  // the last partial group
#endif
    // empty slots: the unused tail of the warp's last chunk
    if (!out.dead && oleft) {
        u64 *z = optr - lane;  // slot 0 of the unused tail
        for (uint32_t k = lane; k < oleft; k += 32)
#pragma unroll
            for (int w = 0; w < RW; ++w)
                *(u64 *)((char *)(z + k) + w * wstride) = 0ull;
    }
    if (!p.count)
        cand1 = cand2 = 0;
    Acc a;
    a.cyc = cnt1;
    a.hash = hs;
    a.cand = cand1;
    a.cyc_next = cnt2;
    a.cand_next = cand2;
    a.paths_next = n_next;
    a.paths_cur = n_in;
    a.out_real = lane == 0 ? written : 0;
    flush<kFBlock>(a, p.sc);
}

template <int NW, bool PACK, int FUSE>
static size_t fused_smem_t(int n)
{
    return ((size_t)n * 2 * NW + ((n + 1) & ~1)) * sizeof(u64) + kFWarps * fused_warp_bytes<NW, PACK, FUSE>();
}

size_t fused_smem(int nw, int n, bool packed, int fuse)
{
    if (fuse == 3)
        return ((size_t)n * 2 * nw + ((n + 1) & ~1)) * sizeof(u64) +
               ((size_t)(n + 1) & ~(size_t)1) * sizeof(NbrSlots) +
               kFWarps * (nw == 1 ? fq_warp_bytes<1>() : fq_warp_bytes<2>());
    if (nw == 1)
        return packed ? (fuse == 2 ? fused_smem_t<1, true, 2>(n) : fused_smem_t<1, true, 1>(n))
                      : (fuse == 2 ? fused_smem_t<1, false, 2>(n) : fused_smem_t<1, false, 1>(n));
    return packed ? (fuse == 2 ? fused_smem_t<2, true, 2>(n) : fused_smem_t<2, true, 1>(n))
                  : (fuse == 2 ? fused_smem_t<2, false, 2>(n) : fused_smem_t<2, false, 1>(n));
}

typedef void (*FusedFn)(const LaunchArgs, const uint32_t);

static FusedFn fused_kernel(int nw, bool pk, int fuse, bool leaf)
{
    if (fuse == 3)
        return !pk || leaf ? nullptr : nw == 1 ? k_expand_fq<1> : nw == 2 ? k_expand_fq<2> : nullptr;
#define FK(N, PK)                                                                          \
    if (nw == N && pk == PK)                                                               \
        return fuse == 2 ? k_expand_fused<N, PK, 2, false>                                 \
                         : (leaf ? k_expand_fused<N, PK, 1, true> : k_expand_fused<N, PK, 1, false>);
    FK(1, true) FK(1, false) FK(2, true) FK(2, false)
#undef FK
    return nullptr;
}

int fused_warps_per_launch(int nw, int n, bool packed, int fuse, bool leaf, int sms)
{
    FusedFn f = fused_kernel(nw, packed, fuse, leaf);
    if (!f)
        return 0;
    const size_t smem = fused_smem(nw, n, packed, fuse);
    if (cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 0;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)f, kFBlock, smem) != cudaSuccess)
        return 0;
    return nb * sms * kFWarps;
}

cudaError_t launch_fused(const LaunchArgs &a, int fuse, bool leaf, uint32_t log_ch, int max_warps, cudaStream_t st)
{
    FusedFn f = fused_kernel(a.g.nw, a.packed != 0, fuse, leaf);
    // one reservation never needs more than one new chunk: <= kFCh2 records (fuse 1 / 2); fuse 3:
    // <= 96 (a child round's output, CC_FQ_DIRECT) or exactly 32 (output-queue flushes)
    if (!f || a.g.n > 128 || (1u << log_ch) < (fuse == 3 ? (1u << kFqMinLogChunk) : (uint32_t)kFCh2) ||
        (a.pg.log_p < log_ch) || max_warps < kFWarps)
        return cudaErrorInvalidValue;
    const size_t smem = fused_smem(a.g.nw, a.g.n, a.packed != 0, fuse);
    cudaError_t e = cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    const u64 tiles = (a.n_in + 31) / 32;
    u64 blocks = std::min<u64>((u64)max_warps / kFWarps, (tiles + kFWarps - 1) / kFWarps);
    if (blocks == 0)
        blocks = 1;
    f<<<(unsigned)blocks, kFBlock, smem, st>>>(a, log_ch);
    return cudaGetLastError();
}

}  // namespace cc
