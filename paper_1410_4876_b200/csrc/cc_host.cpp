// cc_host.cpp -- C ABI (include/chordless.h) and the host orchestrator of the hot path.
//
//   cc_graph_from_csr   CSR validation/normalisation, degree labelling
//                       (kept sequential on the host as the paper does),
//                       relabelling so that internal id == label, forward-pair prefix sums for
//                       Stage 1, adjacency bit rows (the bitmap form of PAPER.md:180 applied to
//                       the graph itself).
//   cc_enumerate        Alg. 4 HostProcess re-designed: instead of |V|-3
//                       blind relaunches over one T/T' pair, a stack of frontier ranges in one
//                       device arena.  Each step expands (a chunk of) the top level into the free
//                       space above it; whole levels are expanded at once while they fit, so the
//                       common case is plain level-synchronous BFS, and it degrades to
//                       depth-first over chunks when the next frontier would exceed the arena
//                       (the RAM<->GPU "data transportation" future work of PAPER.md:455).
//                       Early exit when a level is empty (reading G9).
#include "../../include/chordless.h"
#include "cc_internal.h"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <functional>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

using cc::u64;

namespace {

thread_local std::string g_last_error;

cc_status fail(cc_status s, const std::string &msg)
{
    g_last_error = msg;
    return s;
}

cc_status cuda_fail(cudaError_t e, const char *where)
{
    return fail(CC_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CC_CUDA(call)                                   \
    do {                                                \
        cudaError_t e__ = (call);                       \
        if (e__ != cudaSuccess)                         \
            return cuda_fail(e__, #call);               \
    } while (0)

double now_ms()
{
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

}  // namespace

// the library's private stream-ordered pool (defined below)
namespace {
cudaError_t pool_alloc(void **p, size_t bytes, int device, cudaStream_t st);
cudaMemPool_t lib_pool(int device);
}

// ------------------------------------------------------------------------------ graph
struct DevCopy {
    int device = -1;
    void *buf = nullptr;       // rowptr | col | fwd | pair_prefix | adj | orig | key
    size_t bytes = 0;
    u64 key_seed = 0;
    bool keys_valid = false;
    cc::DevGraph dg{};
};

struct cc_graph {
    int64_t n = 0, m = 0, max_deg = 0;
    std::vector<int32_t> label;     // original id -> label
    std::vector<int32_t> perm;      // label -> original id
    std::vector<uint32_t> irow;     // relabelled CSR (internal id == label)
    std::vector<uint32_t> icol;
    std::vector<uint32_t> ifwd;
    std::vector<u64> pair_prefix;
    int nw = 0;                     // words per bit row; 0 = outside every size class
    bool wide = false;              // 512 < n <= 2015: AoS warp-per-path class (count mode only)
    std::vector<u64> adj;
    double t_build_ms = 0;
    std::mutex mu;
    std::vector<DevCopy> dev;
};

extern "C" void cc_options_init(cc_options *o)
{
    if (!o)
        return;
    std::memset(o, 0, sizeof(*o));
    o->struct_size = sizeof(cc_options);
    o->device = -1;
    o->shard_count = 1;
}

extern "C" const char *cc_last_error(void) { return g_last_error.c_str(); }

extern "C" const char *cc_status_string(cc_status s)
{
    switch (s) {
    case CC_OK: return "CC_OK";
    case CC_ERR_INVALID_ARGUMENT: return "CC_ERR_INVALID_ARGUMENT";
    case CC_ERR_INVALID_VERTEX: return "CC_ERR_INVALID_VERTEX";
    case CC_ERR_SELF_LOOP: return "CC_ERR_SELF_LOOP";
    case CC_ERR_NOT_SYMMETRIC: return "CC_ERR_NOT_SYMMETRIC";
    case CC_ERR_CAPACITY: return "CC_ERR_CAPACITY";
    case CC_ERR_CUDA: return "CC_ERR_CUDA";
    case CC_ERR_NOT_COLLECTED: return "CC_ERR_NOT_COLLECTED";
    case CC_ERR_BUFFER_TOO_SMALL: return "CC_ERR_BUFFER_TOO_SMALL";
    case CC_ERR_TOO_LARGE: return "CC_ERR_TOO_LARGE";
    case CC_ERR_NO_DEVICE: return "CC_ERR_NO_DEVICE";
    }
    return "CC_ERR_UNKNOWN";
}

extern "C" const char *cc_version(void) { return "chordless-b200 0.1 (sm_100a)"; }

// Degree labelling: repeatedly delete a vertex of minimum degree in the
// remaining graph, l(u_i) = i; ties to the lowest original id.  Binary min-heap keyed
// (degree, id) with lazy deletion (a decremented vertex is pushed again; stale entries are
// skipped when popped): O((n + m) log(n + m)) with vector-backed constants.
static void degree_labeling(int64_t n, const std::vector<int64_t> &rp, const std::vector<int32_t> &cl,
                            std::vector<int32_t> &label)
{
    if (n > 0 && n <= 4096) {
        // small graphs: one n-bit set per degree; the next vertex is the lowest set bit of the
        // lowest non-empty degree (ties -> lowest id), O(n^2/64 + m) in all
        const int64_t words = (n + 63) / 64;
        int64_t maxd = 0;
        std::vector<int64_t> d(n);
        for (int64_t v = 0; v < n; ++v) {
            d[v] = rp[v + 1] - rp[v];
            maxd = std::max(maxd, d[v]);
        }
        std::vector<u64> bucket((size_t)(maxd + 1) * words, 0);
        for (int64_t v = 0; v < n; ++v)
            bucket[(size_t)d[v] * words + (v >> 6)] |= 1ull << (v & 63);
        label.assign(n, -1);
        int64_t cur = 0;
        for (int64_t i = 0; i < n; ++i) {
            int32_t u = -1;
            while (u < 0) {
                const u64 *b = &bucket[(size_t)cur * words];
                for (int64_t w = 0; w < words; ++w)
                    if (b[w]) {
                        u = (int32_t)(64 * w + __builtin_ctzll(b[w]));
                        break;
                    }
                if (u < 0)
                    ++cur;
            }
            bucket[(size_t)d[u] * words + (u >> 6)] &= ~(1ull << (u & 63));
            label[u] = (int32_t)i;
            for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
                const int32_t w = cl[k];
                if (label[w] < 0) {
                    bucket[(size_t)d[w] * words + (w >> 6)] &= ~(1ull << (w & 63));
                    --d[w];
                    bucket[(size_t)d[w] * words + (w >> 6)] |= 1ull << (w & 63);
                    cur = std::min(cur, d[w]);
                }
            }
        }
        return;
    }
    typedef std::pair<int64_t, int32_t> Key;
    std::vector<int64_t> d(n);
    std::vector<Key> heap;
    heap.reserve((size_t)n + cl.size());
    for (int64_t v = 0; v < n; ++v) {
        d[v] = rp[v + 1] - rp[v];
        heap.push_back({d[v], (int32_t)v});
    }
    std::make_heap(heap.begin(), heap.end(), std::greater<Key>());
    label.assign(n, -1);
    for (int64_t i = 0; i < n;) {
        std::pop_heap(heap.begin(), heap.end(), std::greater<Key>());
        const Key top = heap.back();
        heap.pop_back();
        const int32_t u = top.second;
        if (label[u] >= 0 || top.first != d[u])
            continue;  // stale entry
        label[u] = (int32_t)i++;
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
            const int32_t w = cl[k];
            if (label[w] < 0) {
                --d[w];
                heap.push_back({d[w], w});
                std::push_heap(heap.begin(), heap.end(), std::greater<Key>());
            }
        }
    }
}

extern "C" cc_status cc_graph_from_csr(int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                                       cc_graph **out)
{
    if (!out)
        return fail(CC_ERR_INVALID_ARGUMENT, "out is NULL");
    if (n < 0 || n > (1 << 20))
        return fail(CC_ERR_INVALID_ARGUMENT, "n must be in [0, 2^20]");
    if (n > 0 && !row_ptr)
        return fail(CC_ERR_INVALID_ARGUMENT, "row_ptr is NULL");
    const double t0 = now_ms();
    if (n > 0) {
        if (row_ptr[0] != 0)
            return fail(CC_ERR_INVALID_ARGUMENT, "row_ptr[0] != 0");
        for (int64_t v = 0; v < n; ++v)
            if (row_ptr[v + 1] < row_ptr[v])
                return fail(CC_ERR_INVALID_ARGUMENT, "row_ptr is decreasing");
        if (row_ptr[n] > 0 && !col_idx)
            return fail(CC_ERR_INVALID_ARGUMENT, "col_idx is NULL");
        if (row_ptr[n] > (int64_t)1 << 31)
            return fail(CC_ERR_INVALID_ARGUMENT, "more than 2^31 adjacency entries");
    }
    // normalise: sort + dedup each row, validate ids and self-loops
    std::vector<int64_t> rp(n + 1, 0);
    std::vector<int32_t> cl;
    cl.reserve(n > 0 ? (size_t)row_ptr[n] : 0);
    for (int64_t v = 0; v < n; ++v) {
        const size_t b = cl.size();
        for (int64_t k = row_ptr[v]; k < row_ptr[v + 1]; ++k) {
            const int32_t w = col_idx[k];
            if (w < 0 || w >= n)
                return fail(CC_ERR_INVALID_VERTEX, "vertex id " + std::to_string(w) + " in row " +
                                                       std::to_string(v) + " outside [0, n)");
            if (w == v)
                return fail(CC_ERR_SELF_LOOP, "self-loop at vertex " + std::to_string(v));
            cl.push_back(w);
        }
        if (!std::is_sorted(cl.begin() + b, cl.end()))
            std::sort(cl.begin() + b, cl.end());
        cl.erase(std::unique(cl.begin() + b, cl.end()), cl.end());
        rp[v + 1] = (int64_t)cl.size();
    }
    // symmetry: w in row v  <=>  v in row w.  Small graphs (every size class that runs, n <=
    // 2015): an n x n bit matrix, O(n^2/64 + m); larger ones: binary search per entry
    const bool small_n = n <= 4096;
    const int64_t mw = (n + 63) / 64;
    std::vector<u64> M(small_n ? (size_t)n * mw : 0, 0);
    if (small_n)
        for (int64_t v = 0; v < n; ++v)
            for (int64_t k = rp[v]; k < rp[v + 1]; ++k)
                M[(size_t)v * mw + (cl[k] >> 6)] |= 1ull << (cl[k] & 63);
    for (int64_t v = 0; v < n; ++v)
        for (int64_t k = rp[v]; k < rp[v + 1]; ++k) {
            const int32_t w = cl[k];
            const bool rev = small_n ? ((M[(size_t)w * mw + (v >> 6)] >> (v & 63)) & 1ull) != 0
                                     : std::binary_search(cl.begin() + rp[w], cl.begin() + rp[w + 1], (int32_t)v);
            if (!rev)
                return fail(CC_ERR_NOT_SYMMETRIC, "edge (" + std::to_string(v) + "," +
                                                      std::to_string(w) + ") has no reverse entry");
        }

    cc_graph *g = new cc_graph();
    g->n = n;
    g->m = (int64_t)cl.size() / 2;
    for (int64_t v = 0; v < n; ++v)
        g->max_deg = std::max<int64_t>(g->max_deg, rp[v + 1] - rp[v]);
    degree_labeling(n, rp, cl, g->label);
    g->perm.assign(n, 0);
    for (int64_t v = 0; v < n; ++v)
        g->perm[g->label[v]] = (int32_t)v;
    // relabelled CSR: row of internal vertex i = labels of the neighbours of perm[i], sorted
    g->irow.assign(n + 1, 0);
    g->icol.resize(cl.size());
    g->ifwd.assign(n, 0);
    g->pair_prefix.assign(n + 1, 0);
    // rows in label space: small graphs scatter the relabelled edges into a label-space bit
    // matrix and read each row back in order (no per-row sort)
    std::vector<u64> LM(small_n ? (size_t)n * mw : 0, 0);
    if (small_n)
        for (int64_t v = 0; v < n; ++v) {
            const int64_t lv = g->label[v];
            for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
                const int32_t lw = g->label[cl[e]];
                LM[(size_t)lv * mw + (lw >> 6)] |= 1ull << (lw & 63);
            }
        }
    for (int64_t i = 0; i < n; ++i) {
        const int32_t v = g->perm[i];
        const uint32_t b = g->irow[i];
        uint32_t k = b;
        if (small_n) {
            for (int64_t w = 0; w < mw; ++w) {
                u64 x = LM[(size_t)i * mw + w];
                while (x) {
                    g->icol[k++] = (uint32_t)(64 * w + __builtin_ctzll(x));
                    x &= x - 1;
                }
            }
        } else {
            for (int64_t e = rp[v]; e < rp[v + 1]; ++e)
                g->icol[k++] = (uint32_t)g->label[cl[e]];
            std::sort(g->icol.begin() + b, g->icol.begin() + k);
        }
        g->irow[i + 1] = k;
        uint32_t f = b;
        while (f < k && g->icol[f] <= (uint32_t)i)
            ++f;
        g->ifwd[i] = f;
        const u64 dplus = k - f;
        g->pair_prefix[i + 1] = g->pair_prefix[i] + dplus * (dplus - 1) / 2;
    }
    int wide_nw = 0;
    if (n > 64 * cc::kMaxWords) {
        // wide class: enough words that v1, v2, vt pack into the spare top bits
        wide_nw = (int)((n + 3 * cc::id_bits((int)n) + 63) / 64);
        if (wide_nw > cc::kWideMaxWords)
            wide_nw = 0;
    }
    if (n <= 64 * cc::kMaxWords || wide_nw) {
        g->nw = wide_nw ? wide_nw : (n > 0 ? (int)((n + 63) / 64) : 1);
        g->wide = wide_nw != 0;
        g->adj.assign((size_t)n * g->nw, 0);
        if (small_n && g->nw >= mw) {
            for (int64_t i = 0; i < n; ++i)
                std::copy(LM.begin() + (size_t)i * mw, LM.begin() + (size_t)(i + 1) * mw,
                          g->adj.begin() + (size_t)i * g->nw);
        } else {
            for (int64_t i = 0; i < n; ++i)
                for (uint32_t k = g->irow[i]; k < g->irow[i + 1]; ++k) {
                    const uint32_t w = g->icol[k];
                    g->adj[(size_t)i * g->nw + (w >> 6)] |= 1ull << (w & 63);
                }
        }
    }
    g->t_build_ms = now_ms() - t0;
    *out = g;
    return CC_OK;
}

extern "C" void cc_graph_free(cc_graph *g)
{
    if (!g)
        return;
    int cur = -1;
    cudaGetDevice(&cur);
    for (auto &d : g->dev)
        if (d.buf) {
            cudaSetDevice(d.device);
            cudaFreeAsync(d.buf, 0);  // stream-ordered: no device-wide synchronisation
        }
    if (cur >= 0)
        cudaSetDevice(cur);
    delete g;
}

extern "C" cc_status cc_graph_info(const cc_graph *g, int64_t *n, int64_t *m, int64_t *max_degree)
{
    if (!g)
        return fail(CC_ERR_INVALID_ARGUMENT, "graph is NULL");
    if (n)
        *n = g->n;
    if (m)
        *m = g->m;
    if (max_degree)
        *max_degree = g->max_deg;
    return CC_OK;
}

extern "C" cc_status cc_graph_labels(const cc_graph *g, int32_t *labels)
{
    if (!g || (!labels && g->n > 0))
        return fail(CC_ERR_INVALID_ARGUMENT, "NULL argument");
    std::copy(g->label.begin(), g->label.end(), labels);
    return CC_OK;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static cc_status upload_graph(cc_graph *g, int device, cudaStream_t st, DevCopy *dc, uint64_t *h2d);

// Upload (once per device) the relabelled graph; recompute keys when the seed changes.
static cc_status ensure_device_graph(cc_graph *g, int device, u64 seed, cudaStream_t st, DevCopy **out,
                                     uint64_t *h2d)
{
    DevCopy *dc = nullptr;
    for (auto &d : g->dev)
        if (d.device == device)
            dc = &d;
    const int64_t n = g->n;
    if (!dc) {
        // built in a local copy and added to g->dev only when every upload succeeded: a failed
        // allocation must not leave a half-built entry that a later call would run on
        DevCopy nd;
        cc_status s = upload_graph(g, device, st, &nd, h2d);
        if (s != CC_OK) {
            if (nd.buf)
                cudaFreeAsync(nd.buf, st);
            return s;
        }
        g->dev.push_back(nd);
        dc = &g->dev.back();
    }
    if (!dc->keys_valid || dc->key_seed != seed) {
        CC_CUDA(cc::launch_keys((u64 *)dc->dg.key, (u64 *)dc->dg.keybyte, dc->dg.orig, (int)n, g->nw, seed, st));
        dc->key_seed = seed;
        dc->keys_valid = true;
    }
    *out = dc;
    return CC_OK;
}

static cc_status upload_graph(cc_graph *g, int device, cudaStream_t st, DevCopy *dc, uint64_t *h2d)
{
    const int64_t n = g->n;
    {
        dc->device = device;
        const size_t s_row = align_up((n + 1) * 4, 256), s_col = align_up(std::max<size_t>(g->icol.size(), 1) * 4, 256),
                     s_fwd = align_up(std::max<int64_t>(n, 1) * 4, 256), s_pp = align_up((n + 1) * 8, 256),
                     s_adj = align_up(std::max<size_t>(g->adj.size(), 1) * 8, 256),
                     s_orig = align_up(std::max<int64_t>(n, 1) * 4, 256), s_key = align_up(std::max<int64_t>(n, 1) * 8, 256),
                     s_kb = g->nw <= cc::kByteTableWords ? align_up((size_t)8 * g->nw * 256 * 8, 256) : 256;
        // wide sparse graphs: the neighbour-mask table of the last-level fusion (cc_internal.h)
        const bool want_nm = g->wide && g->max_deg <= 32;
        const size_t s_nm = want_nm ? align_up((size_t)n * n * 4, 256) : 0;
        dc->bytes = s_row + s_col + s_fwd + s_pp + s_adj + s_orig + s_key + s_kb + s_nm;
        // from the library's pool: a fresh graph per call (the e2e path) then reuses the same
        // memory without cudaMalloc / cudaFree, each of which synchronises the whole device
        CC_CUDA(pool_alloc(&dc->buf, dc->bytes, device, st));
        char *p = (char *)dc->buf;
        auto *rowptr = (uint32_t *)p; p += s_row;
        auto *col = (uint32_t *)p; p += s_col;
        auto *fwd = (uint32_t *)p; p += s_fwd;
        auto *pp = (u64 *)p; p += s_pp;
        auto *adj = (u64 *)p; p += s_adj;
        auto *orig = (int32_t *)p; p += s_orig;
        auto *key = (u64 *)p; p += s_key;
        auto *keybyte = (u64 *)p; p += s_kb;
        auto *nbrmask = want_nm ? (uint32_t *)p : nullptr;
        CC_CUDA(cudaMemcpyAsync(rowptr, g->irow.data(), (n + 1) * 4, cudaMemcpyHostToDevice, st));
        if (!g->icol.empty())
            CC_CUDA(cudaMemcpyAsync(col, g->icol.data(), g->icol.size() * 4, cudaMemcpyHostToDevice, st));
        if (n > 0) {
            CC_CUDA(cudaMemcpyAsync(fwd, g->ifwd.data(), n * 4, cudaMemcpyHostToDevice, st));
            CC_CUDA(cudaMemcpyAsync(orig, g->perm.data(), n * 4, cudaMemcpyHostToDevice, st));
        }
        CC_CUDA(cudaMemcpyAsync(pp, g->pair_prefix.data(), (n + 1) * 8, cudaMemcpyHostToDevice, st));
        if (!g->adj.empty())
            CC_CUDA(cudaMemcpyAsync(adj, g->adj.data(), g->adj.size() * 8, cudaMemcpyHostToDevice, st));
        *h2d += (n + 1) * 4 + g->icol.size() * 4 + n * 8 + (n + 1) * 8 + g->adj.size() * 8;
        dc->dg.n = (int32_t)n;
        dc->dg.nw = g->nw;
        dc->dg.rowptr = rowptr;
        dc->dg.col = col;
        dc->dg.fwd = fwd;
        dc->dg.pair_prefix = pp;
        dc->dg.adj = adj;
        dc->dg.key = key;
        dc->dg.keybyte = keybyte;
        dc->dg.orig = orig;
        dc->dg.nbrmask = nbrmask;
        if (nbrmask) {
            CC_CUDA(cudaMemsetAsync(nbrmask, 0, (size_t)n * n * 4, st));
            CC_CUDA(cc::launch_nbrmask(dc->dg, nbrmask, st));
        }
    }
    return CC_OK;
}

// ------------------------------------------------------------------------------ result
struct cc_result {
    int64_t n = 0;
    std::vector<u64> counts, paths, cand;
    u64 hash = 0;
    cc_stats stats{};
    bool collected = false;
    int device = -1;
    cudaStream_t stream = nullptr;  // cc_options.stream of the enumeration (cc_fetch_cycles uses it)
    int nw = 1;
    void *cyc_buf = nullptr;     // CycleStore s | ids, then adj copy, orig copy
    cc::CycleStore cyc{};
    u64 *adj = nullptr;
    int32_t *orig = nullptr;
    u64 n_cyc = 0;
};

extern "C" void cc_result_free(cc_result *r)
{
    if (!r)
        return;
    if (r->cyc_buf) {
        int cur = -1;
        cudaGetDevice(&cur);
        cudaSetDevice(r->device);
        cudaFreeAsync(r->cyc_buf, r->stream);
        // collect stores can be gigabytes: return them to the driver, not to the pool's cache
        cudaStreamSynchronize(r->stream);
        cudaMemPoolTrimTo(lib_pool(r->device), 256ull << 20);
        if (cur >= 0)
            cudaSetDevice(cur);
    }
    delete r;
}
namespace {

// Scoped device allocation on a stream (stream-ordered allocator).
struct DevBuf {
    void *p = nullptr;
    cudaStream_t st = nullptr;
    cudaMemPool_t trim_pool = nullptr;  // large blocks: give the memory back to the driver
    ~DevBuf()
    {
        if (p)
            cudaFreeAsync(p, st);
        if (p && trim_pool) {
            cudaStreamSynchronize(st);
            cudaMemPoolTrimTo(trim_pool, 64ull << 20);
        }
    }
};

// Per-thread pinned host staging (scratch read-back, page tables).
struct Pinned {
    void *p = nullptr;
    size_t bytes = 0;
    ~Pinned()
    {
        if (p)
            cudaFreeHost(p);
    }
    cudaError_t reserve(size_t b)
    {
        if (b <= bytes)
            return cudaSuccess;
        if (p)
            cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMallocHost(&p, b);
        if (e == cudaSuccess)
            bytes = b;
        return e;
    }
};
thread_local Pinned t_pinned;

// The library's own stream-ordered pool per device (small control blocks, fetch scratch and
// a library-allocated arena when cc_options.workspace is NULL).  Private, so that keeping freed
// blocks cached (release threshold = max) never takes memory from torch or other users of the
// device's default pool; the arena itself is trimmed back to the driver after every call.
cudaMemPool_t lib_pool(int device)
{
    static std::mutex mu;
    static std::vector<std::pair<int, cudaMemPool_t>> pools;
    std::lock_guard<std::mutex> lk(mu);
    for (auto &p : pools)
        if (p.first == device)
            return p.second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
        cudaGetLastError();
        cudaDeviceGetDefaultMemPool(&pool, device);
    } else {
        u64 thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pools.push_back({device, pool});
    return pool;
}

cudaError_t pool_alloc(void **p, size_t bytes, int device, cudaStream_t st)
{
    return cudaMallocFromPoolAsync(p, bytes, lib_pool(device), st);
}

// One frontier level F_t: a list of arena pages, all full except the last.
struct Level {
    std::vector<uint32_t> pages;
    u64 count = 0;
    bool sharded = false;   // paths already partitioned between shards (owned by this one);
                            // set whenever the level is (re)filled: from its parent at commit,
                            // or from a Stage-1 chunk
    double fan = 0;         // observed output slots per input slot of this level's launches (0 = unknown)
    int fan_fuse = -1;      // the launch kind `fan` was observed for (fuse 0 / 1 / 2)
    double fan1 = 0;        // observed |F_{t+1}| / |F_t| (one level), 0 = unknown
    bool shard_now = false; // unsharded level whose expansion does not fit: partition it first
};

}  // namespace

// Copy records [from, from + cnt) of arena page `src` to slots [0, cnt) of page `dst`:
// structure-of-arrays pages (record_bytes / 8 word arrays of P words, then a u32 ids array when
// record_bytes % 8 == 4) or, for the wide class, array-of-structures records.
static cudaError_t copy_records(char *base, u64 page_bytes, uint32_t lp, u64 rec_bytes, bool aos, uint32_t src,
                                u64 from, u64 cnt, uint32_t dst, cudaStream_t st)
{
    const u64 P = 1ull << lp;
    char *ps = base + (u64)src * page_bytes, *pd = base + (u64)dst * page_bytes;
    if (aos)
        return cudaMemcpyAsync(pd, ps + from * rec_bytes, cnt * rec_bytes, cudaMemcpyDeviceToDevice, st);
    const u64 words = rec_bytes / 8;
    cudaError_t e = cudaMemcpy2DAsync(pd, P * 8, ps + from * 8, P * 8, cnt * 8, words, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && rec_bytes % 8)
        e = cudaMemcpyAsync(pd + words * P * 8, ps + words * P * 8 + from * 4, cnt * 4, cudaMemcpyDeviceToDevice, st);
    return e;
}

static cc_status enumerate_impl(const cc_graph *cg, const cc_options *opt_in, cc_result **out,
                                u64 *need_cycles)
{
    const double t_wall0 = now_ms();
    if (!cg || !out)
        return fail(CC_ERR_INVALID_ARGUMENT, "NULL argument");
    cc_options opt;
    cc_options_init(&opt);
    if (opt_in) {
        if (opt_in->struct_size < sizeof(uint32_t) || opt_in->struct_size > sizeof(cc_options))
            return fail(CC_ERR_INVALID_ARGUMENT, "cc_options.struct_size mismatch");
        std::memcpy(&opt, opt_in, opt_in->struct_size);
    }
    if (opt.shard_count < 1 || opt.shard_index >= opt.shard_count)
        return fail(CC_ERR_INVALID_ARGUMENT, "need 0 <= shard_index < shard_count");
    if (opt.root_stride > 1 && opt.root_offset >= opt.root_stride)
        return fail(CC_ERR_INVALID_ARGUMENT, "need root_offset < root_stride");
    cc_graph *g = const_cast<cc_graph *>(cg);
    const int64_t n = g->n;
    if (n > 0 && g->nw == 0)
        return fail(CC_ERR_TOO_LARGE, "n = " + std::to_string(n) + " exceeds the supported size classes (n <= 2015)");

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(CC_ERR_NO_DEVICE, "no CUDA device");
    int device = opt.device;
    if (device < 0)
        CC_CUDA(cudaGetDevice(&device));
    if (device >= ndev)
        return fail(CC_ERR_NO_DEVICE, "device ordinal out of range");
    CC_CUDA(cudaSetDevice(device));
    cudaStream_t st = (cudaStream_t)opt.stream;
    const u64 seed = opt.hash_seed ? opt.hash_seed : 0x1410487600000000ULL;

    std::lock_guard<std::mutex> lk(g->mu);
    cc_result *res = new cc_result();
    std::unique_ptr<cc_result, void (*)(cc_result *)> res_guard(res, cc_result_free);
    res->n = n;
    res->counts.assign(n + 3, 0);
    res->paths.assign(n + 2, 0);
    res->cand.assign(n + 2, 0);
    res->device = device;
    res->stream = st;
    res->nw = std::max(g->nw, 1);
    res->collected = opt.collect != 0;
    cc_stats &S = res->stats;
    S.struct_size = sizeof(cc_stats);
    S.n_words = res->nw;
    S.t_labeling_ms = g->t_build_ms;

    if (n < 3) {  // no cycle possible
        S.t_wall_ms = now_ms() - t_wall0;
        *out = res_guard.release();
        return CC_OK;
    }
    int sms = 0;
    CC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));

    DevCopy *dc = nullptr;
    {
        cc_status s = ensure_device_graph(g, device, seed, st, &dc, &S.h2d_bytes);
        if (s != CC_OK)
            return s;
    }
    const int nw = g->nw;
    // count mode runs on blocked-vertex records (B-mode); collect mode keeps the bitmap S
    const cc::Mode mode = opt.collect ? cc::Mode::S : cc::Mode::B;
    // B-mode records carry v1, v2, vt in the spare top bits of the blocked set when n allows
    const bool wide = g->wide;
    const bool packed = wide || (mode == cc::Mode::B && cc::packable(nw, (int)n));
    // list class: the path's vertex list instead of its blocked set, for sparse
    // wide graphs under a length cap (written paths have <= max(3, max_len - 2) vertices)
    // (collect mode too: the list kernels store each cycle as its vertex list, cc::CycleStore.lw)
    const bool list_ok = wide && opt.max_len >= 4 && opt.max_len <= (uint32_t)cc::kListMaxLen && g->max_deg <= 32;
    if (opt.record_format > 2)
        return fail(CC_ERR_INVALID_ARGUMENT, "record_format must be 0, 1 or 2");
    if (opt.record_format == 2 && !list_ok)
        return fail(CC_ERR_INVALID_ARGUMENT, "record_format 2 (vertex list) needs count mode, 512 < n <= 2015, "
                                             "max degree <= 32 and 4 <= max_len <= " +
                                                 std::to_string(cc::kListMaxLen));
    const bool list = opt.record_format == 2 || (opt.record_format == 0 && list_ok);
    if (wide && opt.collect && !list)
        return fail(CC_ERR_TOO_LARGE, "collect mode above n = " + std::to_string(64 * cc::kMaxWords) +
                                          " needs the vertex-list records: max degree <= 32 and 4 <= max_len <= " +
                                          std::to_string(cc::kListMaxLen) + " (n = " + std::to_string(n) + ")");
    const int rwl = list ? std::max<int>(2, (std::max<int>(3, (int)opt.max_len - 2) + 3) / 4) : 0;
    const u64 rec_bytes = list ? (u64)(rwl + 2) * 8 : (u64)cc::record_bytes(nw, mode, packed);
    S.record_bytes = rec_bytes;
    S.record_format = list ? 2 : 1;

    // ---- frontier arena, split into pages of P = 2^lp records
    DevBuf ws_own;
    ws_own.st = st;
    void *ws = opt.workspace;
    u64 ws_bytes = opt.workspace_bytes;
    if (!ws) {
        if (ws_bytes == 0) {
            size_t fr = 0, tot = 0;
            CC_CUDA(cudaMemGetInfo(&fr, &tot));
            ws_bytes = std::max<u64>(fr / 4, 64ull << 20);
        }
        CC_CUDA(pool_alloc(&ws_own.p, ws_bytes, device, st));
        ws_own.trim_pool = lib_pool(device);
        ws = ws_own.p;
    }
    uint32_t lp = 20;  // 1 Mi records per page, fewer if the arena would have < 64 pages
    while (lp > (uint32_t)cc::kMinLogPage && (ws_bytes / (((u64)1 << lp) * rec_bytes)) < 64)
        --lp;
    const u64 P = (u64)1 << lp;
    const u64 page_bytes = P * rec_bytes;
    const u64 npages = ws_bytes / page_bytes;
    if (npages < 2)
        return fail(CC_ERR_CAPACITY, "workspace of " + std::to_string(ws_bytes) + " B holds fewer than 2 pages of " +
                                         std::to_string(P) + " records");
    S.arena_capacity = npages * P;
    std::vector<uint32_t> free_pages;
    free_pages.reserve(npages);
    for (u64 i = npages; i-- > 0;)
        free_pages.push_back((uint32_t)i);

    // ---- control block: Scratch | page table (in pages, then out pages)
    DevBuf ctrl;
    ctrl.st = st;
    // two Scratch blocks (the second for the launch chained after Stage 1), then the page tables
    const size_t ctrl_bytes = 2 * sizeof(cc::Scratch) + (size_t)2 * npages * 4 + 256;
    CC_CUDA(pool_alloc(&ctrl.p, ctrl_bytes, device, st));
    CC_CUDA(cudaMemsetAsync(ctrl.p, 0, sizeof(cc::Scratch), st));
    cc::Scratch *d_sc = (cc::Scratch *)ctrl.p;
    cc::Scratch *d_sc2 = d_sc + 1;
    uint32_t *d_tab = (uint32_t *)((char *)ctrl.p + 2 * sizeof(cc::Scratch));
    CC_CUDA(t_pinned.reserve(2 * sizeof(cc::Scratch) + (size_t)2 * npages * 4 + 64));
    cc::Scratch *h_sc = (cc::Scratch *)t_pinned.p;
    cc::Scratch *h_sc2 = h_sc + 1;
    uint32_t *h_tab = (uint32_t *)((char *)t_pinned.p + 2 * sizeof(cc::Scratch));

    // ---- collect store
    if (opt.collect) {
        const u64 ccap = opt.collect_capacity ? opt.collect_capacity : (1ull << 22);
        // list class: rwl + 1 words of 16-bit ids per cycle (<= max_len vertices); else S + ids
        const uint32_t lw = list ? (uint32_t)rwl + 1 : 0;
        const size_t s_s = align_up(ccap * (lw ? lw : nw) * 8, 256), s_ids = align_up(ccap * 4, 256),
                     s_adj = align_up((size_t)n * nw * 8, 256), s_orig = align_up((size_t)n * 4, 256);
        CC_CUDA(pool_alloc(&res->cyc_buf, s_s + s_ids + s_adj + s_orig, device, st));
        char *p = (char *)res->cyc_buf;
        res->cyc.s = (u64 *)p;
        res->cyc.ids = (uint32_t *)(p + s_s);
        res->cyc.cap = ccap;
        res->cyc.count = &d_sc->cyc_count;
        res->cyc.lw = lw;
        res->adj = (u64 *)(p + s_s + s_ids);
        res->orig = (int32_t *)(p + s_s + s_ids + s_adj);
        CC_CUDA(cudaMemcpyAsync(res->adj, dc->dg.adj, (size_t)n * nw * 8, cudaMemcpyDeviceToDevice, st));
        CC_CUDA(cudaMemcpyAsync(res->orig, dc->dg.orig, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    }

    cc::LaunchArgs base{};
    base.g = dc->dg;
    base.pg.base = (char *)ws;
    base.pg.page_bytes = page_bytes;
    base.pg.log_p = lp;
    base.pg.in_pages = d_tab;
    base.pg.out_pages = d_tab + npages;
    base.cyc = res->cyc;
    base.sc = d_sc;
    base.collect = opt.collect ? 1 : 0;
    base.root_stride = opt.root_stride;
    base.root_offset = opt.root_offset;
    base.shard_index = opt.shard_index;
    base.shard_count = opt.shard_count;
    // packed bitset records: a fixed id width per word count (6 bits for NW = 1, 8 for NW = 2,
    // cc::packed_id_bits), so the kernels see it as a constant
    base.idb = (uint32_t)(packed && !wide && nw <= 2 ? cc::packed_id_bits(nw, (int)n) : cc::id_bits((int)n));
    base.packed = packed ? 1 : 0;

    const cc::ExpandVariant variant = (mode == cc::Mode::B && g->max_deg <= 4) ? cc::ExpandVariant::Small
                                      : g->max_deg <= 32                      ? cc::ExpandVariant::Thread
                                                                              : cc::ExpandVariant::Warp;
    const size_t gsmem = ((size_t)n * (nw + 1) + (nw <= cc::kByteTableWords ? (size_t)8 * nw * 256 : 0)) * 8;
    const int grid_s1 = (list ? cc::max_blocks_per_sm_list(0, rwl)
                         : wide ? cc::max_blocks_per_sm_wide(0) : cc::max_blocks_per_sm(0, mode, nw, packed, gsmem)) * sms;
    const int grid_ex =
        (list ? cc::max_blocks_per_sm_list(1, rwl)
         : wide ? cc::max_blocks_per_sm_wide(1)
              : cc::max_blocks_per_sm(variant == cc::ExpandVariant::Small ? 4 : variant == cc::ExpandVariant::Thread ? 1 : 2,
                                      mode, nw, packed, cc::expand_smem(mode, nw, (int)n, packed))) * sms;
    const int grid_sf = (list ? cc::max_blocks_per_sm_list(2, rwl)
                         : wide ? cc::max_blocks_per_sm_wide(2) : cc::max_blocks_per_sm(3, mode, nw, packed, 0)) * sms;
    const double maxfan = (double)std::max<int64_t>(g->max_deg - 1, 1);
    // Grid class (count mode, bitset records of <= 2 words, max degree <= 4): large levels are
    // expanded by k_expand_fused (cc_fused.cu), two levels per launch where the length cap allows
    const bool fused_ok = mode == cc::Mode::B && !wide && !list && nw <= 2 && n <= 128 && g->max_deg <= 4 &&
                          std::getenv("CC_NO_FUSED") == nullptr;
    const u64 fused_min = std::getenv("CC_FUSED_MIN") ? std::strtoull(std::getenv("CC_FUSED_MIN"), nullptr, 10)
                                                       : (1ull << 24);
    const bool fq_on = !(std::getenv("CC_FQ") && std::getenv("CC_FQ")[0] == '0');
    int fused_warps[4] = {-1, -1, -1, -1};  // resident warps of the fused kernels: fuse 2, 1, 1 + leaf, 3
    auto fwarps = [&](int fuse, bool leaf) {
        const int i = fuse == 3 ? 3 : fuse == 2 ? 0 : leaf ? 2 : 1;
        if (fused_warps[i] < 0)
            fused_warps[i] = cc::fused_warps_per_launch(nw, (int)n, packed, fuse, leaf, sms);
        return fused_warps[i];
    };
    const uint32_t W = opt.shard_count;
    // Multi-GPU partition: the first frontier level with >= threshold paths is
    // split by content hash.  Deep enough that the heavy-tailed subtree sizes average out (P10x10
    // at W = 8: max/mean shard time 1.37 at 1024 paths per shard, 1.01 at 2^20 -- measured,
    // profiles/), while the levels above it (expanded redundantly by every rank) stay small.
    // Stage 1 is split instead when its pair space alone is large (e.g. K_{150,150}).
    const u64 shard_threshold = (u64)(opt.min_shard_paths ? opt.min_shard_paths : (1u << 20)) * W;
    const u64 s1_shard_threshold = (u64)(opt.min_shard_paths ? opt.min_shard_paths : (1u << 16)) * W;
    const uint32_t max_len = opt.max_len;
    const bool want_paths = max_len == 0 || max_len >= 4;

    cudaEvent_t ev0, ev1, ea, eb, em;
    CC_CUDA(cudaEventCreate(&ev0));
    CC_CUDA(cudaEventCreate(&ev1));
    CC_CUDA(cudaEventCreate(&ea));
    CC_CUDA(cudaEventCreate(&eb));
    CC_CUDA(cudaEventCreate(&em));
    struct EvGuard {
        cudaEvent_t e[5];
        ~EvGuard()
        {
            for (auto x : e)
                cudaEventDestroy(x);
        }
    } evg{{ev0, ev1, ea, eb, em}};
    CC_CUDA(cudaEventRecord(ev0, st));

    u64 cyc_committed = 0;   // collect-store counter after the last committed launch
    u64 in_use = 0, high_water = 0;

    // Launch one kernel over the page list `in` (or a Stage-1 pair range) writing into the
    // free pages; on success the used output pages are returned in `used` and the scratch
    // in *h_sc.  Returns CC_OK, or CC_ERR_CAPACITY with *overflow set when the output did not
    // fit (nothing is committed: the caller retries with less input).
    // Optional per-launch trace (env CC_TRACE=<file>): one CSV line per kernel launch -- the
    // evolution of |T| and |C| per step that the paper plots in Fig. 4.
    struct TraceFile {
        FILE *f = nullptr;
        ~TraceFile()
        {
            if (f)
                fclose(f);
        }
    } trace;
    if (const char *tp = std::getenv("CC_TRACE")) {
        trace.f = std::fopen(tp, "a");
        if (trace.f)
            std::fprintf(trace.f, "kind,level,paths_in,children_out,cycles,candidates,ms,overflow,paths_real,"
                                  "paths_next,out_real,fuse\n");
    }
    enum Kind { STAGE1, EXPAND, FILTER };
    int trace_level = 0;
    // emit: the launch creates paths (children / triplets); leaf: last-level fusion (count the
    // children, write none -- cc::Scratch)
    // fuse (EXPAND only): 0 = k_expand_blocked & co., 1 / 2 = k_expand_fused over 1 / 2 levels
    // with output chunks of 2^log_ch slots.  On success *real_in / *real_out are the paths read and
    // records written (the fused and blocked kernels skip and leave empty slots; the others equal
    // n_in and the output count).
    u64 real_in = 0, real_out = 0;
    auto launch = [&](Kind kind, const uint32_t *in, size_t n_in_pages, u64 n_in, u64 pair_lo, bool emit,
                      bool leaf, bool count, bool filter, std::vector<uint32_t> &used,
                      bool *overflow, int fuse = 0, uint32_t log_ch = 0) -> cc_status {
        *overflow = false;
        const bool writes = emit && !leaf;
        const size_t nfree = free_pages.size();
        // page table: input pages, then every free page (in pop order) as potential output
        for (size_t i = 0; i < n_in_pages; ++i)
            h_tab[i] = in[i];
        for (size_t i = 0; i < nfree; ++i)
            h_tab[npages + i] = free_pages[nfree - 1 - i];
        if (n_in_pages)
            CC_CUDA(cudaMemcpyAsync(d_tab, h_tab, n_in_pages * 4, cudaMemcpyHostToDevice, st));
        if (writes && nfree)
            CC_CUDA(cudaMemcpyAsync(d_tab + npages, h_tab + npages, nfree * 4, cudaMemcpyHostToDevice, st));
        S.h2d_bytes += (n_in_pages + (writes ? nfree : 0)) * 4;
        CC_CUDA(cudaMemsetAsync(d_sc, 0, offsetof(cc::Scratch, cyc_count), st));
        cc::LaunchArgs a = base;
        a.in_lo = pair_lo;
        a.n_in = n_in;
        a.out_off = 0;
        a.out_cap = writes ? nfree * P : 0;
        a.emit = emit ? 1 : 0;
        a.emit_next = leaf ? 0 : 1;
        a.count = count ? 1 : 0;
        a.filter = filter ? 1 : 0;
        if (opt.profile)
            CC_CUDA(cudaEventRecord(ea, st));
        // NVTX range per launch ("expand L<t> f<fuse>", "stage1", "filter L<t>"): profilers can
        // select one level, e.g. ncu --nvtx --nvtx-include "expand L44 f2/" (tools/)
        char nv[48];
        std::snprintf(nv, sizeof(nv), "%s L%d f%d", kind == STAGE1 ? "stage1" : kind == EXPAND ? "expand" : "filter",
                      trace_level, fuse);
        nvtxRangePushA(nv);
        a.tlen = (uint32_t)trace_level;  // vertices per input path of an expansion
        if (list)
            CC_CUDA(cc::launch_list(kind == STAGE1 ? 0 : kind == EXPAND ? 1 : 2, a, rwl, leaf, st,
                                    kind == STAGE1 ? grid_s1 : kind == EXPAND ? grid_ex : grid_sf));
        else if (wide)
            CC_CUDA(cc::launch_wide(kind == STAGE1 ? 0 : kind == EXPAND ? 1 : 2, a, st,
                                    kind == STAGE1 ? grid_s1 : kind == EXPAND ? grid_ex : grid_sf));
        else if (kind == STAGE1)
            CC_CUDA(cc::launch_stage1(a, mode, st, grid_s1));
        else if (kind == EXPAND && fuse)
        {
            // no more warps than a quarter of the free output in chunks (small arenas)
            const u64 cap_warps = std::max<u64>(8, a.out_cap / (4ull << log_ch));
            // two levels on packed records: the full-round queue kernel (k_expand_fq) unless CC_FQ=0
            const int kf = fuse == 2 && packed && fq_on ? 3 : fuse;
            CC_CUDA(cc::launch_fused(a, kf, leaf, log_ch, (int)std::min<u64>((u64)fwarps(kf, leaf), cap_warps), st));
        }
        else if (kind == EXPAND)
            CC_CUDA(cc::launch_expand(a, mode, variant, st, grid_ex));
        else
            CC_CUDA(cc::launch_shard_filter(a, mode, st, grid_sf));
        if (opt.profile)
            CC_CUDA(cudaEventRecord(eb, st));
        nvtxRangePop();
        CC_CUDA(cudaMemcpyAsync(h_sc, d_sc, sizeof(cc::Scratch), cudaMemcpyDeviceToHost, st));
        CC_CUDA(cudaStreamSynchronize(st));
#ifdef CC_CHECKS
        if (const unsigned int fl = cc::fused_check_flags(st))
            return fail(CC_ERR_CUDA, "k_expand_fq bounds check failed (flags " + std::to_string(fl) + ")");
#endif
        S.d2h_bytes += sizeof(cc::Scratch);
        S.launches++;
        float ms = 0;
        if (opt.profile) {
            CC_CUDA(cudaEventElapsedTime(&ms, ea, eb));
            if (kind == STAGE1)
                S.t_stage1_ms += ms;
            else if (kind == EXPAND)
                S.t_expand_ms += ms;
        }
        if (trace.f)
            std::fprintf(trace.f, "%s,%d,%llu,%llu,%llu,%llu,%.6f,%d,%llu,%llu,%llu,%d\n",
                         kind == STAGE1 ? "stage1" : kind == EXPAND ? "expand" : "filter", trace_level,
                         (unsigned long long)n_in, (unsigned long long)h_sc->out_count,
                         (unsigned long long)(h_sc->cycles + h_sc->cycles_next),
                         (unsigned long long)(h_sc->cand + h_sc->cand_next), ms,
                         (h_sc->err || h_sc->out_count > a.out_cap) ? 1 : 0,
                         (unsigned long long)h_sc->paths_cur, (unsigned long long)h_sc->paths_next,
                         (unsigned long long)h_sc->out_real, fuse);
        if (h_sc->err || h_sc->out_count > a.out_cap) {
            *overflow = true;
            if (opt.collect) {  // roll back the cycles this launch stored
                CC_CUDA(cudaMemcpyAsync(&d_sc->cyc_count, &cyc_committed, 8, cudaMemcpyHostToDevice, st));
                CC_CUDA(cudaStreamSynchronize(st));
            }
            return CC_OK;
        }
        cyc_committed = h_sc->cyc_count;
        const bool reports = kind == EXPAND && mode == cc::Mode::B && !wide && !list;
        real_in = reports ? h_sc->paths_cur : n_in;
        real_out = reports ? h_sc->out_real : h_sc->out_count;
        if (kind != FILTER)
            S.paths_written += real_out;
        const u64 npg = (h_sc->out_count + P - 1) / P;
        used.clear();
        for (u64 i = 0; i < npg; ++i) {
            used.push_back(free_pages.back());
            free_pages.pop_back();
        }
        return CC_OK;
    };

    std::vector<Level> levels(n + 3);
    const bool count_tri = opt.shard_index == 0 && (opt.root_stride <= 1 || opt.root_offset == 0) &&
                           (max_len == 0 || max_len >= 3);
    const u64 stage1_total = g->pair_prefix[n];
    S.stage1_pairs = stage1_total;
    u64 s1_next = 0;
    // shard at Stage 1 when the seed space alone is large enough (deterministic: graph-only)
    const bool s1_filter = W > 1 && stage1_total >= s1_shard_threshold;
    int deepest = 2;  // levels 3..deepest may be non-empty
    // small-frontier fast path (cc::SmallArgs): count mode, bitset records, n <= 128, one shard
    const bool small_ok = mode == cc::Mode::B && !wide && !list && nw <= 2 && W == 1 &&
                          std::getenv("CC_NO_SMALL") == nullptr;
    bool small_tried = false;
    std::vector<uint32_t> used;

    while (true) {
        while (deepest >= 3 && levels[deepest].count == 0)
            --deepest;
        if (deepest < 3) {
            // ---- Stage 1 (Alg. 2): the next chunk of forward pairs -> F_3 and triangles
            if (s1_next >= stage1_total)
                break;
            const u64 c = std::min<u64>(stage1_total - s1_next, (u64)free_pages.size() * P);
            if (c == 0)
                return fail(CC_ERR_CAPACITY, "no free arena page for Stage 1");
            // ---- Stage 1 chained with the expansion of all of F_3: both launches are queued
            //      back to back and read back with ONE host round trip (no synchronisation in
            //      between).  The expansion reads Stage 1's output size from the device.  Bitset
            //      count mode outside the small-frontier path (e.g. K_{150,150}), one shard, all
            //      pairs in one chunk.  If the expansion's output overflows, it is discarded and
            //      F_3 continues on the ordinary path.
            const size_t nfree0 = free_pages.size();
            const u64 k1 = (c + P - 1) / P;
            const int d3 = 3;
            const bool emit3 = max_len == 0 || (u64)d3 + 1 < max_len;
            const bool leaf3 = emit3 && max_len != 0 && (u64)d3 + 2 >= max_len;
            const bool chain = mode == cc::Mode::B && !wide && !list && W == 1 && s1_next == 0 && c == stage1_total &&
                               want_paths && !(small_ok && nw <= 2) && nfree0 > k1 &&
                               std::getenv("CC_NO_CHAIN") == nullptr;
            if (chain) {
                for (size_t i = 0; i < nfree0; ++i)
                    h_tab[npages + i] = free_pages[nfree0 - 1 - i];
                CC_CUDA(cudaMemcpyAsync(d_tab + npages, h_tab + npages, nfree0 * 4, cudaMemcpyHostToDevice, st));
                S.h2d_bytes += nfree0 * 4;
                CC_CUDA(cudaMemsetAsync(d_sc, 0, 2 * sizeof(cc::Scratch), st));
                cc::LaunchArgs a1 = base;
                a1.in_lo = 0;
                a1.n_in = c;
                a1.out_off = 0;
                a1.out_cap = k1 * P;
                a1.emit = 1;
                a1.emit_next = 1;
                a1.count = count_tri ? 1 : 0;
                a1.filter = 0;
                cc::LaunchArgs a2 = base;
                a2.sc = d_sc2;
                a2.pg.in_pages = d_tab + npages;  // Stage 1's output pages, in table order
                a2.n_in = c;  // an upper bound, for the grid size; the kernel reads the real count
                a2.n_in_dev = &d_sc->out_count;
                a2.out_off = k1 * P;
                a2.out_cap = emit3 && !leaf3 ? (nfree0 - k1) * P : 0;
                a2.emit = emit3 ? 1 : 0;
                a2.emit_next = leaf3 ? 0 : 1;
                a2.count = 1;
                a2.tlen = 3;
                if (opt.profile)
                    CC_CUDA(cudaEventRecord(ea, st));
                nvtxRangePushA("stage1+expand L3 chained");
                CC_CUDA(cc::launch_stage1(a1, mode, st, grid_s1));
                if (opt.profile)
                    CC_CUDA(cudaEventRecord(em, st));
                CC_CUDA(cc::launch_expand(a2, mode, variant, st, grid_ex));
                if (opt.profile)
                    CC_CUDA(cudaEventRecord(eb, st));
                nvtxRangePop();
                CC_CUDA(cudaMemcpyAsync(h_sc, d_sc, 2 * sizeof(cc::Scratch), cudaMemcpyDeviceToHost, st));
                CC_CUDA(cudaStreamSynchronize(st));
                S.d2h_bytes += 2 * sizeof(cc::Scratch);
                S.launches += 2;
                if (opt.profile) {
                    float m1 = 0, m2 = 0;
                    CC_CUDA(cudaEventElapsedTime(&m1, ea, em));
                    CC_CUDA(cudaEventElapsedTime(&m2, em, eb));
                    S.t_stage1_ms += m1;
                    S.t_expand_ms += m2;
                }
                if (h_sc->err || h_sc->out_count > a1.out_cap)
                    return fail(CC_ERR_CAPACITY, "Stage 1 output overflow (internal sizing error)");
                const bool ok2 = !h_sc2->err && h_sc2->out_count <= a2.out_cap;
                if (trace.f) {
                    std::fprintf(trace.f, "stage1,2,%llu,%llu,%llu,0,0,0,0,0,%llu,0\n", (unsigned long long)c,
                                 (unsigned long long)h_sc->out_count, (unsigned long long)h_sc->cycles,
                                 (unsigned long long)h_sc->out_count);
                    std::fprintf(trace.f, "expand,3,%llu,%llu,%llu,%llu,0,%d,%llu,%llu,%llu,0\n",
                                 (unsigned long long)h_sc->out_count, (unsigned long long)h_sc2->out_count,
                                 (unsigned long long)(h_sc2->cycles + h_sc2->cycles_next),
                                 (unsigned long long)(h_sc2->cand + h_sc2->cand_next), ok2 ? 0 : 1,
                                 (unsigned long long)h_sc2->paths_cur, (unsigned long long)h_sc2->paths_next,
                                 (unsigned long long)h_sc2->out_real);
                }
                s1_next += c;
                S.chunks++;
                S.paths_written += h_sc->out_count;
                res->counts[3] += h_sc->cycles;
                res->hash += h_sc->hash;
                const u64 u1 = (h_sc->out_count + P - 1) / P;
                const u64 n3 = h_sc->out_count;
                // pages of the table in use afterwards: F_3 (if kept) and F_4 (if expanded)
                std::vector<char> keep(nfree0, 0);
                Level &L3 = levels[3];
                Level &L4 = levels[4];
                if (ok2) {
                    S.chunks++;
                    S.rounds = std::max<u64>(S.rounds, 3);
                    const u64 rin = h_sc2->paths_cur, rout = h_sc2->out_real;
                    res->paths[3] += rin;
                    res->cand[3] += h_sc2->cand;
                    S.paths_expanded += rin;
                    res->counts[4] += h_sc2->cycles;
                    res->hash += h_sc2->hash;
                    if (leaf3) {
                        res->paths[4] += h_sc2->paths_next;
                        res->cand[4] += h_sc2->cand_next;
                        res->counts[5] += h_sc2->cycles_next;
                        S.paths_expanded += h_sc2->paths_next;
                        S.leaf_paths += h_sc2->paths_next;
                    }
                    S.paths_written += rout;
                    S.bytes_alg += (rin + rout) * rec_bytes;
                    S.records_levelsync += rin + rout + (leaf3 ? 2 * h_sc2->paths_next : 0);
                    S.slots_moved += n3 + h_sc2->out_count;
                    if (rin > 0)
                        L3.fan1 = (double)(leaf3 ? h_sc2->paths_next : rout) / (double)rin;
                    if (n3 > 0) {
                        L3.fan = (double)h_sc2->out_count / (double)n3;
                        L3.fan_fuse = 0;
                    }
                    const u64 u2 = (h_sc2->out_count + P - 1) / P;
                    L4.pages.clear();
                    for (u64 i = 0; i < u2; ++i) {
                        keep[k1 + i] = 1;
                        L4.pages.push_back(h_tab[npages + k1 + i]);
                    }
                    L4.count = h_sc2->out_count;
                    L4.sharded = true;
                    L4.shard_now = false;
                    in_use += L4.count;
                    high_water = std::max(high_water, std::max<u64>(n3, in_use));
                    deepest = L4.count ? 4 : 2;
                } else {
                    L3.pages.clear();
                    for (u64 i = 0; i < u1; ++i) {
                        keep[i] = 1;
                        L3.pages.push_back(h_tab[npages + i]);
                    }
                    L3.count = n3;
                    L3.sharded = true;
                    L3.shard_now = false;
                    in_use += n3;
                    high_water = std::max(high_water, in_use);
                    deepest = 3;
                }
                // the free list keeps its pop order (table order) minus the pages kept
                std::vector<uint32_t> nf;
                for (size_t i = nfree0; i-- > 0;)
                    if (!keep[i])
                        nf.push_back(h_tab[npages + i]);
                free_pages.swap(nf);
                continue;
            }
            bool of = false;
            trace_level = 2;
            cc_status s = launch(STAGE1, nullptr, 0, c, s1_next, want_paths, false, count_tri, s1_filter, used, &of);
            if (s != CC_OK)
                return s;
            if (of)
                return fail(CC_ERR_CAPACITY, "Stage 1 output overflow (internal sizing error)");
            s1_next += c;
            S.chunks++;
            res->counts[3] += h_sc->cycles;
            res->hash += h_sc->hash;
            Level &L3 = levels[3];
            L3.pages = used;
            L3.count = h_sc->out_count;
            L3.sharded = W == 1 || s1_filter;  // a refill: earlier chunks' flags do not carry over
            L3.shard_now = false;
            in_use += L3.count;
            high_water = std::max(high_water, in_use);
            deepest = 3;
            continue;
        }
        const int d = deepest;
        Level &L = levels[d];
        // ---- small frontiers: the first levels in one cooperative launch (no host round trip
        //      per level); the level where the frontier grows past a page is handed back here
        // two regions of rk contiguous free pages each (the free list is in page order at this
        // point); one page each when contiguity is not available
        size_t rk = std::min<size_t>(16, free_pages.size() / 4);
        if (small_ok && !small_tried && d == 3) {
            const size_t fs = free_pages.size();
            for (size_t i = 0; i < 2 * rk && rk > 1; ++i)
                if (free_pages[fs - 1 - i] != free_pages[fs - 1] + i)
                    rk = 1;
        }
        const u64 small_thr = (u64)std::max<size_t>(rk, 1) * P / (u64)std::max<int64_t>(1, g->max_deg - 1);
        if (small_ok && !small_tried && d == 3 && s1_next >= stage1_total && L.pages.size() == 1 &&
            free_pages.size() >= 2 && L.count <= small_thr) {
            small_tried = true;
            rk = std::max<size_t>(rk, 1);
            const size_t na = (size_t)n + 3;
            DevBuf sm;
            sm.st = st;
            CC_CUDA(pool_alloc(&sm.p, (3 * na + 3) * 8, device, st));
            CC_CUDA(cudaMemsetAsync(sm.p, 0, (3 * na + 3) * 8, st));
            u64 *d_count = (u64 *)sm.p, *d_cyc = d_count + na, *d_cand = d_cyc + na, *d_misc = d_cand + na;
            const u64 c3 = L.count;
            CC_CUDA(cudaMemcpyAsync(d_count + 3, &c3, 8, cudaMemcpyHostToDevice, st));
            std::vector<uint32_t> reg[2];
            for (int r = 0; r < 2; ++r)
                for (size_t i = 0; i < rk; ++i) {
                    reg[r].push_back(free_pages.back());
                    free_pages.pop_back();
                }
            cc::SmallArgs sa{};
            sa.first = L.pages[0];
            sa.region[0] = reg[0][0];
            sa.region[1] = reg[1][0];
            sa.region_cap = (u64)rk * P;
            sa.d0 = 3;
            sa.d_stop = max_len == 0 ? (int)n + 2 : (int)max_len - 2;  // leaf levels stay paged
            sa.max_len = max_len;
            sa.threshold = small_thr;  // the children of a level up to this size fit a region
            sa.count = d_count;
            sa.cyc = d_cyc;
            sa.cand = d_cand;
            sa.hash = d_misc;
            sa.last = (int32_t *)(d_misc + 1);
            sa.err = d_misc + 2;
            cc::LaunchArgs a = base;
            if (opt.profile)
                CC_CUDA(cudaEventRecord(ea, st));
            CC_CUDA(cc::launch_small(a, sa, st, sms));
            if (opt.profile)
                CC_CUDA(cudaEventRecord(eb, st));
            std::vector<u64> h(3 * na + 3);
            CC_CUDA(cudaMemcpyAsync(h.data(), sm.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
            CC_CUDA(cudaStreamSynchronize(st));
            S.d2h_bytes += h.size() * 8;
            S.launches++;
            S.chunks++;
            if (opt.profile) {
                float ms = 0;
                CC_CUDA(cudaEventElapsedTime(&ms, ea, eb));
                S.t_expand_ms += ms;
            }
            const u64 *hc = h.data(), *hy = hc + na, *hd = hy + na, *hm = hd + na;  // count, cyc, cand, misc
            const int last = (int)(int32_t)(hm[1] & 0xffffffffu);
            if (hm[2])
                return fail(CC_ERR_CAPACITY, "small-frontier path overflowed a page (internal sizing error)");
            if (last < 3 || last > (int)n + 2)
                return fail(CC_ERR_CUDA, "small-frontier path returned a bad level");
            res->hash += hm[0];
            for (int t = 3; t < last; ++t) {  // the levels expanded in the cooperative launch
                res->paths[t] += hc[t];
                res->cand[t] += hd[t];
                res->counts[t + 1] += hy[t];
                S.paths_expanded += hc[t];
                S.bytes_alg += (hc[t] + hc[t + 1]) * rec_bytes;
                S.records_levelsync += hc[t] + hc[t + 1];
                S.slots_moved += hc[t] + hc[t + 1];
                S.paths_written += hc[t + 1];
                S.rounds = std::max<u64>(S.rounds, (u64)t);
            }
            // the level `last` (possibly empty) continues on the paged path: it keeps the pages
            // that hold it, every other page goes back to the free list
            std::vector<uint32_t> keep;
            const u64 nlast = hc[last];
            if (last == 3) {
                keep = L.pages;
            } else {
                free_pages.push_back(L.pages[0]);
                keep = reg[(last - 4) & 1];
                keep.resize((size_t)((nlast + P - 1) / P));
            }
            for (int r = 0; r < 2; ++r)
                for (uint32_t pgi : reg[r])
                    if (std::find(keep.begin(), keep.end(), pgi) == keep.end())
                        free_pages.push_back(pgi);
            in_use -= L.count;
            L.pages.clear();
            L.count = 0;
            Level &N = levels[last];
            N.pages = keep;
            N.count = nlast;
            N.sharded = true;  // W == 1 only
            N.shard_now = false;
            in_use += N.count;
            high_water = std::max(high_water, in_use);
            if (N.count == 0) {
                for (uint32_t pgi : N.pages)
                    free_pages.push_back(pgi);
                N.pages.clear();
            }
            deepest = last;
            continue;
        }
        // ---- multi-GPU: partition the first frontier level with >= threshold paths
        if (W > 1 && !L.sharded && (L.count >= shard_threshold || L.shard_now)) {
            bool of = false;
            trace_level = d;
            cc_status s = launch(FILTER, L.pages.data(), L.pages.size(), L.count, 0, true, false, false, false, used,
                                 &of);
            if (s != CC_OK)
                return s;
            if (of)
                return fail(CC_ERR_CAPACITY, "workspace too small for the shard filter");
            for (uint32_t pg : L.pages)
                free_pages.push_back(pg);
            in_use -= L.count;
            L.pages = used;
            L.count = h_sc->out_count;
            in_use += L.count;
            L.sharded = true;
            continue;
        }
        const bool owner = W == 1 || L.sharded || opt.shard_index == 0;
        // children of F_d have d+1 vertices: created iff d+1 < max_len.  Count mode fuses the
        // last level: if they could not have children themselves (d+2 >= max_len) they are
        // counted by this launch and not written
        const bool emit = max_len == 0 || (u64)d + 1 < max_len;
        const bool leaf = emit && (mode == cc::Mode::B || list) && max_len != 0 && (u64)d + 2 >= max_len;
        const bool writes = emit && !leaf;
        // grid class, large levels: k_expand_fused, two levels (F_d -> F_{d+2}) when the
        // grandchildren are written (not the last level under the cap), else one
        const int fuse = fused_ok && L.count >= fused_min ? ((max_len == 0 || (u64)d + 3 < max_len) ? 2 : 1) : 0;
        // F_{d+1} (and F_{d+2}) are empty here (d is the deepest non-empty level); the output
        // level's flags are set when this expansion commits, never before the launch (an
        // overflow may still shard F_d first)
        Level &C = levels[d + (fuse == 2 ? 2 : 1)];
        auto est1 = [&](int t) {
            return levels[t].fan1 > 0 ? levels[t].fan1 : (t > 3 && levels[t - 1].fan1 > 0 ? levels[t - 1].fan1 * 1.3 : maxfan);
        };
        const double fan_cap = fuse == 2 ? maxfan * maxfan : maxfan;
        // ---- choose the input chunk: the last k pages of F_d
        size_t k = L.pages.size();
        if (writes && (W == 1 || L.sharded)) {
            double f = L.fan > 0 && L.fan_fuse == fuse ? L.fan * 1.15
                       : fuse == 2                   ? est1(d) * est1(d + 1) * 1.2
                       : fuse == 1                   ? est1(d) * 1.2
                       : (levels[d - 1].fan > 0 && levels[d - 1].fan_fuse == 0 ? levels[d - 1].fan * 1.5 : maxfan);
            f = std::min(std::max(f, 0.05), fan_cap);
            // keep a reserve so that the child level can expand its first page next (about
            // f pages of grandchildren): without it a high fan-out level fills every free page
            // with children that then cannot be expanded
            const double reserve = (std::ceil(f * 1.2) + 1.0) * (double)P;
            // the fused kernel may leave up to one chunk of empty slots per warp
            const double holes = fuse ? (double)fwarps(fuse, leaf) * 4096.0 : 0.0;
            const double room = std::max((double)P, (double)free_pages.size() * P - reserve - holes);
            // records of the last k pages: (k-1) full pages + the partial last page
            const u64 last_fill = L.count - (u64)(L.pages.size() - 1) * P;
            u64 take = (u64)std::max(1.0, room / f);
            if (take >= L.count)
                k = L.pages.size();
            else if (take <= last_fill)
                k = 1;
            else
                k = 1 + (size_t)((take - last_fill) / P);
        }
        u64 sub = 0;  // > 0: expand only the last `sub` records of the last page (see below)
        for (;;) {
            const u64 last_fill = L.count - (u64)(L.pages.size() - 1) * P;
            u64 c = last_fill + (u64)(k - 1) * P;
            const uint32_t *in = L.pages.data() + (L.pages.size() - k);
            // Less than one page: the tail [last_fill - sub, last_fill) of the last page is copied
            // to a free page of its own and expanded from there; the level keeps the head, so its
            // "all pages full but the last" layout is unchanged.  This is what keeps a tiny arena
            // making progress when one page of a high fan-out level has more children than the
            // free pages hold.
            uint32_t tail_page = UINT32_MAX;
            if (sub) {
                if (free_pages.size() < 2)
                    return fail(CC_ERR_CAPACITY, "workspace too small: no page to split F_" + std::to_string(d));
                tail_page = free_pages.back();
                free_pages.pop_back();
                CC_CUDA(copy_records(base.pg.base, page_bytes, lp, rec_bytes, wide, L.pages.back(), last_fill - sub,
                                     sub, tail_page, st));
                in = &tail_page;
                c = sub;
            }
            bool of = false;
            trace_level = d;
            // output chunk of the fused kernel: about 1/64 of a warp's expected output (at least
            // 512 slots, the largest single reservation, at most 4096), so the empty slots at
            // the warps' ends stay near 1% of the launch's output
            const bool fq = fuse == 2 && packed && fq_on;  // k_expand_fq: smaller reservations
            uint32_t log_ch = fq ? cc::kFqMinLogChunk : 9;
            if (fuse) {
                const double fe = L.fan > 0 && L.fan_fuse == fuse ? L.fan : (fuse == 2 ? est1(d) * est1(d + 1) : est1(d));
                const double warps = std::max(1.0, std::min((double)fwarps(fuse, leaf), (double)c / 32.0));
                const double per = (double)c * fe / (warps * 64.0);
                while (log_ch < 12 && (double)(2u << log_ch) <= per && (2ull << log_ch) <= P)
                    ++log_ch;
            }
            cc_status s = launch(EXPAND, in, 1 + (sub ? 0 : k - 1), c, 0, emit, leaf, owner, false, used, &of, fuse,
                                 log_ch);
            if (tail_page != UINT32_MAX)
                free_pages.push_back(tail_page);  // a copy: the records still live in L's last page
            if (s != CC_OK)
                return s;
            if (of) {
                if (W > 1 && !L.sharded) {
                    // an unsharded level is expanded whole; if its children do not fit, shard it
                    // now (the decision is still a function of the graph only)
                    L.shard_now = true;
                    break;
                }
                if (k == 1) {
                    if (c <= 1)
                        return fail(CC_ERR_CAPACITY, "workspace too small: one path of F_" + std::to_string(d) +
                                                         " needs " + std::to_string(h_sc->out_count) +
                                                         " output records, " +
                                                         std::to_string(free_pages.size() * P) + " free");
                    L.fan = std::max(L.fan_fuse == fuse ? L.fan : 0.0, (double)h_sc->out_count / (double)c);
                    L.fan_fuse = fuse;
                    const double room = (double)(free_pages.size() - 1) * P;
                    sub = std::max<u64>(1, std::min<u64>(c / 2, (u64)(room / (L.fan * 1.15))));
                    continue;
                }
                L.fan = std::max(L.fan_fuse == fuse ? L.fan : 0.0, (double)h_sc->out_count / (double)c);
                L.fan_fuse = fuse;
                const double room = (double)free_pages.size() * P;
                const double want = room / (L.fan * 1.15);
                size_t k2 = want <= last_fill ? 1 : 1 + (size_t)((want - last_fill) / P);
                k = std::max<size_t>(1, std::min(k2, k - 1));
                continue;
            }
            // commit
            S.chunks++;
            S.rounds = std::max<u64>(S.rounds, (u64)d);
            if (owner) {
                res->paths[d] += real_in;
                res->cand[d] += h_sc->cand;
                S.paths_expanded += real_in;
                res->counts[d + 1] += h_sc->cycles;
                res->hash += h_sc->hash;
                if (leaf || fuse == 2) {  // the children: counted here, never written
                    res->paths[d + 1] += h_sc->paths_next;
                    res->cand[d + 1] += h_sc->cand_next;
                    res->counts[d + 2] += h_sc->cycles_next;
                    S.paths_expanded += h_sc->paths_next;
                    if (leaf)
                        S.leaf_paths += h_sc->paths_next;
                }
            }
            // records actually read + written (empty slots excluded), and what a level-synchronous
            // expansion of the same paths reads + writes (each path read once, each
            // child written once; the fused kernel keeps F_{d+1} in shared memory)
            S.bytes_alg += (real_in + real_out) * rec_bytes;
            S.records_levelsync += real_in + real_out + ((leaf || fuse == 2) ? 2 * h_sc->paths_next : 0);
            S.slots_moved += c + h_sc->out_count;
            if (c > 0) {
                L.fan = (double)h_sc->out_count / (double)c;
                L.fan_fuse = fuse;
            }
            if (real_in > 0 && mode == cc::Mode::B && !wide && !list) {
                L.fan1 = (double)(fuse == 2 || leaf ? h_sc->paths_next : real_out) / (double)real_in;
                if (fuse == 2 && h_sc->paths_next > 0)
                    levels[d + 1].fan1 = (double)real_out / (double)h_sc->paths_next;
            }
            if (!sub)
                for (size_t i = 0; i < k; ++i) {
                    free_pages.push_back(L.pages.back());
                    L.pages.pop_back();
                }
            L.count -= c;
            in_use -= c;
            if (h_sc->out_count) {
                C.pages = used;
                C.count = h_sc->out_count;
                C.sharded = L.sharded || W == 1;
                C.shard_now = false;
                in_use += C.count;
                high_water = std::max(high_water, in_use);
                deepest = d + (fuse == 2 ? 2 : 1);
            }
            break;
        }
    }
    S.peak_arena_records = high_water;

    CC_CUDA(cudaEventRecord(ev1, st));
    CC_CUDA(cudaStreamSynchronize(st));
    float tdev = 0;
    CC_CUDA(cudaEventElapsedTime(&tdev, ev0, ev1));
    S.t_dev_ms = tdev;
    for (int64_t k = 0; k <= n; ++k) {
        S.total_cycles += res->counts[k];
        S.candidates += res->cand[k];
    }
    S.triplets = res->paths[3];
    const u64 ncyc = cyc_committed;
    S.cycles_stored = ncyc;
    if (opt.collect) {
        S.bytes_alg += std::min<u64>(ncyc, res->cyc.cap) * rec_bytes;
        if (ncyc > res->cyc.cap) {
            *need_cycles = ncyc;
            return fail(CC_ERR_CAPACITY, "collect capacity " + std::to_string(res->cyc.cap) +
                                             " exceeded: " + std::to_string(ncyc) + " cycles");
        }
        res->n_cyc = ncyc;
    }
    S.t_wall_ms = now_ms() - t_wall0;
    *out = res_guard.release();
    return CC_OK;
}

extern "C" cc_status cc_enumerate(const cc_graph *g, const cc_options *opt, cc_result **out)
{
    u64 need = 0;
    cc_status s = enumerate_impl(g, opt, out, &need);
    if (s == CC_ERR_CAPACITY && need > 0 && opt && opt->collect && opt->collect_capacity == 0) {
        // automatic collect capacity: run again with exactly the capacity needed (the rerun
        // starts from zeroed counters, so nothing is counted twice)
        cc_options o2 = *opt;
        o2.collect_capacity = need;
        s = enumerate_impl(g, &o2, out, &need);
    }
    return s;
}

extern "C" cc_status cc_count_by_length(const cc_result *r, uint64_t *counts, size_t cap, size_t *n_lengths,
                                        uint64_t *set_hash)
{
    if (!r)
        return fail(CC_ERR_INVALID_ARGUMENT, "result is NULL");
    const size_t need = (size_t)r->n + 1;
    if (n_lengths)
        *n_lengths = need;
    if (set_hash)
        *set_hash = r->hash;
    if (counts == nullptr && cap == 0)
        return CC_OK;
    if (!counts || cap < need)
        return fail(CC_ERR_BUFFER_TOO_SMALL, "counts needs n+1 = " + std::to_string(need) + " entries");
    std::copy(r->counts.begin(), r->counts.begin() + need, counts);
    return CC_OK;
}

extern "C" cc_status cc_paths_by_length(const cc_result *r, uint64_t *paths, size_t cap, size_t *n_lengths)
{
    if (!r)
        return fail(CC_ERR_INVALID_ARGUMENT, "result is NULL");
    const size_t need = (size_t)r->n + 1;
    if (n_lengths)
        *n_lengths = need;
    if (paths == nullptr && cap == 0)
        return CC_OK;
    if (!paths || cap < need)
        return fail(CC_ERR_BUFFER_TOO_SMALL, "paths needs n+1 = " + std::to_string(need) + " entries");
    std::copy(r->paths.begin(), r->paths.begin() + need, paths);
    return CC_OK;
}

extern "C" cc_status cc_num_stored_cycles(const cc_result *r, uint64_t *n)
{
    if (!r || !n)
        return fail(CC_ERR_INVALID_ARGUMENT, "NULL argument");
    *n = r->collected ? r->n_cyc : 0;
    return CC_OK;
}

extern "C" cc_status cc_result_stats(const cc_result *r, cc_stats *out)
{
    if (!r || !out)
        return fail(CC_ERR_INVALID_ARGUMENT, "NULL argument");
    const uint32_t sz = out->struct_size;
    if (sz < sizeof(uint32_t) || sz > sizeof(cc_stats))
        return fail(CC_ERR_INVALID_ARGUMENT, "cc_stats.struct_size mismatch");
    std::memcpy(out, &r->stats, sz);
    out->struct_size = sz;
    return CC_OK;
}

// Host side of a device->host copy into the caller's buffer: when `dst` is pageable, the bytes
// stream through two pinned staging buffers -- the DMA of chunk i+1 overlaps the host copy
// (several threads) of chunk i out of the other buffer; pinned (page-locked or registered)
// destinations are copied directly.
static cudaError_t d2h_stream(void *dst, const void *src, size_t bytes, cudaStream_t st)
{
    if (bytes == 0)
        return cudaSuccess;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, dst) == cudaSuccess && at.type == cudaMemoryTypeHost) {
        cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
        return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
    }
    cudaGetLastError();  // pageable memory: cudaPointerGetAttributes may report an error
    constexpr size_t kChunk = 64ull << 20;
    static thread_local Pinned stage;
    cudaError_t e = stage.reserve(2 * kChunk);
    if (e != cudaSuccess)
        return e;
    cudaEvent_t done[2];
    cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming);
    const size_t nch = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t i) {
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        char *buf = (char *)stage.p + (i & 1) * kChunk;
        cudaError_t r = cudaMemcpyAsync(buf, (const char *)src + off, len, cudaMemcpyDeviceToHost, st);
        if (r == cudaSuccess)
            r = cudaEventRecord(done[i & 1], st);
        return r;
    };
    e = issue(0);
    for (size_t i = 0; i < nch && e == cudaSuccess; ++i) {
        if (i + 1 < nch)
            e = issue(i + 1);  // the other buffer was drained by the host copy of chunk i-1
        if (e == cudaSuccess)
            e = cudaEventSynchronize(done[i & 1]);
        if (e != cudaSuccess)
            break;
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        const char *buf = (const char *)stage.p + (i & 1) * kChunk;
        // host copy out of the pinned buffer on 4 threads
        constexpr int kT = 4;
        std::vector<std::thread> th;
        const size_t per = (len + kT - 1) / kT;
        for (int t = 0; t < kT; ++t) {
            const size_t lo = std::min(len, t * per), hi = std::min(len, lo + per);
            if (hi > lo)
                th.emplace_back([=] { std::memcpy((char *)dst + off + lo, buf + lo, hi - lo); });
        }
        for (auto &x : th)
            x.join();
    }
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
    return e;
}

extern "C" cc_status cc_fetch_cycles(const cc_result *r, uint64_t first, uint64_t max_cycles, int32_t *vertices,
                                     size_t vertices_cap, uint64_t *offsets, uint64_t *n_fetched)
{
    if (!r || !offsets || !n_fetched)
        return fail(CC_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!r->collected)
        return fail(CC_ERR_NOT_COLLECTED, "result was enumerated in count-only mode");
    *n_fetched = 0;
    if (first >= r->n_cyc || max_cycles == 0) {
        offsets[0] = 0;
        return CC_OK;
    }
    const u64 cnt = std::min<u64>(max_cycles, r->n_cyc - first);
    int cur = -1;
    CC_CUDA(cudaGetDevice(&cur));
    CC_CUDA(cudaSetDevice(r->device));
    struct Restore {
        int d;
        ~Restore()
        {
            if (d >= 0)
                cudaSetDevice(d);
        }
    } restore{cur};
    // the stream the result was enumerated on (cc_options.stream), so the fetch is ordered after
    // the enumeration without a device-wide synchronisation
    cudaStream_t st = r->stream;
    // offsets (a device scan of the cycle lengths), then the canonical sequences, both copied
    // back through d2h_stream; scratch from the library's stream-ordered pool
    const u64 nblk = (cnt + 1023) / 1024;
    u64 *d_off = nullptr, *d_blk = nullptr;
    int32_t *d_v = nullptr;
    CC_CUDA(pool_alloc((void **)&d_off, (cnt + 1) * 8, r->device, st));
    cudaError_t e = pool_alloc((void **)&d_blk, (nblk + 1) * 8, r->device, st);
    if (e == cudaSuccess)
        e = cc::launch_cycle_offsets(r->cyc, r->nw, first, cnt, d_off, d_blk, st);
    u64 total = 0;
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&total, d_off + cnt, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
        e = cudaStreamSynchronize(st);
    if (e == cudaSuccess && total <= vertices_cap && vertices)
        e = pool_alloc((void **)&d_v, std::max<u64>(total, 1) * 4, r->device, st);
    if (e == cudaSuccess && d_v)
        e = cc::launch_cycle_sequences(r->cyc, r->nw, r->adj, r->orig, first, cnt, d_off, d_v, st);
    if (e == cudaSuccess)
        e = d2h_stream(offsets, d_off, (cnt + 1) * 8, st);
    if (e == cudaSuccess && d_v)
        e = d2h_stream(vertices, d_v, total * 4, st);
    cudaFreeAsync(d_off, st);
    cudaFreeAsync(d_blk, st);
    if (d_v)
        cudaFreeAsync(d_v, st);
    if (e == cudaSuccess)
        e = cudaStreamSynchronize(st);
    if (e != cudaSuccess)
        return cuda_fail(e, "cycle sequences");
    if (total > vertices_cap || !vertices)
        return fail(CC_ERR_BUFFER_TOO_SMALL, "vertices needs " + std::to_string(total) + " entries");
    *n_fetched = cnt;
    return CC_OK;
}
