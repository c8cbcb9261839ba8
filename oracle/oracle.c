/*
 * oracle.c -- CPU oracle for chordless-cycle enumeration (arXiv 1410.4876).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path under paper_1410_4876_b200/.
 *
 * It is deliberately plain and slow: an n x n byte adjacency matrix, an O(n^2)
 * degree labelling, and the paper's sequential algorithm (Alg. 1)
 * run as a recursive depth-first visit per triplet with the literal O(t) chord loop
 * of Alg. 1 line 8.
 *
 * Functions and the passages they follow:
 *   orc_validate         CSR validation (reading R1)
 *   orc_degree_labeling  degree labelling, PAPER.md:53 (§2), ties -> lowest id (reading G1)
 *   orc_triplets         T(G) and triangles, Alg. 1 lines 2-3, PAPER.md:97-101 / PAPER.md:55
 *   orc_enumerate        Alg. 1 lines 4-11, as recursive DFS per triplet
 *                        (the DFS of DCLJ2014); counts, set hash, stats,
 *                        optional cycle list in canonical order
 *   orc_mix              SplitMix64 finaliser used by the set hash
 *
 * Every function is pinned by tests/test_oracle_*.py (brute force over subsets, closed
 * forms, Table 1 counts, invariants).  No parity-unpinned functions.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORC_OK 0
#define ORC_ERR_INVALID_ARGUMENT (-1)
#define ORC_ERR_INVALID_VERTEX (-2)
#define ORC_ERR_SELF_LOOP (-3)
#define ORC_ERR_NOT_SYMMETRIC (-4)
#define ORC_ERR_NO_MEMORY (-5)
#define ORC_ERR_BUFFER_TOO_SMALL (-6)

/* ---------------------------------------------------------------- hash (H-spec) */
uint64_t orc_mix(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

/* ---------------------------------------------------------------- graph */
typedef struct {
    int64_t n;
    unsigned char *adj; /* adj[a*n + b] = 1 iff (a,b) in E */
    int32_t *deg;       /* d_G(v) */
    int32_t **nbr;      /* Adj(v), ascending original id */
    int32_t *nbr_store;
    int32_t *label;     /* l(v), 0-based (reading G2) */
    uint64_t *key;      /* key(v) = mix(seed ^ v) over ORIGINAL ids */
} og_graph;

static void og_free(og_graph *g)
{
    free(g->adj);
    free(g->deg);
    free(g->nbr);
    free(g->nbr_store);
    free(g->label);
    free(g->key);
    memset(g, 0, sizeof(*g));
}

/* Validate and normalise a CSR: ids in range, no self-loops, symmetric; duplicates
 * inside a row are merged.  Builds the adjacency matrix. */
static int og_build(og_graph *g, int64_t n, const int64_t *row_ptr, const int32_t *col)
{
    memset(g, 0, sizeof(*g));
    if (n < 0 || (n > 0 && !row_ptr))
        return ORC_ERR_INVALID_ARGUMENT;
    if (n > 20000)
        return ORC_ERR_INVALID_ARGUMENT; /* the n*n matrix would be silly */
    g->n = n;
    if (n == 0)
        return ORC_OK;
    if (row_ptr[0] != 0)
        return ORC_ERR_INVALID_ARGUMENT;
    for (int64_t v = 0; v < n; v++)
        if (row_ptr[v + 1] < row_ptr[v])
            return ORC_ERR_INVALID_ARGUMENT;
    if (row_ptr[n] > 0 && !col)
        return ORC_ERR_INVALID_ARGUMENT;
    g->adj = (unsigned char *)calloc((size_t)(n * n), 1);
    g->deg = (int32_t *)calloc((size_t)n, sizeof(int32_t));
    g->label = (int32_t *)calloc((size_t)n, sizeof(int32_t));
    g->key = (uint64_t *)calloc((size_t)n, sizeof(uint64_t));
    g->nbr = (int32_t **)calloc((size_t)n, sizeof(int32_t *));
    if (!g->adj || !g->deg || !g->label || !g->key || !g->nbr) {
        og_free(g);
        return ORC_ERR_NO_MEMORY;
    }
    for (int64_t v = 0; v < n; v++) {
        for (int64_t k = row_ptr[v]; k < row_ptr[v + 1]; k++) {
            int64_t w = col[k];
            if (w < 0 || w >= n) {
                og_free(g);
                return ORC_ERR_INVALID_VERTEX;
            }
            if (w == v) {
                og_free(g);
                return ORC_ERR_SELF_LOOP;
            }
            g->adj[v * n + w] = 1;
        }
    }
    for (int64_t a = 0; a < n; a++)
        for (int64_t b = 0; b < n; b++)
            if (g->adj[a * n + b] != g->adj[b * n + a]) {
                og_free(g);
                return ORC_ERR_NOT_SYMMETRIC;
            }
    int64_t total = 0;
    for (int64_t a = 0; a < n; a++) {
        for (int64_t b = 0; b < n; b++)
            g->deg[a] += g->adj[a * n + b];
        total += g->deg[a];
    }
    g->nbr_store = (int32_t *)malloc((size_t)(total > 0 ? total : 1) * sizeof(int32_t));
    if (!g->nbr_store) {
        og_free(g);
        return ORC_ERR_NO_MEMORY;
    }
    int64_t pos = 0;
    for (int64_t a = 0; a < n; a++) {
        g->nbr[a] = g->nbr_store + pos;
        for (int64_t b = 0; b < n; b++)
            if (g->adj[a * n + b])
                g->nbr_store[pos++] = (int32_t)b;
    }
    return ORC_OK;
}

/* Degree labelling: G_1 = G; repeatedly delete a vertex u_i of minimum
 * degree in G_i and set l(u_i) = i.  Ties go to the lowest original id (reading G1).
 * Labels are 0-based (reading G2).  Plain O(n^2) scan. */
static void og_degree_labeling(og_graph *g)
{
    int64_t n = g->n;
    int32_t *d = (int32_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    unsigned char *alive = (unsigned char *)malloc((size_t)(n > 0 ? n : 1));
    for (int64_t v = 0; v < n; v++) {
        d[v] = g->deg[v];
        alive[v] = 1;
    }
    for (int64_t i = 0; i < n; i++) {
        int64_t best = -1;
        for (int64_t v = 0; v < n; v++)
            if (alive[v] && (best < 0 || d[v] < d[best]))
                best = v;
        g->label[best] = (int32_t)i;
        alive[best] = 0;
        for (int32_t k = 0; k < g->deg[best]; k++) {
            int32_t w = g->nbr[best][k];
            if (alive[w])
                d[w]--;
        }
    }
    free(d);
    free(alive);
}

static int og_setup(og_graph *g, int64_t n, const int64_t *row_ptr, const int32_t *col,
                    const int32_t *labels_in, uint64_t seed)
{
    int rc = og_build(g, n, row_ptr, col);
    if (rc != ORC_OK)
        return rc;
    if (labels_in) {
        /* any bijection V -> {0..n-1} defines the cycles uniquely */
        unsigned char *seen = (unsigned char *)calloc((size_t)(n > 0 ? n : 1), 1);
        for (int64_t v = 0; v < n; v++) {
            if (labels_in[v] < 0 || labels_in[v] >= n || seen[labels_in[v]]) {
                free(seen);
                og_free(g);
                return ORC_ERR_INVALID_ARGUMENT;
            }
            seen[labels_in[v]] = 1;
            g->label[v] = labels_in[v];
        }
        free(seen);
    } else {
        og_degree_labeling(g);
    }
    for (int64_t v = 0; v < n; v++)
        g->key[v] = orc_mix(seed ^ (uint64_t)v);
    return ORC_OK;
}

int orc_degree_labeling(int64_t n, const int64_t *row_ptr, const int32_t *col, int32_t *labels)
{
    og_graph g;
    int rc = og_setup(&g, n, row_ptr, col, NULL, 0);
    if (rc != ORC_OK)
        return rc;
    for (int64_t v = 0; v < n; v++)
        labels[v] = g.label[v];
    og_free(&g);
    return ORC_OK;
}

/* ---------------------------------------------------------------- triplets */
/* Alg. 1 lines 2-3:
 *   T(G) = { <x,u,y> : x,y in Adj(u), l(u) < l(x) < l(y), (x,y) not in E }
 *   C    = { <x,u,y> : x,y in Adj(u), l(u) < l(x) < l(y), (x,y) in E }
 * Enumerated in a fixed order: u ascending, then x, y ascending in Adj(u). */
typedef struct {
    int32_t x, u, y;
} og_triplet;

static int64_t og_triplets(const og_graph *g, og_triplet *out, int64_t cap, og_triplet *tri,
                           int64_t tri_cap, int64_t *n_tri)
{
    int64_t nt = 0, nc = 0;
    for (int64_t u = 0; u < g->n; u++) {
        for (int32_t a = 0; a < g->deg[u]; a++) {
            int32_t x = g->nbr[u][a];
            for (int32_t b = 0; b < g->deg[u]; b++) {
                int32_t y = g->nbr[u][b];
                if (!(g->label[u] < g->label[x] && g->label[x] < g->label[y]))
                    continue;
                if (g->adj[(int64_t)x * g->n + y]) {
                    if (tri && nc < tri_cap) {
                        tri[nc].x = x;
                        tri[nc].u = (int32_t)u;
                        tri[nc].y = y;
                    }
                    nc++;
                } else {
                    if (out && nt < cap) {
                        out[nt].x = x;
                        out[nt].u = (int32_t)u;
                        out[nt].y = y;
                    }
                    nt++;
                }
            }
        }
    }
    if (n_tri)
        *n_tri = nc;
    return nt;
}

/* Returns |T(G)| (or an error < 0); writes up to cap triplets (x,u,y) to out and
 * the triangle count to *n_triangles.  labels_in may be NULL (degree labelling). */
int64_t orc_triplets(int64_t n, const int64_t *row_ptr, const int32_t *col, const int32_t *labels_in,
                     int32_t *out, int64_t cap, uint64_t *n_triangles)
{
    og_graph g;
    int rc = og_setup(&g, n, row_ptr, col, labels_in, 0);
    if (rc != ORC_OK)
        return rc;
    int64_t ntri = 0;
    int64_t nt = og_triplets(&g, (og_triplet *)out, cap, NULL, 0, &ntri);
    if (n_triangles)
        *n_triangles = (uint64_t)ntri;
    og_free(&g);
    return nt;
}

/* ---------------------------------------------------------------- enumeration */
typedef struct {
    const og_graph *g;
    uint32_t max_len;
    uint64_t *counts;       /* [n+2] */
    uint64_t set_hash;
    uint64_t *paths_by_len; /* [n+2] paths scanned by the expansion, by vertex count */
    uint64_t candidates;    /* sum over scanned paths of deg(v_t) */
    int32_t *path;          /* current path <v1..vt> */
    /* orc_enumerate_split only: paths of split_len vertices are queued, not visited */
    int split_len;
    int32_t *items;
    int64_t n_items, items_cap;
    /* optional cycle list */
    int32_t *cyc_vertices;
    uint64_t cyc_vertices_cap;
    uint64_t *cyc_offsets;
    uint64_t cyc_cap;
    uint64_t n_cycles;
    uint64_t n_cyc_vertices;
} og_ctx;

static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* Record one chordless cycle <c[0..k-1]>: counts[k]++, set_hash += h(C) where
 * h(C) = mix(sum of key(v) over the cycle's sorted vertex list). */
static void og_record(og_ctx *cx, const int32_t *c, int k)
{
    int32_t tmp[k];
    memcpy(tmp, c, sizeof(int32_t) * (size_t)k);
    qsort(tmp, (size_t)k, sizeof(int32_t), cmp_i32);
    uint64_t s = 0;
    for (int i = 0; i < k; i++)
        s += cx->g->key[tmp[i]];
    cx->counts[k]++;
    cx->set_hash += orc_mix(s);
    if (cx->cyc_offsets) {
        if (cx->n_cycles < cx->cyc_cap && cx->n_cyc_vertices + (uint64_t)k <= cx->cyc_vertices_cap) {
            memcpy(cx->cyc_vertices + cx->n_cyc_vertices, c, sizeof(int32_t) * (size_t)k);
            cx->cyc_offsets[cx->n_cycles + 1] = cx->n_cyc_vertices + (uint64_t)k;
        }
    }
    cx->n_cycles++;
    cx->n_cyc_vertices += (uint64_t)k;
}

/* Alg. 1 lines 7-11 for the path p = path[0..t-1] = <v1..vt>:
 * for each v in Adj(vt): if l(v) > l(v2) and v is not adjacent to v_i, i in {2..t-1}
 * (and v not in p, Alg. 3 line 11 / reading G6), then either v in Adj(v1) -> cycle
 * <p,v>, or <p,v> is a new chordless path that is visited recursively (DFS). */
/* orc_enumerate_split: append the current path of t vertices to the work queue */
static void og_queue(og_ctx *cx, int t)
{
    if (cx->n_items == cx->items_cap) {
        cx->items_cap = cx->items_cap ? 2 * cx->items_cap : 1024;
        cx->items = (int32_t *)realloc(cx->items, (size_t)cx->items_cap * (size_t)t * sizeof(int32_t));
    }
    memcpy(cx->items + cx->n_items * t, cx->path, (size_t)t * sizeof(int32_t));
    cx->n_items++;
}

static void og_visit(og_ctx *cx, int t)
{
    const og_graph *g = cx->g;
    int64_t n = g->n;
    int32_t *p = cx->path;
    int32_t v1 = p[0], v2 = p[1], vt = p[t - 1];
    cx->paths_by_len[t]++;
    cx->candidates += (uint64_t)g->deg[vt];
    for (int32_t k = 0; k < g->deg[vt]; k++) {
        int32_t v = g->nbr[vt][k];
        if (!(g->label[v] > g->label[v2]))
            continue;
        int in_p = 0;
        for (int i = 0; i < t; i++)
            if (p[i] == v)
                in_p = 1;
        if (in_p)
            continue;
        int chord = 0;
        for (int i = 1; i <= t - 2; i++) /* v_2 .. v_{t-1} (1-based) */
            if (g->adj[(int64_t)v * n + p[i]]) {
                chord = 1;
                break;
            }
        if (chord)
            continue;
        p[t] = v;
        if (g->adj[(int64_t)v * n + v1]) {
            og_record(cx, p, t + 1);
        } else if (cx->max_len == 0 || (uint32_t)(t + 1) < cx->max_len) {
            if (cx->split_len > 0 && t + 1 == cx->split_len)
                og_queue(cx, t + 1);  /* visited later by a worker thread */
            else
                og_visit(cx, t + 1);
        }
    }
}

typedef struct {
    og_ctx cx;
    const og_triplet *trip;
    int64_t n_trip;
    uint64_t stride, offset;
    int tid, nthreads;
} og_worker;

static void *og_worker_main(void *arg)
{
    og_worker *w = (og_worker *)arg;
    int64_t r = 0;
    for (int64_t i = 0; i < w->n_trip; i++) {
        /* root sample: keep <x,u,y> iff mix(x<<42 | u<<21 | y) % stride == offset
         * (original ids) */
        uint64_t rkey = ((uint64_t)w->trip[i].x << 42) | ((uint64_t)w->trip[i].u << 21) |
                        (uint64_t)w->trip[i].y;
        if (w->stride > 1 && orc_mix(rkey) % w->stride != w->offset)
            continue;
        if (r++ % w->nthreads != w->tid)
            continue;
        w->cx.path[0] = w->trip[i].x;
        w->cx.path[1] = w->trip[i].u;
        w->cx.path[2] = w->trip[i].y;
        og_visit(&w->cx, 3);
    }
    return NULL;
}

/*
 * Enumerate every chordless cycle of G exactly once (Alg. 1).
 *   max_len      0 = no cap; else only cycles with <= max_len vertices (reading G14)
 *   seed         hash seed (0 -> default 0x1410487600000000)
 *   labels_in    optional bijection V -> {0..n-1}; NULL = degree labelling
 *   nthreads     roots are dealt round-robin to threads (sums are order-independent)
 *   root_stride, root_offset   only roots <x,u,y> with mix(x<<42|u<<21|y) % stride == offset
 *                are expanded (bounded samples); triangles are counted iff offset == 0
 *   counts[n+1], paths_by_len[n+1] are written; cycle list optional (nthreads must be 1).
 */
int orc_enumerate(int64_t n, const int64_t *row_ptr, const int32_t *col, uint32_t max_len,
                  uint64_t seed, const int32_t *labels_in, int nthreads, uint64_t root_stride,
                  uint64_t root_offset, uint64_t *counts, uint64_t *set_hash, uint64_t *paths_by_len,
                  uint64_t *candidates, int32_t *cyc_vertices, uint64_t cyc_vertices_cap,
                  uint64_t *cyc_offsets, uint64_t cyc_cap, uint64_t *n_cycles)
{
    if (seed == 0)
        seed = 0x1410487600000000ULL;
    if (nthreads < 1 || root_stride < 1 || root_offset >= root_stride)
        return ORC_ERR_INVALID_ARGUMENT;
    if (cyc_offsets && nthreads != 1)
        return ORC_ERR_INVALID_ARGUMENT;
    og_graph g;
    int rc = og_setup(&g, n, row_ptr, col, labels_in, seed);
    if (rc != ORC_OK)
        return rc;
    for (int64_t k = 0; k <= n; k++) {
        counts[k] = 0;
        if (paths_by_len)
            paths_by_len[k] = 0;
    }
    *set_hash = 0;
    if (candidates)
        *candidates = 0;
    if (cyc_offsets && cyc_cap > 0)
        cyc_offsets[0] = 0;
    uint64_t total_cycles = 0, total_vertices = 0;

    /* Alg. 1 lines 2-3 */
    int64_t ntri = 0;
    int64_t nt = og_triplets(&g, NULL, 0, NULL, 0, &ntri);
    og_triplet *trip = (og_triplet *)malloc((size_t)(nt > 0 ? nt : 1) * sizeof(og_triplet));
    og_triplet *tri = (og_triplet *)malloc((size_t)(ntri > 0 ? ntri : 1) * sizeof(og_triplet));
    og_triplets(&g, trip, nt, tri, ntri, &ntri);

    og_worker *ws = (og_worker *)calloc((size_t)nthreads, sizeof(og_worker));
    for (int i = 0; i < nthreads; i++) {
        og_ctx *cx = &ws[i].cx;
        cx->g = &g;
        cx->max_len = max_len;
        cx->counts = (uint64_t *)calloc((size_t)n + 2, sizeof(uint64_t));
        cx->paths_by_len = (uint64_t *)calloc((size_t)n + 2, sizeof(uint64_t));
        cx->path = (int32_t *)calloc((size_t)n + 2, sizeof(int32_t));
        if (i == 0 && cyc_offsets) {
            cx->cyc_vertices = cyc_vertices;
            cx->cyc_vertices_cap = cyc_vertices_cap;
            cx->cyc_offsets = cyc_offsets;
            cx->cyc_cap = cyc_cap;
        }
        ws[i].trip = trip;
        ws[i].n_trip = nt;
        ws[i].stride = root_stride;
        ws[i].offset = root_offset;
        ws[i].tid = i;
        ws[i].nthreads = nthreads;
    }
    /* triangles: Alg. 1 line 2 puts them straight into C (counted once, by thread 0) */
    if (root_offset == 0 && (max_len == 0 || max_len >= 3)) {
        for (int64_t i = 0; i < ntri; i++) {
            int32_t c[3] = {tri[i].x, tri[i].u, tri[i].y};
            og_record(&ws[0].cx, c, 3);
        }
    }
    /* Alg. 1 lines 4-11: expand every triplet (only when cycles of length >= 4 are wanted) */
    if (max_len == 0 || max_len >= 4) {
        if (nthreads == 1) {
            og_worker_main(&ws[0]);
        } else {
            pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
            for (int i = 0; i < nthreads; i++)
                pthread_create(&th[i], NULL, og_worker_main, &ws[i]);
            for (int i = 0; i < nthreads; i++)
                pthread_join(th[i], NULL);
            free(th);
        }
    }
    for (int i = 0; i < nthreads; i++) {
        og_ctx *cx = &ws[i].cx;
        for (int64_t k = 0; k <= n; k++) {
            counts[k] += cx->counts[k];
            if (paths_by_len)
                paths_by_len[k] += cx->paths_by_len[k];
        }
        *set_hash += cx->set_hash;
        if (candidates)
            *candidates += cx->candidates;
        total_cycles += cx->n_cycles;
        total_vertices += cx->n_cyc_vertices;
        free(cx->counts);
        free(cx->paths_by_len);
        free(cx->path);
    }
    if (n_cycles)
        *n_cycles = total_cycles;
    free(ws);
    free(trip);
    free(tri);
    og_free(&g);
    if (cyc_offsets && (total_cycles > cyc_cap || total_vertices > cyc_vertices_cap))
        return ORC_ERR_BUFFER_TOO_SMALL;
    return ORC_OK;
}

/* Validation only (error kinds of SPEC.md:48 / S:34). */
int orc_validate(int64_t n, const int64_t *row_ptr, const int32_t *col)
{
    og_graph g;
    int rc = og_build(&g, n, row_ptr, col);
    if (rc == ORC_OK)
        og_free(&g);
    return rc;
}

/* ---------------------------------------------------------------- parallel driver (large runs)
 * The same visits as orc_enumerate, scheduled for many threads when there are few triplets
 * (a grid has ~n of them, with very unequal subtrees): Alg. 1 runs on one thread down to the
 * paths of split_len vertices, which are queued instead of visited; nthreads workers then take
 * queued paths one at a time (shared counter) and finish each with the same og_visit.  Every
 * path is visited exactly once and every sum is order-independent, so the outputs equal
 * orc_enumerate's (pinned by tests/test_oracle_pins.py).  Count mode only.  */
typedef struct {
    og_ctx cx;
    og_ctx *root;
    int64_t *next;
} og_split_worker;

static void *og_split_main(void *arg)
{
    og_split_worker *w = (og_split_worker *)arg;
    const og_ctx *r = w->root;
    const int L = r->split_len;
    for (;;) {
        int64_t i = __atomic_fetch_add(w->next, 1, __ATOMIC_RELAXED);
        if (i >= r->n_items)
            break;
        memcpy(w->cx.path, r->items + i * L, (size_t)L * sizeof(int32_t));
        og_visit(&w->cx, L);
    }
    return NULL;
}

int orc_enumerate_split(int64_t n, const int64_t *row_ptr, const int32_t *col, uint32_t max_len,
                        uint64_t seed, int nthreads, int split_len, uint64_t *counts, uint64_t *set_hash,
                        uint64_t *paths_by_len, uint64_t *candidates)
{
    if (seed == 0)
        seed = 0x1410487600000000ULL;
    if (nthreads < 1 || split_len < 4)
        return ORC_ERR_INVALID_ARGUMENT;
    og_graph g;
    int rc = og_setup(&g, n, row_ptr, col, NULL, seed);
    if (rc != ORC_OK)
        return rc;
    int64_t ntri = 0;
    int64_t nt = og_triplets(&g, NULL, 0, NULL, 0, &ntri);
    og_triplet *trip = (og_triplet *)malloc((size_t)(nt > 0 ? nt : 1) * sizeof(og_triplet));
    og_triplet *tri = (og_triplet *)malloc((size_t)(ntri > 0 ? ntri : 1) * sizeof(og_triplet));
    og_triplets(&g, trip, nt, tri, ntri, &ntri);
    og_split_worker *ws = (og_split_worker *)calloc((size_t)nthreads + 1, sizeof(og_split_worker));
    for (int i = 0; i <= nthreads; i++) {
        og_ctx *cx = &ws[i].cx;
        cx->g = &g;
        cx->max_len = max_len;
        cx->counts = (uint64_t *)calloc((size_t)n + 2, sizeof(uint64_t));
        cx->paths_by_len = (uint64_t *)calloc((size_t)n + 2, sizeof(uint64_t));
        cx->path = (int32_t *)calloc((size_t)n + 2, sizeof(int32_t));
    }
    og_ctx *root = &ws[nthreads].cx; /* the single-threaded prefix phase */
    root->split_len = split_len;
    if (max_len == 0 || max_len >= 3) {
        for (int64_t i = 0; i < ntri; i++) {
            int32_t c[3] = {tri[i].x, tri[i].u, tri[i].y};
            og_record(root, c, 3);
        }
    }
    if (max_len == 0 || max_len >= 4) {
        for (int64_t i = 0; i < nt; i++) {
            root->path[0] = trip[i].x;
            root->path[1] = trip[i].u;
            root->path[2] = trip[i].y;
            og_visit(root, 3);
        }
    }
    int64_t next = 0;
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int i = 0; i < nthreads; i++) {
        ws[i].root = root;
        ws[i].next = &next;
        pthread_create(&th[i], NULL, og_split_main, &ws[i]);
    }
    for (int i = 0; i < nthreads; i++)
        pthread_join(th[i], NULL);
    free(th);
    for (int64_t k = 0; k <= n; k++) {
        counts[k] = 0;
        if (paths_by_len)
            paths_by_len[k] = 0;
    }
    *set_hash = 0;
    if (candidates)
        *candidates = 0;
    for (int i = 0; i <= nthreads; i++) {
        og_ctx *cx = &ws[i].cx;
        for (int64_t k = 0; k <= n; k++) {
            counts[k] += cx->counts[k];
            if (paths_by_len)
                paths_by_len[k] += cx->paths_by_len[k];
        }
        *set_hash += cx->set_hash;
        if (candidates)
            *candidates += cx->candidates;
        free(cx->counts);
        free(cx->paths_by_len);
        free(cx->path);
        free(cx->items);
    }
    free(ws);
    free(trip);
    free(tri);
    og_free(&g);
    return ORC_OK;
}
