/*
 * TEST INFRASTRUCTURE — CPU oracle for the VQhull hot path.
 *
 * A plain-C restatement of the reference algorithm (VQhull, arxiv 2510.09417,
 * /root/reference/proj).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library, and only as the CHECKER; the product
 * (paper_2510_09417_b200) never links or calls it.
 *
 * Pinned against the reference: tests/test_oracle.py compares every function
 * here with oracle/_ref/libvqhull_ref.so (the reference compiled from its own
 * sources) and with the committed golden vectors under tests/golden/.
 *
 * Build: oracle/Makefile, -O2 -ffp-contract=off (the reference's own
 * CMakeLists.txt:17 flag), so every predicate rounds exactly like the
 * reference's scalar and vector paths.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double x, y; } opt_point;

/* ---------------------------------------------------------------------------
 * Predicates — kernels.hpp:19-45 (EdgeFrame, frame_left_of, frame_offset,
 * prefer_farthest).  Evaluated with the exact same expressions and operand
 * order; FP contraction is off for this translation unit.
 * ------------------------------------------------------------------------- */
typedef struct {
    double px, py, qx, qy, dx, dy;
} edge_frame;

static edge_frame frame_make(double px, double py, double qx, double qy) {
    edge_frame e = {px, py, qx, qy, qx - px, qy - py}; /* kernels.hpp:23-25 */
    return e;
}

static int frame_left_of(double ux, double uy, const edge_frame* e) {
    return (e->px - ux) * (e->qy - uy) > (e->py - uy) * (e->qx - ux); /* :28-30 */
}

static double frame_offset(double ux, double uy, const edge_frame* e) {
    return e->dy * ux - e->dx * uy; /* :32-34 */
}

/* Canonical farthest order, kernels.hpp:41-45: smaller offset wins; an exact
 * tie falls to the lexicographically smaller point. */
static int prefer_farthest(double co, double cx, double cy, double io,
                           double ix, double iy) {
    if (co != io) return co < io;
    return cx < ix || (cx == ix && cy < iy);
}

/* SideTracker, extract_core.hpp:308-334 */
typedef struct {
    edge_frame f;
    int present;
    double off, x, y;
} side_tracker;

static void tracker_consider(side_tracker* t, double x, double y) {
    const double g = frame_offset(x, y, &t->f);
    if (!t->present || prefer_farthest(g, x, y, t->off, t->x, t->y)) {
        t->present = 1;
        t->off = g;
        t->x = x;
        t->y = y;
    }
}

/* ---------------------------------------------------------------------------
 * find_extremes — geometry.cpp:7-36.  lo: min x, ties to min y, then first
 * index; hi: max x, ties to max y, then first index.  Returns 1 on n == 0
 * (the reference throws std::invalid_argument).
 * ------------------------------------------------------------------------- */
int oracle_find_extremes(const double* xs, const double* ys, size_t n,
                         size_t* lo_out, size_t* hi_out) {
    if (n == 0) return 1;
    size_t lo = 0, hi = 0;
    double lo_x = xs[0], hi_x = xs[0];
    for (size_t i = 1; i < n; ++i) {
        const double x = xs[i];
        if (x < lo_x) {
            lo_x = x;
            lo = i;
        } else if (x == lo_x) {
            if (ys[i] < ys[lo]) lo = i;
        }
        if (x > hi_x) {
            hi_x = x;
            hi = i;
        } else if (x == hi_x && i != hi) {
            if (ys[i] > ys[hi]) hi = i;
        }
    }
    *lo_out = lo;
    *hi_out = hi;
    return 0;
}

/* ---------------------------------------------------------------------------
 * One partition pass — the contract of extract_subsets (extract.hpp:14-24,
 * 75-82), restated as the scalar path extract_small (extract_core.hpp:518-537):
 * points left of A are written forward from 0, points left of B (and not of
 * A: kernels.hpp:91) backward from n; r1/r2 follow the canonical order.  The
 * order INSIDE each side differs from the reference's vector path, which the
 * reference itself leaves unspecified; the multisets and r1/r2 are identical.
 * `scratch` must hold 2n doubles.
 * ------------------------------------------------------------------------- */
typedef struct {
    size_t w_l, w_r;
    int has_r1, has_r2;
    opt_point r1, r2;
} extract_outcome;

static extract_outcome extract_pass(double* xs, double* ys, size_t n,
                                    const edge_frame* a, const edge_frame* b,
                                    double* scratch) {
    extract_outcome o;
    side_tracker t1 = {*a, 0, 0, 0, 0}, t2 = {*b, 0, 0, 0, 0};
    double* tx = scratch;
    double* ty = scratch + n;
    memcpy(tx, xs, n * sizeof(double));
    memcpy(ty, ys, n * sizeof(double));
    size_t wl = 0, wr = n;
    for (size_t i = 0; i < n; ++i) {
        const double x = tx[i], y = ty[i];
        if (frame_left_of(x, y, a)) {
            xs[wl] = x;
            ys[wl] = y;
            ++wl;
            tracker_consider(&t1, x, y);
        } else if (frame_left_of(x, y, b)) {
            --wr;
            xs[wr] = x;
            ys[wr] = y;
            tracker_consider(&t2, x, y);
        }
    }
    o.w_l = wl;
    o.w_r = wr;
    o.has_r1 = t1.present;
    o.has_r2 = t2.present;
    o.r1.x = t1.x; o.r1.y = t1.y;
    o.r2.x = t2.x; o.r2.y = t2.y;
    return o;
}

int oracle_extract_subsets(double* xs, double* ys, size_t n, const double* ea,
                           const double* eb, size_t* w_l, size_t* w_r,
                           double* r1, int* has_r1, double* r2, int* has_r2) {
    const edge_frame a = frame_make(ea[0], ea[1], ea[2], ea[3]);
    const edge_frame b = frame_make(eb[0], eb[1], eb[2], eb[3]);
    double* scratch = (double*)malloc((2 * n + 2) * sizeof(double));
    if (!scratch) return 1;
    const extract_outcome o = extract_pass(xs, ys, n, &a, &b, scratch);
    free(scratch);
    *w_l = o.w_l;
    *w_r = o.w_r;
    *has_r1 = o.has_r1;
    *has_r2 = o.has_r2;
    r1[0] = o.r1.x; r1[1] = o.r1.y;
    r2[0] = o.r2.x; r2[1] = o.r2.y;
    return 0;
}

/* ---------------------------------------------------------------------------
 * Quickhull driver — hull.cpp:119-190 (chain_iterative, explicit stack) with
 * assemble_chain (hull.cpp:59-73) and the convex_hull bootstrap (:207-267).
 * The recursive driver (:78-115) computes the identical sequence; only the
 * explicit-stack form is restated.
 * ------------------------------------------------------------------------- */
typedef struct {
    size_t lo, hi;
    opt_point p, r, q;
    int phase;
    size_t abs_wl, abs_wr;
    opt_point r1, r2;
    size_t c1;
} frame_t;

typedef struct {
    double* xs;
    double* ys;
    double* scratch;
    /* optional per-call trace (points, s1, s2, chain2_moved) */
    uint64_t* trace;
    size_t trace_cap, trace_len;
} hull_ctx;

static size_t assemble_chain(hull_ctx* c, size_t lo, opt_point r, size_t c1,
                             size_t abs_wr, size_t c2, size_t trace_idx) {
    c->xs[lo + c1] = r.x;
    c->ys[lo + c1] = r.y;
    if (c2 > 0) {
        const size_t dst = lo + c1 + 1;
        memmove(c->xs + dst, c->xs + abs_wr, c2 * sizeof(double));
        memmove(c->ys + dst, c->ys + abs_wr, c2 * sizeof(double));
    }
    if (c->trace && trace_idx < c->trace_cap) c->trace[4 * trace_idx + 3] = c2;
    return c1 + 1 + c2;
}

static size_t record_call(hull_ctx* c, size_t m, size_t s1, size_t s2) {
    const size_t id = c->trace_len++;
    if (c->trace && id < c->trace_cap) {
        c->trace[4 * id + 0] = m;
        c->trace[4 * id + 1] = s1;
        c->trace[4 * id + 2] = s2;
        c->trace[4 * id + 3] = 0;
    }
    return id;
}

/* Returns the chain length, or (size_t)-1 on allocation failure. */
static size_t chain_iterative(hull_ctx* c, size_t lo, size_t hi, opt_point p,
                              opt_point r, opt_point q) {
    size_t cap = 64, top = 0;
    frame_t* st = (frame_t*)malloc(cap * sizeof(frame_t));
    if (!st) return (size_t)-1;
    size_t* tix = (size_t*)malloc(cap * sizeof(size_t));
    if (!tix) { free(st); return (size_t)-1; }
    memset(&st[0], 0, sizeof(frame_t));
    st[0].lo = lo; st[0].hi = hi; st[0].p = p; st[0].r = r; st[0].q = q;
    top = 1;
    size_t ret = 0;
    while (top > 0) {
        frame_t* f = &st[top - 1];
        if (f->phase == 0) {
            const size_t m = f->hi - f->lo;
            if (m <= 1) { /* hull.cpp:83 — the single point is r itself */
                ret = m;
                --top;
                continue;
            }
            const edge_frame ea = frame_make(f->p.x, f->p.y, f->r.x, f->r.y);
            const edge_frame eb = frame_make(f->r.x, f->r.y, f->q.x, f->q.y);
            const extract_outcome o = extract_pass(c->xs + f->lo, c->ys + f->lo,
                                                   m, &ea, &eb, c->scratch);
            const size_t s1 = o.w_l, s2 = m - o.w_r;
            f->abs_wl = f->lo + o.w_l;
            f->abs_wr = f->lo + o.w_r;
            tix[top - 1] = record_call(c, m, s1, s2);
            f->r1 = o.r1;
            f->r2 = o.r2;
            f->phase = 1;
            if (s1 > 0) {
                if (top == cap) {
                    cap *= 2;
                    frame_t* ns = (frame_t*)realloc(st, cap * sizeof(frame_t));
                    size_t* nt = (size_t*)realloc(tix, cap * sizeof(size_t));
                    if (!ns || !nt) { free(ns ? ns : st); free(nt ? nt : tix); return (size_t)-1; }
                    st = ns; tix = nt;
                    f = &st[top - 1];
                }
                frame_t* ch = &st[top++];
                memset(ch, 0, sizeof(frame_t));
                ch->lo = f->lo; ch->hi = f->abs_wl;
                ch->p = f->p; ch->r = f->r1; ch->q = f->r;
            } else {
                ret = 0;
            }
        } else if (f->phase == 1) {
            f->c1 = ret;
            f->phase = 2;
            if (f->abs_wr < f->hi) {
                if (top == cap) {
                    cap *= 2;
                    frame_t* ns = (frame_t*)realloc(st, cap * sizeof(frame_t));
                    size_t* nt = (size_t*)realloc(tix, cap * sizeof(size_t));
                    if (!ns || !nt) { free(ns ? ns : st); free(nt ? nt : tix); return (size_t)-1; }
                    st = ns; tix = nt;
                    f = &st[top - 1];
                }
                frame_t* ch = &st[top++];
                memset(ch, 0, sizeof(frame_t));
                ch->lo = f->abs_wr; ch->hi = f->hi;
                ch->p = f->r; ch->r = f->r2; ch->q = f->q;
            } else {
                ret = 0;
            }
        } else {
            ret = assemble_chain(c, f->lo, f->r, f->c1, f->abs_wr, ret,
                                 tix[top - 1]);
            --top;
        }
    }
    free(st);
    free(tix);
    return ret;
}

/* convex_hull (hull.cpp:207-267) on a private copy; writes the vertex
 * coordinates clockwise from the leftmost(-lowest) point.  out_* need room
 * for n entries.  Returns 0, or 1 on allocation failure. */
static int hull_coords(const double* xs_in, const double* ys_in, size_t n,
                       double* out_x, double* out_y, size_t* out_count,
                       uint64_t* trace, size_t trace_cap, size_t* trace_len) {
    *out_count = 0;
    if (trace_len) *trace_len = 0;
    if (n == 0) return 0;
    hull_ctx c;
    memset(&c, 0, sizeof c);
    c.xs = (double*)malloc(n * sizeof(double));
    c.ys = (double*)malloc(n * sizeof(double));
    c.scratch = (double*)malloc(2 * n * sizeof(double));
    c.trace = trace;
    c.trace_cap = trace_cap;
    if (!c.xs || !c.ys || !c.scratch) {
        free(c.xs); free(c.ys); free(c.scratch);
        return 1;
    }
    memcpy(c.xs, xs_in, n * sizeof(double));
    memcpy(c.ys, ys_in, n * sizeof(double));

    size_t ilo = 0, ihi = 0;
    oracle_find_extremes(c.xs, c.ys, n, &ilo, &ihi);
    const opt_point p = {c.xs[ilo], c.ys[ilo]};
    const opt_point q = {c.xs[ihi], c.ys[ihi]};

    /* bootstrap: degenerate triangle p, q, p (hull.cpp:228-235) */
    const edge_frame ea = frame_make(p.x, p.y, q.x, q.y);
    const edge_frame eb = frame_make(q.x, q.y, p.x, p.y);
    const extract_outcome o = extract_pass(c.xs, c.ys, n, &ea, &eb, c.scratch);
    const size_t s1 = o.w_l, s2 = n - o.w_r;
    record_call(&c, n, s1, s2);

    size_t c1 = 0, c2 = 0;
    int fail = 0;
    if (s1 > 0) {
        c1 = chain_iterative(&c, 0, o.w_l, p, o.r1, q);
        if (c1 == (size_t)-1) fail = 1;
    }
    if (!fail && s2 > 0) {
        c2 = chain_iterative(&c, o.w_r, n, q, o.r2, p);
        if (c2 == (size_t)-1) fail = 1;
    }
    if (!fail) {
        size_t k = 0;
        out_x[k] = p.x; out_y[k] = p.y; ++k;
        for (size_t i = 0; i < c1; ++i) { out_x[k] = c.xs[i]; out_y[k] = c.ys[i]; ++k; }
        if (!(q.x == p.x && q.y == p.y)) { out_x[k] = q.x; out_y[k] = q.y; ++k; }
        for (size_t i = 0; i < c2; ++i) {
            out_x[k] = c.xs[o.w_r + i]; out_y[k] = c.ys[o.w_r + i]; ++k;
        }
        *out_count = k;
    }
    if (trace_len) *trace_len = c.trace_len;
    free(c.xs); free(c.ys); free(c.scratch);
    return fail;
}

int oracle_convex_hull(const double* xs, const double* ys, size_t n,
                       double* out_x, double* out_y, size_t* out_count) {
    return hull_coords(xs, ys, n, out_x, out_y, out_count, NULL, 0, NULL);
}

/* Traced hull: per-call records {points, s1, s2, chain2_moved} in the
 * reference's order (hull.hpp:26-36) and the byte model (bench.cpp:16-21). */
int oracle_trace_hull(const double* xs, const double* ys, size_t n,
                      uint64_t* calls, size_t calls_cap, size_t* n_calls,
                      uint64_t* model_bytes, size_t* hull_size) {
    double* hx = (double*)malloc((n + 1) * sizeof(double));
    double* hy = (double*)malloc((n + 1) * sizeof(double));
    if (!hx || !hy) { free(hx); free(hy); return 1; }
    int own = 0;
    if (!calls) {
        calls_cap = n + 2;
        calls = (uint64_t*)malloc(4 * calls_cap * sizeof(uint64_t));
        if (!calls) { free(hx); free(hy); return 1; }
        own = 1;
    }
    size_t len = 0;
    const int rc = hull_coords(xs, ys, n, hx, hy, hull_size, calls, calls_cap, &len);
    uint64_t bytes = 8 * (uint64_t)n;
    for (size_t i = 0; i < len && i < calls_cap; ++i)
        bytes += 16 * (calls[4 * i] + calls[4 * i + 1] + calls[4 * i + 2]) +
                 16 * calls[4 * i + 3];
    *model_bytes = bytes;
    *n_calls = len;
    if (own) free(calls);
    free(hx); free(hy);
    return rc;
}

/* ---------------------------------------------------------------------------
 * vqhull_compute semantics — vqhull_c.cpp:26-64: argument checks (return 1),
 * hull, then every vertex maps to the FIRST input index holding equal
 * coordinates (== comparison, so +0.0 and -0.0 match, :11-22 and :57).
 * The reference uses an n-entry unordered_multimap; this restatement sorts the
 * h vertices and scans the input once (same result, O(n log h), h memory).
 * ------------------------------------------------------------------------- */
typedef struct {
    double x, y;
    size_t v;
} vkey;

static int vkey_cmp(const void* a, const void* b) {
    const vkey* u = (const vkey*)a;
    const vkey* w = (const vkey*)b;
    if (u->x < w->x) return -1;
    if (u->x > w->x) return 1;
    if (u->y < w->y) return -1;
    if (u->y > w->y) return 1;
    return 0;
}

int oracle_compute(const double* xs, const double* ys, size_t n, int workers,
                   uint64_t* out_indices, size_t* out_count) {
    if (!out_count || workers < 1) return 1;
    *out_count = 0;
    if (n == 0) return 0;
    if (!xs || !ys || !out_indices) return 1;
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(xs[i]) || !isfinite(ys[i])) return 1;

    double* hx = (double*)malloc(n * sizeof(double));
    double* hy = (double*)malloc(n * sizeof(double));
    if (!hx || !hy) { free(hx); free(hy); return 1; }
    size_t h = 0;
    if (oracle_convex_hull(xs, ys, n, hx, hy, &h)) { free(hx); free(hy); return 1; }

    vkey* keys = (vkey*)malloc((h ? h : 1) * sizeof(vkey));
    uint64_t* best = (uint64_t*)malloc((h ? h : 1) * sizeof(uint64_t));
    if (!keys || !best) { free(hx); free(hy); free(keys); free(best); return 1; }
    for (size_t v = 0; v < h; ++v) {
        keys[v].x = hx[v];
        keys[v].y = hy[v];
        keys[v].v = v;
        best[v] = (uint64_t)n;
    }
    qsort(keys, h, sizeof(vkey), vkey_cmp);
    for (size_t i = 0; i < n; ++i) {
        size_t a = 0, b = h;
        const vkey probe = {xs[i], ys[i], 0};
        while (a < b) { /* lower bound */
            const size_t mid = a + (b - a) / 2;
            if (vkey_cmp(&keys[mid], &probe) < 0) a = mid + 1; else b = mid;
        }
        /* hull vertices are pairwise distinct, so at most one key matches */
        if (a < h && keys[a].x == xs[i] && keys[a].y == ys[i]) {
            const size_t v = keys[a].v;
            if (best[v] == (uint64_t)n) best[v] = i;
        }
    }
    int rc = 0;
    for (size_t v = 0; v < h; ++v) {
        if (best[v] == (uint64_t)n) { rc = 1; break; } /* cannot happen */
        out_indices[v] = best[v];
    }
    if (!rc) *out_count = h;
    free(hx); free(hy); free(keys); free(best);
    return rc;
}

/* FNV-1a-64 over the index list, every index a little-endian u64 — the hash
 * used for the golden index lists. */
uint64_t oracle_fnv1a64_u64(const uint64_t* v, size_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n; ++i) {
        uint64_t x = v[i];
        for (int b = 0; b < 8; ++b) {
            h ^= (x >> (8 * b)) & 0xffu;
            h *= 0x100000001b3ull;
        }
    }
    return h;
}
