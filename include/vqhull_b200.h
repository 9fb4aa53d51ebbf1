/*
 * vqhull_b200.h — C ABI of the B200-native VQhull hot path.
 *
 * Drop-in boundary.  The first entry point is the reference's own flat C
 * interface, same name, signature, ownership and return codes
 * (reference: proj/include/vqhull/vqhull_c.h:23-24, proj/src/vqhull_c.cpp:26-64);
 * a program linked against libvqhull_b200.so instead of the reference's
 * libvqhull.a gets the identical clockwise first-occurrence index list,
 * computed on the GPU.  The vqhull_cuda_* entry points expose the same
 * computation on device-resident arrays (the reference's C++ seam:
 * convex_hull, hull.hpp:58; find_extremes, geometry.hpp:135-138;
 * extract_subsets, extract.hpp:79-82) for callers that already hold the
 * points in HBM.
 *
 * All functions are reentrant (an internal per-device engine is guarded by a
 * mutex) and synchronous with respect to the caller: on return, outputs are
 * written.  Streams are passed as void* (a cudaStream_t), NULL = default stream.
 *
 * Return codes: 0 success; 1 invalid arguments (exactly the reference's
 * conditions: out_count NULL, workers < 1, NULL arrays with n > 0, a
 * non-finite coordinate); 2 unsupported size (n >= 2^32 - 1 points per
 * device); 3 CUDA error (see vqhull_cuda_last_error()); 4 (sharded merge
 * only) retry the shards with a margin floor.
 */
#ifndef VQHULL_B200_H
#define VQHULL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VQHULL_OK 0
#define VQHULL_EINVAL 1
#define VQHULL_ESIZE 2
#define VQHULL_ECUDA 3
#define VQHULL_ERETRY 4  /* sharded merge: recompute the shards with a margin floor */

/* Replaces vqhull_compute (vqhull_c.h:23-24, vqhull_c.cpp:26-64).
 * xs, ys: n host coordinates (pageable or pinned).  out_indices: host array
 * with room for n entries; receives the input indices of the hull vertices,
 * clockwise from the leftmost(-lowest) point; equal coordinates resolve to
 * the first occurrence.  `workers` is validated (>= 1) as in the reference;
 * the GPU path does not use it. */
int vqhull_compute(const double* xs, const double* ys, size_t n, int workers,
                   size_t* out_indices, size_t* out_count);

/* Same computation on device-resident arrays.  d_xs, d_ys: device pointers
 * (not modified).  out_indices: host OR device pointer with room for n
 * uint64 entries.  Replaces convex_hull (hull.hpp:58) + the index mapping of
 * vqhull_c.cpp:46-61. */
int vqhull_cuda_hull(const double* d_xs, const double* d_ys, uint64_t n,
                     uint64_t* out_indices, uint64_t* out_count, void* stream);

/* Same, 32-bit indices written to a DEVICE buffer, no host round trip of the
 * index list (the bench's device-resident leg).  *out_count is host memory. */
int vqhull_cuda_hull_u32(const double* d_xs, const double* d_ys, uint64_t n,
                         uint32_t* d_out_indices, uint64_t* out_count, void* stream);

/* find_extremes (geometry.cpp:7-36) on device arrays: lo = leftmost (ties:
 * lowest y, then first index), hi = rightmost (ties: highest y, then first
 * index).  Returns 1 for n == 0 (the reference throws). */
int vqhull_cuda_find_extremes(const double* d_xs, const double* d_ys, uint64_t n,
                              uint64_t* lo, uint64_t* hi, void* stream);

/* extract_subsets (extract.hpp:75-82) on device arrays, in place: afterwards
 * [0, *w_l) holds exactly the points left of edge_a, [*w_r, n) exactly the
 * points left of edge_b and not of edge_a, the middle is unspecified.
 * edge = {px, py, qx, qy} (host).  r1/r2 (host, 2 doubles) receive the
 * farthest point of each side in the canonical order (kernels.hpp:36-45);
 * has_r1/has_r2 say whether the side is non-empty. */
int vqhull_cuda_extract_subsets(double* d_xs, double* d_ys, uint64_t n,
                                const double* edge_a, const double* edge_b,
                                uint64_t* w_l, uint64_t* w_r, double* r1,
                                int* has_r1, double* r2, int* has_r2,
                                void* stream);

/* Statistics of the last vqhull_cuda_hull* / vqhull_compute call on this
 * thread's device engine. */
typedef struct vqhull_stats {
    uint64_t n;                 /* points */
    uint64_t hull_size;         /* vertices */
    uint32_t levels;            /* recursion levels processed on device */
    uint32_t launches;          /* kernels launched by the call */
    uint64_t survivors_root;    /* points written by the fused root pass */
    uint64_t level_points;      /* sum over levels of points partitioned by K2 */
    uint64_t finisher_points;   /* points handed to the warp finisher */
    uint64_t finisher_segments;
    uint64_t segments;          /* K2 segments over all levels */
    uint64_t bytes_moved;       /* algorithmic HBM bytes */
    /* per-kernel device time (ms), valid when timing is enabled */
    float ms_extremes;
    float ms_bootstrap;
    float ms_root_partition;
    float ms_levels;            /* all K2 launches */
    float ms_finisher;
    float ms_other;             /* planner, tile map, emission */
    float ms_total;             /* first kernel start .. last kernel end */
    uint32_t timing_valid;
    uint64_t bytes_extremes;    /* algorithmic bytes per kernel family */
    uint64_t bytes_bootstrap;
    uint64_t bytes_root_partition;
    uint64_t bytes_levels;
    uint64_t bytes_finisher;
    uint32_t root_filtered;     /* 2 (default): split root = octagon from a 1/16
                                   sample, one filter pass over every point (exact
                                   p, q of the survivors), level 1 over the
                                   survivors; 1: exact extremes pass + level 1
                                   behind the octagon filter in one pass;
                                   0: find_extremes + bootstrap + fused levels 1+2 */
    uint32_t root_filter_on;    /* the octagon filter could drop points (coordinate
                                   magnitudes in range) */
    uint32_t root_reruns;       /* 1: a split-root survivor lay beyond 2^12 x the
                                   polygon's scale, the call was rerun unfiltered */
    uint32_t tail_launches;     /* launches of the persistent recursion kernel */
    uint32_t tail_levels;       /* levels it processed */
    uint64_t shard_tested;      /* last vqhull_cuda_shard_candidates: points certified */
    uint64_t shard_candidates;  /* ... and the candidates it kept */
    uint32_t shard_cert_vertices; /* vertices of the certificate polygon (0: none) */
    uint32_t pad0;
} vqhull_stats;

int vqhull_cuda_get_stats(vqhull_stats* out);

/* Enable (1) / disable (0) per-kernel CUDA-event timing inside the engine. */
int vqhull_cuda_set_timing(int enable);

/* Output-offset mode of the partition kernels.  0 (default): each tile
 * claims its place in S1/S2 with one packed atomic — no tile waits for
 * another; survivors inside S1/S2 follow claim order, which the reference
 * leaves unspecified (extract.hpp:14-18).  1: decoupled look-back, survivors
 * keep input order (order-preserving compaction).  Hull outputs are identical
 * in both modes.  The environment variable VQHULL_STABLE=1 sets the default. */
int vqhull_cuda_set_stable(int stable);

/* Root stage: 0 (default, fast mode with 16-byte aligned inputs) one pass for
 * the 8 exact directional extremes, then level 1 behind their octagon filter;
 * 1: find_extremes, bootstrap arg-max and the fused levels-1+2 pass.  The
 * recursion is the reference's in both; hull outputs are identical.  The
 * environment variable VQHULL_ROOT=reference sets 1. */
int vqhull_cuda_set_root_reference(int reference);

/* Root stage, all three giving identical hulls: 0 (default) split root —
 * octagon from a 1/16 sample, one filter pass over every point (survivors,
 * exact p and q), level 1 over the survivors; 1 one-pass octagon root (exact
 * extremes pass, then level 1 behind the filter); 2 = set_root_reference(1).
 * Returns 1 for another mode.  VQHULL_ROOT=octagon|reference sets 1|2. */
int vqhull_cuda_set_root_mode(int mode);

/* The filter pass's fast inner test (a drop region verified inside the
 * filter polygon, tested before the chord test): -1 = automatic (the sample
 * pass picks the region of largest area, default), 0 = the box only,
 * 1 = box | octagon, 2 = box | disk, 3 = the disk alone (what the automatic
 * choice takes when the disk covers the box; a forced region that does not
 * exist for the input falls back to the automatic choice).  The hull never
 * depends on it; tests use it to show that.  Returns VQHULL_EINVAL outside
 * -1..3. */
int vqhull_cuda_set_filter_inner(int mode);

/* Frees this thread's device engine buffers (points, level tables) and
 * trims the memory pool; the next call re-allocates.  For callers that need
 * the device memory back between hulls. */
int vqhull_cuda_trim(void);

/* Human-readable description of the last CUDA error (thread-local). */
const char* vqhull_cuda_last_error(void);

/* 1 when a CUDA device is usable from this library. */
int vqhull_cuda_available(void);

/* ---- sharded hull ----------------------------
 * Exact by construction: each shard sends every point it cannot prove to be
 * deep inside its own local hull (a margin argument), and the
 * merge runs the ordinary recursion over the union; the result equals the
 * reference's global recursion over all points.
 *
 * Local stage on this device: hull of the shard d_xs/d_ys[0, n) (global
 * indices offset + i), then its candidates, sorted by global index and packed
 * as 3-double rows: row 0 = {count, M_eff, A} (count = -1: the shard holds a
 * non-finite coordinate), rows 1.. = {x, y, global index as uint64 bits}.
 * d_pack: device buffer of cap_rows + 1 rows (NULL: only *count); the first
 * min(count, cap_rows) candidates are written.  margin_floor: 0, or the value
 * a merge returned with VQHULL_ERETRY. */
int vqhull_cuda_shard_candidates(const double* d_xs, const double* d_ys, uint64_t n, uint64_t offset,
                                 double margin_floor, double* d_pack, uint64_t cap_rows,
                                 uint64_t* count, void* stream);

/* The last vqhull_cuda_shard_candidates' pack again, with room for cap_rows
 * candidates (after a first pack that was too small). */
int vqhull_cuda_shard_repack(double* d_pack, uint64_t cap_rows, void* stream);

/* Merge on this device: nranks packs in offset order, pack r at
 * d_packs + 3 * r * stride_rows.  out_indices (host or device, room for all
 * candidates) receives the global clockwise first-occurrence list.
 * VQHULL_ERETRY: recompute every shard with *margin_floor and merge again. */
int vqhull_cuda_merge_candidates(const double* d_packs, uint32_t nranks, uint64_t stride_rows,
                                 uint64_t* out_indices, uint64_t* out_count, double* margin_floor,
                                 void* stream);

/* Single-process multi-GPU hull of HOST arrays: num_shards contiguous shards,
 * shard s on device s mod (device count), each with its own H2D, local hull
 * and candidates; peer copies to device 0, merge there.  64-bit indices: n
 * may exceed 2^32 - 1 when every shard stays below it.  vqhull_compute uses
 * this path when VQHULL_GPUS is set (its value = shards) or n needs it. */
int vqhull_cuda_hull_multi(const double* xs, const double* ys, uint64_t n, int num_shards,
                           uint64_t* out_indices, uint64_t* out_count);

/* Library version string. */
const char* vqhull_b200_version(void);

/* Dataset generators (tooling, not the hot path): the reference's counter-
 * based splitmix64 streams (dataset.cpp:32-75) plus the harness-defined
 * square (BASELINE config 2: x = 2U(2i)-1, y = 2U(2i+1)-1).  Fills points
 * [first, first+n) of the (kind, seed) sequence into host xs/ys using
 * `threads` host threads.  kind: 0 kuzmin, 1 circle, 2 disk, 3 square. */
int vqhull_generate(int kind, uint64_t seed, uint64_t first, uint64_t n,
                    double* xs, double* ys, int threads);

#ifdef __cplusplus
}
#endif

#endif /* VQHULL_B200_H */
