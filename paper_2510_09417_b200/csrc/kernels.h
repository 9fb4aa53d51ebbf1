// Host-side launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "hull_types.cuh"

namespace vqb {

void launch_extremes(const double* xs, const double* ys, uint64_t n, void* partials,
                     uint32_t* ticket, RootInfo* root, int grid, cudaStream_t st);
void launch_bootstrap(const double* xs, const double* ys, uint64_t n, void* partials,
                      uint32_t* ticket, RootInfo* root, int grid, cudaStream_t st);
size_t partial_bytes(int grid);
void print_sample_trace();
uint32_t sample_mask(uint64_t n);
void fin_trace(bool on);
void print_fin_trace();
void upload_root_consts(const RootInfo* d_root, cudaStream_t st);
cudaError_t launch_root_partition(const RootArgs& a, int grid, bool stable, cudaStream_t st);
cudaError_t launch_level(const LevelArgs& a, bool general, bool stable, int grid, cudaStream_t st);
void launch_planner(const ChildRec* slots, uint32_t nslots, const LevelInfo* prev, uint32_t nslots_bound,
                    SegRec* segs, FinRec* fins, uint8_t* kind, uint32_t* link, LevelInfo* info,
                    uint32_t* flags, void* aggs, void* incs, uint32_t epoch, uint32_t* ctr,
                    uint32_t* seg_pcnt, uint32_t* seg_done, unsigned long long* seg_ctr,
                    int max_grid, cudaStream_t st, LevelInfo* next_info = nullptr);
void launch_tilemap(const SegRec* segs, const LevelInfo* info, uint32_t* tile_seg,
                    uint32_t ntiles_hint, cudaStream_t st);
void launch_finisher(const FinRec* fins, const LevelInfo* info, uint32_t fin_cap, const double* ix,
                     const double* iy, const uint32_t* iid, uint32_t* chain, uint32_t* fin_count,
                     uint32_t nfin_hint, int max_grid, cudaStream_t st);
// batch finisher (finisher.cu): several segments per CTA, nodes named by their apex
void launch_finisher_batch(const FinRec* fins, const LevelInfo* info, uint32_t fin_cap, const double* ix,
                           const double* iy, const uint32_t* iid, uint32_t* chain, uint32_t* fin_count,
                           uint32_t nfin_hint, int max_grid, cudaStream_t st);
int occupancy_finisher_batch();
void launch_size(uint32_t nslots, const uint8_t* kind, const uint32_t* link,
                 const uint32_t* fin_count, const uint32_t* child_size, uint32_t* size,
                 cudaStream_t st);
void launch_emit(uint32_t nslots, const uint8_t* kind, const uint32_t* link,
                 const ChildRec* slots, const FinRec* fins, const uint32_t* fin_count,
                 const uint32_t* chain, const uint32_t* start, const uint32_t* child_size,
                 uint32_t* child_start, uint32_t* out, cudaStream_t st);
void launch_poly_sample(const double* xs, const double* ys, uint64_t n, void* partials,
                        uint32_t* ticket, unsigned long long* keys, RootInfo* root,
                        unsigned long long* side_ctr, int grid, bool with_pq, cudaStream_t st);
cudaError_t launch_root_filtered(const RootArgs& a, int grid, cudaStream_t st);
void launch_emit_small(const EmitAll& e, const RootInfo* root, const uint32_t* chain, uint32_t* out,
                       uint32_t* h_out, cudaStream_t st);
void launch_legacy_poly(RootInfo* root, unsigned long long* side_ctr, cudaStream_t st);
void launch_poly_frame(const RootInfo* root, const uint32_t* size2, uint32_t* start2, uint32_t* out,
                       uint32_t* h_out, cudaStream_t st);
size_t plan_agg_bytes();
int occupancy_root(bool stable);
int occupancy_level(bool stable);
int occupancy_finisher();

int occupancy_filtered();
cudaError_t launch_root_filter(const FilterArgs& a, int grid, cudaStream_t st);
int occupancy_filter();
size_t filter_partial_bytes(int grid);
int occupancy_poly_sample();
int occupancy_extremes();
int occupancy_bootstrap();
uint32_t read_and_clear_fault();
uint32_t* fault_word_ptr();  // device address of the fault word (async copies)
void set_filter_inner(int mode);  // -1 auto (K_S picks), else force 0 box / 1 octagon / 2 disk when valid
void launch_tiny(const TinyArgs& a, cudaStream_t st);
size_t tail_smem_bytes();
int occupancy_tail();
cudaError_t launch_tail(const TailArgs& a, int grid, cudaStream_t st);
int kc_prepare();  // clusters of the cluster recursion the device can host (0: none)
cudaError_t launch_cluster_tail(const TailArgs& a, cudaStream_t st);

// sharded hull (shard.cu)
void launch_cert_build(const uint32_t* hull, uint32_t h, const double* xs, const double* ys, double floor_m,
                       CertHead* head, CertRec* rec, float* asc, uint32_t* tab, cudaStream_t st);
void launch_certify(const double* xs, const double* ys, const uint32_t* ids, uint64_t n_host,
                    const uint32_t* n_dev, const CertHead* head, const CertRec* rec, const float* asc,
                    const uint32_t* tab, double* rx, double* ry, uint32_t* rid, uint32_t* rcount,
                    unsigned long long* amax_bits, int grid, cudaStream_t st);
size_t sort_temp_bytes(uint32_t n);
cudaError_t launch_sort_ids(void* temp, size_t temp_bytes, const uint32_t* keys_in, uint32_t* keys_out,
                            uint32_t* vals_in, uint32_t* vals_out, uint32_t n, int end_bit, cudaStream_t st);
void launch_pack(const double* rx, const double* ry, const uint32_t* sorted_id, const uint32_t* perm,
                 uint32_t count, uint32_t cap, uint64_t offset, double* pack, cudaStream_t st);
void launch_merge_gather(const double* packs, uint64_t stride_rows, const uint64_t* starts, uint32_t nranks,
                         uint64_t total, double* mx, double* my, uint64_t* mg, uint32_t* unsorted,
                         cudaStream_t st);
void launch_map_gidx(const uint32_t* pos, uint64_t h, const uint64_t* mg, uint64_t* out, cudaStream_t st);

}  // namespace vqb
