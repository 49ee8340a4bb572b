// ts_kernels.cuh -- kernel launch interfaces shared by the translation units.
#pragma once
#include "ts_common.cuh"

namespace ts {

struct Counters {
    unsigned long long m;        // accepted triangles
    unsigned long long e;        // tile entries
    unsigned long long key_and;  // AND / OR of accepted depth keys (pass selection)
    unsigned long long key_or;
    unsigned long long key_min;
    unsigned long long key_max;
    long long err[4];            // first non-finite index per group
    unsigned long long n_flagged;
    unsigned long long n_frec;       // fragment records emitted by the training forward
    unsigned long long frec_over;    // 1: the record buffer overflowed (backward falls back)
    unsigned long long blend_done;   // blend CTAs finished (the fix-up's end-of-flags signal)
    unsigned long long pad[2];
};

// One composited fragment of a training forward, in (tile, batch, entry-major)
// order, for the streaming backward: the transmittance and the accumulated
// colour in front of it (fp64), its pixel, source triangle and ordinal in the
// pixel's list.  pix = ~0u marks a hole (a passing pair that was not composited).
struct __align__(16) FragRec {
    double T;
    double C[3];
    unsigned pix, src, ord, pad;
};
static_assert(sizeof(FragRec) == 48, "FragRec layout");

struct PreOut {
    Rec64* rec;                // (N) fp64 records (accepted only)
    short4* bbox;              // (N) clipped pixel bbox (0s if culled)
    unsigned long long* key;   // (N) depth bits
    unsigned* tcount;          // (N) tiles touched
    unsigned* flag;            // (N) accepted
    float* area;               // (N) per_triangle_area, nullable
    double* depth;             // (N) centroid depth, nullable
    Counters* ctr;
};

struct FastPreOut {
    RecF* rec;                 // (N) fast records (accepted with tiles only)
    RecB* recb;                // (N) backward records, nullable (training forwards)
    RecC* recc;                // (N) fp64 colour / opacity / sigma, nullable (training forwards)
    short4* bbox;              // (N)
    unsigned long long* key;
    unsigned* tcount;
    unsigned* flag;
    float* area;
    double* depth;
    Counters* ctr;
    float* max_weight;         // zeroed per triangle (nullable): the blend accumulates into them
    int* pixel_count;
};

struct FastBlendOut {
    float* image;
    float* alpha_map;
    float* max_weight;
    int* pixel_count;
    int* last_src;
    int* n_frag;
    float* t_final;
    double* t_final64;         // training forward only
    int* last_pos;
    int2* flags;               // (pixel, flag position) of guard-band pixels
    Counters* ctr;
    // fragment emission (render(collect_fragments=True), render.py:383-399):
    // fragment i of pixel p goes to frag_off[p] + i; null = no emission
    const long long* frag_off;
    int* frag_tri;             // source id
    double* frag_w;            // blend weight T * alpha
    double* frag_z;            // camera-space depth of the triangle
    const unsigned long long* zkey;  // (N) fp64 bit pattern of the centroid depth
    // training forwards: fragment records for the streaming backward (null = none)
    FragRec* frec;
    unsigned long long frec_cap;
    double* c_total64;         // (P,3) unclipped colour incl. T_final * background
    const RecC* recc;          // training forwards: fp64 colours of the sources
    const int* tile_order;     // blend order of the tiles (longest first), null = tile id order
};

struct BlendOut {
    float* image;
    float* alpha_map;
    float* max_weight;
    int* pixel_count;
    int* last_src;
    int* n_frag;
    double* t_final;
    int* last_pos;
};

// ts_exact.cu
// project_scene dump: PROJ_ROW doubles per depth-sorted accepted triangle (see k_projection_dump)
constexpr int PROJ_ROW = 64;
void launch_projection_dump(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                            const unsigned* sorted_src, long long m, double* rows, double* area_full,
                            cudaStream_t st);
void launch_preprocess(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                       const PreOut& out, cudaStream_t st);
void launch_blend_exact(const Cam& cam, const Opts& opt, const Rec64* rec, const int* tile_start,
                        const int* ent_src, const BlendOut& out, cudaStream_t st);
void launch_blend_bwd_exact(const Cam& cam, const Opts& opt, const Rec64* rec, const int* tile_start,
                            const int* ent_src, const double* t_final, const int* last_pos,
                            const float* d_image, double* sgrad, cudaStream_t st);
void launch_chain_bwd(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                      const unsigned* flag, const double* sgrad, const ts_grads& g, int accumulate,
                      cudaStream_t st);
void launch_chain_bwd32(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                        const unsigned* flag, const float* sgrad, const ts_grads& g, int accumulate,
                        cudaStream_t st);

// ts_fast.cu
void launch_preprocess_fast(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                            const FastPreOut& out, cudaStream_t st);
void launch_blend_fast(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype, const RecF* rec,
                       const short4* bbox, const int* tile_start, const unsigned* ent_src, const FastBlendOut& out,
                       cudaStream_t st);
void launch_fixup_fwd(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype, const RecF* rec,
                      const int* tile_start, const unsigned* ent_src, const FastBlendOut& out,
                      cudaStream_t st);

// ts_blend.cu: render-only forward blend (dense pair evaluation)
void launch_blend_dense(const Cam& cam, const Opts& opt, bool acc64, const RecF* rec, const int* tile_start,
                        const unsigned* ent_src, const FastBlendOut& out, cudaStream_t st);

// ts_bwd.cu: dense backward blend
void launch_blend_bwd_dense(const Cam& cam, const Opts& opt, const RecF* rec, const RecB* recb, const RecC* recc,
                            const int* tile_start, const unsigned* ent_src, const double* t_final,
                            const int* last_pos, const float* d_image, const int* n_frag, const long long* frag_off,
                            const double* fg_dw, const double* fg_dz, const unsigned long long* run_if, double* sgrad,
                            cudaStream_t st);
// ts_bwd_stream.cu: streaming backward over the training forward's fragment records
// with frag_off: the fragment-gradient terms too (frag_w: the fragments' blend weights from
// ts_collect_fragments of the same forward; sw: scratch of F doubles)
void launch_bwd_stream(const Cam& cam, const Opts& opt, const RecF* rec, const RecB* recb, const RecC* recc,
                       const FragRec* frec, const Counters* ctr, unsigned long long cap, const double* c_total,
                       const float* d_image, double* sgrad, cudaStream_t st, const long long* frag_off = nullptr,
                       const double* frag_w = nullptr, const double* fg_dw = nullptr, const double* fg_dz = nullptr,
                       double* sw = nullptr);

// ts_chain.cu: fp32-parameter chain to the 59 parameter gradients (false: not applicable)
// deferred multi-view chain (ts_backward_screen / ts_chain_views)
constexpr int TS_MAX_CHAIN_VIEWS = 8;
struct ChainViews {
    Cam cam[TS_MAX_CHAIN_VIEWS];
    const unsigned* flag[TS_MAX_CHAIN_VIEWS];
    const double* sgrad[TS_MAX_CHAIN_VIEWS];
    int n;
};
void launch_chain_multi(const ChainViews& cv, const Opts& opt, const ts_soup& soup, const ts_grads& g,
                        int accumulate, cudaStream_t st, long long lo = 0, long long hi = -1);
bool chain_bwd_fast_ok(const ts_soup& soup, int dtype, const ts_grads& g);
// triangles [lo, hi) (hi < 0: all); lo a multiple of 64
bool launch_chain_bwd_fast(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype, const unsigned* flag,
                           const double* sgrad, const ts_grads& g, int accumulate, cudaStream_t st, long long lo = 0,
                           long long hi = -1);

// ts_sort.cu
struct SortScratch {
    unsigned* hist;     // RADIX * max_blocks
    unsigned* bsums;    // max_blocks + 1
    int max_blocks;
};
size_t sort_scratch_bytes(int max_blocks);
int sort_grid(long long count, int max_blocks);

// compaction of accepted triangles: keys_c[pos] = key[i], vals_c[pos] = i
void compact_accepted(long long n, const unsigned* flag, const unsigned long long* key,
                      unsigned long long* keys_c, unsigned* vals_c, const SortScratch& s,
                      cudaStream_t st);
// stable LSD radix sort of (key, value) pairs over bits [bit_lo, bit_hi).
// Returns 0 if the result is in (keys, vals), 1 if in (keys_alt, vals_alt).
int radix_sort_u64(long long count, unsigned long long* keys, unsigned* vals,
                   unsigned long long* keys_alt, unsigned* vals_alt, int bit_lo, int bit_hi,
                   const SortScratch& s, cudaStream_t st);
int radix_sort_u32(long long count, unsigned* keys, unsigned* vals, unsigned* keys_alt,
                   unsigned* vals_alt, int bit_lo, int bit_hi, const SortScratch& s,
                   cudaStream_t st);
// offs[m] = exclusive scan over m of tcount[sorted_src[m]]; rank_of[sorted_src[m]] = m
void rank_offsets(long long m, const unsigned* sorted_src, const unsigned* tcount, unsigned* offs,
                  int* rank_of, const SortScratch& s, cudaStream_t st);
// tile duplication in depth-rank order: tkey = tile id, tval = source id
void duplicate_entries(long long m, const unsigned* sorted_src, const short4* bbox, const unsigned* offs,
                       int ntx, unsigned* tkey, unsigned* tval, long long cap, unsigned* overflow,
                       cudaStream_t st);
// tile_start[t] = first entry of tile t (CSR), tile_start[ntiles] = E
void tile_ranges(long long e, const unsigned* tkey, int ntiles, int* tile_start, cudaStream_t st);
// same with the entry count read on the device (min(cap, *de))
void tile_ranges_dev(long long cap, const unsigned long long* de, const unsigned* tkey, int ntiles, int* tile_start,
                     cudaStream_t st);
// entry_rank[pos] = rank_of[ent_src[pos]]
void entries_to_rank(long long e, const unsigned* ent_src, const int* rank_of, int* out,
                     cudaStream_t st);
void bbox_dump(long long n, const short4* bbox, int* out, cudaStream_t st);

// build_tile_lists for any tile size: cnt (m int32) per-triangle tile counts and
// off (m+1 int64) their scan; then the CSR (start[ntiles+1], entry[e]) from
// bbox (m x 4 int64, rank order); kv = 4 u32 scratch arrays of e items
void tile_lists_count(long long m, const long long* bbox, int ts, int* cnt, long long* off, void* cs_scratch,
                      cudaStream_t st);
void tile_lists_fill(long long m, long long e, const long long* bbox, int ts, int ntx, int ntiles,
                     const long long* off, unsigned* const kv[4], const SortScratch& s, long long* start,
                     long long* entry, cudaStream_t st);
// onesweep radix sort (32-bit keys), scratch from onesweep_scratch_bytes
size_t onesweep_scratch_bytes(long long max_count, int max_passes);
int onesweep_sort_u32(long long count, unsigned* keys, unsigned* vals, unsigned* keys_alt,
                      unsigned* vals_alt, int nbits, void* scratch, cudaStream_t st);
// ts_optim.cu: fused Adam step (bad: device int64[4], first non-finite triangle per group)
void launch_adam_step(float* const params[4], const float* const grads[4], long long n, float* m, float* v,
                      long long* t, const double lrs[4], long long* bad, double* ibc, cudaStream_t st);

// ts_density.cu: adaptive density control (density.py:27-263)
void launch_stats_accum(long long n, const float* maxw, const int* pixcnt, const float* area, int min_pixels,
                        int first, double* acc_maxw, int* acc_views, double* acc_area, cudaStream_t st);
void launch_prune_mark(long long n, const double* acc_maxw, const int* acc_views, const void* opacity, int is_f64,
                       double tau_prune, int min_views, double opacity_dead, unsigned char* flags,
                       cudaStream_t st);
size_t sample_scratch_bytes(long long n);
void launch_sample_candidates(long long n, const long long* pool, const long long* kept, const void* param,
                              int is_f64, int inverse, const double* expo, long long count, long long* picked,
                              void* scratch, const SortScratch& ss, cudaStream_t st);
void launch_pick_info(long long count, const long long* picked, const long long* pool, const long long* kept,
                      const double* acc_area, long long n_views, const void* vertices, int is_f64, long long* src,
                      double* mean_area, unsigned char* degen, cudaStream_t st);
void launch_gather_rows(long long n_out, const long long* origin, const void* src, void* dst, int width,
                        int elem_bytes, cudaStream_t st);
void launch_child_vertices(long long n_child, const long long* parent, const int* code, const double* uni,
                           double max_noise_factor, const void* src, void* dst, int is_f64, cudaStream_t st);
// ts_sort.cu: in-order indices of the zero flags; *n_kept = their count (device)
void compact_unflagged(long long n, const unsigned char* flags, long long* kept, long long* n_kept,
                       const SortScratch& s, cudaStream_t st);

// ts_io.cu: binary PLY body pack / unpack (scene_io.py:382-455)
void launch_ply_pack(long long n, const void* vertices, const void* sh, int is_f64, unsigned char* vout,
                     void* fout, cudaStream_t st);
void launch_ply_unpack(long long n_face, long long n_vertex, const unsigned char* vin, const void* fin,
                       double sigma, int is_f64, void* vertices, void* opacity, void* sig, void* sh,
                       unsigned long long* bad, cudaStream_t st);

// ts_loss.cu: distortion loss over fragment CSR lists, fragment depth map
size_t distortion_scratch_bytes(long long npix);
void launch_distortion_loss(long long npix, const long long* off, const double* w, const double* z,
                            long long image_size, double* out, double* d_w, double* d_z, void* scratch,
                            cudaStream_t st);
// normal loss (cam: fx, fy, cx, cy, R[9] row-major, t[3])
size_t normal_scratch_bytes(long long n, long long npix);
void launch_normal_loss(const float* v, long long n, const long long* off, const int* ftri, const double* w,
                        long long nfrag, const double* depth, int H, int W, const double cam[16], double* out,
                        double* d_vertices, double* d_w, void* scratch, cudaStream_t st);
void launch_fragment_depth(long long npix, const long long* off, const double* w, const double* z, double* depth,
                           cudaStream_t st);
// ts_loss.cu: photometric loss (L1 + D-SSIM) and gradient
size_t photometric_scratch_bytes(int H, int W);
void launch_photometric_loss(const float* x, const float* y, int H, int W, double lam, double* out, float* d_image,
                             void* scratch, bool ssim_only, cudaStream_t st);

// ts_bin.cu: tile-first binning (chunk x tile counts, scan, fill; per-tile exact depth sort).
// bucket: one (32-bit range-reduced depth key, source) record per tile entry.
void bin_tiles_fill(long long n, const short4* bbox, const unsigned long long* key64, int ntx, int ntiles,
                    unsigned* tcnt, unsigned* mat, int* tile_start, uint2* bucket, const Counters* ctr,
                    long long cap, unsigned* overflow, int* big_list, cudaStream_t st, int* tile_order = nullptr);
size_t bin_matrix_bytes(long long n, int ntiles);
int bin_max_tiles();
void bin_tiles_sort(long long n, int ntiles, const int* tile_start, const uint2* bucket,
                    const unsigned long long* key64, unsigned* ent_src, unsigned* const scratch[4],
                    const int* big_list, cudaStream_t st, const int* tile_order = nullptr);
// count = min(cap, *dcount), read on the device
int onesweep_sort_u32_dev(long long cap, const unsigned long long* dcount, unsigned* keys, unsigned* vals,
                          unsigned* keys_alt, unsigned* vals_alt, int nbits, void* scratch, cudaStream_t st);
// depth keys of all n triangles (culled -> 2^kbits_cap - 1), reduction from the counters
void depth_keys(long long n, const unsigned* flag, const unsigned long long* key, const Counters* ctr, int kbits_cap,
                unsigned* k32, unsigned* vals, cudaStream_t st);
void compact_accepted32(long long n, const unsigned* flag, const unsigned long long* key,
                        unsigned long long kmin, int shift, unsigned* keys_c, unsigned* vals_c,
                        const SortScratch& s, cudaStream_t st);
void fix_depth_runs(long long m, const unsigned* k32, unsigned* vals, const unsigned long long* key64,
                    cudaStream_t st, unsigned skip_key = 0xffffffffu);

// CSR offsets (n+1, int64) from int32 counts; scratch from count_scan_scratch_bytes
size_t count_scan_scratch_bytes(long long n);
void count_scan_i64(long long n, const int* cnt, long long* off, void* scratch, cudaStream_t st);
// *bad += number of i in [0, n] with a[i] != b[i]
void offsets_mismatch(long long n, const long long* a, const long long* b, unsigned long long* bad, cudaStream_t st);

}  // namespace ts
