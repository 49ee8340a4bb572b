// ts_api.cu -- C ABI (include/trisplat_b200.h): context, scratch management
// and the per-view pipeline.
//
//   ts_forward  = render()          render.py:364-432
//   ts_backward = render_backward() backward.py:93-211
//
// Pipeline per view (one stream):
//   preprocess (project, cull, edges, bbox, colour, depth key)       1 kernel
//   -- one host sync: M, E, depth-key range, non-finite indices --
//   compaction of accepted triangles (range-reduced 32-bit depth key) 3 kernels
//   onesweep radix sort on depth (+ exact tie-run fix)               <= 6 kernels
//   rank offsets, tile duplication in depth-rank order               4 kernels
//   onesweep radix sort on tile id (stable)                          <= 3 kernels
//   tile ranges                                                      1 kernel
//   blend (fast: fp32 + guard band, then exact fix-up; or exact fp64) 1-2 kernels
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ts_kernels.cuh"

namespace ts {
std::atomic<long long> g_launches{0};
}

using namespace ts;

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

struct ts_context {
    int device = 0;
    // per-triangle scratch (capacity in triangles)
    long long cap_n = -1;
    void* tri_buf = nullptr;
    size_t tri_bytes = 0, ent_bytes = 0, pix_bytes = 0, os_bytes = 0;  // (ts_workspace_bytes)
    unsigned long long* key = nullptr;
    unsigned* tcount = nullptr;
    unsigned* flag = nullptr;
    unsigned long long* keys_c = nullptr;  // also used as 2 x u32 key arrays
    unsigned* vals_c = nullptr;
    unsigned long long* keys_alt = nullptr;
    unsigned* vals_alt = nullptr;
    unsigned* offs = nullptr;
    int* rank_of = nullptr;
    double* depth = nullptr;
    short4* bbox = nullptr;
    DevBuf rec64, recf, recb, recc, sg64, sg32;
    DevBuf frag_off, cs_scratch;  // expected fragment CSR offsets + scan scratch
    DevBuf tl_cnt, tl_off, tl_cs, tl_kv;  // ts_tile_lists scratch
    DevBuf adam_ibc;                      // Adam bias corrections of the current step
    DevBuf fsw;                           // per fragment: suffix of dw * w (fragment-gradient backward)
    // deferred chain (ts_backward_screen / ts_chain_views): per pending view its
    // screen-space gradients, cull flags and camera
    DevBuf slot_sg[TS_MAX_CHAIN_VIEWS], slot_flag[TS_MAX_CHAIN_VIEWS];
    Cam slot_cam[TS_MAX_CHAIN_VIEWS];
    int n_slots = 0;
    ts_soup slot_soup{};
    Opts slot_opt{};
    DevBuf frec, ctot;            // training forward: fragment records + final unclipped colour
    unsigned long long frec_cap = 0;
    long long frec_hint = 0;      // largest fragment-record count seen (record-buffer sizing)
    bool frec_ready = false;      // the last forward wrote fragment records
    // ts_set_option: cross-check paths for tests (defaults are the product path)
    bool opt_legacy_binning = false;  // global depth sort + tile duplication instead of tile-first binning
    bool opt_tile_backward = false;   // tile backward instead of the streaming backward
    // per-entry scratch
    long long cap_e = -1;
    void* ent_buf = nullptr;
    unsigned *tkey = nullptr, *tval = nullptr, *tkey_alt = nullptr, *tval_alt = nullptr;
    unsigned *tscr0 = nullptr, *tscr1 = nullptr;  // tile-sort scratch (tiles longer than shared memory)
    unsigned* tcnt = nullptr;                      // per-tile entry counts
    int* big_list = nullptr;                       // tiles for the long-tile sort, count at [ntiles]
    int* tile_order = nullptr;                     // blend order of the tiles (longest first)
    uint2* bucket = nullptr;                       // (reduced depth key, source) of every tile entry, unsorted
    DevBuf binmat;                                 // chunk x tile count matrix of the binning
    DevBuf lossbuf;                                // photometric loss scratch
    DevBuf densbuf;                                // density control: sampling keys / sort scratch
    bool sorted_valid = false;                     // sorted_src holds the global depth order
    // per-pixel scratch
    long long cap_p = -1, cap_tiles = -1;
    void* pix_buf = nullptr;
    double* t_final = nullptr;
    float* t_final32 = nullptr;
    int* last_pos = nullptr;
    int* nfrag = nullptr;       // composited fragments per pixel of the last forward
    int2* flags = nullptr;
    int* tile_start = nullptr;
    // sort scratch
    void* sort_buf = nullptr;
    SortScratch sort{};
    void* os_buf = nullptr;
    long long os_cap = -1;
    // counters
    Counters* d_ctr = nullptr;
    Counters* h_ctr = nullptr;   // readback of the last frame's counters
    Counters* h_init = nullptr;  // initial counters (never a copy destination: async frames overlap)
    unsigned* d_sticky = nullptr;  // entry-capacity overflow since the last ts_forward_status (device view)
    unsigned* h_sticky = nullptr;  // the same word, page-locked and mapped: an asynchronous forward sees
                                   // an earlier frame's overflow without a host synchronisation
    // last forward
    bool have_fwd = false;
    bool have_bwd_state = false;
    int precision = 0;
    Cam cam{};
    Opts opt{};
    ts_soup soup{};
    int dtype = 0;
    long long n = 0, m = 0, e = 0;
    long long e_hint = 0;  // largest entry count seen (entry-buffer sizing)
    long long wcap = 0;    // working entry capacity of the last forward
    const unsigned* sorted_src = nullptr;
    const unsigned* ent_src = nullptr;
    int sgrad_kind = 0;  // 0 none, 1 fp64, 2 fp32
    // asynchronous forwards (ts_set_async): no host synchronization per frame
    bool async_mode = false;
    bool pending = false;
    bool last_validate = true;
    // stage profiling
    bool profile = false;
    cudaEvent_t ev[TS_NUM_STAGES][2] = {};
    bool ev_used[TS_NUM_STAGES] = {};
};

static int cuda_err(cudaError_t e) {
    if (e != cudaSuccess) {
        fprintf(stderr, "[trisplat_b200] CUDA error: %s\n", cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? TS_ERR_OOM : TS_ERR_CUDA;
    }
    return TS_OK;
}
#define TS_CHECK(x)                   \
    do {                              \
        int _rc = cuda_err((x));      \
        if (_rc != TS_OK) return _rc; \
    } while (0)

// Every entry point runs on the context's device and restores the caller's
// current device afterwards (torch keeps its own notion of the current device).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(const ts_context* c) {
        if (!c) return;
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != c->device && cudaSetDevice(c->device) == cudaSuccess) prev = cur;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static void stage_begin(ts_context* c, int s, cudaStream_t st) {
    if (c->profile) {
        cudaEventRecord(c->ev[s][0], st);
        c->ev_used[s] = true;
    }
}
static void stage_end(ts_context* c, int s, cudaStream_t st) {
    if (c->profile) cudaEventRecord(c->ev[s][1], st);
}

static int ensure(DevBuf& b, size_t bytes) {
    if (bytes <= b.bytes) return TS_OK;
    size_t cap = bytes + bytes / 4 + 4096;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    TS_CHECK(cudaMalloc(&b.p, cap));
    b.bytes = cap;
    return TS_OK;
}

static int ensure_tri(ts_context* c, long long n) {
    if (n <= c->cap_n) return TS_OK;
    long long cap = n + n / 4 + 1024;
    if (c->tri_buf) cudaFree(c->tri_buf);
    c->tri_buf = nullptr;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    size_t o_key = take(8 * cap), o_tc = take(4 * cap), o_fl = take(4 * cap), o_kc = take(8 * cap),
           o_vc = take(4 * cap), o_ka = take(8 * cap), o_va = take(4 * cap), o_of = take(4 * (cap + 1)),
           o_rk = take(4 * cap), o_dp = take(8 * cap), o_bb = take(8 * cap);
    TS_CHECK(cudaMalloc(&c->tri_buf, off));
    c->tri_bytes = off;
    char* b = (char*)c->tri_buf;
    c->key = (unsigned long long*)(b + o_key);
    c->tcount = (unsigned*)(b + o_tc);
    c->flag = (unsigned*)(b + o_fl);
    c->keys_c = (unsigned long long*)(b + o_kc);
    c->vals_c = (unsigned*)(b + o_vc);
    c->keys_alt = (unsigned long long*)(b + o_ka);
    c->vals_alt = (unsigned*)(b + o_va);
    c->offs = (unsigned*)(b + o_of);
    c->rank_of = (int*)(b + o_rk);
    c->depth = (double*)(b + o_dp);
    c->bbox = (short4*)(b + o_bb);
    c->cap_n = cap;
    return TS_OK;
}

static int ensure_ent(ts_context* c, long long e) {
    if (e <= c->cap_e) return TS_OK;
    long long cap = e + e / 4 + 4096;
    if (c->ent_buf) cudaFree(c->ent_buf);
    c->ent_buf = nullptr;
    size_t one = align_up(4 * cap, 256);
    TS_CHECK(cudaMalloc(&c->ent_buf, 8 * one));
    c->ent_bytes = 8 * one;
    char* b = (char*)c->ent_buf;
    c->tkey = (unsigned*)b;
    c->tval = (unsigned*)(b + one);
    c->tkey_alt = (unsigned*)(b + 2 * one);
    c->tval_alt = (unsigned*)(b + 3 * one);
    c->tscr0 = (unsigned*)(b + 4 * one);
    c->tscr1 = (unsigned*)(b + 5 * one);
    c->bucket = (uint2*)(b + 6 * one);
    c->cap_e = cap;
    return TS_OK;
}

static int ensure_pix(ts_context* c, long long p, long long ntiles) {
    if (p <= c->cap_p && ntiles <= c->cap_tiles) return TS_OK;
    if (c->pix_buf) cudaFree(c->pix_buf);
    c->pix_buf = nullptr;
    long long cp = p > c->cap_p ? p : c->cap_p;
    long long ct = ntiles > c->cap_tiles ? ntiles : c->cap_tiles;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    size_t o_tf = take(8 * cp), o_t32 = take(4 * cp), o_lp = take(4 * cp), o_fg = take(8 * cp),
           o_ts = take(4 * (ct + 1)), o_nf = take(4 * cp), o_tc = take(4 * (ct + 1)), o_bl = take(4 * (ct + 1)),
           o_or = take(4 * (ct + 1));
    TS_CHECK(cudaMalloc(&c->pix_buf, off));
    c->pix_bytes = off;
    char* b = (char*)c->pix_buf;
    c->t_final = (double*)(b + o_tf);
    c->t_final32 = (float*)(b + o_t32);
    c->last_pos = (int*)(b + o_lp);
    c->flags = (int2*)(b + o_fg);
    c->tile_start = (int*)(b + o_ts);
    c->nfrag = (int*)(b + o_nf);
    c->tcnt = (unsigned*)(b + o_tc);
    c->big_list = (int*)(b + o_bl);
    c->tile_order = (int*)(b + o_or);
    // flagged-pixel list entries start empty (pixel -1); the fix-up empties each
    // entry it consumes, so the list is clean for the next frame
    TS_CHECK(cudaMemset(c->flags, 0xff, 8 * (size_t)cp));
    TS_CHECK(cudaDeviceSynchronize());
    c->cap_p = cp;
    c->cap_tiles = ct;
    return TS_OK;
}

static int ensure_os(ts_context* c, long long count) {
    if (count <= c->os_cap) return TS_OK;
    long long cap = count + count / 4 + 4096;
    if (c->os_buf) cudaFree(c->os_buf);
    c->os_buf = nullptr;
    TS_CHECK(cudaMalloc(&c->os_buf, onesweep_scratch_bytes(cap, 4)));
    c->os_bytes = onesweep_scratch_bytes(cap, 4);
    c->os_cap = cap;
    return TS_OK;
}

static void build_cam_opts(const ts_camera* cam, const ts_options* opt, Cam& c, Opts& o) {
    c.fx = cam->fx;
    c.fy = cam->fy;
    c.cx = cam->cx;
    c.cy = cam->cy;
    c.z_near = cam->z_near;
    for (int k = 0; k < 9; k++) c.R[k] = cam->R[k];
    for (int k = 0; k < 3; k++) c.t[k] = cam->t[k];
    for (int b = 0; b < 3; b++)
        c.cc[b] = -(cam->R[0 * 3 + b] * cam->t[0] + cam->R[1 * 3 + b] * cam->t[1] + cam->R[2 * 3 + b] * cam->t[2]);
    c.width = cam->width;
    c.height = cam->height;
    c.ntx = (cam->width + TILE - 1) / TILE;
    c.nty = (cam->height + TILE - 1) / TILE;
    o.mode = opt->mode;
    o.sh_degree = opt->sh_degree;
    o.ncoef = (opt->sh_degree + 1) * (opt->sh_degree + 1);
    o.solid = opt->solid;
    o.validate = opt->validate;
    o.tau_cutoff = opt->tau_cutoff;
    o.tau_contrib = opt->tau_contrib;
    for (int k = 0; k < 3; k++) o.bg[k] = opt->background[k];
}

static int bit_length(unsigned long long x) { return x ? 64 - __builtin_clzll(x) : 0; }

extern "C" {

const char* ts_version(void) { return "trisplat_b200 0.2.0 (sm_100a)"; }

const char* ts_error_string(int code) {
    switch (code) {
        case TS_OK: return "ok";
        case TS_ERR_INVALID_ARG: return "invalid argument";
        case TS_ERR_CUDA: return "CUDA error";
        case TS_ERR_OOM: return "out of device memory";
        case TS_ERR_NO_FORWARD: return "ts_backward called without a preceding ts_forward";
        case TS_ERR_NONFINITE: return "non-finite triangle parameters";
        case TS_ERR_TILE_SIZE: return "only tile_size=16 is supported";
        case TS_ERR_FRAGMENTS: return "fragment gradients do not match this scene/camera";
        case TS_ERR_NO_BWD_STATE: return "the preceding ts_forward ran with keep_backward=0";
        case TS_ERR_CAPACITY: return "tile-entry capacity exceeded by an asynchronous forward (repeat the frame)";
        default: return "unknown error";
    }
}

int ts_context_create(ts_context** out, int device) {
    if (!out) return TS_ERR_INVALID_ARG;
    int prev_device = -1;
    cudaGetDevice(&prev_device);
    TS_CHECK(cudaSetDevice(device));
    struct Restore {
        int d;
        ~Restore() {
            if (d >= 0) cudaSetDevice(d);
        }
    } restore{prev_device};
    ts_context* c = new ts_context();
    c->device = device;
    c->sort.max_blocks = 1184;  // 8 x 148 SMs
    size_t sb = sort_scratch_bytes(c->sort.max_blocks);
    int rc = cuda_err(cudaMalloc(&c->sort_buf, sb + 1024));
    if (rc) {
        delete c;
        return rc;
    }
    c->sort.hist = (unsigned*)c->sort_buf;
    c->sort.bsums = c->sort.hist + 256 * (size_t)c->sort.max_blocks + 32;
    rc = cuda_err(cudaMalloc(&c->d_ctr, sizeof(Counters)));
    if (!rc) rc = cuda_err(cudaMallocHost(&c->h_ctr, sizeof(Counters)));
    if (!rc) rc = cuda_err(cudaMallocHost(&c->h_init, sizeof(Counters)));
    if (!rc) {
        memset(c->h_init, 0, sizeof(Counters));
        c->h_init->key_and = ~0ull;
        c->h_init->key_min = ~0ull;
        for (int k = 0; k < 4; k++) c->h_init->err[k] = 0x7fffffffffffffffLL;
    }
    if (!rc) rc = cuda_err(cudaHostAlloc((void**)&c->h_sticky, sizeof(unsigned), cudaHostAllocMapped));
    if (!rc) {
        *(volatile unsigned*)c->h_sticky = 0u;
        rc = cuda_err(cudaHostGetDevicePointer((void**)&c->d_sticky, c->h_sticky, 0));
    }
    if (rc) {
        delete c;
        return rc;
    }
    *out = c;
    return TS_OK;
}

int ts_context_destroy(ts_context* c) {
    DeviceGuard device_guard(c);
    if (!c) return TS_OK;
    cudaFree(c->tri_buf);
    cudaFree(c->ent_buf);
    cudaFree(c->pix_buf);
    for (DevBuf* b : {&c->fsw, &c->adam_ibc, &c->tl_cnt, &c->tl_off, &c->tl_cs, &c->tl_kv, &c->rec64, &c->recf, &c->recb, &c->recc, &c->sg64, &c->sg32, &c->frag_off, &c->cs_scratch, &c->frec,
                      &c->ctot, &c->binmat, &c->lossbuf, &c->densbuf})
        cudaFree(b->p);
    for (int k = 0; k < TS_MAX_CHAIN_VIEWS; k++) {
        cudaFree(c->slot_sg[k].p);
        cudaFree(c->slot_flag[k].p);
    }
    cudaFree(c->sort_buf);
    cudaFree(c->os_buf);
    cudaFree(c->d_ctr);
    cudaFreeHost(c->h_sticky);
    cudaFreeHost(c->h_ctr);
    cudaFreeHost(c->h_init);
    for (int k = 0; k < TS_NUM_STAGES; k++)
        if (c->ev[k][0]) {
            cudaEventDestroy(c->ev[k][0]);
            cudaEventDestroy(c->ev[k][1]);
        }
    delete c;
    return TS_OK;
}

int64_t ts_launch_count(ts_context*) { return g_launches.load(); }

int ts_profile(ts_context* c, int enable) {
    DeviceGuard device_guard(c);
    if (!c) return TS_ERR_INVALID_ARG;
    if (enable && !c->ev[0][0])
        for (int k = 0; k < TS_NUM_STAGES; k++) {
            TS_CHECK(cudaEventCreate(&c->ev[k][0]));
            TS_CHECK(cudaEventCreate(&c->ev[k][1]));
        }
    c->profile = enable != 0;
    return TS_OK;
}

int ts_stage_times(ts_context* c, float* ms, int n) {
    DeviceGuard device_guard(c);
    if (!c || !ms) return TS_ERR_INVALID_ARG;
    for (int k = 0; k < n && k < TS_NUM_STAGES; k++) {
        ms[k] = 0.f;
        if (c->profile && c->ev_used[k]) {
            TS_CHECK(cudaEventSynchronize(c->ev[k][1]));
            TS_CHECK(cudaEventElapsedTime(&ms[k], c->ev[k][0], c->ev[k][1]));
        }
    }
    return TS_OK;
}

// Global depth order of the current forward (np.lexsort((idx, z)),
// render.py:276) into sorted_src: 24-bit range-reduced keys while ties stay
// rare (n < 2^22), else 32-bit; exact (z64, idx) order restored inside runs of
// equal reduced keys.  Used by the legacy binning and the debug dumps.
static void global_depth_order(ts_context* c, long long n, cudaStream_t st) {
    const int kcap = n < (1ll << 22) ? 24 : 31;
    unsigned* k32 = (unsigned*)c->keys_c;
    unsigned* k32_alt = (unsigned*)c->keys_alt;
    depth_keys(n, c->flag, c->key, c->d_ctr, kcap, k32, c->vals_c, st);
    int par = onesweep_sort_u32(n, k32, c->vals_c, k32_alt, c->vals_alt, kcap, c->os_buf, st);
    c->sorted_src = par ? c->vals_alt : c->vals_c;
    fix_depth_runs(n, par ? k32_alt : k32, (unsigned*)c->sorted_src, c->key, st, (1u << kcap) - 1u);
    g_launches += 2 + 3 * ((kcap + 7) / 8);
    c->sorted_valid = true;
}

// Binning + blend of the current forward, sized from host capacities and the
// device counters of the preprocess (no host round trip).  Default: tile-first
// binning (ts_bin.cu) -- per-tile counts, scan, bucket fill, then every tile's
// list sorted by exact (z, idx) in shared memory.  TS_OPT_LEGACY_BINNING: global depth
// sort, rank offsets, tile duplication, stable radix sort by tile, ranges.
static int enqueue_tail(ts_context* c, const Cam& cm, const Opts& op, const ts_options* opt, const ts_soup* soup,
                        const ts_forward_out* out, cudaStream_t st) {
    const bool fast = opt->precision == 0;
    const long long n = soup->n;
    const int ntiles = cm.ntx * cm.nty;
    c->sorted_valid = false;
    // working capacity: the largest entry count seen so far with headroom
    // (the sort grids follow it); more entries raise the sticky overflow flag
    const long long wcap = c->e_hint > 0 ? std::min<long long>(c->cap_e, c->e_hint + c->e_hint / 4 + 4096)
                                         : c->cap_e;
    const int* order = nullptr;  // blend order of the tiles (tile-first binning only)
    if (n > 0 && !c->opt_legacy_binning && ntiles <= bin_max_tiles()) {
        stage_begin(c, TS_STAGE_BINNING, st);
        bin_tiles_fill(n, c->bbox, c->key, cm.ntx, ntiles, c->tcnt, (unsigned*)c->binmat.p, c->tile_start,
                       c->bucket, c->d_ctr, wcap, c->d_sticky, c->big_list, st, c->tile_order);
        order = c->tile_order;
        stage_end(c, TS_STAGE_BINNING, st);
        stage_begin(c, TS_STAGE_DEPTH_SORT, st);
        unsigned* const scr[4] = {c->tkey_alt, c->tval_alt, c->tscr0, c->tscr1};
        bin_tiles_sort(n, ntiles, c->tile_start, c->bucket, c->key, c->tval, scr, c->big_list, st, c->tile_order);
        stage_end(c, TS_STAGE_DEPTH_SORT, st);
        c->ent_src = c->tval;
        c->sorted_src = c->vals_c;
        c->wcap = wcap;
        g_launches += 6;
    } else if (n > 0) {
        stage_begin(c, TS_STAGE_DEPTH_SORT, st);
        global_depth_order(c, n, st);
        stage_end(c, TS_STAGE_DEPTH_SORT, st);

        // tile duplication in rank order + stable sort by tile id (render.py:315-361)
        stage_begin(c, TS_STAGE_BINNING, st);
        rank_offsets(n, c->sorted_src, c->tcount, c->offs, nullptr, c->sort, st);
        duplicate_entries(n, c->sorted_src, c->bbox, c->offs, cm.ntx, c->tkey, c->tval, wcap, c->d_sticky, st);
        const int tbits = bit_length((unsigned long long)(ntiles > 1 ? ntiles - 1 : 0));
        int par = onesweep_sort_u32_dev(wcap, &c->d_ctr->e, c->tkey, c->tval, c->tkey_alt, c->tval_alt, tbits,
                                        c->os_buf, st);
        const unsigned* skey = par ? c->tkey_alt : c->tkey;
        c->ent_src = par ? c->tval_alt : c->tval;
        tile_ranges_dev(wcap, &c->d_ctr->e, skey, ntiles, c->tile_start, st);
        c->wcap = wcap;
        g_launches += 5 + 3 * ((tbits + 7) / 8);
        stage_end(c, TS_STAGE_BINNING, st);
    } else {
        c->sorted_src = c->vals_c;
        c->sorted_valid = true;
        c->ent_src = c->tval;
        TS_CHECK(cudaMemsetAsync(c->tile_start, 0, sizeof(int) * (ntiles + 1), st));
    }

    if (fast) {
        FastBlendOut bo{out->image, out->alpha_map, out->max_weight, out->pixel_count, out->last_src,
                        c->nfrag, c->t_final32, opt->keep_backward ? c->t_final : nullptr, c->last_pos,
                        c->flags, c->d_ctr};
        bo.tile_order = order;
        if (opt->keep_backward) {
            bo.recc = (const RecC*)c->recc.p;
            if (!c->opt_tile_backward && c->frec.p) {
                bo.frec = (FragRec*)c->frec.p;
                bo.frec_cap = c->frec_cap;
                bo.c_total64 = (double*)c->ctot.p;
            }
        }
        stage_begin(c, TS_STAGE_BLEND, st);
        launch_blend_dense(cm, op, opt->keep_backward != 0, (const RecF*)c->recf.p, c->tile_start, c->ent_src, bo, st);
        stage_end(c, TS_STAGE_BLEND, st);
        stage_begin(c, TS_STAGE_FIXUP, st);
        launch_fixup_fwd(cm, op, *soup, opt->param_dtype, (const RecF*)c->recf.p, c->tile_start, c->ent_src,
                         bo, st);
        stage_end(c, TS_STAGE_FIXUP, st);
        g_launches += 2;
    } else {
        BlendOut bo{out->image, out->alpha_map, out->max_weight, out->pixel_count, out->last_src,
                    c->nfrag, c->t_final, c->last_pos};
        stage_begin(c, TS_STAGE_BLEND, st);
        launch_blend_exact(cm, op, (const Rec64*)c->rec64.p, c->tile_start, (const int*)c->ent_src, bo, st);
        stage_end(c, TS_STAGE_BLEND, st);
        g_launches += 1;
    }
    const long long P = (long long)cm.width * cm.height;
    if (out->n_frag && P) TS_CHECK(cudaMemcpyAsync(out->n_frag, c->nfrag, 4 * P, cudaMemcpyDeviceToDevice, st));
    return cuda_err(cudaGetLastError());
}

// Host view of the counters of the last forward (after the stream has run it):
// result fields, non-finite report, entry-capacity check.
static int finish_forward(ts_context* c, ts_forward_result* res, bool validate) {
    const Counters& h = *c->h_ctr;
    c->m = (long long)h.m;
    c->e = (long long)h.e;
    c->e_hint = std::max(c->e_hint, c->e);
    if (res) {
        res->n_visible = (int64_t)h.m;
        res->n_entries = (int64_t)h.e;
        res->n_flagged = (int64_t)h.n_flagged;
        for (int k = 0; k < 4; k++) res->err_index[k] = h.err[k] == 0x7fffffffffffffffLL ? -1 : h.err[k];
    }
    if (validate)
        for (int k = 0; k < 4; k++)
            if (h.err[k] != 0x7fffffffffffffffLL) return TS_ERR_NONFINITE;
    if (c->e >= (1ll << 31)) return TS_ERR_INVALID_ARG;
    return TS_OK;
}

int ts_forward(ts_context* c, const ts_camera* cam, const ts_options* opt, const ts_soup* soup,
               const ts_forward_out* out, ts_forward_result* res, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !cam || !opt || !soup || !out) return TS_ERR_INVALID_ARG;
    if (opt->tile_size != TILE) return TS_ERR_TILE_SIZE;
    if (cam->width < 1 || cam->height < 1 || soup->n < 0 || opt->sh_degree < 0 || opt->sh_degree > 3)
        return TS_ERR_INVALID_ARG;
    if (soup->n >= (1ll << 31) || cam->width > 32000 || cam->height > 32000) return TS_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (c->async_mode && *(volatile unsigned*)c->h_sticky) {
        // an earlier asynchronous frame outgrew the tile-entry capacity (its tile lists
        // were emptied): report it here, before more frames are enqueued, whether or
        // not the caller polls ts_forward_status (which grows the capacity and clears it)
        return TS_ERR_CAPACITY;
    }
    c->have_fwd = false;
    c->have_bwd_state = false;
    for (int k = 0; k < TS_NUM_STAGES; k++) c->ev_used[k] = false;
    Cam cm;
    Opts op;
    build_cam_opts(cam, opt, cm, op);
    const bool fast = opt->precision == 0;
    const long long n = soup->n;
    const long long P = (long long)cam->width * cam->height;
    const int ntiles = cm.ntx * cm.nty;
    const long long n1 = n > 0 ? n : 1;
    int rc = ensure_tri(c, n1);
    if (rc) return rc;
    if ((rc = ensure_pix(c, P, ntiles))) return rc;
    if (fast) {
        if ((rc = ensure(c->recf, sizeof(RecF) * n1))) return rc;
        if (opt->keep_backward && (rc = ensure(c->recb, sizeof(RecB) * n1))) return rc;
        if (opt->keep_backward && (rc = ensure(c->recc, sizeof(RecC) * n1))) return rc;
    } else {
        if ((rc = ensure(c->rec64, sizeof(Rec64) * n1))) return rc;
    }
    // tile-entry capacity: the last frame's count with headroom, at least 4 per triangle
    if ((rc = ensure_ent(c, std::max<long long>(4 * n1 + 4096, c->e_hint + c->e_hint / 2)))) return rc;
    if ((rc = ensure_os(c, std::max<long long>(n1, c->cap_e) + 1))) return rc;
    if ((rc = ensure(c->binmat, bin_matrix_bytes(n1, cm.ntx * cm.nty)))) return rc;
    c->frec_ready = false;
    if (fast && opt->keep_backward) {
        // fragment records of the training forward (~6.5 per tile entry here; the
        // largest count seen with headroom once one frame has run)
        const long long want = c->frec_hint > 0 ? c->frec_hint + c->frec_hint / 4 + 4096
                                                : std::max<long long>(8 * std::max<long long>(c->e_hint, n1), 1ll << 20);
        if ((rc = ensure(c->frec, sizeof(FragRec) * (size_t)want))) return rc;
        c->frec_cap = c->frec.bytes / sizeof(FragRec);
        if ((rc = ensure(c->ctot, sizeof(double) * 3 * (size_t)P))) return rc;
    }
    TS_CHECK(cudaMemcpyAsync(c->d_ctr, c->h_init, sizeof(Counters), cudaMemcpyHostToDevice, st));
    if (!fast) {  // (the fast preprocess zeroes them per triangle)
        if (out->max_weight && n) TS_CHECK(cudaMemsetAsync(out->max_weight, 0, sizeof(float) * n, st));
        if (out->pixel_count && n) TS_CHECK(cudaMemsetAsync(out->pixel_count, 0, sizeof(int) * n, st));
    }
    stage_begin(c, TS_STAGE_PREPROCESS, st);
    if (fast) {
        FastPreOut po{(RecF*)c->recf.p, opt->keep_backward ? (RecB*)c->recb.p : nullptr,
                      opt->keep_backward ? (RecC*)c->recc.p : nullptr, c->bbox, c->key,
                      c->tcount, c->flag, out->area, nullptr, c->d_ctr, out->max_weight, out->pixel_count};
        launch_preprocess_fast(cm, op, *soup, opt->param_dtype, po, st);
    } else {
        PreOut po{(Rec64*)c->rec64.p, c->bbox, c->key, c->tcount, c->flag, out->area, nullptr, c->d_ctr};
        launch_preprocess(cm, op, *soup, opt->param_dtype, po, st);
    }
    stage_end(c, TS_STAGE_PREPROCESS, st);
    g_launches += n > 0 ? 1 : 0;
    if ((rc = enqueue_tail(c, cm, op, opt, soup, out, st))) return rc;
    // (asynchronous forwards read the counters back in ts_forward_status only)
    if (!c->async_mode)
        TS_CHECK(cudaMemcpyAsync(c->h_ctr, c->d_ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    c->have_fwd = true;
    c->have_bwd_state = !fast || opt->keep_backward;
    c->frec_ready = fast && opt->keep_backward && !c->opt_tile_backward;
    c->precision = opt->precision;
    c->cam = cm;
    c->opt = op;
    c->soup = *soup;
    c->dtype = opt->param_dtype;
    c->n = n;
    c->last_validate = opt->validate != 0;
    if (c->async_mode) {
        // the caller checks the frame later with ts_forward_status()
        c->pending = true;
        if (res) memset(res, 0xff, sizeof(*res));
        return TS_OK;
    }
    TS_CHECK(cudaStreamSynchronize(st));
    if (c->frec_ready) c->frec_hint = std::max<long long>(c->frec_hint, (long long)c->h_ctr->n_frec);
    const bool e_over = c->h_ctr->e > (unsigned long long)c->wcap;
    const bool f_over = c->frec_ready && c->h_ctr->frec_over;
    if (e_over || f_over) {
        TS_CHECK(cudaMemsetAsync(c->d_sticky, 0, sizeof(unsigned), st));
        // more tile entries than the capacity, or more fragment records than the
        // record buffer (first training frame of a scene): grow and redo binning + blend
        const long long e = (long long)c->h_ctr->e;
        c->e_hint = std::max(c->e_hint, e);
        if ((rc = ensure_ent(c, e + e / 4 + 4096))) return rc;
        if ((rc = ensure_os(c, std::max<long long>(n1, c->cap_e) + 1))) return rc;
        if (f_over) {
            const long long f = c->frec_hint;
            if ((rc = ensure(c->frec, sizeof(FragRec) * (size_t)(f + f / 4 + 4096)))) return rc;
            c->frec_cap = c->frec.bytes / sizeof(FragRec);
        }
        // n_flagged, n_frec, frec_over, blend_done
        static_assert(offsetof(Counters, blend_done) == offsetof(Counters, n_flagged) + 24, "counter order");
        TS_CHECK(cudaMemsetAsync(&c->d_ctr->n_flagged, 0, 4 * sizeof(unsigned long long), st));
        if (out->max_weight && n) TS_CHECK(cudaMemsetAsync(out->max_weight, 0, sizeof(float) * n, st));
        if (out->pixel_count && n) TS_CHECK(cudaMemsetAsync(out->pixel_count, 0, sizeof(int) * n, st));
        if ((rc = enqueue_tail(c, cm, op, opt, soup, out, st))) return rc;
        TS_CHECK(cudaMemcpyAsync(c->h_ctr, c->d_ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
        TS_CHECK(cudaStreamSynchronize(st));
    }
    rc = finish_forward(c, res, opt->validate != 0);
    if (rc) {  // a failed frame leaves no state a backward could read
        c->have_fwd = false;
        c->have_bwd_state = false;
        c->frec_ready = false;
    }
    return rc;
}

int ts_set_async(ts_context* c, int enable) {
    DeviceGuard device_guard(c);
    if (!c) return TS_ERR_INVALID_ARG;
    c->async_mode = enable != 0;
    return TS_OK;
}

int ts_forward_status(ts_context* c, ts_forward_result* res, void* stream) {
    DeviceGuard device_guard(c);
    if (!c) return TS_ERR_INVALID_ARG;
    if (!c->have_fwd) return TS_ERR_NO_FORWARD;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned sticky = 0;
    TS_CHECK(cudaMemcpyAsync(c->h_ctr, c->d_ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    TS_CHECK(cudaMemcpyAsync(&sticky, c->d_sticky, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    TS_CHECK(cudaStreamSynchronize(st));
    c->pending = false;
    if (c->frec_ready) c->frec_hint = std::max<long long>(c->frec_hint, (long long)c->h_ctr->n_frec);
    if (sticky) {
        TS_CHECK(cudaMemsetAsync(c->d_sticky, 0, sizeof(unsigned), st));
        finish_forward(c, res, false);
        // the next forward sizes its entry buffer from the largest count seen
        c->e_hint = std::max<long long>(c->e_hint, c->e) * 2;
        c->have_bwd_state = false;
        c->frec_ready = false;
        return TS_ERR_CAPACITY;
    }
    const int rc = finish_forward(c, res, c->last_validate);
    if (rc) {
        c->have_bwd_state = false;
        c->frec_ready = false;
    }
    return rc;
}

int ts_set_option(ts_context* c, int option, int64_t value) {
    DeviceGuard device_guard(c);
    if (!c) return TS_ERR_INVALID_ARG;
    switch (option) {
        case TS_OPT_LEGACY_BINNING: c->opt_legacy_binning = value != 0; return TS_OK;
        case TS_OPT_TILE_BACKWARD: c->opt_tile_backward = value != 0; return TS_OK;
        default: return TS_ERR_INVALID_ARG;
    }
}

static int backward_impl(ts_context* c, const float* d_image, const ts_grads* grads, int accumulate,
                         const long long* frag_off, const double* fg_dw, const double* fg_dz, void* stream,
                         int n_chunks = 0, const int64_t* bounds = nullptr, void* const* events = nullptr,
                         const double* frag_w = nullptr, long long n_frag_total = 0);

int ts_backward(ts_context* c, const float* d_image, const ts_grads* grads, int accumulate,
                void* stream) {
    DeviceGuard device_guard(c);
    return backward_impl(c, d_image, grads, accumulate, nullptr, nullptr, nullptr, stream);
}

int ts_backward_chunked(ts_context* c, const float* d_image, const ts_grads* grads, int accumulate, int n_chunks,
                        const int64_t* bounds, void* const* events, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || n_chunks < 1 || !bounds || !events) return TS_ERR_INVALID_ARG;
    if (bounds[0] != 0 || bounds[n_chunks] != c->n) return TS_ERR_INVALID_ARG;
    for (int k = 0; k < n_chunks; k++) {
        if (bounds[k + 1] < bounds[k] || (bounds[k] & 63) || !events[k]) return TS_ERR_INVALID_ARG;
    }
    return backward_impl(c, d_image, grads, accumulate, nullptr, nullptr, nullptr, stream, n_chunks, bounds, events);
}

// expected fragment CSR offsets of the last forward into c->frag_off; returns F
static int fragment_offsets(ts_context* c, cudaStream_t st, long long* total) {
    const long long P = (long long)c->cam.width * c->cam.height;
    int rc;
    if ((rc = ensure(c->frag_off, sizeof(long long) * (P + 1)))) return rc;
    if ((rc = ensure(c->cs_scratch, count_scan_scratch_bytes(P)))) return rc;
    count_scan_i64(P, c->nfrag, (long long*)c->frag_off.p, c->cs_scratch.p, st);
    g_launches += 3;
    long long f = 0;
    TS_CHECK(cudaMemcpyAsync(&f, (long long*)c->frag_off.p + P, sizeof(long long), cudaMemcpyDeviceToHost, st));
    TS_CHECK(cudaStreamSynchronize(st));
    *total = f;
    return TS_OK;
}

int ts_fragment_offsets(ts_context* c, int64_t* offsets, int64_t* n_fragments, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !n_fragments) return TS_ERR_INVALID_ARG;
    if (!c->have_fwd) return TS_ERR_NO_FORWARD;
    cudaStream_t st = (cudaStream_t)stream;
    long long f = 0;
    int rc = fragment_offsets(c, st, &f);
    if (rc) return rc;
    const long long P = (long long)c->cam.width * c->cam.height;
    if (offsets)
        TS_CHECK(cudaMemcpyAsync(offsets, c->frag_off.p, sizeof(long long) * (P + 1), cudaMemcpyDeviceToDevice, st));
    *n_fragments = (int64_t)f;
    return TS_OK;
}

int ts_collect_fragments(ts_context* c, const int64_t* offsets, int32_t* triangle, double* weight, double* depth,
                         void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !offsets || !triangle || !weight || !depth) return TS_ERR_INVALID_ARG;
    if (!c->have_fwd) return TS_ERR_NO_FORWARD;
    if (c->precision != 0) return TS_ERR_INVALID_ARG;  // fragment lists come from the fast path's fp64 replay
    cudaStream_t st = (cudaStream_t)stream;
    // re-composite with fp64 weights and emit every composited fragment
    // (rasterize_forward collect branch, _kernels.py:107-116); statistics and
    // images are not touched, flagged pixels are re-emitted by the fix-up
    TS_CHECK(cudaMemsetAsync(&c->d_ctr->n_flagged, 0, sizeof(unsigned long long), st));
    TS_CHECK(cudaMemsetAsync(&c->d_ctr->blend_done, 0, sizeof(unsigned long long), st));
    FastBlendOut bo{};
    bo.t_final = c->t_final32;
    bo.t_final64 = nullptr;
    bo.last_pos = c->last_pos;
    bo.n_frag = c->nfrag;
    bo.flags = c->flags;
    bo.ctr = c->d_ctr;
    bo.frag_off = (const long long*)offsets;
    bo.frag_tri = triangle;
    bo.frag_w = weight;
    bo.frag_z = depth;
    bo.zkey = c->key;
    if (c->have_bwd_state) {
        // a training forward: its fp64-compositing dense blend again, emitting each
        // pixel's fragments into its CSR list (no records, images or statistics)
        bo.recc = (const RecC*)c->recc.p;
        launch_blend_dense(c->cam, c->opt, true, (const RecF*)c->recf.p, c->tile_start, c->ent_src, bo, st);
    } else {
        launch_blend_fast(c->cam, c->opt, c->soup, c->dtype, (const RecF*)c->recf.p, c->bbox, c->tile_start,
                          c->ent_src, bo, st);
    }
    launch_fixup_fwd(c->cam, c->opt, c->soup, c->dtype, (const RecF*)c->recf.p, c->tile_start, c->ent_src, bo, st);
    g_launches += 2;
    return cuda_err(cudaGetLastError());
}

int ts_backward_fragments(ts_context* c, const float* d_image, const int64_t* offsets, const double* weight,
                          const double* d_weight, const double* d_depth, const ts_grads* grads, int accumulate,
                          void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !d_image || !grads || !offsets || !d_weight || !d_depth) return TS_ERR_INVALID_ARG;
    if (!c->have_fwd) return TS_ERR_NO_FORWARD;
    if (!c->have_bwd_state) return TS_ERR_NO_BWD_STATE;
    if (c->precision != 0) return TS_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    long long f = 0;
    int rc = fragment_offsets(c, st, &f);
    if (rc) return rc;
    const long long P = (long long)c->cam.width * c->cam.height;
    // the layout must be the CSR of this scene/camera (backward.py:130-136)
    TS_CHECK(cudaMemsetAsync(&c->d_ctr->pad[0], 0, sizeof(unsigned long long), st));
    offsets_mismatch(P, (const long long*)offsets, (const long long*)c->frag_off.p, &c->d_ctr->pad[0], st);
    g_launches += 1;
    unsigned long long bad = 0;
    TS_CHECK(cudaMemcpyAsync(&bad, &c->d_ctr->pad[0], sizeof(bad), cudaMemcpyDeviceToHost, st));
    TS_CHECK(cudaStreamSynchronize(st));
    if (bad) return TS_ERR_FRAGMENTS;
    return backward_impl(c, d_image, grads, accumulate, (const long long*)offsets, d_weight, d_depth, stream, 0,
                         nullptr, nullptr, weight, f);
}

// Screen-space part of a fast-path backward (the blend backward into the
// per-triangle fp64 rows sg, zeroed first): the streaming backward over the
// training forward's fragment records, or the tile backward.
static int screen_backward_fast(ts_context* c, const float* d_image, double* sg, const long long* frag_off,
                                const double* fg_dw, const double* fg_dz, const double* frag_w,
                                long long n_frag_total, cudaStream_t st) {
    int rc;
    stage_begin(c, TS_STAGE_BLEND_BWD, st);
    if (c->n > 0) TS_CHECK(cudaMemsetAsync(sg, 0, sizeof(double) * SG_STRIDE * c->n, st));
    if (c->frec_ready && (!frag_off || frag_w)) {
        // streaming backward over the forward's fragment records (with the
        // fragment-gradient terms when the caller passes the fragments' weights);
        // the tile backward runs instead only if the record buffer overflowed
        if (frag_off && (rc = ensure(c->fsw, sizeof(double) * (size_t)(n_frag_total > 0 ? n_frag_total : 1))))
            return rc;
        launch_bwd_stream(c->cam, c->opt, (const RecF*)c->recf.p, (const RecB*)c->recb.p, (const RecC*)c->recc.p,
                          (const FragRec*)c->frec.p, c->d_ctr, c->frec_cap, (const double*)c->ctot.p, d_image,
                          sg, st, frag_off, frag_w, fg_dw, fg_dz, frag_off ? (double*)c->fsw.p : nullptr);
        launch_blend_bwd_dense(c->cam, c->opt, (const RecF*)c->recf.p, (const RecB*)c->recb.p,
                               (const RecC*)c->recc.p, c->tile_start,
                               c->ent_src, c->t_final, c->last_pos, d_image, c->nfrag, frag_off, fg_dw, fg_dz,
                               &c->d_ctr->frec_over, sg, st);
        g_launches += frag_off ? 1 : 0;
    } else
        launch_blend_bwd_dense(c->cam, c->opt, (const RecF*)c->recf.p, (const RecB*)c->recb.p,
                               (const RecC*)c->recc.p, c->tile_start,
                               c->ent_src, c->t_final, c->last_pos, d_image, c->nfrag, frag_off, fg_dw, fg_dz,
                               nullptr, sg, st);
    stage_end(c, TS_STAGE_BLEND_BWD, st);
    return TS_OK;
}

static int backward_impl(ts_context* c, const float* d_image, const ts_grads* grads, int accumulate,
                         const long long* frag_off, const double* fg_dw, const double* fg_dz, void* stream,
                         int n_chunks, const int64_t* bounds, void* const* events, const double* frag_w,
                         long long n_frag_total) {
    if (!c || !d_image || !grads) return TS_ERR_INVALID_ARG;
    if (!c->have_fwd) return TS_ERR_NO_FORWARD;
    if (!c->have_bwd_state) return TS_ERR_NO_BWD_STATE;
    cudaStream_t st = (cudaStream_t)stream;
    const long long n1 = c->n > 0 ? c->n : 1;
    int rc;
    c->ev_used[TS_STAGE_BLEND_BWD] = c->ev_used[TS_STAGE_CHAIN_BWD] = false;
    if (c->precision == 0) {
        if ((rc = ensure(c->sg64, sizeof(double) * SG_STRIDE * n1))) return rc;
        double* sg = (double*)c->sg64.p;
        if ((rc = screen_backward_fast(c, d_image, sg, frag_off, fg_dw, fg_dz, frag_w, n_frag_total, st))) return rc;
        stage_begin(c, TS_STAGE_CHAIN_BWD, st);
        if (n_chunks > 0 && chain_bwd_fast_ok(c->soup, c->dtype, *grads)) {
            // the chain in triangle ranges, an event after each: the caller's
            // collective on a bucket can start while the next range computes
            for (int k = 0; k < n_chunks; k++) {
                launch_chain_bwd_fast(c->cam, c->opt, c->soup, c->dtype, c->flag, sg, *grads, accumulate, st, bounds[k],
                                      bounds[k + 1]);
                TS_CHECK(cudaEventRecord((cudaEvent_t)events[k], st));
            }
            g_launches += n_chunks - 1;
        } else {
            if (!launch_chain_bwd_fast(c->cam, c->opt, c->soup, c->dtype, c->flag, sg, *grads, accumulate, st))
                launch_chain_bwd(c->cam, c->opt, c->soup, c->dtype, c->flag, sg, *grads, accumulate, st);
            for (int k = 0; k < n_chunks; k++) TS_CHECK(cudaEventRecord((cudaEvent_t)events[k], st));
        }
        stage_end(c, TS_STAGE_CHAIN_BWD, st);
        c->sgrad_kind = 1;
    } else {
        if ((rc = ensure(c->sg64, sizeof(double) * SG_STRIDE * n1))) return rc;
        double* sg = (double*)c->sg64.p;
        stage_begin(c, TS_STAGE_BLEND_BWD, st);
        if (c->n > 0) TS_CHECK(cudaMemsetAsync(sg, 0, sizeof(double) * SG_STRIDE * c->n, st));
        launch_blend_bwd_exact(c->cam, c->opt, (const Rec64*)c->rec64.p, c->tile_start, (const int*)c->ent_src,
                               c->t_final, c->last_pos, d_image, sg, st);
        stage_end(c, TS_STAGE_BLEND_BWD, st);
        stage_begin(c, TS_STAGE_CHAIN_BWD, st);
        launch_chain_bwd(c->cam, c->opt, c->soup, c->dtype, c->flag, sg, *grads, accumulate, st);
        for (int k = 0; k < n_chunks; k++) TS_CHECK(cudaEventRecord((cudaEvent_t)events[k], st));
        stage_end(c, TS_STAGE_CHAIN_BWD, st);
        c->sgrad_kind = 1;
    }
    g_launches += 2;
    TS_CHECK(cudaGetLastError());
    return TS_OK;
}

int ts_backward_screen(ts_context* c, const float* d_image, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !d_image) return TS_ERR_INVALID_ARG;
    if (!c->have_fwd) return TS_ERR_NO_FORWARD;
    if (!c->have_bwd_state) return TS_ERR_NO_BWD_STATE;
    // fast path, fp32 parameters with 16-byte aligned blocks (the chain's staged loads)
    if (c->precision != 0 || c->dtype != 0 || (((uintptr_t)c->soup.sh | (uintptr_t)c->soup.vertices) & 15))
        return TS_ERR_INVALID_ARG;
    if (c->n_slots >= TS_MAX_CHAIN_VIEWS) return TS_ERR_INVALID_ARG;  // ts_chain_views first
    if (c->n_slots > 0 && (c->soup.n != c->slot_soup.n || c->soup.vertices != c->slot_soup.vertices ||
                           c->soup.sh != c->slot_soup.sh || c->opt.mode != c->slot_opt.mode ||
                           c->opt.ncoef != c->slot_opt.ncoef))
        return TS_ERR_INVALID_ARG;  // every pending view renders the same soup with the same options
    cudaStream_t st = (cudaStream_t)stream;
    const long long n1 = c->n > 0 ? c->n : 1;
    const int k = c->n_slots;
    int rc;
    if ((rc = ensure(c->slot_sg[k], sizeof(double) * SG_STRIDE * n1))) return rc;
    if ((rc = ensure(c->slot_flag[k], sizeof(unsigned) * n1))) return rc;
    c->ev_used[TS_STAGE_BLEND_BWD] = c->ev_used[TS_STAGE_CHAIN_BWD] = false;
    if ((rc = screen_backward_fast(c, d_image, (double*)c->slot_sg[k].p, nullptr, nullptr, nullptr, nullptr, 0, st)))
        return rc;
    if (c->n > 0)
        TS_CHECK(cudaMemcpyAsync(c->slot_flag[k].p, c->flag, sizeof(unsigned) * c->n, cudaMemcpyDeviceToDevice, st));
    c->slot_cam[k] = c->cam;
    if (k == 0) {
        c->slot_soup = c->soup;
        c->slot_opt = c->opt;
    }
    c->n_slots = k + 1;
    g_launches += 1;
    return cuda_err(cudaGetLastError());
}

int ts_pending_views(ts_context* c) { return c ? c->n_slots : 0; }

int ts_reserve(ts_context* c, int64_t n, int width, int height, int64_t entries, int keep_backward) {
    DeviceGuard device_guard(c);
    if (!c || n < 0 || width < 1 || height < 1 || width > 32000 || height > 32000 || n >= (1ll << 31))
        return TS_ERR_INVALID_ARG;
    const long long n1 = n > 0 ? n : 1;
    const long long P = (long long)width * height;
    const int ntiles = ((width + TILE - 1) / TILE) * ((height + TILE - 1) / TILE);
    const long long e = entries > 0 ? entries : 4 * n1 + 4096;
    c->e_hint = std::max<long long>(c->e_hint, e);  // the forwards' working capacity follows it
    int rc;
    if ((rc = ensure_tri(c, n1)) || (rc = ensure_pix(c, P, ntiles)) ||
        (rc = ensure(c->recf, sizeof(RecF) * n1)) ||
        (rc = ensure_ent(c, std::max<long long>(4 * n1 + 4096, c->e_hint + c->e_hint / 2))) ||
        (rc = ensure_os(c, std::max<long long>(n1, c->cap_e) + 1)) || (rc = ensure(c->binmat, bin_matrix_bytes(n1, ntiles))))
        return rc;
    if (keep_backward) {
        const long long f = std::max<long long>(c->frec_hint, 8 * std::max<long long>(c->e_hint, n1));
        c->frec_hint = std::max<long long>(c->frec_hint, f);
        if ((rc = ensure(c->recb, sizeof(RecB) * n1)) || (rc = ensure(c->recc, sizeof(RecC) * n1)) ||
            (rc = ensure(c->sg64, sizeof(double) * SG_STRIDE * n1)) ||
            (rc = ensure(c->frec, sizeof(FragRec) * (size_t)(f + f / 4 + 4096))) ||
            (rc = ensure(c->ctot, sizeof(double) * 3 * (size_t)P)))
            return rc;
        c->frec_cap = c->frec.bytes / sizeof(FragRec);
    }
    return TS_OK;
}

int64_t ts_workspace_bytes(ts_context* c) {
    if (!c) return 0;
    int64_t t = (int64_t)(c->tri_bytes + c->ent_bytes + c->pix_bytes + c->os_bytes);
    for (const DevBuf* b : {&c->fsw, &c->adam_ibc, &c->tl_cnt, &c->tl_off, &c->tl_cs, &c->tl_kv, &c->rec64, &c->recf,
                            &c->recb, &c->recc, &c->sg64, &c->sg32, &c->frag_off, &c->cs_scratch, &c->frec, &c->ctot,
                            &c->binmat, &c->lossbuf, &c->densbuf})
        t += (int64_t)b->bytes;
    for (int k = 0; k < TS_MAX_CHAIN_VIEWS; k++) t += (int64_t)(c->slot_sg[k].bytes + c->slot_flag[k].bytes);
    return t;
}


int ts_chain_views(ts_context* c, const ts_grads* grads, int accumulate, int n_chunks, const int64_t* bounds,
                   void* const* events, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !grads) return TS_ERR_INVALID_ARG;
    if (c->n_slots == 0) return TS_ERR_NO_BWD_STATE;
    if (!chain_bwd_fast_ok(c->slot_soup, 0, *grads)) return TS_ERR_INVALID_ARG;
    const long long n = c->slot_soup.n;
    if (n_chunks > 0) {
        if (!bounds || !events || bounds[0] != 0 || bounds[n_chunks] != n) return TS_ERR_INVALID_ARG;
        for (int k = 0; k < n_chunks; k++)
            if (bounds[k + 1] < bounds[k] || (bounds[k] & 63) || !events[k]) return TS_ERR_INVALID_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    ChainViews cv{};
    cv.n = c->n_slots;
    for (int k = 0; k < cv.n; k++) {
        cv.cam[k] = c->slot_cam[k];
        cv.flag[k] = (const unsigned*)c->slot_flag[k].p;
        cv.sgrad[k] = (const double*)c->slot_sg[k].p;
    }
    c->ev_used[TS_STAGE_CHAIN_BWD] = false;
    stage_begin(c, TS_STAGE_CHAIN_BWD, st);
    if (n_chunks > 0) {
        for (int k = 0; k < n_chunks; k++) {
            launch_chain_multi(cv, c->slot_opt, c->slot_soup, *grads, accumulate, st, bounds[k], bounds[k + 1]);
            TS_CHECK(cudaEventRecord((cudaEvent_t)events[k], st));
        }
        g_launches += n_chunks;
    } else {
        launch_chain_multi(cv, c->slot_opt, c->slot_soup, *grads, accumulate, st);
        g_launches += 1;
    }
    stage_end(c, TS_STAGE_CHAIN_BWD, st);
    c->n_slots = 0;
    return cuda_err(cudaGetLastError());
}

int ts_photometric_loss(ts_context* c, const float* rendered, const float* target, int height, int width,
                        double lambda_dssim, double* out, float* d_image, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !rendered || !target || !out || height < 1 || width < 1) return TS_ERR_INVALID_ARG;
    int rc;
    if ((rc = ensure(c->lossbuf, photometric_scratch_bytes(height, width)))) return rc;
    launch_photometric_loss(rendered, target, height, width, lambda_dssim, out, d_image, c->lossbuf.p, false,
                            (cudaStream_t)stream);
    g_launches += 3;
    return cuda_err(cudaGetLastError());
}

int ts_distortion_loss(ts_context* c, const int64_t* offsets, const double* weight, const double* depth,
                       int64_t n_pixels, int64_t image_size, double* out, double* d_weight, double* d_depth,
                       void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !offsets || !out || n_pixels < 0) return TS_ERR_INVALID_ARG;
    int rc;
    if ((rc = ensure(c->lossbuf, distortion_scratch_bytes(n_pixels)))) return rc;
    launch_distortion_loss(n_pixels, (const long long*)offsets, weight, depth,
                           image_size > 0 ? image_size : n_pixels, out, d_weight, d_depth, c->lossbuf.p,
                           (cudaStream_t)stream);
    g_launches += n_pixels > 0 ? 2 : 1;
    return cuda_err(cudaGetLastError());
}

int ts_normal_loss(ts_context* c, const float* vertices, int64_t n, const int64_t* offsets,
                   const int32_t* triangle, const double* weight, int64_t n_fragments, const double* depth,
                   const ts_camera* cam, double* out, double* d_vertices, double* d_weight, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !cam || !out || n < 0 || n_fragments < 0 || !offsets || !depth) return TS_ERR_INVALID_ARG;
    if ((n > 0 && !vertices) || (n_fragments > 0 && (!triangle || !weight))) return TS_ERR_INVALID_ARG;
    const long long npix = (long long)cam->width * cam->height;
    int rc;
    if ((rc = ensure(c->lossbuf, normal_scratch_bytes(n, npix)))) return rc;
    double cm[16] = {cam->fx, cam->fy, cam->cx, cam->cy};
    for (int k = 0; k < 9; k++) cm[4 + k] = cam->R[k];
    for (int k = 0; k < 3; k++) cm[13 + k] = cam->t[k];
    launch_normal_loss(vertices, n, (const long long*)offsets, triangle, weight, n_fragments, depth, cam->height,
                       cam->width, cm, out, d_vertices, d_weight, c->lossbuf.p, (cudaStream_t)stream);
    g_launches += 5;
    return cuda_err(cudaGetLastError());
}

int ts_fragment_depth(ts_context* c, const int64_t* offsets, const double* weight, const double* depth,
                      int64_t n_pixels, double* out_depth, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !offsets || !out_depth || n_pixels < 0) return TS_ERR_INVALID_ARG;
    launch_fragment_depth(n_pixels, (const long long*)offsets, weight, depth, out_depth, (cudaStream_t)stream);
    g_launches += n_pixels > 0 ? 1 : 0;
    return cuda_err(cudaGetLastError());
}

int ts_adam_step(ts_context* c, float* vertices, float* opacity, float* sigma, float* sh, int64_t n,
                 const ts_grads* grads, float* m, float* v, int64_t* t, const double* lrs, int64_t* bad,
                 void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !grads || !lrs || !bad || !t || n < 0) return TS_ERR_INVALID_ARG;
    if (n > 0 && (!vertices || !opacity || !sigma || !sh || !m || !v)) return TS_ERR_INVALID_ARG;
    int rc;
    if ((rc = ensure(c->adam_ibc, 2 * sizeof(double)))) return rc;
    float* const params[4] = {vertices, opacity, sigma, sh};
    const float* const g[4] = {grads->d_vertices, grads->d_opacity, grads->d_sigma, grads->d_sh};
    launch_adam_step(params, g, n, m, v, (long long*)t, lrs, (long long*)bad, (double*)c->adam_ibc.p,
                     (cudaStream_t)stream);
    g_launches += n > 0 ? 2 : 0;
    return cuda_err(cudaGetLastError());
}

// ---------------- density control (density.py:27-263) ----------------
int ts_view_stats_accumulate(ts_context* c, int64_t n, const float* max_weight, const int32_t* pixel_count,
                             const float* area, int min_pixels, int first, double* acc_max_weight,
                             int32_t* acc_views, double* acc_area, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || n < 0) return TS_ERR_INVALID_ARG;
    if (n > 0 && (!max_weight || !pixel_count || !area || !acc_max_weight || !acc_views || !acc_area))
        return TS_ERR_INVALID_ARG;
    launch_stats_accum(n, max_weight, pixel_count, area, min_pixels, first, acc_max_weight, acc_views, acc_area,
                       (cudaStream_t)stream);
    g_launches += n > 0 ? 1 : 0;
    return cuda_err(cudaGetLastError());
}

int ts_prune_mark(ts_context* c, int64_t n, const double* acc_max_weight, const int32_t* acc_views,
                  const void* opacity, int dtype, double tau_prune, int min_views, double opacity_dead,
                  uint8_t* flags, int64_t* kept, int64_t* n_kept, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || n < 0 || !n_kept || (dtype != 0 && dtype != 1)) return TS_ERR_INVALID_ARG;
    if (n > 0 && (!acc_max_weight || !acc_views || !opacity || !flags || !kept)) return TS_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    launch_prune_mark(n, acc_max_weight, acc_views, opacity, dtype, tau_prune, min_views, opacity_dead, flags, st);
    compact_unflagged(n, flags, (long long*)kept, (long long*)n_kept, c->sort, st);
    g_launches += n > 0 ? 4 : 0;
    return cuda_err(cudaGetLastError());
}

int ts_sample_candidates(ts_context* c, int64_t n_pool, const int64_t* pool, const int64_t* kept,
                         const void* param, int dtype, int criterion, const double* exponential, int64_t count,
                         int64_t* picked, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || n_pool < 0 || count < 0 || count > n_pool || (dtype != 0 && dtype != 1)) return TS_ERR_INVALID_ARG;
    if (criterion != TS_SAMPLE_INVERSE_SIGMA && criterion != TS_SAMPLE_OPACITY) return TS_ERR_INVALID_ARG;
    if (count == 0) return TS_OK;
    if (!param || !exponential || !picked) return TS_ERR_INVALID_ARG;
    if (n_pool > 0xffffffffLL) return TS_ERR_CAPACITY;
    int rc;
    if ((rc = ensure(c->densbuf, sample_scratch_bytes(n_pool)))) return rc;
    launch_sample_candidates(n_pool, (const long long*)pool, (const long long*)kept, param, dtype,
                             criterion == TS_SAMPLE_INVERSE_SIGMA, exponential, count, (long long*)picked,
                             c->densbuf.p, c->sort, (cudaStream_t)stream);
    g_launches += 3 + 3 * 8;
    return cuda_err(cudaGetLastError());
}

int ts_pick_info(ts_context* c, int64_t count, const int64_t* picked, const int64_t* pool, const int64_t* kept,
                 const double* acc_area, int64_t n_views, const void* vertices, int dtype, int64_t* source,
                 double* mean_area, uint8_t* degenerate, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || count < 0 || (dtype != 0 && dtype != 1)) return TS_ERR_INVALID_ARG;
    if (count > 0 && (!picked || !acc_area || !vertices || !source || !mean_area || !degenerate))
        return TS_ERR_INVALID_ARG;
    launch_pick_info(count, (const long long*)picked, (const long long*)pool, (const long long*)kept, acc_area,
                     n_views, vertices, dtype, (long long*)source, mean_area, degenerate, (cudaStream_t)stream);
    g_launches += count > 0 ? 1 : 0;
    return cuda_err(cudaGetLastError());
}

int ts_gather_rows(ts_context* c, int64_t n_out, const int64_t* origin, const void* src, void* dst, int width,
                   int elem_bytes, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || n_out < 0 || width < 0 || (elem_bytes != 4 && elem_bytes != 8)) return TS_ERR_INVALID_ARG;
    if (n_out > 0 && width > 0 && (!origin || !src || !dst)) return TS_ERR_INVALID_ARG;
    launch_gather_rows(n_out, (const long long*)origin, src, dst, width, elem_bytes, (cudaStream_t)stream);
    g_launches += (n_out > 0 && width > 0) ? 1 : 0;
    return cuda_err(cudaGetLastError());
}

int ts_child_vertices(ts_context* c, int64_t n_child, const int64_t* parent, const int32_t* code,
                      const double* uniforms, double max_noise_factor, const void* src_vertices, void* dst_vertices,
                      int dtype, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || n_child < 0 || (dtype != 0 && dtype != 1)) return TS_ERR_INVALID_ARG;
    if (n_child > 0 && (!parent || !code || !src_vertices || !dst_vertices)) return TS_ERR_INVALID_ARG;
    launch_child_vertices(n_child, (const long long*)parent, code, uniforms, max_noise_factor, src_vertices,
                          dst_vertices, dtype, (cudaStream_t)stream);
    g_launches += n_child > 0 ? 1 : 0;
    return cuda_err(cudaGetLastError());
}

// ---------------- model I/O: binary PLY body (scene_io.py:382-455) ----------------
int ts_ply_pack(ts_context* c, const void* vertices, const void* sh, int dtype, int64_t n, uint8_t* vertex_bytes,
                void* face_bytes, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || n < 0 || (dtype != 0 && dtype != 1)) return TS_ERR_INVALID_ARG;
    if (n > 0 && (!vertices || !sh || !vertex_bytes || !face_bytes)) return TS_ERR_INVALID_ARG;
    if (n > (1LL << 31) / 3) return TS_ERR_CAPACITY;  // int32 vertex indices
    if (((uintptr_t)vertex_bytes & 15) || ((uintptr_t)face_bytes & 15)) return TS_ERR_INVALID_ARG;
    launch_ply_pack(n, vertices, sh, dtype, vertex_bytes, face_bytes, (cudaStream_t)stream);
    g_launches += n > 0 ? 1 : 0;
    return cuda_err(cudaGetLastError());
}

int ts_ply_unpack(ts_context* c, const uint8_t* vertex_bytes, int64_t n_vertex, const void* face_bytes,
                  int64_t n_face, double sigma, int dtype, void* vertices, void* opacity, void* sigma_out, void* sh,
                  uint64_t* bad, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || n_vertex < 0 || n_face < 0 || !bad || (dtype != 0 && dtype != 1)) return TS_ERR_INVALID_ARG;
    if (n_face > 0 && (!vertex_bytes || !face_bytes || !vertices || !opacity || !sigma_out || !sh))
        return TS_ERR_INVALID_ARG;
    if ((uintptr_t)face_bytes & 15) return TS_ERR_INVALID_ARG;
    launch_ply_unpack(n_face, n_vertex, vertex_bytes, face_bytes, sigma, dtype, vertices, opacity, sigma_out, sh,
                      (unsigned long long*)bad, (cudaStream_t)stream);
    g_launches += n_face > 0 ? 1 : 0;
    return cuda_err(cudaGetLastError());
}

int ts_ssim(ts_context* c, const float* x, const float* y, int height, int width, double* out, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !x || !y || !out || height < 1 || width < 1) return TS_ERR_INVALID_ARG;
    int rc;
    if ((rc = ensure(c->lossbuf, photometric_scratch_bytes(height, width)))) return rc;
    launch_photometric_loss(x, y, height, width, 1.0, out, nullptr, c->lossbuf.p, true, (cudaStream_t)stream);
    g_launches += 2;
    return cuda_err(cudaGetLastError());
}

int ts_debug_copy(ts_context* c, int what, void* dst, size_t bytes, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !dst) return TS_ERR_INVALID_ARG;
    if (!c->have_fwd) return TS_ERR_NO_FORWARD;
    cudaStream_t st = (cudaStream_t)stream;
    int ntiles = c->cam.ntx * c->cam.nty;
    switch (what) {
        case TS_DUMP_SORTED_IDX:
            if (bytes < 4 * (size_t)c->m) return TS_ERR_INVALID_ARG;
            if (!c->sorted_valid) global_depth_order(c, c->n, st);
            if (c->m) TS_CHECK(cudaMemcpyAsync(dst, c->sorted_src, 4 * c->m, cudaMemcpyDeviceToDevice, st));
            return TS_OK;
        case TS_DUMP_TILE_START:
            if (bytes < 4 * (size_t)(ntiles + 1)) return TS_ERR_INVALID_ARG;
            TS_CHECK(cudaMemcpyAsync(dst, c->tile_start, 4 * (ntiles + 1), cudaMemcpyDeviceToDevice, st));
            return TS_OK;
        case TS_DUMP_ENTRY_RANK:
            if (bytes < 4 * (size_t)c->e) return TS_ERR_INVALID_ARG;
            if (!c->sorted_valid) global_depth_order(c, c->n, st);
            rank_offsets(c->n, c->sorted_src, c->tcount, c->offs, c->rank_of, c->sort, st);
            entries_to_rank(c->e, c->ent_src, c->rank_of, (int*)dst, st);
            return cuda_err(cudaGetLastError());
        case TS_DUMP_BBOX:
            if (bytes < 16 * (size_t)c->n) return TS_ERR_INVALID_ARG;
            bbox_dump(c->n, c->bbox, (int*)dst, st);
            return cuda_err(cudaGetLastError());
        case TS_DUMP_DEPTH:
            if (bytes < 8 * (size_t)c->n) return TS_ERR_INVALID_ARG;
            // the depth key is the fp64 bit pattern of the centroid depth (0 if culled)
            if (c->n) TS_CHECK(cudaMemcpyAsync(dst, c->key, 8 * c->n, cudaMemcpyDeviceToDevice, st));
            return TS_OK;
        case TS_DUMP_SGRAD: {
            if (bytes < 8 * SG_STRIDE * (size_t)c->n || !c->sgrad_kind) return TS_ERR_INVALID_ARG;
            if (!c->n) return TS_OK;
            if (c->sgrad_kind == 1) {
                TS_CHECK(cudaMemcpyAsync(dst, c->sg64.p, 8 * SG_STRIDE * c->n, cudaMemcpyDeviceToDevice, st));
            } else {
                // widen fp32 -> fp64 through a host bounce (debug only)
                size_t cnt = (size_t)SG_STRIDE * c->n;
                float* h32 = (float*)malloc(4 * cnt);
                double* h64 = (double*)malloc(8 * cnt);
                TS_CHECK(cudaMemcpyAsync(h32, c->sg32.p, 4 * cnt, cudaMemcpyDeviceToHost, st));
                TS_CHECK(cudaStreamSynchronize(st));
                for (size_t k = 0; k < cnt; k++) h64[k] = h32[k];
                TS_CHECK(cudaMemcpyAsync(dst, h64, 8 * cnt, cudaMemcpyHostToDevice, st));
                TS_CHECK(cudaStreamSynchronize(st));
                free(h32);
                free(h64);
            }
            return TS_OK;
        }
        case TS_DUMP_FRAGREC: {
            // fragment records of the last training forward (48 B each, count first)
            unsigned long long nrec = 0;
            TS_CHECK(cudaMemcpyAsync(&nrec, &c->d_ctr->n_frec, sizeof(nrec), cudaMemcpyDeviceToHost, st));
            TS_CHECK(cudaStreamSynchronize(st));
            if (!c->frec_ready) nrec = 0;
            nrec = std::min<unsigned long long>(nrec, c->frec_cap);
            if (bytes < 8 + sizeof(FragRec) * nrec) return TS_ERR_INVALID_ARG;
            TS_CHECK(cudaMemcpyAsync(dst, &nrec, 8, cudaMemcpyHostToDevice, st));
            if (nrec)
                TS_CHECK(cudaMemcpyAsync((char*)dst + 8, c->frec.p, sizeof(FragRec) * nrec, cudaMemcpyDeviceToDevice,
                                         st));
            TS_CHECK(cudaStreamSynchronize(st));
            return TS_OK;
        }
        case TS_DUMP_PROJECTION: {
            // project_scene of the last forward: PROJ_ROW doubles per depth-sorted
            // accepted triangle, then area_full (N doubles)
            if (bytes < 8 * ((size_t)PROJ_ROW * c->m + (size_t)c->n)) return TS_ERR_INVALID_ARG;
            if (!c->sorted_valid) global_depth_order(c, c->n, st);
            double* rows = (double*)dst;
            launch_projection_dump(c->cam, c->opt, c->soup, c->dtype, c->sorted_src, c->m, rows,
                                   rows + (size_t)PROJ_ROW * c->m, st);
            g_launches += 1;
            return cuda_err(cudaGetLastError());
        }
        default:
            return TS_ERR_INVALID_ARG;
    }
}

int ts_tile_lists(ts_context* c, const int64_t* bbox, int64_t m, int tile_size, int width, int height,
                  int64_t* tile_start, int64_t* entry_tri, int64_t* n_entries, void* stream) {
    DeviceGuard device_guard(c);
    if (!c || !n_entries || m < 0 || tile_size < 1 || width < 0 || height < 0 || (m > 0 && !bbox))
        return TS_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const long long ntx = (width + tile_size - 1) / tile_size, nty = (height + tile_size - 1) / tile_size;
    if (ntx * nty >= (1ll << 31)) return TS_ERR_INVALID_ARG;
    const int ntiles = (int)(ntx * nty);
    const long long m1 = m > 0 ? m : 1;
    int rc;
    if ((rc = ensure(c->tl_cnt, sizeof(int) * m1))) return rc;
    if ((rc = ensure(c->tl_off, sizeof(long long) * (m1 + 1)))) return rc;
    if ((rc = ensure(c->tl_cs, count_scan_scratch_bytes(m1)))) return rc;
    tile_lists_count(m, (const long long*)bbox, tile_size, (int*)c->tl_cnt.p, (long long*)c->tl_off.p, c->tl_cs.p, st);
    long long e = 0;
    TS_CHECK(cudaMemcpyAsync(&e, (long long*)c->tl_off.p + m, sizeof(e), cudaMemcpyDeviceToHost, st));
    TS_CHECK(cudaStreamSynchronize(st));
    *n_entries = e;
    if (!tile_start || (e > 0 && !entry_tri)) return TS_OK;  // size query
    if (e >= (1ll << 32)) return TS_ERR_INVALID_ARG;
    const long long e1 = e > 0 ? e : 1;
    if ((rc = ensure(c->tl_kv, 4 * sizeof(unsigned) * (size_t)e1))) return rc;
    unsigned* kv0 = (unsigned*)c->tl_kv.p;
    unsigned* const kv[4] = {kv0, kv0 + e1, kv0 + 2 * e1, kv0 + 3 * e1};
    tile_lists_fill(m, e, (const long long*)bbox, tile_size, (int)ntx, ntiles, (const long long*)c->tl_off.p, kv,
                    c->sort, (long long*)tile_start, (long long*)entry_tri, st);
    g_launches += 6;
    return cuda_err(cudaGetLastError());
}

int ts_flagged_pixels(ts_context* c, int64_t* n_flagged) {
    DeviceGuard device_guard(c);
    if (!c || !n_flagged) return TS_ERR_INVALID_ARG;
    *n_flagged = (int64_t)c->h_ctr->n_flagged;
    return TS_OK;
}

}  // extern "C"
