// ts_blend.cu -- render-only forward blend (rasterize_forward, _kernels.py:59-132)
// as dense (entry, pixel) pair evaluation.
//
// CTA per 16x16 tile, 256 threads.  The tile's entry list (depth-rank order)
// is consumed in batches of DB entries:
//   1. stage    -- records to shared memory; per entry the rectangle
//                  bbox ∩ tile and an exclusive scan of the rectangle areas;
//   2. evaluate -- the S = Σ area (entry, pixel) pairs of the batch are split
//                  into 256 equal contiguous ranges, one per thread, so every
//                  lane evaluates a pixel that lies inside its entry's bbox
//                  (the reference's per-pixel bbox test, _kernels.py:87-95,
//                  costs nothing and no lane idles).  A pair whose r = phi/phi_s
//                  passes the lower end of the contribution band stores its
//                  fp32 alpha in s_al[entry][pixel] and sets bit `entry` of the
//                  pixel's batch mask (NaN alpha = r inside the band);
//   3. composite -- thread = pixel walks its mask bits in ascending entry
//                  (= depth) order: front-to-back compositing with the guard
//                  band of ts_fast.cu, per-entry max weight / pixel count in
//                  shared memory, one global atomic per (entry, tile).
// Pixels whose decision falls inside a guard band stop and are flagged for
// the exact fp64 fix-up (k_fixup_fwd), exactly as in k_blend_render.
#include "ts_kernels.cuh"

namespace ts {

namespace {
constexpr float T_MIN_F = 1e-4f;
constexpr float ALPHA_CLAMP_F = 0.99f;

}  // namespace


// DB entries per batch at most, PCAP (entry, pixel) pairs per batch at most.
// Records live in a ring of 2*DB slots (slot = tile-list position mod 2*DB),
// split into the evaluation part (first 96 B of RecF) and the tail (last 32 B:
// f0, f1, rgb, bbox); source ids in a ring of 4*DB.  While batch [b, b+nb) is
// processed, the records of [b+nb, b+nb+DB) and the ids up to b+3*DB are in
// flight (cp.async).

template <int DB, int PCAP>
struct DenseSmem {
    static constexpr int RR = 2 * DB, SR = 4 * DB, NW = DB / 32;
    EvalRec ev[RR];
    TailRec tail[RR];
    float r[PCAP];                 // per pair: fp32 r; NaN = inside the contribution band
    unsigned mask[NW][256];        // per pixel: bit j = entry j passes (r >= r_lo)
    unsigned srcq[SR];
    float4 col[DB];                // rgb, f0
    float f1[DB];
    int S[DB + 1];                 // first pair of entry j
    int H[DB + 1];                 // first row unit of entry j (row-interval evaluation)
    double inva[DB][3];            // 1 / a_e0 per edge (0 if a_e0 == 0)
    unsigned geo[DB];              // cx0 | cy0<<4 | w<<8 | magic<<16
    int2 kb[DB];                   // pair of pixel (lx, ly) = x + ly * y + lx
    unsigned maxw[DB];
    int pix[DB];
    // per-pixel compositing state (pixels migrate between threads every batch)
    float T[256], C[3][256], eps[256];
    int last[256], cnt[256], flag[256];  // flag: -1 live, >= 0 flag position, -2 outside the image
    int hist[DB + 1], cursor[DB + 1];
    int perm[256];
    double xc[TILE], yc[TILE];     // pixel centres of the tile (fp64)
    int nb;
};

template <int DB, int PCAP, bool SORT, bool ROWS>
__global__ void __launch_bounds__(256) k_blend_dense(Cam cam, Opts opt, const RecF* __restrict__ rec,
                                                     const int* __restrict__ tile_start,
                                                     const unsigned* __restrict__ ent_src,
                                                     FastBlendOut out) {
    using SM = DenseSmem<DB, PCAP>;
    constexpr int RR = SM::RR, SR = SM::SR, NW = SM::NW;
    extern __shared__ __align__(16) unsigned char s_dyn[];
    SM& sm = *reinterpret_cast<SM*>(s_dyn);

    const int tid = threadIdx.x;
    const unsigned lane = tid & 31, warp = tid >> 5;
    const int t = blockIdx.x;
    const int tx = t % cam.ntx, ty = t / cam.ntx;
    const int X0 = tx * TILE, Y0 = ty * TILE;
    const int s = tile_start[t], e = tile_start[t + 1];
    const float tau = (float)opt.tau_contrib;
    const int mode = opt.mode;
    {
        const int px = X0 + (tid & 15), py = Y0 + (tid >> 4);
        sm.T[tid] = 1.f;
        sm.C[0][tid] = sm.C[1][tid] = sm.C[2][tid] = 0.f;
        sm.eps[tid] = 0.f;
        sm.last[tid] = -1;
        sm.cnt[tid] = 0;
        sm.flag[tid] = (px < cam.width && py < cam.height) ? -1 : -2;
    }
    if (tid < DB) {
        sm.maxw[tid] = 0u;
        sm.pix[tid] = 0;
    }
    if (tid < TILE) sm.xc[tid] = (double)(X0 + tid) + 0.5;
    else if (tid < 2 * TILE) sm.yc[tid - TILE] = (double)(Y0 + tid - TILE) + 0.5;
    auto fetch_rec = [&](int p, int q) {  // 16-byte chunk q of the record at list position p
        const float4* g = reinterpret_cast<const float4*>(rec + sm.srcq[p & (SR - 1)]) + q;
        const int slot = p & (RR - 1);
        if (q < 6) cp_async16(reinterpret_cast<float4*>(&sm.ev[slot]) + q, g);
        else cp_async16(reinterpret_cast<float4*>(&sm.tail[slot]) + (q - 6), g);
    };
    // prologue: ids of [s, s+3DB), then records of [s, s+DB)
    int shi = min(s + 3 * DB, e), rhi = min(s + DB, e);
    for (int p = s + tid; p < shi; p += 256) cp_async4(&sm.srcq[p & (SR - 1)], ent_src + p);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    for (int c = tid; c < (rhi - s) * 8; c += 256) fetch_rec(s + (c >> 3), c & 7);
    cp_async_commit();
    int nb = 0;
    for (int b = s; b < e; b += nb) {
        cp_async_wait_all();
        const bool my_done = sm.flag[tid] != -1 || sm.T[tid] < T_MIN_F;
        if (__syncthreads_count(!my_done) == 0) break;
        const int navail = min(DB, e - b);
        {  // ids two batches ahead
            const int nshi = min(b + 3 * DB, e);
            for (int p = shi + tid; p < nshi; p += 256) cp_async4(&sm.srcq[p & (SR - 1)], ent_src + p);
            shi = max(shi, nshi);
        }
        // ---- 1. rectangles, scan, batch size (warp 0); clear masks / histogram ----
#pragma unroll
        for (int w = 0; w < NW; w++) sm.mask[w][tid] = 0u;
        if (tid <= DB) sm.hist[tid] = sm.cursor[tid] = 0;
        if (warp == 0) {
            int cx0[NW], cy0[NW], w[NW], h[NW], incl[NW];
            bool valid[NW];
            int carry = 0;
#pragma unroll
            for (int hf = 0; hf < NW; hf++) {
                const int j = (int)lane + 32 * hf;
                valid[hf] = j < navail;
                cx0[hf] = cy0[hf] = w[hf] = h[hf] = 0;
                if (valid[hf]) {
                    const int slot = (b + j) & (RR - 1);
                    const float4 t0 = reinterpret_cast<const float4*>(&sm.tail[slot])[0];
                    const int4 t1 = reinterpret_cast<const int4*>(&sm.tail[slot])[1];
                    const int bx0 = (short)(t1.y & 0xffff), bx1 = (short)(t1.y >> 16);
                    const int by0 = (short)(t1.z & 0xffff), by1 = (short)(t1.z >> 16);
                    cx0[hf] = max(bx0 - X0, 0);
                    cy0[hf] = max(by0 - Y0, 0);
                    w[hf] = max(min(bx1 - X0, TILE) - cx0[hf], 0);
                    h[hf] = max(min(by1 - Y0, TILE) - cy0[hf], 0);
                    sm.col[j] = make_float4(t0.z, t0.w, __int_as_float(t1.x), t0.x);
                    sm.f1[j] = t0.y;
                }
                int a = w[hf] * h[hf];
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, a, off);
                    if ((int)lane >= off) a += y;
                }
                incl[hf] = a + carry;
                carry = __shfl_sync(0xffffffffu, incl[hf], 31);
            }
            if constexpr (ROWS) {
                int hcarry = 0;
#pragma unroll
                for (int hf = 0; hf < NW; hf++) {
                    const int j = (int)lane + 32 * hf;
                    int a = h[hf];
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, a, off);
                        if ((int)lane >= off) a += y;
                    }
                    sm.H[j + 1] = a + hcarry;
                    hcarry += __shfl_sync(0xffffffffu, a, 31);
                    if (valid[hf]) {
                        const EvalRec& r = sm.ev[(b + j) & (RR - 1)];
#pragma unroll
                        for (int q = 0; q < 3; q++) {
                            const double ae = r.a[3 * q];
                            sm.inva[j][q] = ae != 0.0 ? 1.0 / ae : 0.0;
                        }
                    }
                }
                if (lane == 0) sm.H[0] = 0;
            }
            // batch = longest prefix of entries whose pairs fit in PCAP (>= 1 entry)
            int n = 0;
            bool full = true;
#pragma unroll
            for (int hf = 0; hf < NW; hf++) {
                const unsigned bm = __ballot_sync(0xffffffffu, valid[hf] && incl[hf] <= PCAP);
                if (full) n += __popc(bm);
                full = full && bm == 0xffffffffu;
            }
            n = max(n, 1);
#pragma unroll
            for (int hf = 0; hf < NW; hf++) {
                const int j = (int)lane + 32 * hf;
                const int excl = incl[hf] - w[hf] * h[hf];
                sm.S[j + 1] = incl[hf];
                const unsigned magic = w[hf] ? (32768u + (unsigned)w[hf] - 1u) / (unsigned)w[hf] : 0u;
                sm.geo[j] = (unsigned)cx0[hf] | ((unsigned)cy0[hf] << 4) | ((unsigned)w[hf] << 8) | (magic << 16);
                sm.kb[j] = make_int2(excl - cy0[hf] * w[hf] - cx0[hf], w[hf]);
            }
            if (lane == 0) {
                sm.S[0] = 0;
                sm.nb = n;
            }
        }
        __syncthreads();
        nb = sm.nb;
        {  // records of the next window [b+nb, b+nb+DB) (their ids arrived in an earlier batch)
            const int nrhi = min(b + nb + DB, e);
            for (int c = tid; c < (nrhi - rhi) * 8; c += 256) fetch_rec(rhi + (c >> 3), c & 7);
            rhi = max(rhi, nrhi);
            cp_async_commit();
        }
        if constexpr (ROWS) {
            // ---- 2. evaluate by row units (entry j, row ly): the pixels of the row with
            //         r >= r_lo form an interval (intersection of three half-planes),
            //         solved in fp64 and widened by a margin far above its rounding
            //         error; only the pixels inside are evaluated, with the exact
            //         per-pixel formula, so every decision matches the pair evaluation ----
            const int U = sm.H[nb];
            for (int u = tid; u < U; u += 256) {
                int j = 0;
#pragma unroll
                for (int step = DB / 2; step > 0; step >>= 1)
                    if (j + step < nb && sm.H[j + step] <= u) j += step;
                const unsigned g = sm.geo[j];
                const int w = (g >> 8) & 31, cx0 = g & 15, cy0 = (g >> 4) & 15;
                const int ly = cy0 + (u - sm.H[j]);
                const EvalRec& r = sm.ev[(b + j) & (RR - 1)];
                const double pcy = sm.yc[ly];
                const double rlo = r.r_lo;
                const double D0 = fma(r.a[1], pcy, r.a[2]);
                const double D1 = fma(r.a[4], pcy, r.a[5]);
                const double D2 = fma(r.a[7], pcy, r.a[8]);
                const double a0 = r.a[0], a3 = r.a[3], a6 = r.a[6];
                int xl = cx0, xr = cx0 + w - 1;
                const double xoff = (double)X0 + 0.5;
                auto clip = [&](double ae, double De, double inv) {
                    if (ae == 0.0) {
                        if (De < rlo) xr = -1;  // l_e == D_e exactly
                        return;
                    }
                    const double t = (rlo - De) * inv - xoff;  // l_e >= r_lo  <=>  x >= t (ae > 0)
                    const double eps = 1e-9 + 1e-12 * fabs(t + xoff);
                    if (ae > 0.0) {
                        const double tc = fmin(fmax(t - eps, -2.0), 18.0);  // NaN -> no bound
                        xl = max(xl, (int)ceil(tc));
                    } else {
                        const double tc = fmax(fmin(t + eps, 18.0), -2.0);
                        xr = min(xr, (int)floor(tc));
                    }
                };
                clip(a0, D0, sm.inva[j][0]);
                clip(a3, D1, sm.inva[j][1]);
                clip(a6, D2, sm.inva[j][2]);
                if (xl <= xr) {
                    const int2 kbj = sm.kb[j];
                    const double rhi = r.r_hi;
                    const unsigned bit = 1u << (j & 31);
                    unsigned* mrow = &sm.mask[j >> 5][ly * TILE];
                    float* rrow = &sm.r[kbj.x + ly * kbj.y];
                    for (int x = xl; x <= xr; x++) {
                        const double pcx = sm.xc[x];
                        const double l0 = fma(a0, pcx, D0);
                        const double l1 = fma(a3, pcx, D1);
                        const double l2 = fma(a6, pcx, D2);
                        const double m01 = l0 < l1 ? l0 : l1;
                        const double rr = m01 < l2 ? m01 : l2;
                        if (rr >= rlo) {
                            rrow[x] = rr > rhi ? (float)rr : __int_as_float(0x7fc00000);
                            atomicOr(&mrow[x], bit);
                        }
                    }
                }
            }
        } else {
        // ---- 2. evaluate: warp w takes a contiguous range of pairs, 32 consecutive
        //         pairs per step (lane-uniform control flow, broadcast record loads) ----
        {
            const int total = sm.S[nb];
            const int chunk = ((total + 255) >> 8) << 5;
            const int k0 = (int)warp * chunk;
            const int kE = min(k0 + chunk, total);
            int jb = 0;
            if (k0 < kE) {
#pragma unroll
                for (int step = DB / 2; step > 0; step >>= 1)
                    if (jb + step < nb && sm.S[jb + step] <= k0) jb += step;
            }
            for (int kb = k0; kb < kE; kb += 32) {
                const int k = kb + (int)lane;
                int sj;
                const int j = pair_step_entry(sm.S, nb, kb, jb, sj);
                if (k < kE) {
                    const unsigned g = sm.geo[j];
                    const int w = (g >> 8) & 31;
                    const int local = k - sj;
                    const int dy = (int)(((unsigned)local * (g >> 16)) >> 15);
                    const int qx = (int)(g & 15) + local - dy * w;
                    const int qy = (int)((g >> 4) & 15) + dy;
                    const double pcx = sm.xc[qx], pcy = sm.yc[qy];
                    const EvalRec& r = sm.ev[(b + j) & (RR - 1)];
                    const double l0 = fma(r.a[0], pcx, fma(r.a[1], pcy, r.a[2]));
                    const double l1 = fma(r.a[3], pcx, fma(r.a[4], pcy, r.a[5]));
                    const double l2 = fma(r.a[6], pcx, fma(r.a[7], pcy, r.a[8]));
                    const double m01 = l0 < l1 ? l0 : l1;
                    const double rr = m01 < l2 ? m01 : l2;
                    if (rr >= r.r_lo) {
                        sm.r[k] = rr > r.r_hi ? (float)rr : __int_as_float(0x7fc00000);
                        atomicOr(&sm.mask[j >> 5][qy * TILE + qx], 1u << (j & 31));
                    }
                }
            }
        }
        }
        __syncthreads();
        // ---- 3. order live pixels by pass count (descending) so the lanes of a warp
        //         composite lists of similar length ----
        int nact = 256;
        if constexpr (SORT) {
            int npass = 0;
            if (!my_done) {
#pragma unroll
                for (int w = 0; w < NW; w++) npass += __popc(sm.mask[w][tid]);
                if (npass) atomicAdd(&sm.hist[DB - npass], 1);
            }
            __syncthreads();
            // every warp scans the (DB+1)-bin histogram itself
            int hv[NW + 1], off[NW + 1], carry = 0;
#pragma unroll
            for (int hf = 0; hf <= NW; hf++) {
                const int bin = (int)lane + 32 * hf;
                hv[hf] = bin <= DB ? sm.hist[bin] : 0;
                int incl = hv[hf];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if ((int)lane >= o) incl += y;
                }
                off[hf] = incl - hv[hf] + carry;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
            nact = carry;
            const int bin = DB - npass;
            int o = 0;
#pragma unroll
            for (int hf = 0; hf <= NW; hf++) {
                const int v = __shfl_sync(0xffffffffu, off[hf], bin & 31);
                if ((bin >> 5) == hf) o = v;
            }
            if (npass) sm.perm[o + atomicAdd(&sm.cursor[bin], 1)] = tid;
            __syncthreads();
        }
        // ---- 4. composite: thread -> live pixel, passing entries in depth order ----
        if (tid < nact && (SORT || !my_done)) {
            const int pp = SORT ? sm.perm[tid] : tid;
            const int plx = pp & 15, ply = pp >> 4;
            float T = sm.T[pp], C0 = sm.C[0][pp], C1 = sm.C[1][pp], C2 = sm.C[2][pp], epsT = sm.eps[pp];
            int last = sm.last[pp], cnt = sm.cnt[pp], flag_pos = -1;
            bool stop = false;
#pragma unroll
            for (int wd = 0; wd < NW; wd++) {
                unsigned m = sm.mask[wd][pp];
                while (m) {
                    const int j = wd * 32 + __ffs(m) - 1;
                    m &= m - 1;
                    const int2 kb = sm.kb[j];
                    const float rv = sm.r[kb.x + ply * kb.y + plx];
                    if (isnan(rv)) {
                        flag_pos = b + j;
                        stop = true;
                        break;
                    }
                    const float4 col = sm.col[j];
                    const float f1 = sm.f1[j];
                    float a, ea;
                    if (mode == 0) {
                        const float lg = fast_lg2(fminf(rv, 1.f));
                        const float arg = fmaf(col.w, lg, f1);
                        a = fast_ex2(arg);
                        ea = 5e-7f + col.w * (6e-7f + 2.4e-7f * fabsf(lg)) + 1.2e-7f * fabsf(arg);
                    } else {
                        const float x = rv * col.w;
                        a = __fdividef(f1, 1.0f + fast_ex2(fminf(x, 1009.9f)));
                        ea = 8e-7f + 1.2e-7f * fabsf(x);
                    }
                    a = fminf(a, ALPHA_CLAMP_F);
                    const float wgt = T * a;
                    const float tn = fmaf(-T, a, T);
                    const float en = fmaf(ea * a, __frcp_rn(1.f - a), epsT + 2.4e-7f);
                    const float ew = epsT + ea + 1.2e-7f;
                    if (fabsf(tn - T_MIN_F) <= fmaf(2.f * en, tn, 1e-11f) ||
                        fabsf(wgt - tau) <= fmaf(2.f * ew, wgt, 1e-9f)) {
                        flag_pos = b + j;
                        stop = true;
                        break;
                    }
                    C0 = fmaf(wgt, col.x, C0);
                    C1 = fmaf(wgt, col.y, C1);
                    C2 = fmaf(wgt, col.z, C2);
                    last = b + j;
                    cnt++;
                    T = tn;
                    epsT = en;
                    red_max_shared(&sm.maxw[j], __float_as_uint(wgt));
                    if (wgt > tau) red_add_shared(&sm.pix[j], 1);
                    if (T < T_MIN_F) {
                        stop = true;
                        break;
                    }
                }
                if (stop) break;
            }
            sm.T[pp] = T;
            sm.C[0][pp] = C0;
            sm.C[1][pp] = C1;
            sm.C[2][pp] = C2;
            sm.eps[pp] = epsT;
            sm.last[pp] = last;
            sm.cnt[pp] = cnt;
            if (flag_pos >= 0) sm.flag[pp] = flag_pos;
        }
        __syncthreads();
        if (tid < nb) {
            const unsigned src = sm.srcq[(b + tid) & (SR - 1)];
            if (sm.maxw[tid] && out.max_weight) atomicMax((unsigned*)out.max_weight + src, sm.maxw[tid]);
            if (sm.pix[tid] && out.pixel_count) atomicAdd(out.pixel_count + src, sm.pix[tid]);
            sm.maxw[tid] = 0u;
            sm.pix[tid] = 0;
        }
    }
    cp_async_wait_all();
    __syncthreads();
    const int flag_pos = sm.flag[tid];
    if (flag_pos != -2) {
        const int p = (Y0 + (tid >> 4)) * cam.width + X0 + (tid & 15);
        if (flag_pos >= 0) {
            unsigned long long k = atomicAdd(&out.ctr->n_flagged, 1ull);
            out.flags[k] = make_int2(p, flag_pos);
        } else {
            const float T = sm.T[tid];
            const int last = sm.last[tid];
            if (out.image) {
                out.image[p * 3 + 0] = fminf(fmaxf(fmaf(T, (float)opt.bg[0], sm.C[0][tid]), 0.f), 1.f);
                out.image[p * 3 + 1] = fminf(fmaxf(fmaf(T, (float)opt.bg[1], sm.C[1][tid]), 0.f), 1.f);
                out.image[p * 3 + 2] = fminf(fmaxf(fmaf(T, (float)opt.bg[2], sm.C[2][tid]), 0.f), 1.f);
            }
            if (out.alpha_map) out.alpha_map[p] = 1.f - T;
            out.t_final[p] = T;
            if (out.t_final64) out.t_final64[p] = (double)T;
            out.last_pos[p] = last;
            if (out.n_frag) out.n_frag[p] = sm.cnt[tid];
            if (out.last_src) out.last_src[p] = last >= 0 ? (int)ent_src[last] : -1;
        }
    }
}

template <int DB, int PCAP, bool SORT, bool ROWS>
static void launch_dense(const Cam& cam, const Opts& opt, const RecF* rec, const int* tile_start,
                         const unsigned* ent_src, const FastBlendOut& out, cudaStream_t st) {
    const int dyn = (int)sizeof(DenseSmem<DB, PCAP>);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_blend_dense<DB, PCAP, SORT, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        attr = true;
    }
    const int ntiles = cam.ntx * cam.nty;
    k_blend_dense<DB, PCAP, SORT, ROWS><<<ntiles, 256, dyn, st>>>(cam, opt, rec, tile_start, ent_src, out);
}

void launch_blend_dense(const Cam& cam, const Opts& opt, const RecF* rec, const short4* bbox,
                        const int* tile_start, const unsigned* ent_src, const FastBlendOut& out,
                        cudaStream_t st) {
    (void)bbox;
    static const int variant = [] {
        const char* v = getenv("TS_DENSE_VARIANT");
        return v ? atoi(v) : 0;
    }();
    if (variant == 1)
        launch_dense<64, 2048, false, false>(cam, opt, rec, tile_start, ent_src, out, st);
    else if (variant == 2)
        launch_dense<32, 2048, false, false>(cam, opt, rec, tile_start, ent_src, out, st);
    else if (variant == 3)
        launch_dense<64, 4096, false, true>(cam, opt, rec, tile_start, ent_src, out, st);
    else
        launch_dense<64, 4096, false, false>(cam, opt, rec, tile_start, ent_src, out, st);
}

}  // namespace ts
