// ts_blend.cu -- forward blend (rasterize_forward, _kernels.py:59-132) as dense
// (entry, pixel) pair evaluation.
//
// CTA per 16x16 tile, 256 threads, thread = pixel for compositing.  The tile's
// entry list (depth-rank order) is consumed in batches of at most DB entries /
// PCAP pairs:
//   1. geometry  -- records arrive in a cp.async ring one batch ahead (source
//                   ids two batches ahead).  Thread (entry j = tid/4, rows
//                   4q..4q+3) clips every row of the rectangle bbox ∩ tile to
//                   the span of pixel centres that can pass r >= r_lo (three
//                   half-planes, fp64, widened by 1e-6 px: a superset of the
//                   passing pixels); pairs = pixels of the spans, numbered
//                   entry-major, row by row.  Scans over the 4 threads of an
//                   entry and over entries give the segment (entry, row) table,
//                   the batch size (<= PCAP pairs) and the pair-word tables;
//   2. evaluate  -- the batch's pairs are split over the warps, 32 consecutive
//                   pairs per step, so every lane evaluates a pixel inside its
//                   entry's bbox (the reference's per-pixel bbox test,
//                   _kernels.py:87-95, costs nothing) and near its pass
//                   region (~2.5x fewer pairs than the rectangles).  A pair whose
//                   r = phi/phi_s passes the lower end of the contribution band
//                   stores r (NaN = inside the band) and sets bit `entry` of the
//                   pixel's batch mask;
//   3. composite -- thread = pixel walks its bits in ascending entry (= depth)
//                   order, front to back; per-entry max weight / pixel count in
//                   shared memory, one global atomic per (entry, tile).
// Render forwards (ACC64 = false) composite in fp32 with the decision guard
// band of ts_fast.cu; training forwards (ACC64 = true) use the reference's
// alpha in fp64 and fp64 transmittance, so the saved T_final is the one the
// backward recursion needs.  Any undecided decision flags the pixel for the
// exact fp64 fix-up (k_fixup_fwd).
#include <type_traits>

#include "ts_kernels.cuh"

namespace ts {

namespace {
constexpr float T_MIN_F = 1e-4f;
constexpr float ALPHA_CLAMP_F = 0.99f;

// 32-bit shared-memory addressing for the compositing loop (through the
// generic struct reference the compiler rebuilds the shared window address
// every iteration)
__device__ __forceinline__ int lds_s32(unsigned a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds_f32(unsigned a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float2 lds_f32x2(unsigned a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds_f32x4(unsigned a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void red_s_max(unsigned a, unsigned v) {
    asm volatile("red.shared.max.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_s_add(unsigned a, int v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
}  // namespace

template <int DB, int PCAP, bool ACC64>
struct DenseSmem {
    static constexpr int RR = 2 * DB, SR = 4 * DB, NW = DB / 32;
    using Real = typename std::conditional<ACC64, double, float>::type;
    EvalRec ev[RR];
    TailRec tail[RR];
    RecC rc[ACC64 ? RR : 1];       // training forwards: fp64 colour, opacity, sigma of the ring slots
    Real r[PCAP];                  // per pair: render: alpha (clamped); training: r; NaN = inside the band
    float2 eq[ACC64 ? 1 : PCAP];   // render: relative error increments of the fp32 weight and transmittance
    unsigned mask[NW][256];        // per pixel: bit j = entry j passes (r >= r_lo)
    unsigned srcq[SR];
    float4 col[DB];                // rgb, f0
    float f1[DB];
    unsigned seg[DB * TILE];       // segment s (one row of one entry): first pair | j<<13 | row<<19 | xa<<23
    int rowtab[DB][TILE];          // row ly of entry j: its first pair minus its first column (pair = rowtab + lx)
    unsigned starts[PCAP / 32];    // bit (k & 31) of word k >> 5: a segment starts at pair k
    int jfirst[PCAP / 32];         // segment holding pair 32 w
    unsigned ein[DB];              // per entry: inclusive (pairs<<16 | segments) within its warp
    __align__(16) unsigned wtot[8];  // per warp: (pairs<<16 | segments) of its 8 entries
    int total;                     // pairs of the batch
    unsigned pbits[ACC64 ? PCAP / 32 : 1];      // training: pair k passes (the others' record slots are holes)
    unsigned long long rbase;                   // first record of the batch (~0: none)
    unsigned maxw[DB];
    int pix[DB];
    double xc[TILE], yc[TILE];     // pixel centres of the tile (fp64)
};

template <int DB, int PCAP, bool ACC64, int MINB>
__global__ void __launch_bounds__(256, MINB) k_blend_dense(Cam cam, Opts opt, const RecF* __restrict__ rec,
                                                     const int* __restrict__ tile_start,
                                                     const unsigned* __restrict__ ent_src, FastBlendOut out) {
    TS_PDL_ENTRY();
    using SM = DenseSmem<DB, PCAP, ACC64>;
    using Real = typename SM::Real;
    constexpr int RR = SM::RR, SR = SM::SR, NW = SM::NW;
    extern __shared__ __align__(16) unsigned char s_dyn[];
    SM& sm = *reinterpret_cast<SM*>(s_dyn);

    const int tid = threadIdx.x;
    const unsigned lane = tid & 31, warp = tid >> 5;
    const int t = out.tile_order ? __ldg(out.tile_order + blockIdx.x) : (int)blockIdx.x;
    const int tx = t % cam.ntx, ty = t / cam.ntx;
    const int X0 = tx * TILE, Y0 = ty * TILE;
    const int lx = tid & 15, ly = tid >> 4;
    const int px = X0 + lx, py = Y0 + ly;
    const bool inside = px < cam.width && py < cam.height;
    const int s = tile_start[t], e = tile_start[t + 1];
    const float tau = (float)opt.tau_contrib;
    const int mode = opt.mode;
    // per-pixel compositing state (thread = pixel)
    Real T = 1, C0 = 0, C1 = 0, C2 = 0;
    float epsT = 0.f;  // relative error bound of the fp32 transmittance
    int last = -1, cnt = 0, flag_pos = -1;
    bool done = !inside;
    long long fbase = 0;  // collect_fragments: the pixel's first CSR slot
    if constexpr (ACC64)
        if (out.frag_tri && inside) fbase = out.frag_off[py * cam.width + px];
    if (tid < DB) {
        sm.maxw[tid] = 0u;
        sm.pix[tid] = 0;
    }
    if (tid < TILE) sm.xc[tid] = (double)(X0 + tid) + 0.5;
    else if (tid < 2 * TILE) sm.yc[tid - TILE] = (double)(Y0 + tid - TILE) + 0.5;
    auto fetch_rec = [&](int p, int q) {  // 16-byte chunk q of the record at list position p
        const unsigned src = sm.srcq[p & (SR - 1)];
        const float4* g = reinterpret_cast<const float4*>(rec + src) + q;
        const int slot = p & (RR - 1);
        if (q < 6) cp_async16(reinterpret_cast<float4*>(&sm.ev[slot]) + q, g);
        else cp_async16(reinterpret_cast<float4*>(&sm.tail[slot]) + (q - 6), g);
        if constexpr (ACC64) {
            if (q < 3) cp_async16(reinterpret_cast<double2*>(&sm.rc[slot]) + q, reinterpret_cast<const double2*>(out.recc + src) + q);
        }
    };
    // prologue: ids of [s, s+3DB), then records of [s, s+DB)
    int shi = min(s + 3 * DB, e), rhi = min(s + DB, e);
    for (int p = s + tid; p < shi; p += 256) cp_async4(&sm.srcq[p & (SR - 1)], ent_src + p);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    for (int c = tid; c < (rhi - s) * 8; c += 256) fetch_rec(s + (c >> 3), c & 7);
    cp_async_commit();
    if (tid < PCAP / 32) sm.starts[tid] = 0u;
    int nb = 0, pb = 0, pnb = 0;  // (pb, pnb): previous batch, statistics not yet flushed
    for (int b = s; b < e; b += nb) {
        cp_async_wait_all();
        if (__syncthreads_count(!done) == 0) break;
        const int navail = min(DB, e - b);
        if (tid < pnb) {  // per-entry statistics of the previous batch (complete since the barrier)
            const unsigned src = sm.srcq[(pb + tid) & (SR - 1)];
            if (sm.maxw[tid] && out.max_weight) red_gmax_u32((unsigned*)out.max_weight + src, sm.maxw[tid]);
            if (sm.pix[tid] && out.pixel_count) red_gadd_s32(out.pixel_count + src, sm.pix[tid]);
            sm.maxw[tid] = 0u;
            sm.pix[tid] = 0;
        }
        {  // ids two batches ahead
            const int nshi = min(b + 3 * DB, e);
            for (int p = shi + tid; p < nshi; p += 256) cp_async4(&sm.srcq[p & (SR - 1)], ent_src + p);
            shi = max(shi, nshi);
        }
        // ---- 1. geometry: thread (entry j, rows 4q..4q+3); clear the masks ----
        static_assert(DB == 64 && PCAP <= 8192, "geometry layout: 4 threads per entry, 13-bit pair ids");
#pragma unroll
        for (int w = 0; w < NW; w++) sm.mask[w][tid] = 0u;
        {
            const int j = tid >> 2, q = tid & 3;
            const bool vj = j < navail;
            const int slot = (b + j) & (RR - 1);
            // rows cy0 + q + 4m of the rectangle (strided: the 4 threads share its rows evenly)
            int xa[4], len[4], cy0 = 0;
#pragma unroll
            for (int m = 0; m < 4; m++) xa[m] = len[m] = 0;
            if (vj) {
                const float4 t0 = reinterpret_cast<const float4*>(&sm.tail[slot])[0];
                const int4 t1 = reinterpret_cast<const int4*>(&sm.tail[slot])[1];
                const int bx0 = (short)(t1.y & 0xffff), bx1 = (short)(t1.y >> 16);
                const int by0 = (short)(t1.z & 0xffff), by1 = (short)(t1.z >> 16);
                const int cx0 = max(bx0 - X0, 0), cx1 = min(bx1 - X0, TILE) - 1;
                cy0 = max(by0 - Y0, 0);
                const int cy1 = min(by1 - Y0, TILE) - 1;
                if (q == 0) {
                    sm.col[j] = make_float4(t0.z, t0.w, __int_as_float(t1.x), t0.x);
                    sm.f1[j] = t0.y;
                }
                if (cy0 + q <= cy1 && cx0 <= cx1) {
                    const EvalRec& R = sm.ev[slot];
                    const double rlo = R.r_lo, xl = sm.xc[0], y0 = sm.yc[cy0 + q];
                    // per edge, the bound on the tile-local pixel index is linear in the
                    // row: lx >= / <= tb0 + m * sl (a0 > 0 / < 0) with tb0 = (r_lo -
                    // l(xl, y0)) / a0 and sl the change per 4 rows, in fp32 with a margin
                    // covering the fp32 rounding (1e-3 px + 2^-20 of the magnitudes);
                    // edges with |a0| tiny or a0 == 0 do not narrow the rows
                    // (a superset of the passing pixels either way)
                    float tb0[3], sl[3], mg[3];
                    bool up[3], dn[3];
#pragma unroll
                    for (int ed = 0; ed < 3; ed++) {
                        const double a0 = R.a[3 * ed], a1 = R.a[3 * ed + 1];
                        const double n0 = rlo - fma(a0, xl, fma(a1, y0, R.a[3 * ed + 2]));
                        const float inv = rcp_approx((float)a0);  // (1 ulp; |a0| < 2^-126: inf, not finite)
                        tb0[ed] = (float)n0 * inv;
                        sl[ed] = (float)(-4.0 * a1) * inv;
                        const bool fin = fabsf(inv) < 1e30f && fabsf(tb0[ed]) < 1e6f && fabsf(sl[ed]) < 1e4f;
                        mg[ed] = 1e-3f + 9.6e-7f * (fabsf(tb0[ed]) + 4.f * fabsf(sl[ed]));
                        up[ed] = a0 > 0.0 && fin;
                        dn[ed] = a0 < 0.0 && fin;
                    }
                    const int nrow = (cy1 - cy0 - q) / 4 + 1;
#pragma unroll
                    for (int m = 0; m < 4; m++) {
                        if (m >= nrow) break;
                        int lo = cx0, hi = cx1;
#pragma unroll
                        for (int ed = 0; ed < 3; ed++) {
                            const float tb = fminf(fmaxf(fmaf((float)m, sl[ed], tb0[ed]), -64.f), 64.f);
                            lo = up[ed] ? max(lo, __float2int_ru(tb - mg[ed])) : lo;
                            hi = dn[ed] ? min(hi, __float2int_rd(tb + mg[ed])) : hi;
                        }
                        xa[m] = lo;
                        len[m] = max(hi - lo + 1, 0);
                    }
                }
            }
            // row-major pair / segment numbering within the entry: row cy0 + q + 4m
            // follows all rows of levels < m and the rows of level m with smaller q
            unsigned lev[4], exl[4];
#pragma unroll
            for (int m = 0; m < 4; m++) {
                const unsigned vm = ((unsigned)len[m] << 16) | (unsigned)(len[m] > 0);
                unsigned x = vm;
                const unsigned y1 = __shfl_up_sync(0xffffffffu, x, 1);
                if (q >= 1) x += y1;
                const unsigned y2 = __shfl_up_sync(0xffffffffu, x, 2);
                if (q >= 2) x += y2;
                exl[m] = x - vm;
                lev[m] = __shfl_sync(0xffffffffu, x, (int)lane | 3);
            }
            const unsigned et = lev[0] + lev[1] + lev[2] + lev[3];  // entry total (pairs<<16 | segments)
            // scans: entries within the warp, warps
            unsigned ei = et;
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, ei, off);
                if ((int)lane >= off) ei += y;
            }
            if (q == 0) sm.ein[j] = ei;
            if (lane == 31) sm.wtot[warp] = ei;
            __syncthreads();
            unsigned wpre = 0, all = 0;
            {
                const uint4 wa = reinterpret_cast<const uint4*>(sm.wtot)[0];
                const uint4 wb = reinterpret_cast<const uint4*>(sm.wtot)[1];
                const unsigned wt[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
                for (int w2 = 0; w2 < 8; w2++) {
                    wpre += w2 < (int)warp ? wt[w2] : 0u;
                    all += wt[w2];
                }
            }
            // batch = longest prefix of entries whose pairs fit in PCAP (>= 1 entry)
            int n = 0;
            {
                if ((all >> 16) <= (unsigned)PCAP) {
                    n = navail;
                } else {
                    unsigned cum = 0;
                    for (int w2 = 0; w2 < 8; w2++) {
                        const unsigned wt = sm.wtot[w2];
                        if (((cum + wt) >> 16) <= (unsigned)PCAP && (w2 + 1) * 8 <= navail) {
                            cum += wt;
                            n += 8;
                            continue;
                        }
                        for (int u = 0; u < 8; u++) {
                            const int jj = w2 * 8 + u;
                            if (jj >= navail || ((cum + sm.ein[jj]) >> 16) > (unsigned)PCAP) break;
                            n++;
                        }
                        break;
                    }
                    n = max(n, 1);
                }
            }
            nb = n;
            if (j < n) {
                unsigned base = wpre + ei - et;  // the entry's first (pair, segment)
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    if (len[m] > 0) {
                        const int ly2 = cy0 + q + 4 * m;
                        const unsigned pm = base + exl[m];
                        const unsigned P0 = pm >> 16, S0 = pm & 0xffffu;
                        TS_ASSERT(P0 + (unsigned)len[m] <= (unsigned)PCAP && S0 < (unsigned)(DB * TILE) && ly2 < TILE);
                        sm.rowtab[j][ly2] = (int)P0 - xa[m];
                        sm.seg[S0] = P0 | ((unsigned)j << 13) | ((unsigned)ly2 << 19) | ((unsigned)xa[m] << 23);
                        atomicOr(&sm.starts[P0 >> 5], 1u << (P0 & 31));
                        // a segment (<= 16 pairs) holds at most one word start
                        const unsigned wq = (P0 + 31) >> 5;
                        if ((wq << 5) <= P0 + (unsigned)len[m] - 1u) {
                            TS_ASSERT(wq < (unsigned)(PCAP / 32));
                            sm.jfirst[wq] = (int)S0;
                        }
                    }
                    base += lev[m];
                }
                if (j == n - 1 && q == 0) sm.total = (int)((wpre + ei) >> 16);
            }
        }
        __syncthreads();
        {  // records of the next window [b+nb, b+nb+DB) (their ids arrived in an earlier batch)
            const int nrhi = min(b + nb + DB, e);
            for (int c = tid; c < (nrhi - rhi) * 8; c += 256) fetch_rec(rhi + (c >> 3), c & 7);
            rhi = max(rhi, nrhi);
            cp_async_commit();
        }
        // ---- 2. evaluate: warp w takes a contiguous range of pairs, 32 consecutive
        //         pairs per step (lane-uniform control flow, broadcast record loads) ----
        // training records: one slot per pair of the batch (record of pair k at
        // rbase + k; pairs that fail the test -- ~0.1 % -- become holes), reserved
        // here so the atomic's round trip overlaps the evaluation
        unsigned long long rb_res = 0;
        if constexpr (ACC64)
            if (out.frec && tid == 0) rb_res = atomicAdd(&out.ctr->n_frec, (unsigned long long)sm.total);
        {
            const int total = sm.total;
            const int chunk = ((total + 255) >> 8) << 5;
            const int k0 = (int)warp * chunk;
            const int kE = min(k0 + chunk, total);
            for (int kb = k0; kb < kE; kb += 32) {
                const int k = kb + (int)lane;
                bool pass = false;
                // segment of pair k: the word's first segment plus the segment starts in (kb, k]
                const int sk = sm.jfirst[kb >> 5] + __popc(sm.starts[kb >> 5] & ((2u << lane) - 2u));
                if (k < kE) {
                    const unsigned sg = sm.seg[sk];
                    const int j = (int)((sg >> 13) & 63u);
                    const int qx = (int)(sg >> 23) + k - (int)(sg & 0x1fffu);
                    const int qy = (int)((sg >> 19) & 15u);
                    const double pcx = sm.xc[qx], pcy = sm.yc[qy];
                    const EvalRec& r = sm.ev[(b + j) & (RR - 1)];
                    const double l0 = fma(r.a[0], pcx, fma(r.a[1], pcy, r.a[2]));
                    const double l1 = fma(r.a[3], pcx, fma(r.a[4], pcy, r.a[5]));
                    const double l2 = fma(r.a[6], pcx, fma(r.a[7], pcy, r.a[8]));
                    const double m01 = l0 < l1 ? l0 : l1;
                    const double rr = m01 < l2 ? m01 : l2;
                    pass = rr >= r.r_lo;
                    if (pass) {
                        if constexpr (ACC64) {
                            sm.r[k] = rr > r.r_hi ? (Real)rr : (Real)__int_as_float(0x7fc00000);
                        } else {
                            // render: the fp32 alpha and its error bound here, densely
                            // (not in the per-pixel compositing loop)
                            float a = __int_as_float(0x7fc00000), ea = 0.f;
                            if (rr > r.r_hi) {
                                const float rv = (float)rr;
                                const float4 col = sm.col[j];
                                const float f1 = sm.f1[j];
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
                            }
                            sm.r[k] = a;
                            // error increments of the weight T a (ea + 1.2e-7) and of the
                            // transmittance T (1 - a) (ea a / (1 - a) + 2.4e-7; 1 - a >= 0.01)
                            sm.eq[k] = make_float2(ea + 1.2e-7f, fmaf(ea * a, rcp_approx(1.f - a), 2.4e-7f));
                        }
                        atomicOr(&sm.mask[j >> 5][qy * TILE + qx], 1u << (j & 31));
                    }
                }
                if constexpr (ACC64) {
                    const unsigned pb = __ballot_sync(0xffffffffu, pass);
                    if (lane == 0) sm.pbits[kb >> 5] = pb;
                }
            }
        }
        if constexpr (ACC64) {
            if (out.frec && tid == 0) {
                unsigned long long base = rb_res;
                if (base + (unsigned long long)sm.total > out.frec_cap) {
                    out.ctr->frec_over = 1ull;
                    base = ~0ull;
                }
                sm.rbase = base;
            }
        }
        __syncthreads();
        if (tid < PCAP / 32) sm.starts[tid] = 0u;  // for the next batch (read by the evaluation only)
        if constexpr (ACC64) {
            // the slots of pairs that failed the contribution test are holes
            if (out.frec && sm.rbase != ~0ull) {
                const int total = sm.total;
                for (int wi = tid; wi < ((total + 31) >> 5); wi += 256) {
                    const int nv = min(32, total - 32 * wi);
                    unsigned miss = ~sm.pbits[wi] & (nv == 32 ? 0xffffffffu : ((1u << nv) - 1u));
                    while (miss) {
                        const int k = 32 * wi + __ffs(miss) - 1;
                        miss &= miss - 1;
                        out.frec[sm.rbase + k].pix = ~0u;
                    }
                }
            }
        }
        // ---- 3. composite: thread = pixel, passing entries in depth order ----
        static_assert(NW <= 2, "64-bit pixel masks");
        unsigned long long mm = sm.mask[0][tid];
        if constexpr (NW == 2) mm |= (unsigned long long)sm.mask[1][tid] << 32;
        unsigned long long rb = ~0ull;
        if constexpr (ACC64)
            if (out.frec) rb = sm.rbase;
        // training records: passing pairs this pixel does not composite are holes
        auto mark_holes = [&](unsigned long long hm) {
            while (hm) {
                const int j = __ffsll((long long)hm) - 1;
                hm &= hm - 1;
                const int kh = sm.rowtab[j][ly] + lx;
                const int slot = kh;
                TS_ASSERT(kh >= 0 && kh < sm.total && rb + slot < out.frec_cap);
                out.frec[rb + slot].pix = ~0u;
            }
        };
        if constexpr (!ACC64) {
            // render: walk the two mask words; 32-bit shared addressing
            if (!done) {
                const unsigned sb = (unsigned)__cvta_generic_to_shared(s_dyn);
                const unsigned s_rt = sb + (unsigned)offsetof(SM, rowtab) + 4u * (unsigned)ly;
                const unsigned s_r = sb + (unsigned)offsetof(SM, r), s_eq = sb + (unsigned)offsetof(SM, eq);
                const unsigned s_col = sb + (unsigned)offsetof(SM, col);
                const unsigned s_mw = sb + (unsigned)offsetof(SM, maxw), s_px = sb + (unsigned)offsetof(SM, pix);
                unsigned w = (unsigned)mm, w1 = (unsigned)(mm >> 32);
                int jb = 0;
                while (true) {
                    if (w == 0) {
                        if (jb != 0 || w1 == 0) break;
                        w = w1;
                        jb = 32;
                    }
                    const int j = jb + __ffs(w) - 1;
                    w &= w - 1;
                    const int kp = lds_s32(s_rt + 64u * (unsigned)j) + lx;
                    TS_ASSERT(kp >= 0 && kp < sm.total && ((sm.mask[j >> 5][tid] >> (j & 31)) & 1u));
                    const float a = lds_f32(s_r + 4u * (unsigned)kp);  // alpha (clamped); NaN = in the band
                    if (isnan(a)) {
                        flag_pos = b + j;
                        done = true;
                        break;
                    }
                    const float2 eq = lds_f32x2(s_eq + 8u * (unsigned)kp);
                    const float wgt = T * a;
                    const float tn = fmaf(-T, a, T);
                    // relative error bounds of tn and of wgt (the tests keep a 2x margin)
                    const float en = epsT + eq.y, ew = epsT + eq.x;
                    if (fabsf(tn - T_MIN_F) <= fmaf(2.f * en, tn, 1e-11f) ||
                        fabsf(wgt - tau) <= fmaf(2.f * ew, wgt, 1e-9f)) {
                        flag_pos = b + j;
                        done = true;
                        break;
                    }
                    const float4 col = lds_f32x4(s_col + 16u * (unsigned)j);
                    C0 = fmaf(wgt, col.x, C0);
                    C1 = fmaf(wgt, col.y, C1);
                    C2 = fmaf(wgt, col.z, C2);
                    last = b + j;
                    cnt++;
                    T = tn;
                    epsT = en;
                    if (wgt > tau) red_s_add(s_px + 4u * (unsigned)j, 1);
                    red_s_max(s_mw + 4u * (unsigned)j, __float_as_uint(wgt));
                    if (T < T_MIN_F) {
                        done = true;
                        break;
                    }
                }
            }
        } else
        if (done) {
            if (rb != ~0ull) mark_holes(mm);
        } else {
            {
                while (mm) {
                    const int j = __ffsll((long long)mm) - 1;
                    mm &= mm - 1;
                    const int kp = sm.rowtab[j][ly] + lx;
                    TS_ASSERT(kp >= 0 && kp < sm.total && ((sm.mask[j >> 5][tid] >> (j & 31)) & 1u));
                const Real rv = sm.r[kp];
                    if (isnan(rv)) {  // r inside the contribution band
                        flag_pos = b + j;
                        done = true;
                        mm |= 1ull << j;
                        break;
                    }
                    const float4 col = sm.col[j];
                    float wout;
                    if constexpr (ACC64) {
                        // the reference's alpha (_kernels.py:43-56) and transmittance in fp64
                        const RecC& rcj = sm.rc[(b + j) & (RR - 1)];
                        const double2 os = make_double2(rcj.opa, rcj.sig);
                        double a;
                        if (mode == 0) {
                            const double rc = fmin((double)rv, 1.0);
                            a = os.x * (os.y == 1.0 ? rc : pow(rc, os.y));
                        } else {
                            double x = (double)rv * sm.ev[(b + j) & (RR - 1)].phis / os.y;
                            if (x > 700.0) x = 700.0;
                            a = os.x * (1.0 / (1.0 + exp(x)));
                        }
                        if (a > ALPHA_CLAMP) a = ALPHA_CLAMP;
                        const double wd64 = __dmul_rn(T, a);
                        const double tn = __dmul_rn(T, __dsub_rn(1.0, a));
                        // r differs from the reference's by ~1e-13 relative
                        if (fabs(tn - T_MIN) <= 1e-9 * tn || fabs(wd64 - opt.tau_contrib) <= 1e-9 * wd64) {
                            flag_pos = b + j;
                            done = true;
                            mm |= 1ull << j;
                            break;
                        }
                        if (rb != ~0ull) {
                            const int kr = kp;
                            const int slot = kr;
                            TS_ASSERT(rb + slot < out.frec_cap);
                            double4* fr = reinterpret_cast<double4*>(out.frec + rb + slot);
                            fr[0] = make_double4((double)T, (double)C0, (double)C1, (double)C2);
                            reinterpret_cast<uint4*>(fr + 1)[0] =
                                make_uint4((unsigned)(py * cam.width + px), sm.srcq[(b + j) & (SR - 1)], (unsigned)cnt, 0u);
                        }
                        if (out.frag_tri) {  // collect_fragments: fragment cnt of this pixel's CSR list
                            const long long fi = fbase + cnt;
                            const unsigned src = sm.srcq[(b + j) & (SR - 1)];
                            out.frag_tri[fi] = (int)src;
                            out.frag_w[fi] = wd64;
                            out.frag_z[fi] = __longlong_as_double((long long)__ldg(out.zkey + src));
                        }
                        C0 += wd64 * rcj.rgb[0];
                        C1 += wd64 * rcj.rgb[1];
                        C2 += wd64 * rcj.rgb[2];
                        last = b + j;
                        cnt++;
                        T = tn;
                        wout = (float)wd64;
                        if (wd64 > opt.tau_contrib) red_add_shared(&sm.pix[j], 1);
                    } else {
                        const float a = (float)rv;  // alpha of the evaluation (clamped)
                        const float wgt = T * a;
                        const float tn = fmaf(-T, a, T);
                        // relative error bounds of tn and of wgt (the tests keep a 2x margin)
                        const float2 eq = sm.eq[kp];
                        const float en = epsT + eq.y, ew = epsT + eq.x;
                        if (fabsf(tn - T_MIN_F) <= fmaf(2.f * en, tn, 1e-11f) ||
                            fabsf(wgt - tau) <= fmaf(2.f * ew, wgt, 1e-9f)) {
                            flag_pos = b + j;
                            done = true;
                            break;
                        }
                        C0 = fmaf(wgt, col.x, C0);
                        C1 = fmaf(wgt, col.y, C1);
                        C2 = fmaf(wgt, col.z, C2);
                        last = b + j;
                        cnt++;
                        T = tn;
                        epsT = en;
                        wout = wgt;
                        if (wgt > tau) red_add_shared(&sm.pix[j], 1);
                    }
                    red_max_shared(&sm.maxw[j], __float_as_uint(wout));
                    if (T < (Real)T_MIN) {
                        done = true;
                        break;
                    }
                }
            }
            if (done && rb != ~0ull) mark_holes(mm);
        }
        pb = b;
        pnb = nb;
    }
    __syncthreads();
    if (tid < pnb) {
        const unsigned src = sm.srcq[(pb + tid) & (SR - 1)];
        if (sm.maxw[tid] && out.max_weight) red_gmax_u32((unsigned*)out.max_weight + src, sm.maxw[tid]);
        if (sm.pix[tid] && out.pixel_count) red_gadd_s32(out.pixel_count + src, sm.pix[tid]);
    }
    cp_async_wait_all();
    if (inside) {
        const int p = py * cam.width + px;
        if (flag_pos >= 0) {
            unsigned long long k = atomicAdd(&out.ctr->n_flagged, 1ull);
            out.flags[k] = make_int2(p, flag_pos);  // (pixel >= 0: the entry is published)
            __threadfence();
        } else {
            if (out.image) {
                out.image[p * 3 + 0] = (float)fmin(fmax(C0 + T * (Real)opt.bg[0], (Real)0), (Real)1);
                out.image[p * 3 + 1] = (float)fmin(fmax(C1 + T * (Real)opt.bg[1], (Real)0), (Real)1);
                out.image[p * 3 + 2] = (float)fmin(fmax(C2 + T * (Real)opt.bg[2], (Real)0), (Real)1);
            }
            if (out.alpha_map) out.alpha_map[p] = (float)(1 - T);
            out.t_final[p] = (float)T;
            if (out.t_final64) out.t_final64[p] = (double)T;
            if (out.c_total64) {
                out.c_total64[p * 3 + 0] = (double)C0 + (double)T * opt.bg[0];
                out.c_total64[p * 3 + 1] = (double)C1 + (double)T * opt.bg[1];
                out.c_total64[p * 3 + 2] = (double)C2 + (double)T * opt.bg[2];
            }
            out.last_pos[p] = last;
            if (out.n_frag) out.n_frag[p] = cnt;
            if (out.last_src) out.last_src[p] = last >= 0 ? (int)ent_src[last] : -1;
        }
    }
    // this tile's flags are published: count the CTA (k_fixup_fwd ends when all have)
    __syncthreads();
    if (tid == 0) atomicAdd(&out.ctr->blend_done, 1ull);
}

template <int DB, int PCAP, bool ACC64, int MINB>
static void launch_dense(const Cam& cam, const Opts& opt, const RecF* rec, const int* tile_start,
                         const unsigned* ent_src, const FastBlendOut& out, cudaStream_t st) {
    const int dyn = (int)sizeof(DenseSmem<DB, PCAP, ACC64>);
    smem_optin((const void*)k_blend_dense<DB, PCAP, ACC64, MINB>, dyn);
    launch_pdl(k_blend_dense<DB, PCAP, ACC64, MINB>, dim3(cam.ntx * cam.nty), dim3(256), dyn, st, cam, opt, rec,
               tile_start, ent_src, out);
}

// render forwards (fp32 compositing with the guard band) and training forwards
// (fp64 alpha / transmittance with the RecC colours, fragment records): 4 CTAs
// per SM (64 registers, no spills; 5 at 48 registers spill)
void launch_blend_dense(const Cam& cam, const Opts& opt, bool acc64, const RecF* rec, const int* tile_start,
                        const unsigned* ent_src, const FastBlendOut& out, cudaStream_t st) {
    if (acc64) launch_dense<64, 2048, true, 4>(cam, opt, rec, tile_start, ent_src, out, st);
    else launch_dense<64, 2048, false, 4>(cam, opt, rec, tile_start, ent_src, out, st);
}

}  // namespace ts
