// ts_bwd.cu -- dense backward blend (rasterize_backward, _kernels.py:181-318).
//
// CTA per 16x16 tile, 256 threads, thread = pixel for the per-pixel pass.
// The tile's entry list is walked BACK TO FRONT from the largest saved last
// contributor of the tile, in batches of at most DB entries / PCAP pairs:
//   1. stage    -- records (evaluation part, tail, backward record) arrive in a
//                  cp.async ring one batch ahead; warp 0 builds the rectangles
//                  bbox ∩ tile and their pair scan, entry jj of the batch being
//                  list position bend-1-jj (so ascending bits = back to front);
//   2. evaluate -- the batch's (entry, pixel) pairs are split over the warps,
//                  32 consecutive pairs per step; a pair at or before the
//                  pixel's last contributor (_kernels.py:226-243) with
//                  r >= r_lo sets the pixel's bit and stores r (fp32, argmax
//                  edge in the two low mantissa bits; NaN = contribution band);
//   3. per pixel -- the pixel walks its bits back to front with the
//                  reference's recursion (_kernels.py:245-318): T_k from the
//                  saved T_final, suffix colour S, dL/dalpha, the window and
//                  edge-chain derivatives (fp64 where they cancel), and adds
//                  the 12 screen-space gradients of the fragment to per-entry
//                  shared accumulators;
//   4. flush    -- one fp64 global atomic per (entry, component) and tile.
#include "ts_kernels.cuh"

namespace ts {

template <int DB, int PCAP, int GCAP>
struct BwdSmem {
    static constexpr int RR = 2 * DB, SR = 4 * DB, NW = DB / 32;
    EvalRec ev[RR];
    TailRec tail[RR];
    RecB rb[RR];
    float r[PCAP];               // per pair: r (edge in the low 2 bits); NaN = inside the band
    unsigned mask[NW][256];      // per pixel: bit jj = entry jj contributes
    unsigned srcq[SR];
    float4 col[DB];              // rgb, f0
    float4 par[DB];              // opacity, sigma, 1/opacity, 1/phi_s
    float f1[DB];
    int S[DB + 1];
    unsigned geo[DB];
    int2 kb[DB];
    double g[GCAP][13];          // per contributing pair (entry-major rank): 12 screen-space gradients
    unsigned pbits[PCAP / 32];   // pair k contributes
    int wpre[PCAP / 32 + 1];     // contributing pairs before word w
    double xc[TILE], yc[TILE];
    int last[256];
    int nb, np, hi;
};

template <int DB, int PCAP, int GCAP>
__global__ void __launch_bounds__(256, 2) k_blend_bwd_dense(Cam cam, Opts opt, const RecF* __restrict__ rec,
                                                         const RecB* __restrict__ recb,
                                                         const int* __restrict__ tile_start,
                                                         const unsigned* __restrict__ ent_src,
                                                         const double* __restrict__ t_final,
                                                         const int* __restrict__ last_pos,
                                                         const float* __restrict__ d_image,
                                                         const int* __restrict__ n_frag,
                                                         const long long* __restrict__ frag_off,
                                                         const double* __restrict__ fg_dw,
                                                         const double* __restrict__ fg_dz,
                                                         double* __restrict__ sgrad) {
    using SM = BwdSmem<DB, PCAP, GCAP>;
    constexpr int RR = SM::RR, SR = SM::SR, NW = SM::NW;
    extern __shared__ __align__(16) unsigned char s_dyn[];
    SM& sm = *reinterpret_cast<SM*>(s_dyn);

    const int tid = threadIdx.x;
    const unsigned lane = tid & 31, warp = tid >> 5;
    const int t = blockIdx.x;
    const int tx = t % cam.ntx, ty = t / cam.ntx;
    const int X0 = tx * TILE, Y0 = ty * TILE;
    const int lx = tid & 15, ly = tid >> 4;
    const int px = X0 + lx, py = Y0 + ly;
    const bool inside = px < cam.width && py < cam.height;
    const int s = tile_start[t];
    const int mode = opt.mode;
    // per-pixel state (the pixel stays with its thread)
    int my_last = -1;
    double T = 1.0, S0 = 0.0, S1 = 0.0, S2 = 0.0;
    double d0 = 0.0, d1 = 0.0, d2 = 0.0;
    // upstream fragment gradients (backward.py:122-142): fragment k of the pixel
    // is fg_*[fbase + k], visited back to front
    const bool has_fg = fg_dw != nullptr;
    const int NC = has_fg ? 13 : 12;
    long long fbase = 0;
    int fk = -1;
    double sw = 0.0;
    if (inside) {
        const int p = py * cam.width + px;
        if (has_fg) {
            fbase = frag_off[p];
            fk = n_frag[p] - 1;
        }
        my_last = last_pos[p];
        T = t_final[p];
        d0 = d_image[p * 3 + 0];
        d1 = d_image[p * 3 + 1];
        d2 = d_image[p * 3 + 2];
    }
    S0 = T * opt.bg[0];
    S1 = T * opt.bg[1];
    S2 = T * opt.bg[2];
    sm.last[tid] = my_last;
    if (tid < TILE) sm.xc[tid] = (double)(X0 + tid) + 0.5;
    else if (tid < 2 * TILE) sm.yc[tid - TILE] = (double)(Y0 + tid - TILE) + 0.5;
    if (tid == 0) sm.hi = -1;
    __syncthreads();
    if (my_last >= 0) atomicMax(&sm.hi, my_last);
    __syncthreads();
    const int hi = sm.hi;
    if (hi < s) return;

    auto fetch_rec = [&](int p, int q) {  // 16-byte chunk q of (RecF, RecB) at list position p
        const unsigned src = sm.srcq[p & (SR - 1)];
        const int slot = p & (RR - 1);
        if (q < 6)
            cp_async16(reinterpret_cast<float4*>(&sm.ev[slot]) + q, reinterpret_cast<const float4*>(rec + src) + q);
        else if (q < 8)
            cp_async16(reinterpret_cast<float4*>(&sm.tail[slot]) + (q - 6),
                       reinterpret_cast<const float4*>(rec + src) + q);
        else
            cp_async16(reinterpret_cast<float4*>(&sm.rb[slot]) + (q - 8),
                       reinterpret_cast<const float4*>(recb + src) + (q - 8));
    };
    // prologue: ids of [hi+1-3DB, hi], then records of [hi+1-DB, hi]
    int slo = max(s, hi + 1 - 3 * DB), rlo = max(s, hi + 1 - DB);
    for (int p = slo + tid; p <= hi; p += 256) cp_async4(&sm.srcq[p & (SR - 1)], ent_src + p);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    for (int c = tid; c < (hi + 1 - rlo) * 16; c += 256) fetch_rec(rlo + (c >> 4), c & 15);
    cp_async_commit();

    int nb = 0;
    for (int bend = hi + 1; bend > s; bend -= nb) {
        cp_async_wait_all();
        __syncthreads();
        const int navail = min(DB, bend - s);
        {  // ids two batches ahead (lower positions)
            const int nslo = max(s, bend - 3 * DB);
            for (int p = nslo + tid; p < slo; p += 256) cp_async4(&sm.srcq[p & (SR - 1)], ent_src + p);
            slo = min(slo, nslo);
        }
        // ---- 1. rectangles + pair scan (warp 0); entry jj <-> position bend-1-jj ----
#pragma unroll
        for (int w = 0; w < NW; w++) sm.mask[w][tid] = 0u;
        if (warp == 0) {
            int cx0[NW], cy0[NW], w[NW], h[NW], incl[NW];
            bool valid[NW];
            int carry = 0;
#pragma unroll
            for (int hf = 0; hf < NW; hf++) {
                const int jj = (int)lane + 32 * hf;
                valid[hf] = jj < navail;
                cx0[hf] = cy0[hf] = w[hf] = h[hf] = 0;
                if (valid[hf]) {
                    const int slot = (bend - 1 - jj) & (RR - 1);
                    const float4 t0 = reinterpret_cast<const float4*>(&sm.tail[slot])[0];
                    const int4 t1 = reinterpret_cast<const int4*>(&sm.tail[slot])[1];
                    const int bx0 = (short)(t1.y & 0xffff), bx1 = (short)(t1.y >> 16);
                    const int by0 = (short)(t1.z & 0xffff), by1 = (short)(t1.z >> 16);
                    cx0[hf] = max(bx0 - X0, 0);
                    cy0[hf] = max(by0 - Y0, 0);
                    w[hf] = max(min(bx1 - X0, TILE) - cx0[hf], 0);
                    h[hf] = max(min(by1 - Y0, TILE) - cy0[hf], 0);
                    sm.col[jj] = make_float4(t0.z, t0.w, __int_as_float(t1.x), t0.x);
                    sm.f1[jj] = t0.y;
                    const RecB& rb = sm.rb[slot];
                    const float o = rb.opa;
                    sm.par[jj] = make_float4(o, rb.sig, 1.f / o, (float)(1.0 / sm.ev[slot].phis));
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
                const int jj = (int)lane + 32 * hf;
                const int excl = incl[hf] - w[hf] * h[hf];
                sm.S[jj + 1] = incl[hf];
                const unsigned magic = w[hf] ? (32768u + (unsigned)w[hf] - 1u) / (unsigned)w[hf] : 0u;
                sm.geo[jj] = (unsigned)cx0[hf] | ((unsigned)cy0[hf] << 4) | ((unsigned)w[hf] << 8) | (magic << 16);
                sm.kb[jj] = make_int2(excl - cy0[hf] * w[hf] - cx0[hf], w[hf]);
            }
            if (lane == 0) {
                sm.S[0] = 0;
                sm.nb = n;
            }
        }
        __syncthreads();
        nb = sm.nb;
        {  // records of the next window [bend-nb-DB, bend-nb)
            const int nrlo = max(s, bend - nb - DB);
            for (int c = tid; c < (rlo - nrlo) * 16; c += 256) fetch_rec(nrlo + (c >> 4), c & 15);
            rlo = min(rlo, nrlo);
            cp_async_commit();
        }
        // ---- 2. evaluate ----
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
                bool pass = false;
                int sj;
                const int jj = pair_step_entry(sm.S, nb, kb, jb, sj);
                if (k < kE) {
                    const unsigned g = sm.geo[jj];
                    const int w = (g >> 8) & 31;
                    const int local = k - sj;
                    const int dy = (int)(((unsigned)local * (g >> 16)) >> 15);
                    const int qx = (int)(g & 15) + local - dy * w;
                    const int qy = (int)((g >> 4) & 15) + dy;
                    const int p = qy * TILE + qx;
                    if (bend - 1 - jj <= sm.last[p]) {
                        const double pcx = sm.xc[qx], pcy = sm.yc[qy];
                        const EvalRec& r = sm.ev[(bend - 1 - jj) & (RR - 1)];
                        const double l0 = fma(r.a[0], pcx, fma(r.a[1], pcy, r.a[2]));
                        const double l1 = fma(r.a[3], pcx, fma(r.a[4], pcy, r.a[5]));
                        const double l2 = fma(r.a[6], pcx, fma(r.a[7], pcy, r.a[8]));
                        // argmax of phi = argmin of phi/phi_s, ties -> lowest edge (_kernels.py:36-42)
                        double rr = l0;
                        unsigned edge = 0;
                        if (l1 < rr) { rr = l1; edge = 1; }
                        if (l2 < rr) { rr = l2; edge = 2; }
                        if (rr >= r.r_lo) {
                            sm.r[k] = rr > r.r_hi ? __uint_as_float((__float_as_uint((float)rr) & ~3u) | edge)
                                                  : __int_as_float(0x7fc00000);
                            atomicOr(&sm.mask[jj >> 5][p], 1u << (jj & 31));
                            pass = true;
                        }
                    }
                }
                const unsigned pb = __ballot_sync(0xffffffffu, pass);
                if (lane == 0) sm.pbits[kb >> 5] = pb;
            }
        }
        __syncthreads();
        // ---- 2b. ranks of contributing pairs; the batch keeps the longest prefix of
        //          entries whose contributing pairs fit in GCAP (the rest is
        //          re-evaluated with the next batch) ----
        if (warp == 0) {
            constexpr int NWD = PCAP / 32;
            const int total = sm.S[nb];
            const int nwd = (total + 31) >> 5;
            int carry = 0;
#pragma unroll
            for (int q = 0; q < NWD / 32; q++) {
                const int wi = (int)lane + 32 * q;
                int c = wi < nwd ? __popc(sm.pbits[wi]) : 0;
                int incl = c;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, off);
                    if ((int)lane >= off) incl += y;
                }
                sm.wpre[wi] = incl - c + carry;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0) sm.wpre[NWD] = carry;
            __syncwarp();
            // contributing pairs before the end of entry jj
            int n = 0;
            bool full = true;
#pragma unroll
            for (int hf = 0; hf < NW; hf++) {
                const int jj = (int)lane + 32 * hf;
                int rk = 0x7fffffff;
                if (jj < nb) {
                    const int ke = sm.S[jj + 1];
                    const int wi = ke >> 5;
                    rk = sm.wpre[wi] + (wi < nwd ? __popc(sm.pbits[wi] & ((1u << (ke & 31)) - 1u)) : 0);
                }
                const unsigned bm = __ballot_sync(0xffffffffu, jj < nb && rk <= GCAP);
                if (full) n += __popc(bm);
                full = full && bm == 0xffffffffu;
            }
            if (lane == 0) sm.np = max(n, 1);
        }
        __syncthreads();
        const int np = sm.np;
        // ---- 3. per pixel, back to front ----
        if (my_last >= 0) {
#pragma unroll
            for (int wd = 0; wd < NW; wd++) {
                const int lim = np - 32 * wd;
                unsigned m = lim <= 0 ? 0u : (lim >= 32 ? sm.mask[wd][tid] : sm.mask[wd][tid] & ((1u << lim) - 1u));
                while (m) {
                    const int jj = wd * 32 + __ffs(m) - 1;
                    m &= m - 1;
                    const int slot = (bend - 1 - jj) & (RR - 1);
                    const int2 kbj = sm.kb[jj];
                    const int kk = kbj.x + ly * kbj.y + lx;
                    const float rv = sm.r[kk];
                    const EvalRec& er = sm.ev[slot];
                    const float4 par = sm.par[jj];  // o, sigma, 1/o, 1/phi_s
                    const double pcx = sm.xc[lx], pcy = sm.yc[ly];
                    // alpha with the reference formula in fp64 (_kernels.py:43-56): the
                    // transmittance recursion divides by 1 - alpha
                    int edge;
                    double r64;
                    if (!isnan(rv)) {
                        edge = (int)(__float_as_uint(rv) & 3u);
                        r64 = fma(er.a[3 * edge], pcx, fma(er.a[3 * edge + 1], pcy, er.a[3 * edge + 2]));
                    } else {  // r inside the contribution band: argmax edge and r in fp64
                        const double l0 = fma(er.a[0], pcx, fma(er.a[1], pcy, er.a[2]));
                        const double l1 = fma(er.a[3], pcx, fma(er.a[4], pcy, er.a[5]));
                        const double l2 = fma(er.a[6], pcx, fma(er.a[7], pcy, er.a[8]));
                        r64 = l0;
                        edge = 0;
                        if (l1 < r64) { r64 = l1; edge = 1; }
                        if (l2 < r64) { r64 = l2; edge = 2; }
                    }
                    const double o64 = (double)par.x, sg64 = (double)par.y;
                    const double rc = fmin(r64, 1.0);
                    double ae;
                    if (mode == 0) ae = r64 <= 0.0 ? 0.0 : o64 * (sg64 == 1.0 ? rc : pow(rc, sg64));
                    else ae = o64 / (1.0 + exp(fmin(r64 * er.phis / sg64, 700.0)));
                    if (ae < ALPHA_MIN) {  // (band pairs only) not composited: the slot adds nothing
                        const int sz = sm.wpre[kk >> 5] + __popc(sm.pbits[kk >> 5] & ((1u << (kk & 31)) - 1u));
#pragma unroll
                        for (int c = 0; c < 13; c++) sm.g[sz][c] = 0.0;
                        continue;
                    }
                    const bool clamped = ae > ALPHA_CLAMP;
                    const double a = clamped ? ALPHA_CLAMP : ae;
                    const float lgr = mode == 0 ? fast_lg2((float)rc) : 0.f;
                    const float4 col = sm.col[jj];
                    const double inv1m = 1.0 / (1.0 - a);
                    const double tb = T * inv1m;
                    const double w = tb * a;
                    double g[13];
                    g[8] = w * d0;
                    g[9] = w * d1;
                    g[10] = w * d2;
                    double ga = d0 * (tb * col.x - S0 * inv1m) + d1 * (tb * col.y - S1 * inv1m) +
                                d2 * (tb * col.z - S2 * inv1m);
                    g[12] = 0.0;
                    if (has_fg) {
                        const double u = fg_dw[fbase + fk];
                        ga += u * tb - sw * inv1m;
                        sw += u * w;
                        g[12] = fg_dz[fbase + fk];
                        fk--;
                    }
                    S0 = fma(w, (double)col.x, S0);
                    S1 = fma(w, (double)col.y, S1);
                    S2 = fma(w, (double)col.z, S2);
                    T = tb;
#pragma unroll
                    for (int c = 0; c < 8; c++) g[c] = 0.0;
                    g[11] = 0.0;
                    if (!clamped) {
                        const double window = a * (double)par.z;
                        g[6] = ga * window;  // d/d opacity = g_alpha * alpha / o
                        const double g_win = (double)par.x * ga;
                        const double phi = r64 * er.phis;
                        double g_phi;
                        if (mode == 0) {
                            g[7] = g_win * window * ((double)lgr * 0.6931471805599453);
                            const double g_r = g_win * (double)par.y * window / rc;
                            if (r64 >= 1.0) {
                                g_phi = 0.0;
                            } else {
                                g_phi = g_r * (double)par.w;
                                g[11] = -g_r * r64 * (double)par.w;
                            }
                        } else {
                            const double E = exp(fmin(phi / (double)par.y, 700.0));
                            const double ww = E / ((1.0 + E) * (1.0 + E));
                            const double is = 1.0 / (double)par.y;
                            g[7] = g_win * ww * phi * is * is;
                            g_phi = -g_win * ww * is;
                        }
                        const RecB& rb = sm.rb[slot];
                        const TailRec& tr = sm.tail[slot];
                        const int ib = edge == 2 ? 0 : edge + 1;
                        const double ax = rb.qx[edge], ay = rb.qy[edge], bx = rb.qx[ib], by = rb.qy[ib];
                        const double pxr = (double)(px - tr.ox) + 0.5, pyr = (double)(py - tr.oy) + 0.5;
                        const double sl = rb.sl[edge], ul = rb.ul[edge], vl = rb.vl[edge];
                        const double gax = (g_phi * (sl * (pyr - by) + phi * ul));
                        const double gay = (g_phi * (sl * (bx - pxr) + phi * vl));
                        const double gbx = (g_phi * (sl * (ay - pyr) - phi * ul));
                        const double gby = (g_phi * (sl * (pxr - ax) - phi * vl));
                        g[0] = edge == 0 ? gax : (ib == 0 ? gbx : 0.0);
                        g[1] = edge == 0 ? gay : (ib == 0 ? gby : 0.0);
                        g[2] = edge == 1 ? gax : (ib == 1 ? gbx : 0.0);
                        g[3] = edge == 1 ? gay : (ib == 1 ? gby : 0.0);
                        g[4] = edge == 2 ? gax : (ib == 2 ? gbx : 0.0);
                        g[5] = edge == 2 ? gay : (ib == 2 ? gby : 0.0);
                    }
                    const int slot_g = sm.wpre[kk >> 5] + __popc(sm.pbits[kk >> 5] & ((1u << (kk & 31)) - 1u));
#pragma unroll
                    for (int c = 0; c < 13; c++) sm.g[slot_g][c] = g[c];
                }
            }
        }
        __syncthreads();
        // ---- 4. flush: per (entry, component) an fp64 sum over the entry's
        //         contributing pairs in a fixed order, one global atomic ----
        for (int c = tid; c < np * NC; c += 256) {
            const int jj = c / NC, comp = c - jj * NC;
            auto rank = [&](int k) {
                const int wi = k >> 5;
                return sm.wpre[wi] + ((k & 31) ? __popc(sm.pbits[wi] & ((1u << (k & 31)) - 1u)) : 0);
            };
            const int r0 = rank(sm.S[jj]), r1 = rank(sm.S[jj + 1]);
            double v = 0.0;
            for (int q = r0; q < r1; q++) v += sm.g[q][comp];
            if (v != 0.0) atomicAdd(sgrad + (size_t)sm.srcq[(bend - 1 - jj) & (SR - 1)] * SG_STRIDE + comp, v);
        }
        nb = np;
    }
    cp_async_wait_all();
}

template <int DB, int PCAP, int GCAP>
static void launch_bwd_dense(const Cam& cam, const Opts& opt, const RecF* rec, const RecB* recb,
                             const int* tile_start, const unsigned* ent_src, const double* t_final,
                             const int* last_pos, const float* d_image, const int* n_frag,
                             const long long* frag_off, const double* fg_dw, const double* fg_dz, double* sgrad,
                             cudaStream_t st) {
    const int dyn = (int)sizeof(BwdSmem<DB, PCAP, GCAP>);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_blend_bwd_dense<DB, PCAP, GCAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        attr = true;
    }
    const int ntiles = cam.ntx * cam.nty;
    k_blend_bwd_dense<DB, PCAP, GCAP><<<ntiles, 256, dyn, st>>>(cam, opt, rec, recb, tile_start, ent_src, t_final,
                                                           last_pos, d_image, n_frag, frag_off, fg_dw, fg_dz, sgrad);
}

void launch_blend_bwd_dense(const Cam& cam, const Opts& opt, const RecF* rec, const RecB* recb,
                            const int* tile_start, const unsigned* ent_src, const double* t_final,
                            const int* last_pos, const float* d_image, const int* n_frag, const long long* frag_off,
                            const double* fg_dw, const double* fg_dz, double* sgrad, cudaStream_t st) {
    launch_bwd_dense<64, 2048, 512>(cam, opt, rec, recb, tile_start, ent_src, t_final, last_pos, d_image, n_frag,
                                    frag_off, fg_dw, fg_dz, sgrad, st);
}

}  // namespace ts
