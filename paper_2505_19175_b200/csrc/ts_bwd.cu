// ts_bwd.cu -- dense backward blend (rasterize_backward, _kernels.py:181-318).
//
// CTA per 16x16 tile, 256 threads.  The tile's entry list is walked BACK TO
// FRONT from the largest saved last contributor of the tile, in batches of at
// most DB entries / PCAP pairs; entry jj of a batch is list position bend-1-jj,
// so ascending bits = back to front.  Per batch:
//   1. stage    -- records (evaluation part, tail, backward record) arrive in a
//                  cp.async ring one batch ahead; warp 0 builds the rectangles
//                  bbox ∩ tile and their pair scan;
//   2. evaluate -- dense over the batch's (entry, pixel) pairs, 32 consecutive
//                  pairs per warp step: a pair at or before the pixel's last
//                  contributor (_kernels.py:226-243) is composited iff
//                  alpha >= 1/255 with the reference's alpha in fp64
//                  (_kernels.py:43-56); it stores r (fp32, argmax edge in the
//                  two low mantissa bits) and alpha (fp64), and sets the pixel's
//                  bit and the pair's bit;
//   3. slots    -- composited pairs get entry-major slots (prefix popcounts);
//                  the batch keeps the longest prefix of entries whose slots
//                  fit in GCAP (the rest is re-evaluated with the next batch);
//   4. recursion -- thread = pixel walks its bits back to front with the only
//                  sequential part of the reference (_kernels.py:255-275):
//                  T_k = T_{k+1} / (1 - alpha_k) from the saved T_final, the
//                  suffix colour S and (frag_grads) the suffix weight sum; it
//                  stores T_k, S behind fragment k and the fragment's upstream
//                  terms in the fragment's slot;
//   5. gradients -- dense over slots, 32 per warp step: dL/dalpha, window and
//                  edge-chain derivatives (fp64 where they cancel,
//                  _kernels.py:276-318) per slot in fp64, a segmented warp
//                  reduction (fp32 partials) over the slots of one entry, and
//                  one fp64 global atomic per (entry, component) and warp step.
#include "ts_kernels.cuh"

namespace ts {

namespace {
struct __align__(16) BwdSlot {
    double tb;             // transmittance in front of the fragment
    double s0, s1, s2;     // suffix colour behind the fragment
    int k;                 // pair index
    int jp;                // entry | pixel << 8
    double u, sw, dz;      // frag_grads: d_weight, suffix weight sum, d_depth
};
}  // namespace

template <int DB, int PCAP, int GCAP>
struct BwdSmem {
    static constexpr int RR = 2 * DB, SR = 4 * DB, NW = DB / 32;
    EvalRec ev[RR];
    TailRec tail[RR];
    RecB rb[RR];
    RecC rc[RR];                 // fp64 colour, opacity, sigma
    double al[PCAP];             // per pair: unclamped alpha (fp64)
    float r[PCAP];               // per pair: r (edge in the low 2 bits)
    BwdSlot slot[GCAP];
    unsigned mask[NW][256];      // per pixel: bit jj = entry jj composited
    unsigned srcq[SR];
    double4 par[DB];             // opacity, sigma, 1/opacity, 1/phi_s (fp64)
    int S[DB + 1];
    unsigned starts[PCAP / 32];  // bit (k & 31) of word k >> 5: an entry starts at pair k
    int jfirst[PCAP / 32];       // entry holding pair 32 w
    unsigned geo[DB];
    int2 kb[DB];
    unsigned pbits[PCAP / 32];   // pair k composited
    int wpre[PCAP / 32 + 1];     // composited pairs before word w
    float d[3][256];             // upstream image gradient per pixel
    double xc[TILE], yc[TILE];
    int last[256];
    int nb, np, hi;
};

template <int DB, int PCAP, int GCAP, int MINB>
__global__ void __launch_bounds__(256, MINB) k_blend_bwd_dense(Cam cam, Opts opt, const RecF* __restrict__ rec,
                                                            const RecB* __restrict__ recb,
                                                            const RecC* __restrict__ recc,
                                                            const int* __restrict__ tile_start,
                                                            const unsigned* __restrict__ ent_src,
                                                            const double* __restrict__ t_final,
                                                            const int* __restrict__ last_pos,
                                                            const float* __restrict__ d_image,
                                                            const int* __restrict__ n_frag,
                                                            const long long* __restrict__ frag_off,
                                                            const double* __restrict__ fg_dw,
                                                            const double* __restrict__ fg_dz,
                                                            const unsigned long long* __restrict__ run_if,
                                                            double* __restrict__ sgrad) {
    TS_PDL_ENTRY();
    if (run_if && *run_if == 0ull) return;  // the streaming backward handled this frame
    using SM = BwdSmem<DB, PCAP, GCAP>;
    constexpr int RR = SM::RR, SR = SM::SR, NW = SM::NW;
    extern __shared__ __align__(16) unsigned char s_dyn[];
    SM& sm = *reinterpret_cast<SM*>(s_dyn);

    const int tid = threadIdx.x;
    const unsigned lane = tid & 31, warp = tid >> 5;
    const int t = blockIdx.x;
    const int tx = t % cam.ntx, ty = t / cam.ntx;
    const int X0 = tx * TILE, Y0 = ty * TILE;
    const int px = X0 + (tid & 15), py = Y0 + (tid >> 4);
    const bool inside = px < cam.width && py < cam.height;
    const int s = tile_start[t];
    const int mode = opt.mode;
    // per-pixel recursion state (thread = pixel)
    int my_last = -1;
    double T = 1.0;
    // upstream fragment gradients (backward.py:122-142): fragment k of the
    // pixel is fg_*[fbase + k], visited back to front
    const bool has_fg = fg_dw != nullptr;
    long long fbase = 0;
    int fk = -1;
    double sw = 0.0;
    float d0 = 0.f, d1 = 0.f, d2 = 0.f;
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
    double S0 = T * opt.bg[0], S1 = T * opt.bg[1], S2 = T * opt.bg[2];
    sm.d[0][tid] = d0;
    sm.d[1][tid] = d1;
    sm.d[2][tid] = d2;
    sm.last[tid] = my_last;
    if (tid < TILE) sm.xc[tid] = (double)(X0 + tid) + 0.5;
    else if (tid < 2 * TILE) sm.yc[tid - TILE] = (double)(Y0 + tid - TILE) + 0.5;
    if (tid == 0) sm.hi = -1;
    __syncthreads();
    if (my_last >= 0) atomicMax(&sm.hi, my_last);
    __syncthreads();
    const int hi = sm.hi;
    if (hi < s) return;

    constexpr int NCH = 15;  // 16-byte chunks per entry: RecF 8, RecB 4, RecC 3
    auto fetch_rec = [&](int p, int q) {  // 16-byte chunk q of (RecF, RecB, RecC) at list position p
        const unsigned src = sm.srcq[p & (SR - 1)];
        const int slot = p & (RR - 1);
        if (q < 6)
            cp_async16(reinterpret_cast<float4*>(&sm.ev[slot]) + q, reinterpret_cast<const float4*>(rec + src) + q);
        else if (q < 8)
            cp_async16(reinterpret_cast<float4*>(&sm.tail[slot]) + (q - 6),
                       reinterpret_cast<const float4*>(rec + src) + q);
        else if (q < 12)
            cp_async16(reinterpret_cast<float4*>(&sm.rb[slot]) + (q - 8),
                       reinterpret_cast<const float4*>(recb + src) + (q - 8));
        else
            cp_async16(reinterpret_cast<float4*>(&sm.rc[slot]) + (q - 12),
                       reinterpret_cast<const float4*>(recc + src) + (q - 12));
    };
    auto rank = [&](int k) {  // composited pairs before pair k
        const int wi = k >> 5;
        return sm.wpre[wi] + ((k & 31) ? __popc(sm.pbits[wi] & ((1u << (k & 31)) - 1u)) : 0);
    };
    // prologue: ids of [hi+1-3DB, hi], then records of [hi+1-DB, hi]
    int slo = max(s, hi + 1 - 3 * DB), rlo = max(s, hi + 1 - DB);
    for (int p = slo + tid; p <= hi; p += 256) cp_async4(&sm.srcq[p & (SR - 1)], ent_src + p);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    for (int c = tid; c < (hi + 1 - rlo) * NCH; c += 256) fetch_rec(rlo + c / NCH, c % NCH);
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
                    const int4 t1 = reinterpret_cast<const int4*>(&sm.tail[slot])[1];
                    const int bx0 = (short)(t1.y & 0xffff), bx1 = (short)(t1.y >> 16);
                    const int by0 = (short)(t1.z & 0xffff), by1 = (short)(t1.z >> 16);
                    cx0[hf] = max(bx0 - X0, 0);
                    cy0[hf] = max(by0 - Y0, 0);
                    w[hf] = max(min(bx1 - X0, TILE) - cx0[hf], 0);
                    h[hf] = max(min(by1 - Y0, TILE) - cy0[hf], 0);
                    const RecC& rc = sm.rc[slot];
                    sm.par[jj] = make_double4(rc.opa, rc.sig, 1.0 / rc.opa, 1.0 / sm.ev[slot].phis);
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
            // pair-word tables of the batch (entries < n): entry starts and the
            // entry holding the first pair of every 32-pair word
            for (int w = (int)lane; w < PCAP / 32; w += 32) sm.starts[w] = 0u;
            __syncwarp();
#pragma unroll
            for (int hf = 0; hf < NW; hf++) {
                const int jq = (int)lane + 32 * hf;
                if (jq < n) {
                    const int excl = incl[hf] - w[hf] * h[hf];
                    atomicOr(&sm.starts[excl >> 5], 1u << (excl & 31));
                    for (int wq = (excl + 31) >> 5; wq <= ((incl[hf] - 1) >> 5); wq++) sm.jfirst[wq] = jq;
                }
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
            for (int c = tid; c < (rlo - nrlo) * NCH; c += 256) fetch_rec(nrlo + c / NCH, c % NCH);
            rlo = min(rlo, nrlo);
            cp_async_commit();
        }
        // ---- 2. evaluate (dense pairs): r, argmax edge, fp64 alpha, composited? ----
        {
            const int total = sm.S[nb];
            const int chunk = ((total + 255) >> 8) << 5;
            const int k0 = (int)warp * chunk;
            const int kE = min(k0 + chunk, total);
            for (int kb = k0; kb < kE; kb += 32) {
                const int k = kb + (int)lane;
                bool comp = false;
                // entry of pair k: the word's first entry plus the entry starts in (kb, k]
                const int jj = sm.jfirst[kb >> 5] + __popc(sm.starts[kb >> 5] & ((2u << lane) - 2u));
                const int sj = sm.S[jj];
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
                            const double4 par = sm.par[jj];
                            const double o64 = par.x, sg64 = par.y;
                            double ae;
                            if (mode == 0) {
                                const double rc = fmin(rr, 1.0);
                                ae = rr <= 0.0 ? 0.0 : o64 * (sg64 == 1.0 ? rc : pow(rc, sg64));
                            } else {
                                ae = o64 / (1.0 + exp(fmin(rr * r.phis / sg64, 700.0)));
                            }
                            // outside the band alpha >= 1/255 holds by construction
                            if (rr > r.r_hi || ae >= ALPHA_MIN) {
                                comp = true;
                                sm.r[k] = __uint_as_float((__float_as_uint((float)rr) & ~3u) | edge);
                                sm.al[k] = ae;
                                atomicOr(&sm.mask[jj >> 5][p], 1u << (jj & 31));
                            }
                        }
                    }
                }
                const unsigned pb = __ballot_sync(0xffffffffu, comp);
                if (lane == 0) sm.pbits[kb >> 5] = pb;
            }
        }
        __syncthreads();
        // ---- 3. slots: prefix popcounts; the batch keeps the longest prefix of
        //         entries whose composited pairs fit in GCAP ----
        if (warp == 0) {
            constexpr int NWD = PCAP / 32;
            const int total = sm.S[nb];
            const int nwd = (total + 31) >> 5;
            int carry = 0;
#pragma unroll
            for (int q = 0; q < NWD / 32; q++) {
                const int wi = (int)lane + 32 * q;
                const int c = wi < nwd ? __popc(sm.pbits[wi]) : 0;
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
        // ---- 4. recursion (thread = pixel), back to front over entries < np ----
        if (my_last >= 0) {
#pragma unroll
            for (int wd = 0; wd < NW; wd++) {
                const int lim = np - 32 * wd;
                unsigned m = lim <= 0 ? 0u : (lim >= 32 ? sm.mask[wd][tid] : sm.mask[wd][tid] & ((1u << lim) - 1u));
                while (m) {
                    const int jj = wd * 32 + __ffs(m) - 1;
                    m &= m - 1;
                    const int2 kbj = sm.kb[jj];
                    const int k = kbj.x + (tid >> 4) * kbj.y + (tid & 15);
                    double a = sm.al[k];
                    if (a > ALPHA_CLAMP) a = ALPHA_CLAMP;
                    const double tb = T / (1.0 - a);
                    const double w = tb * a;
                    BwdSlot& sl = sm.slot[rank(k)];
                    sl.tb = tb;
                    sl.s0 = S0;
                    sl.s1 = S1;
                    sl.s2 = S2;
                    sl.k = k;
                    sl.jp = jj | (tid << 8);
                    if (has_fg) {
                        const double u = fg_dw[fbase + fk];
                        sl.u = u;
                        sl.sw = sw;
                        sl.dz = fg_dz[fbase + fk];
                        sw += u * w;
                        fk--;
                    }
                    const double* col = sm.rc[(bend - 1 - jj) & (RR - 1)].rgb;
                    S0 = fma(w, col[0], S0);
                    S1 = fma(w, col[1], S1);
                    S2 = fma(w, col[2], S2);
                    T = tb;
                }
            }
        }
        __syncthreads();
        // ---- 5. gradients, dense over the np entries' slots ----
        {
            const int nslot = rank(sm.S[np]);
            for (int q0 = (int)warp * 32; q0 < nslot; q0 += 256) {
                const int q = q0 + (int)lane;
                const bool act = q < nslot;
                double g[13];
#pragma unroll
                for (int c = 0; c < 13; c++) g[c] = 0.0;
                int jj = -1 - (int)lane;  // unique keys for idle lanes
                if (act) {
                    const BwdSlot& sl = sm.slot[q];
                    jj = sl.jp & 255;
                    const int pix = sl.jp >> 8;
                    const int k = sl.k;
                    const int slot = (bend - 1 - jj) & (RR - 1);
                    const double4 par = sm.par[jj];  // o, sigma, 1/o, 1/phi_s
                    const double* col = sm.rc[slot].rgb;
                    const double ae = sm.al[k];
                    const bool clamped = ae > ALPHA_CLAMP;
                    const double a = clamped ? ALPHA_CLAMP : ae;
                    const double inv1m = 1.0 / (1.0 - a);
                    const double tb = sl.tb;
                    const double w = tb * a;
                    const double dd0 = sm.d[0][pix], dd1 = sm.d[1][pix], dd2 = sm.d[2][pix];
                    g[8] = w * dd0;
                    g[9] = w * dd1;
                    g[10] = w * dd2;
                    double ga = dd0 * (tb * col[0] - sl.s0 * inv1m) + dd1 * (tb * col[1] - sl.s1 * inv1m) +
                                dd2 * (tb * col[2] - sl.s2 * inv1m);
                    if (has_fg) {
                        ga += sl.u * tb - sl.sw * inv1m;
                        g[12] = sl.dz;
                    }
                    if (!clamped) {
                        const float rv = sm.r[k];
                        const int edge = (int)(__float_as_uint(rv) & 3u);
                        const EvalRec& er = sm.ev[slot];
                        const int lx = pix & 15, ly = pix >> 4;
                        const double pcx = sm.xc[lx], pcy = sm.yc[ly];
                        // fp64 r of the argmax edge for the chain (phi = r * phi_s)
                        const double r64 = fma(er.a[3 * edge], pcx, fma(er.a[3 * edge + 1], pcy, er.a[3 * edge + 2]));
                        const double window = a * par.z;
                        g[6] = ga * window;  // d/d opacity = g_alpha * alpha / o
                        const double g_win = par.x * ga;
                        const double phi = r64 * er.phis;
                        double g_phi;
                        if (mode == 0) {
                            const double rc = fmin(r64, 1.0);
                            g[7] = g_win * window * log(rc);
                            const double g_r = g_win * par.y * window / rc;
                            if (r64 >= 1.0) {
                                g_phi = 0.0;
                            } else {
                                g_phi = g_r * par.w;
                                g[11] = -g_r * r64 * par.w;
                            }
                        } else {
                            const double E = exp(fmin(phi / par.y, 700.0));
                            const double ww = E / ((1.0 + E) * (1.0 + E));
                            const double is = 1.0 / par.y;
                            g[7] = g_win * ww * phi * is * is;
                            g_phi = -g_win * ww * is;
                        }
                        const RecB& rb = sm.rb[slot];
                        const TailRec& tr = sm.tail[slot];
                        const int ib = edge == 2 ? 0 : edge + 1;
                        const double ax = rb.q[edge].x, ay = rb.q[edge].y, bx = rb.q[ib].x, by = rb.q[ib].y;
                        const double pxr = (double)(X0 + lx - tr.ox) + 0.5, pyr = (double)(Y0 + ly - tr.oy) + 0.5;
                        double sl_, ul, vl;
                        rb_edge(rb.q[edge], rb.q[ib], rb.esign, edge, sl_, ul, vl);
                        const double gax = g_phi * (sl_ * (pyr - by) + phi * ul);
                        const double gay = g_phi * (sl_ * (bx - pxr) + phi * vl);
                        const double gbx = g_phi * (sl_ * (ay - pyr) - phi * ul);
                        const double gby = g_phi * (sl_ * (pxr - ax) - phi * vl);
                        g[0] = edge == 0 ? gax : (ib == 0 ? gbx : 0.0);
                        g[1] = edge == 0 ? gay : (ib == 0 ? gby : 0.0);
                        g[2] = edge == 1 ? gax : (ib == 1 ? gbx : 0.0);
                        g[3] = edge == 1 ? gay : (ib == 1 ? gby : 0.0);
                        g[4] = edge == 2 ? gax : (ib == 2 ? gbx : 0.0);
                        g[5] = edge == 2 ? gay : (ib == 2 ? gby : 0.0);
                    }
                }
                // segmented fp64 reduction: slots of one entry are consecutive, so a
                // lane adds the lanes below it with the same entry; the first lane of
                // each run ends with the run's sum.  Only as many levels as the
                // longest run needs.
                double* gf = g;
                const int jprev = __shfl_up_sync(0xffffffffu, jj, 1);
                const bool head = lane == 0 || jprev != jj;
                const unsigned heads = __ballot_sync(0xffffffffu, head);
                const unsigned later = heads & ~((2u << lane) - 1u);
                const int runlen = head ? (later ? __ffs(later) - 1 : 32) - (int)lane : 0;
                const int maxrun = __reduce_max_sync(0xffffffffu, runlen);
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    if (off >= maxrun) break;
                    const int jo = __shfl_down_sync(0xffffffffu, jj, off);
                    const bool same = (int)lane + off < 32 && jo == jj;
#pragma unroll
                    for (int c = 0; c < 13; c++) {
                        const double v = __shfl_down_sync(0xffffffffu, gf[c], off);
                        if (same) gf[c] += v;
                    }
                }
                if (act && head) {
                    double* dst = sgrad + (size_t)sm.srcq[(bend - 1 - jj) & (SR - 1)] * SG_STRIDE;
#pragma unroll
                    for (int c = 0; c < 13; c++)
                        if (gf[c] != 0.0) atomicAdd(dst + c, gf[c]);
                }
            }
        }
        nb = np;
    }
    cp_async_wait_all();
}

template <int DB, int PCAP, int GCAP, int MINB>
static void launch_bwd_dense(const Cam& cam, const Opts& opt, const RecF* rec, const RecB* recb, const RecC* recc,
                             const int* tile_start, const unsigned* ent_src, const double* t_final,
                             const int* last_pos, const float* d_image, const int* n_frag,
                             const long long* frag_off, const double* fg_dw, const double* fg_dz,
                             const unsigned long long* run_if, double* sgrad, cudaStream_t st) {
    const int dyn = (int)sizeof(BwdSmem<DB, PCAP, GCAP>);
    smem_optin((const void*)k_blend_bwd_dense<DB, PCAP, GCAP, MINB>, dyn);
    const int ntiles = cam.ntx * cam.nty;
    launch_pdl(k_blend_bwd_dense<DB, PCAP, GCAP, MINB>, dim3(ntiles), dim3(256), dyn, st, cam, opt, rec, recb, recc,
               tile_start, ent_src, t_final, last_pos, d_image, n_frag, frag_off, fg_dw, fg_dz, run_if, sgrad);
}

void launch_blend_bwd_dense(const Cam& cam, const Opts& opt, const RecF* rec, const RecB* recb, const RecC* recc,
                            const int* tile_start, const unsigned* ent_src, const double* t_final,
                            const int* last_pos, const float* d_image, const int* n_frag, const long long* frag_off,
                            const double* fg_dw, const double* fg_dz, const unsigned long long* run_if, double* sgrad,
                            cudaStream_t st) {
    // 3 CTAs per SM (measured against 64-entry batches at 2 CTAs per SM)
    launch_bwd_dense<32, 1024, 384, 3>(cam, opt, rec, recb, recc, tile_start, ent_src, t_final, last_pos, d_image, n_frag,
                                           frag_off, fg_dw, fg_dz, run_if, sgrad, st);
}

}  // namespace ts
