// ts_bwd_stream.cu -- streaming backward blend (rasterize_backward,
// _kernels.py:181-318) over the fragment records of the training forward.
//
// The training forward (k_blend_dense, fp64 compositing, + k_fixup_fwd)
// writes one FragRec per composited fragment, grouped by (tile, entry): the
// transmittance T_k and the colour C_k accumulated in front of the fragment,
// its pixel and source triangle.  With the pixel's final unclipped colour C_N
// (incl. T_N * background) the reference's back-to-front recursion becomes a
// closed form per fragment:
//     w_k = T_k alpha_k,   S_k = C_N - C_k - w_k c_k   (suffix colour),
//     dL/dalpha_k = sum_c d_c (T_k c_k - S_k / (1 - alpha_k)),
// so every fragment is independent: one lane per record, r / argmax edge /
// alpha recomputed in fp64 from the triangle's records (fp64 colour, opacity
// and sigma from its RecC), the window and edge chain as in k_blend_bwd_dense,
// per warp step the components in shared memory, one lane per (run of records
// of one triangle, component) summing its run in fp64 and adding it with one
// atomic.  No tile loop, no
// CTA barrier.  If the forward's record buffer overflowed, this kernel does
// nothing and the tile backward runs instead.
#include "ts_kernels.cuh"

namespace ts {

#ifndef TS_BWD_MINB
#define TS_BWD_MINB 4  // CTAs per SM (64 registers, no spills with the shared-memory components; 80 at 3)
#endif
#ifndef TS_BWD_GRID
#define TS_BWD_GRID 4  // CTAs per SM in the launch (one resident wave; 4 x 64 registers: 1.13 -> 0.97 ms at C3 against 3 x 80)
#endif

// Upstream gradients on the fragments' blend weights and depths (render_backward
// with frag_grads, _kernels.py:262-272), addressed through the fragment CSR:
// record (pixel p, ordinal k) is fragment off[p] + k.  sw[i] = sum over the
// pixel's later fragments of dw * w (k_frag_suffix).
struct FragGrads {
    const long long* off;
    const double* dw;
    const double* dz;
    const double* sw;
};

// sw[i] = sum_{i < k < end(p)} dw[k] w[k] per pixel p (the reference's running
// `sw`, _kernels.py:265-268, back to front).  Eight lanes per pixel (four pixels per
// warp), 32-fragment chunks from the list's back end, each lane holding four
// consecutive fragments: the suffix inside the lane is serial, across the group a
// 3-step suffix scan of the lane totals, plus the sum of the later chunks.
__global__ void __launch_bounds__(256) k_frag_suffix(long long npix, const long long* __restrict__ off,
                                                     const double* __restrict__ w, const double* __restrict__ dw,
                                                     double* __restrict__ sw) {
    const long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    const unsigned lane = threadIdx.x & 31, gl = lane & 7;
    const unsigned gmask = 0xffu << (lane & 24);
    if (p >= npix) return;  // whole groups leave together
    const long long lo = off[p], hi = off[p + 1];
    double carry = 0.0;  // sum over the chunks after the current one
    for (long long top = hi; top > lo; top -= 32) {
        const long long base = top - 32 > lo ? top - 32 : lo;
        const long long kf = base + 4 * gl;
        double x[4], t = 0.0;
#pragma unroll
        for (int r = 0; r < 4; r++) {
            x[r] = kf + r < top ? dw[kf + r] * w[kf + r] : 0.0;
            t += x[r];
        }
        // inclusive suffix scan of the lane totals: lane L gets sum_{L <= j < 8} t_j
        double v = t;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const double y = __shfl_down_sync(gmask, v, o, 8);
            if ((int)gl + o < 8) v += y;
        }
        double after = carry + (v - t);  // everything after this lane's last fragment
#pragma unroll
        for (int r = 3; r >= 0; r--) {
            if (kf + r < top) sw[kf + r] = after;
            after += x[r];
        }
        carry += __shfl_sync(gmask, v, 0, 8);
    }
}

template <bool FRAG>
__global__ void __launch_bounds__(256, TS_BWD_MINB) k_bwd_stream(Cam cam, Opts opt, const RecF* __restrict__ rec,
                                                 const RecB* __restrict__ recb, const RecC* __restrict__ recc,
                                                 const FragRec* __restrict__ frec, const Counters* __restrict__ ctr,
                                                 unsigned long long cap, const double* __restrict__ c_total,
                                                 const float* __restrict__ d_image, double* __restrict__ sgrad,
                                                 FragGrads fg) {
    constexpr int NG = FRAG ? 13 : 12;  // reduced components: gq[6] go gsig grgb[3] gphis (+ gz)
    TS_PDL_ENTRY();
    if (ctr->frec_over) return;
    const unsigned long long total = ctr->n_frec;
    const long long n = (long long)(total < cap ? total : cap);
    const unsigned lane = threadIdx.x & 31;
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const int mode = opt.mode;
    // per warp: the step's per-record components (component-major, padded) and
    // its runs (first lane, triangle)
    __shared__ double s_red[8][NG][33];
    __shared__ unsigned s_run[8][33];
    __shared__ unsigned s_rkey[8][32];
    const int wl = threadIdx.x >> 5;
    // (interleaved 32-record steps: measured faster than one contiguous range per warp)
    for (long long q0 = gw * 32; q0 < n; q0 += nw * 32) {
        const long long q = q0 + lane;
        // the lane's components go straight to its shared-memory column (short
        // register live ranges: 64 registers, 4 CTAs per SM)
        double* gsl = &s_red[wl][0][lane];
#pragma unroll
        for (int c = 0; c < NG; c++) gsl[c * 33] = 0.0;
#define GF(c, v) (gsl[(c) * 33] = (v))
        unsigned key = 0xffffffffu - lane;  // unique keys for idle lanes and holes
        bool act = false;
        if (q < n) {
            const double2 ta = __ldg(reinterpret_cast<const double2*>(frec + q));
            const double2 tb2 = __ldg(reinterpret_cast<const double2*>(frec + q) + 1);
            const double4 tc = make_double4(ta.x, ta.y, tb2.x, tb2.y);
            const uint4 ids = __ldg(reinterpret_cast<const uint4*>(frec + q) + 2);  // pix, src, ordinal
            if (ids.x != 0xffffffffu) {
                act = true;
                const unsigned pix = ids.x, src = ids.y;
                key = src;
                const RecF& R = rec[src];
                const RecB& B = recb[src];
                const RecC& Cc = recc[src];
                const int px = (int)(pix % (unsigned)cam.width), py = (int)(pix / (unsigned)cam.width);
                const double pcx = px + 0.5, pcy = py + 0.5;
                // the record's edge functions and phi_s as five 16-byte loads
                const double2* ra = reinterpret_cast<const double2*>(R.a);
                const double2 a01 = __ldg(ra), a23 = __ldg(ra + 1), a45 = __ldg(ra + 2), a67 = __ldg(ra + 3);
                const double2 a8p = __ldg(ra + 4);  // (a[8], phis)
                const double l0 = fma(a01.x, pcx, fma(a01.y, pcy, a23.x));
                const double l1 = fma(a23.y, pcx, fma(a45.x, pcy, a45.y));
                const double l2 = fma(a67.x, pcx, fma(a67.y, pcy, a8p.x));
                // argmax of phi = argmin of phi/phi_s, ties -> lowest edge (_kernels.py:36-42)
                double r64 = l0;
                int edge = 0;
                if (l1 < r64) { r64 = l1; edge = 1; }
                if (l2 < r64) { r64 = l2; edge = 2; }
                const double phis = a8p.y;
                const double2 osg = __ldg(reinterpret_cast<const double2*>(&Cc.opa));
                const double o = osg.x, sg = osg.y;
                const double rc = fmin(r64, 1.0);
                double ae;
                if (mode == 0) ae = o * (sg == 1.0 ? rc : pow(rc, sg));
                else ae = o / (1.0 + exp(fmin(r64 * phis / sg, 700.0)));
                const bool clamped = ae > ALPHA_CLAMP;
                const double a = clamped ? ALPHA_CLAMP : ae;
                const double inv1m = 1.0 / (1.0 - a);
                const double tb = tc.x;
                const double w = tb * a;
                const double2 c01 = __ldg(reinterpret_cast<const double2*>(Cc.rgb));
                const double2 c2io = __ldg(reinterpret_cast<const double2*>(Cc.rgb + 2));  // (rgb[2], inv_opa)
                const double c0 = c01.x, c1 = c01.y, c2 = c2io.x;
                const double s0 = __ldg(c_total + pix * 3 + 0) - tc.y - w * c0;
                const double s1 = __ldg(c_total + pix * 3 + 1) - tc.z - w * c1;
                const double s2 = __ldg(c_total + pix * 3 + 2) - tc.w - w * c2;
                const double d0 = __ldg(d_image + pix * 3 + 0), d1 = __ldg(d_image + pix * 3 + 1),
                             d2 = __ldg(d_image + pix * 3 + 2);
                GF(8, w * d0);
                GF(9, w * d1);
                GF(10, w * d2);
                double ga = d0 * (tb * c0 - s0 * inv1m) + d1 * (tb * c1 - s1 * inv1m) + d2 * (tb * c2 - s2 * inv1m);
                if constexpr (FRAG) {
                    const long long fi = __ldg(fg.off + pix) + ids.z;
                    ga += __ldg(fg.dw + fi) * tb - __ldg(fg.sw + fi) * inv1m;
                    GF(12, __ldg(fg.dz + fi));
                }
                if (!clamped) {
                    // (reciprocals of the opacity and of phi_s precomputed per triangle: the
                    // products differ from the quotients by <= 1 ulp)
                    const double inv_o = c2io.y, inv_phis = __ldg(&B.inv_phis);
                    const double window = a * inv_o;
                    GF(6, ga * window);  // d/d opacity = g_alpha * alpha / o
                    const double g_win = o * ga;
                    const double phi = r64 * phis;
                    double g_phi;
                    if (mode == 0) {
                        GF(7, g_win * window * log(rc));
                        // window / rc = rc^(sigma - 1): 1 for sigma = 1
                        const double g_r = g_win * sg * (sg == 1.0 ? 1.0 : window / rc);
                        if (r64 >= 1.0) {
                            g_phi = 0.0;
                        } else {
                            g_phi = g_r * inv_phis;
                            GF(11, -g_r * r64 * inv_phis);
                        }
                    } else {
                        const double E = exp(fmin(phi / sg, 700.0));
                        const double ww = E / ((1.0 + E) * (1.0 + E));
                        const double is = 1.0 / sg;
                        GF(7, g_win * ww * phi * is * is);
                        g_phi = -g_win * ww * is;
                    }
                    const int ib = edge == 2 ? 0 : edge + 1;
                    const double2 qa = __ldg(&B.q[edge]), qb = __ldg(&B.q[ib]);
                    const double ax = qa.x, ay = qa.y, bx = qb.x, by = qb.y;
                    const unsigned oxy = __ldg(reinterpret_cast<const unsigned*>(&R.ox));  // (ox, oy) shorts
                    const double pxr = (double)(px - (int)(short)(oxy & 0xffffu)) + 0.5;
                    const double pyr = (double)(py - (int)(short)(oxy >> 16)) + 0.5;
                    double sl, ul, vl;
                    rb_edge(qa, qb, __ldg(&B.esign), edge, sl, ul, vl);
                    const double gax = g_phi * (sl * (pyr - by) + phi * ul);
                    const double gay = g_phi * (sl * (bx - pxr) + phi * vl);
                    const double gbx = g_phi * (sl * (ay - pyr) - phi * ul);
                    const double gby = g_phi * (sl * (pxr - ax) - phi * vl);
                    GF(0, edge == 0 ? gax : (ib == 0 ? gbx : 0.0));
                    GF(1, edge == 0 ? gay : (ib == 0 ? gby : 0.0));
                    GF(2, edge == 1 ? gax : (ib == 1 ? gbx : 0.0));
                    GF(3, edge == 1 ? gay : (ib == 1 ? gby : 0.0));
                    GF(4, edge == 2 ? gax : (ib == 2 ? gbx : 0.0));
                    GF(5, edge == 2 ? gay : (ib == 2 ? gby : 0.0));
                }
            }
        }
        // segmented reduction over consecutive records of one triangle
        const unsigned kprev = __shfl_up_sync(0xffffffffu, key, 1);
        const bool head = lane == 0 || kprev != key;
        const unsigned heads = __ballot_sync(0xffffffffu, head);
        {
            // run r = lanes [s_run[r], s_run[r+1]); lane L sums components of the
            // (run, component) items L, L+32, ... and adds each sum with one atomic
            const int nr = __popc(heads);
            const int r = __popc(heads & ((2u << lane) - 1u)) - 1;
            if (head) {
                s_run[wl][r] = lane;
                s_rkey[wl][r] = act ? key : 0xffffffffu;
            }
            if (lane == 0) s_run[wl][nr] = 32;
            __syncwarp();
            for (int item = lane; item < nr * NG; item += 32) {
                const int rr = item / NG, c = item - rr * NG;
                const unsigned k = s_rkey[wl][rr];
                if (k == 0xffffffffu) continue;
                const int lo = s_run[wl][rr], hi = s_run[wl][rr + 1];
                double acc = 0.0;
                for (int j = lo; j < hi; j++) acc += s_red[wl][c][j];
                if (acc != 0.0) atomicAdd(sgrad + (size_t)k * SG_STRIDE + c, acc);  // (component 12 = SG_GZ)
            }
            __syncwarp();
        }
#undef GF
    }
}

void launch_bwd_stream(const Cam& cam, const Opts& opt, const RecF* rec, const RecB* recb, const RecC* recc,
                       const FragRec* frec, const Counters* ctr, unsigned long long cap, const double* c_total,
                       const float* d_image, double* sgrad, cudaStream_t st, const long long* frag_off,
                       const double* frag_w, const double* fg_dw, const double* fg_dz, double* sw) {
    const dim3 grid(sm_count() * TS_BWD_GRID);
    if (!frag_off) {
        launch_pdl(k_bwd_stream<false>, grid, dim3(256), 0, st, cam, opt, rec, recb, recc, frec, ctr, cap, c_total,
                   d_image, sgrad, FragGrads{});
        return;
    }
    const long long npix = (long long)cam.width * cam.height;
    if (npix > 0) k_frag_suffix<<<(unsigned)((npix + 31) / 32), 256, 0, st>>>(npix, frag_off, frag_w, fg_dw, sw);
    launch_pdl(k_bwd_stream<true>, grid, dim3(256), 0, st, cam, opt, rec, recb, recc, frec, ctr, cap, c_total, d_image,
               sgrad, FragGrads{frag_off, fg_dw, fg_dz, sw});
}

}  // namespace ts
