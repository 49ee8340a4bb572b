// ts_exact.cu -- fp64 kernels that reproduce the reference arithmetic exactly.
//
// Compiled with -fmad=false (and every op written with explicit _rn
// intrinsics in ts_common.cuh), so products and sums round separately as in
// the numba reference.  Kernels:
//   k_preprocess       render.py:159-190, 193-250, 271-273, 292-302; soup.py:67-77
//   k_blend_exact      _kernels.py:59-132 (+ stats of render.py:411-418)
//   k_blend_bwd_exact  _kernels.py:181-318
//   k_chain_bwd        backward.py:59-90, 158-210; sh.py:55-100
#include "ts_kernels.cuh"

namespace ts {

// ---------------------------------------------------------------------------
// k_preprocess: one thread per source triangle.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_preprocess(Cam cam, Opts opt, const T* __restrict__ verts,
                                                    const T* __restrict__ opacity,
                                                    const T* __restrict__ sigma,
                                                    const T* __restrict__ sh, long long n,
                                                    PreOut out) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = false;
    unsigned long long key = 0;
    unsigned tcount = 0;
    if (i < n) {
        double v[9];
#pragma unroll
        for (int k = 0; k < 9; k++) v[k] = (double)verts[i * 9 + k];
        double o_raw = (double)opacity[i];
        double sg = (double)sigma[i];
        if (opt.validate) {
            bool fv = true;
#pragma unroll
            for (int k = 0; k < 9; k++) fv &= isfinite(v[k]);
            if (!fv) atomicMin(&out.ctr->err[0], i);
            if (!isfinite(o_raw)) atomicMin(&out.ctr->err[1], i);
            if (!isfinite(sg)) atomicMin(&out.ctr->err[2], i);
            bool fs = true;
            for (int k = 0; k < 48; k++) fs &= isfinite((double)sh[i * 48 + k]);
            if (!fs) atomicMin(&out.ctr->err[3], i);
        }
        Proj64 p;
        project64(v, cam, p);
        if (out.area) out.area[i] = p.valid_z ? (float)p.area : 0.0f;
        if (out.depth) out.depth[i] = p.z;
        ok = accepted(p);
        short4 bb = make_short4(0, 0, 0, 0);
        if (ok) {
            double o = opt.solid ? 1.0 : o_raw;
            Edge64 E;
            edge_bbox64(p.q, p.phis, o, sg, opt.mode, opt.tau_cutoff, cam.width, cam.height, E);
            bb = make_short4((short)E.bb[0], (short)E.bb[1], (short)E.bb[2], (short)E.bb[3]);
            Rec64 r;
#pragma unroll
            for (int e = 0; e < 3; e++) {
                r.nx[e] = E.nx[e];
                r.ny[e] = E.ny[e];
                r.d[e] = E.d[e];
                r.qx[e] = p.q[e * 2];
                r.qy[e] = p.q[e * 2 + 1];
            }
            r.phis = p.phis;
            r.sig = sg;
            r.opa = o;
            r.bx0 = (int)E.bb[0];
            r.bx1 = (int)E.bb[1];
            r.by0 = (int)E.bb[2];
            r.by1 = (int)E.bb[3];
            r.esign = E.esign;
            r.pad[0] = r.pad[1] = r.pad[2] = 0;
            // view-dependent colour, render.py:292-302
            double u[3];
#pragma unroll
            for (int b = 0; b < 3; b++)
                u[b] = TS_S(TS_D(TS_A(TS_A(v[b], v[3 + b]), v[6 + b]), 3.0), cam.cc[b]);
            double un = __dsqrt_rn(TS_A(TS_A(TS_M(u[0], u[0]), TS_M(u[1], u[1])), TS_M(u[2], u[2])));
            un = un > 1e-12 ? un : 1e-12;
            double basis[16];
            sh_basis16(TS_D(u[0], un), TS_D(u[1], un), TS_D(u[2], un), basis);
            for (int ch = 0; ch < 3; ch++) {
                double acc = 0.0;
                for (int c = 0; c < opt.ncoef; c++)
                    acc = TS_A(acc, TS_M(basis[c], (double)sh[i * 48 + c * 3 + ch]));
                double raw = TS_A(acc, 0.5);
                r.rgb[ch] = raw < 0.0 ? 0.0 : (raw > 1.0 ? 1.0 : raw);
            }
            out.rec[i] = r;
            tcount = (unsigned)tiles_touched(r.bx0, r.bx1, r.by0, r.by1);
            key = (unsigned long long)__double_as_longlong(p.z);
        }
        out.bbox[i] = bb;
        out.flag[i] = ok ? 1u : 0u;
        out.tcount[i] = tcount;
        out.key[i] = key;
    }
    // block-aggregated counters
    unsigned long long kmin = ok ? key : ~0ull, kmax = ok ? key : 0ull;
    unsigned cnt = ok ? 1u : 0u;
    unsigned long long tc = tcount;
    for (int off = 16; off > 0; off >>= 1) {
        unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, off);
        unsigned long long b = __shfl_xor_sync(0xffffffffu, kmax, off);
        kmin = a < kmin ? a : kmin;
        kmax = b > kmax ? b : kmax;
        cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        tc += __shfl_xor_sync(0xffffffffu, tc, off);
    }
    if ((threadIdx.x & 31) == 0 && cnt) {
        atomicMin(&out.ctr->key_min, kmin);
        atomicMax(&out.ctr->key_max, kmax);
        atomicAdd(&out.ctr->m, (unsigned long long)cnt);
        atomicAdd(&out.ctr->e, tc);
    }
}

void launch_preprocess(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                       const PreOut& out, cudaStream_t st) {
    long long n = soup.n;
    if (n <= 0) return;
    unsigned grid = (unsigned)((n + 255) / 256);
    if (dtype == 1)
        k_preprocess<double><<<grid, 256, 0, st>>>(cam, opt, (const double*)soup.vertices,
                                                   (const double*)soup.opacity,
                                                   (const double*)soup.sigma,
                                                   (const double*)soup.sh, n, out);
    else
        k_preprocess<float><<<grid, 256, 0, st>>>(cam, opt, (const float*)soup.vertices,
                                                  (const float*)soup.opacity,
                                                  (const float*)soup.sigma, (const float*)soup.sh,
                                                  n, out);
}

// ---------------------------------------------------------------------------
// k_blend_exact: one CTA per 16x16 tile, one thread per pixel, fp64.
// ---------------------------------------------------------------------------
constexpr int BATCH = 32;

__global__ void __launch_bounds__(256) k_blend_exact(Cam cam, Opts opt, const Rec64* __restrict__ rec,
                                                     const int* __restrict__ tile_start,
                                                     const int* __restrict__ ent_src,
                                                     BlendOut out) {
    __shared__ Rec64 s_rec[BATCH];
    __shared__ int s_src[BATCH];
    __shared__ unsigned s_maxw[BATCH];
    __shared__ int s_pix[BATCH];
    const int t = blockIdx.x;
    const int tx = t % cam.ntx, ty = t / cam.ntx;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int px = tx * TILE + lx, py = ty * TILE + ly;
    const bool inside = px < cam.width && py < cam.height;
    const double pcx = px + 0.5, pcy = py + 0.5;
    double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
    int last = -1, cnt = 0;
    bool done = !inside;
    const int s = tile_start[t], e = tile_start[t + 1];
    const unsigned lane = threadIdx.x & 31;
    if (threadIdx.x < BATCH) { s_maxw[threadIdx.x] = 0u; s_pix[threadIdx.x] = 0; }
    for (int b = s; b < e; b += BATCH) {
        if (__syncthreads_count(!done) == 0) break;
        int nb = min(BATCH, e - b);
        if (threadIdx.x < nb) {
            int src = ent_src[b + threadIdx.x];
            s_src[threadIdx.x] = src;
            s_rec[threadIdx.x] = rec[src];
        }
        __syncthreads();
        for (int j = 0; j < nb; j++) {
            const Rec64& r = s_rec[j];
            bool contrib = false;
            double w = 0.0;
            if (!done && px >= r.bx0 && px < r.bx1 && py >= r.by0 && py < r.by1) {
                double rr, phi;
                int edge;
                double alpha = fragment_alpha64(pcx, pcy, r, opt.mode, rr, phi, edge);
                if (alpha > ALPHA_CLAMP) alpha = ALPHA_CLAMP;
                if (alpha >= ALPHA_MIN) {
                    w = TS_M(T, alpha);
                    C0 = TS_A(C0, TS_M(w, r.rgb[0]));
                    C1 = TS_A(C1, TS_M(w, r.rgb[1]));
                    C2 = TS_A(C2, TS_M(w, r.rgb[2]));
                    contrib = true;
                    last = b + j;
                    cnt++;
                    T = TS_M(T, TS_S(1.0, alpha));
                    if (T < T_MIN) done = true;
                }
            }
            unsigned any = __ballot_sync(0xffffffffu, contrib);
            if (any) {
                unsigned wb = contrib ? __float_as_uint((float)w) : 0u;
                unsigned mx = __reduce_max_sync(0xffffffffu, wb);
                unsigned pc = __popc(__ballot_sync(0xffffffffu, contrib && w > opt.tau_contrib));
                if (lane == 0) {
                    atomicMax(&s_maxw[j], mx);
                    if (pc) atomicAdd(&s_pix[j], (int)pc);
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < nb) {
            int src = s_src[threadIdx.x];
            if (s_maxw[threadIdx.x] && out.max_weight)
                atomicMax((unsigned*)out.max_weight + src, s_maxw[threadIdx.x]);
            if (s_pix[threadIdx.x] && out.pixel_count)
                atomicAdd(out.pixel_count + src, s_pix[threadIdx.x]);
            s_maxw[threadIdx.x] = 0u;
            s_pix[threadIdx.x] = 0;
        }
    }
    if (inside) {
        int p = py * cam.width + px;
        double i0 = TS_A(C0, TS_M(T, opt.bg[0]));
        double i1 = TS_A(C1, TS_M(T, opt.bg[1]));
        double i2 = TS_A(C2, TS_M(T, opt.bg[2]));
        if (out.image) {
            out.image[p * 3 + 0] = (float)fmin(fmax(i0, 0.0), 1.0);
            out.image[p * 3 + 1] = (float)fmin(fmax(i1, 0.0), 1.0);
            out.image[p * 3 + 2] = (float)fmin(fmax(i2, 0.0), 1.0);
        }
        if (out.alpha_map) out.alpha_map[p] = (float)TS_S(1.0, T);
        out.t_final[p] = T;
        out.last_pos[p] = last;
        if (out.n_frag) out.n_frag[p] = cnt;
        if (out.last_src) out.last_src[p] = last >= 0 ? ent_src[last] : -1;
    }
}

void launch_blend_exact(const Cam& cam, const Opts& opt, const Rec64* rec, const int* tile_start,
                        const int* ent_src, const BlendOut& out, cudaStream_t st) {
    int ntiles = cam.ntx * cam.nty;
    k_blend_exact<<<ntiles, 256, 0, st>>>(cam, opt, rec, tile_start, ent_src, out);
}

// ---------------------------------------------------------------------------
// k_blend_bwd_exact: back-to-front from the saved last contributor.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

__global__ void __launch_bounds__(256) k_blend_bwd_exact(Cam cam, Opts opt, const Rec64* __restrict__ rec,
                                                         const int* __restrict__ tile_start,
                                                         const int* __restrict__ ent_src,
                                                         const double* __restrict__ t_final,
                                                         const int* __restrict__ last_pos,
                                                         const float* __restrict__ d_image,
                                                         double* __restrict__ sgrad) {
    __shared__ Rec64 s_rec[BATCH];
    __shared__ int s_src[BATCH];
    __shared__ int s_hi;
    const int t = blockIdx.x;
    const int tx = t % cam.ntx, ty = t / cam.ntx;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int px = tx * TILE + lx, py = ty * TILE + ly;
    const bool inside = px < cam.width && py < cam.height;
    const double pcx = px + 0.5, pcy = py + 0.5;
    const unsigned lane = threadIdx.x & 31;
    const int s = tile_start[t];
    int my_last = -1;
    double T = 1.0, d0 = 0.0, d1 = 0.0, d2 = 0.0;
    if (inside) {
        int p = py * cam.width + px;
        my_last = last_pos[p];
        T = t_final[p];
        d0 = d_image[p * 3 + 0];
        d1 = d_image[p * 3 + 1];
        d2 = d_image[p * 3 + 2];
    }
    double S0 = TS_M(T, opt.bg[0]), S1 = TS_M(T, opt.bg[1]), S2 = TS_M(T, opt.bg[2]);
    if (threadIdx.x == 0) s_hi = -1;
    __syncthreads();
    if (my_last >= 0) atomicMax(&s_hi, my_last);
    __syncthreads();
    const int hi = s_hi;
    for (int bend = hi + 1; bend > s; bend -= BATCH) {
        int bstart = max(s, bend - BATCH);
        int nb = bend - bstart;
        __syncthreads();
        if (threadIdx.x < nb) {
            int src = ent_src[bstart + threadIdx.x];
            s_src[threadIdx.x] = src;
            s_rec[threadIdx.x] = rec[src];
        }
        __syncthreads();
        for (int j = nb - 1; j >= 0; j--) {
            const Rec64& r = s_rec[j];
            const int pos = bstart + j;
            double g[12];
#pragma unroll
            for (int k = 0; k < 12; k++) g[k] = 0.0;
            bool act = false;
            if (pos <= my_last && px >= r.bx0 && px < r.bx1 && py >= r.by0 && py < r.by1) {
                double rr, phi;
                int edge;
                double alpha = fragment_alpha64(pcx, pcy, r, opt.mode, rr, phi, edge);
                bool clamped = false;
                if (alpha > ALPHA_CLAMP) { alpha = ALPHA_CLAMP; clamped = true; }
                if (alpha >= ALPHA_MIN) {
                    act = true;
                    double one_m = TS_S(1.0, alpha);
                    double tb = TS_D(T, one_m);
                    double w = TS_M(tb, alpha);
                    g[SG_GRGB + 0] = TS_M(w, d0);
                    g[SG_GRGB + 1] = TS_M(w, d1);
                    g[SG_GRGB + 2] = TS_M(w, d2);
                    double ga = TS_M(d0, TS_S(TS_M(tb, r.rgb[0]), TS_D(S0, one_m)));
                    ga = TS_A(ga, TS_M(d1, TS_S(TS_M(tb, r.rgb[1]), TS_D(S1, one_m))));
                    ga = TS_A(ga, TS_M(d2, TS_S(TS_M(tb, r.rgb[2]), TS_D(S2, one_m))));
                    S0 = TS_A(S0, TS_M(w, r.rgb[0]));
                    S1 = TS_A(S1, TS_M(w, r.rgb[1]));
                    S2 = TS_A(S2, TS_M(w, r.rgb[2]));
                    T = tb;
                    if (!clamped) {
                        g[SG_GO] = TS_M(ga, TS_D(alpha, r.opa));
                        double g_win = TS_M(r.opa, ga);
                        double g_phi;
                        if (opt.mode == 0) {
                            double window = pow(rr, r.sig);
                            g[SG_GSIG] = TS_M(TS_M(g_win, window), log(rr));
                            double g_r = TS_M(TS_M(g_win, r.sig), pow(rr, TS_S(r.sig, 1.0)));
                            if (rr >= 1.0) {
                                g_phi = 0.0;
                            } else {
                                g_phi = TS_D(g_r, r.phis);
                                g[SG_GPHIS] = TS_D(TS_M(-g_r, phi), TS_M(r.phis, r.phis));
                            }
                        } else {
                            double window = rr;
                            g[SG_GSIG] = TS_D(TS_M(TS_M(TS_M(g_win, window), TS_S(1.0, window)), phi),
                                              TS_M(r.sig, r.sig));
                            g_phi = TS_D(TS_M(TS_M(-g_win, window), TS_S(1.0, window)), r.sig);
                        }
                        int ia = edge, ib = (edge + 1) % 3;
                        double ax = r.qx[ia], ay = r.qy[ia], bx = r.qx[ib], by = r.qy[ib];
                        double ex = TS_S(bx, ax), ey = TS_S(by, ay);
                        double ell = __dsqrt_rn(TS_A(TS_M(ex, ex), TS_M(ey, ey)));
                        double sgn = ((r.esign >> edge) & 1) ? -1.0 : 1.0;
                        double inv_l = TS_D(1.0, ell);
                        double inv_l2 = TS_M(inv_l, inv_l);
                        double gax = TS_S(TS_M(TS_M(sgn, TS_S(pcy, by)), inv_l), TS_M(TS_M(phi, TS_S(ax, bx)), inv_l2));
                        double gay = TS_S(TS_M(TS_M(sgn, TS_S(bx, pcx)), inv_l), TS_M(TS_M(phi, TS_S(ay, by)), inv_l2));
                        double gbx = TS_S(TS_M(TS_M(sgn, TS_S(ay, pcy)), inv_l), TS_M(TS_M(phi, TS_S(bx, ax)), inv_l2));
                        double gby = TS_S(TS_M(TS_M(sgn, TS_S(pcx, ax)), inv_l), TS_M(TS_M(phi, TS_S(by, ay)), inv_l2));
                        g[SG_GQ + ia * 2] = TS_M(g_phi, gax);
                        g[SG_GQ + ia * 2 + 1] = TS_M(g_phi, gay);
                        g[SG_GQ + ib * 2] = TS_M(g_phi, gbx);
                        g[SG_GQ + ib * 2 + 1] = TS_M(g_phi, gby);
                    }
                }
            }
            if (__any_sync(0xffffffffu, act)) {
#pragma unroll
                for (int k = 0; k < 12; k++) g[k] = warp_sum(g[k]);
                if (lane == 0) {
                    double* dst = sgrad + (size_t)s_src[j] * SG_STRIDE;
#pragma unroll
                    for (int k = 0; k < 12; k++)
                        if (g[k] != 0.0) atomicAdd(dst + k, g[k]);
                }
            }
        }
    }
}

void launch_blend_bwd_exact(const Cam& cam, const Opts& opt, const Rec64* rec, const int* tile_start,
                            const int* ent_src, const double* t_final, const int* last_pos,
                            const float* d_image, double* sgrad, cudaStream_t st) {
    int ntiles = cam.ntx * cam.nty;
    k_blend_bwd_exact<<<ntiles, 256, 0, st>>>(cam, opt, rec, tile_start, ent_src, t_final, last_pos,
                                              d_image, sgrad);
}

// ---------------------------------------------------------------------------
// k_chain_bwd: screen-space grads -> 59 parameter grads, one thread per source.
// ---------------------------------------------------------------------------
template <typename T, typename G>
__global__ void __launch_bounds__(128) k_chain_bwd(Cam cam, Opts opt, const T* __restrict__ verts,
                                                   const T* __restrict__ sh,
                                                   const unsigned* __restrict__ flag,
                                                   const G* __restrict__ sgrad, long long n,
                                                   ts_grads grads, int accumulate) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double dv[9], dsh[48], dop = 0.0, dsig = 0.0;
#pragma unroll
    for (int k = 0; k < 9; k++) dv[k] = 0.0;
#pragma unroll
    for (int k = 0; k < 48; k++) dsh[k] = 0.0;
    if (flag[i]) {
        const G* sg = sgrad + (size_t)i * SG_STRIDE;
        double gq[6];
#pragma unroll
        for (int k = 0; k < 6; k++) gq[k] = sg[SG_GQ + k];
        dop = sg[SG_GO];
        dsig = sg[SG_GSIG];
        double grgb[3] = {sg[SG_GRGB], sg[SG_GRGB + 1], sg[SG_GRGB + 2]};
        double gphis = sg[SG_GPHIS], gz = sg[SG_GZ];
        double v[9];
#pragma unroll
        for (int k = 0; k < 9; k++) v[k] = (double)verts[i * 9 + k];
        Proj64 p;
        project64(v, cam, p);
        const double* q = p.q;
        if (opt.mode == 0) {
            // _phis_q_grad, backward.py:59-90
            double e1x = q[2] - q[0], e1y = q[3] - q[1];
            double e2x = q[4] - q[0], e2y = q[5] - q[1];
            double cross = e1x * e2y - e1y * e2x;
            double sgn = (cross > 0) - (cross < 0);
            double d12x = q[2] - q[4], d12y = q[3] - q[5];
            double d20x = q[4] - q[0], d20y = q[5] - q[1];
            double d01x = q[0] - q[2], d01y = q[1] - q[3];
            double perim = sqrt(d12x * d12x + d12y * d12y) + sqrt(d20x * d20x + d20y * d20y) +
                           sqrt(d01x * d01x + d01y * d01y);
            double area = fabs(cross) / 2.0;
            double dcross[6] = {q[3] - q[5], q[4] - q[2], q[5] - q[1],
                                q[0] - q[4], q[1] - q[3], q[2] - q[0]};
            double dperim[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int a = 0; a < 3; a++) {
#pragma unroll
                for (int jj = 1; jj <= 2; jj++) {
                    int b = (a + jj) % 3;
                    double dx = q[a * 2] - q[b * 2], dy = q[a * 2 + 1] - q[b * 2 + 1];
                    double nd = sqrt(dx * dx + dy * dy);
                    dperim[a * 2] += dx / nd;
                    dperim[a * 2 + 1] += dy / nd;
                }
            }
            double coef_a = -2.0 / perim;
            double coef_p = 2.0 * area / (perim * perim);
#pragma unroll
            for (int k = 0; k < 6; k++) gq[k] += gphis * (coef_a * (0.5 * sgn * dcross[k]) + coef_p * dperim[k]);
        }
        // projection Jacobian, backward.py:181-190
        double dxc[9];
#pragma unroll
        for (int k = 0; k < 3; k++) {
            double zc = p.xc[k * 3 + 2];
            dxc[k * 3 + 0] = cam.fx * gq[k * 2] / zc;
            dxc[k * 3 + 1] = cam.fy * gq[k * 2 + 1] / zc;
            dxc[k * 3 + 2] = (-cam.fx * p.xc[k * 3] * gq[k * 2] - cam.fy * p.xc[k * 3 + 1] * gq[k * 2 + 1]) / (zc * zc) +
                             gz / 3.0;
        }
#pragma unroll
        for (int k = 0; k < 3; k++)
#pragma unroll
            for (int b = 0; b < 3; b++)
                dv[k * 3 + b] = dxc[k * 3] * cam.R[b] + dxc[k * 3 + 1] * cam.R[3 + b] + dxc[k * 3 + 2] * cam.R[6 + b];
        // colour path, backward.py:192-205
        double u[3];
#pragma unroll
        for (int b = 0; b < 3; b++)
            u[b] = TS_S(TS_D(TS_A(TS_A(v[b], v[3 + b]), v[6 + b]), 3.0), cam.cc[b]);
        double un = __dsqrt_rn(TS_A(TS_A(TS_M(u[0], u[0]), TS_M(u[1], u[1])), TS_M(u[2], u[2])));
        un = un > 1e-12 ? un : 1e-12;
        double vd[3] = {TS_D(u[0], un), TS_D(u[1], un), TS_D(u[2], un)};
        double basis[16];
        sh_basis16(vd[0], vd[1], vd[2], basis);
        double coef[48];
        for (int k = 0; k < 48; k++) coef[k] = (double)sh[i * 48 + k];
        double d_raw[3];
        for (int ch = 0; ch < 3; ch++) {
            double acc = 0.0;
            for (int c = 0; c < opt.ncoef; c++) acc = TS_A(acc, TS_M(basis[c], coef[c * 3 + ch]));
            double raw = TS_A(acc, 0.5);
            d_raw[ch] = (raw > 0.0 && raw < 1.0) ? grgb[ch] : 0.0;
        }
        for (int c = 0; c < opt.ncoef; c++)
            for (int ch = 0; ch < 3; ch++) dsh[c * 3 + ch] = basis[c] * d_raw[ch];
        double gb[16][3];
        sh_basis_grad16(vd[0], vd[1], vd[2], gb);
        double ddir[3];
        for (int dd = 0; dd < 3; dd++) {
            double acc = 0.0;
            for (int ch = 0; ch < 3; ch++)
                for (int c = 0; c < opt.ncoef; c++) acc += d_raw[ch] * coef[c * 3 + ch] * gb[c][dd];
            ddir[dd] = acc;
        }
        double dot = vd[0] * ddir[0] + vd[1] * ddir[1] + vd[2] * ddir[2];
#pragma unroll
        for (int b = 0; b < 3; b++) {
            double du = (ddir[b] - vd[b] * dot) / un;
#pragma unroll
            for (int k = 0; k < 3; k++) dv[k * 3 + b] += du / 3.0;
        }
    }
    float* gv = grads.d_vertices + i * 9;
    float* gs = grads.d_sh + i * 48;
    if (accumulate) {
#pragma unroll
        for (int k = 0; k < 9; k++) gv[k] += (float)dv[k];
        grads.d_opacity[i] += (float)dop;
        grads.d_sigma[i] += (float)dsig;
        for (int k = 0; k < 48; k++) gs[k] += (float)dsh[k];
    } else {
#pragma unroll
        for (int k = 0; k < 9; k++) gv[k] = (float)dv[k];
        grads.d_opacity[i] = (float)dop;
        grads.d_sigma[i] = (float)dsig;
        for (int k = 0; k < 48; k++) gs[k] = (float)dsh[k];
    }
}

template <typename G>
static void chain_impl(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                       const unsigned* flag, const G* sgrad, const ts_grads& g, int accumulate,
                       cudaStream_t st) {
    long long n = soup.n;
    if (n <= 0) return;
    unsigned grid = (unsigned)((n + 127) / 128);
    if (dtype == 1)
        k_chain_bwd<double, G><<<grid, 128, 0, st>>>(cam, opt, (const double*)soup.vertices,
                                                     (const double*)soup.sh, flag, sgrad, n, g,
                                                     accumulate);
    else
        k_chain_bwd<float, G><<<grid, 128, 0, st>>>(cam, opt, (const float*)soup.vertices,
                                                    (const float*)soup.sh, flag, sgrad, n, g,
                                                    accumulate);
}

void launch_chain_bwd(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                      const unsigned* flag, const double* sgrad, const ts_grads& g, int accumulate,
                      cudaStream_t st) {
    chain_impl<double>(cam, opt, soup, dtype, flag, sgrad, g, accumulate, st);
}

void launch_chain_bwd32(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                        const unsigned* flag, const float* sgrad, const ts_grads& g, int accumulate,
                        cudaStream_t st) {
    chain_impl<float>(cam, opt, soup, dtype, flag, sgrad, g, accumulate, st);
}


// ---------------------------------------------------------------------------
// k_projection_dump: project_scene (render.py:253-312) for the depth-sorted
// accepted triangles of the last forward, every field of SceneProjection in
// the reference's fp64 operation order (this TU has no FMA contraction).
// Row m (PROJ_ROW doubles) of `rows`: xc[9] q[6] z area phis nrm[6] doff[3]
// esign[3] sig opa rgb[3] raw_rgb[3] basis[16] viewdir[3] u_norm bbox[4];
// area_full[i] for every source (render.py:271-272).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(128) k_projection_dump(Cam cam, Opts opt, const T* __restrict__ verts,
                                                         const T* __restrict__ opacity,
                                                         const T* __restrict__ sigma, const T* __restrict__ sh,
                                                         const unsigned* __restrict__ sorted_src, long long m,
                                                         long long n, double* __restrict__ rows,
                                                         double* __restrict__ area_full) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) {
        double v[9];
#pragma unroll
        for (int a = 0; a < 9; a++) v[a] = (double)verts[k * 9 + a];
        Proj64 p;
        project64(v, cam, p);
        area_full[k] = p.valid_z ? p.area : 0.0;
    }
    if (k >= m) return;
    const long long i = sorted_src[k];
    double v[9];
#pragma unroll
    for (int a = 0; a < 9; a++) v[a] = (double)verts[i * 9 + a];
    Proj64 p;
    project64(v, cam, p);
    const double o = opt.solid ? 1.0 : (double)opacity[i];
    const double sg = (double)sigma[i];
    Edge64 E;
    edge_bbox64(p.q, p.phis, o, sg, opt.mode, opt.tau_cutoff, cam.width, cam.height, E);
    double* r = rows + k * PROJ_ROW;
    int c = 0;
#pragma unroll
    for (int a = 0; a < 9; a++) r[c++] = p.xc[a];
#pragma unroll
    for (int a = 0; a < 6; a++) r[c++] = p.q[a];
    r[c++] = p.z;
    r[c++] = p.area;
    r[c++] = p.phis;
#pragma unroll
    for (int e = 0; e < 3; e++) {
        r[c++] = E.nx[e];
        r[c++] = E.ny[e];
    }
#pragma unroll
    for (int e = 0; e < 3; e++) r[c++] = E.d[e];
#pragma unroll
    for (int e = 0; e < 3; e++) r[c++] = ((E.esign >> e) & 1) ? -1.0 : 1.0;
    r[c++] = sg;
    r[c++] = o;
    // view direction from the camera centre to the world centroid, SH colour
    double u[3];
#pragma unroll
    for (int b = 0; b < 3; b++) u[b] = TS_S(TS_D(TS_A(TS_A(v[b], v[3 + b]), v[6 + b]), 3.0), cam.cc[b]);
    double un = __dsqrt_rn(TS_A(TS_A(TS_M(u[0], u[0]), TS_M(u[1], u[1])), TS_M(u[2], u[2])));
    un = un > 1e-12 ? un : 1e-12;
    const double dir[3] = {TS_D(u[0], un), TS_D(u[1], un), TS_D(u[2], un)};
    double basis[16];
    sh_basis16(dir[0], dir[1], dir[2], basis);
    double raw[3];
    for (int ch = 0; ch < 3; ch++) {
        double acc = 0.0;
        for (int cc = 0; cc < opt.ncoef; cc++) acc = TS_A(acc, TS_M(basis[cc], (double)sh[i * 48 + cc * 3 + ch]));
        raw[ch] = TS_A(acc, 0.5);
    }
#pragma unroll
    for (int ch = 0; ch < 3; ch++) r[c++] = raw[ch] < 0.0 ? 0.0 : (raw[ch] > 1.0 ? 1.0 : raw[ch]);
#pragma unroll
    for (int ch = 0; ch < 3; ch++) r[c++] = raw[ch];
#pragma unroll
    for (int a = 0; a < 16; a++) r[c++] = basis[a];
#pragma unroll
    for (int b = 0; b < 3; b++) r[c++] = dir[b];
    r[c++] = un;
#pragma unroll
    for (int a = 0; a < 4; a++) r[c++] = (double)E.bb[a];
    while (c < PROJ_ROW) r[c++] = 0.0;
}

void launch_projection_dump(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                            const unsigned* sorted_src, long long m, double* rows, double* area_full,
                            cudaStream_t st) {
    const long long n = soup.n;
    const long long cnt = n > m ? n : m;
    if (cnt <= 0) return;
    const unsigned grid = (unsigned)((cnt + 127) / 128);
    if (dtype == 1)
        k_projection_dump<double><<<grid, 128, 0, st>>>(cam, opt, (const double*)soup.vertices,
                                                        (const double*)soup.opacity, (const double*)soup.sigma,
                                                        (const double*)soup.sh, sorted_src, m, n, rows, area_full);
    else
        k_projection_dump<float><<<grid, 128, 0, st>>>(cam, opt, (const float*)soup.vertices,
                                                       (const float*)soup.opacity, (const float*)soup.sigma,
                                                       (const float*)soup.sh, sorted_src, m, n, rows, area_full);
}

}  // namespace ts
