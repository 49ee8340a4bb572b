// ts_fast.cu -- the fast (default) path: fp64 edge functions, fp32 alpha and
// compositing, with a guard band around every discrete decision of the
// reference compositor and an exact fp64 fix-up for the rare pixels whose
// decision falls inside it.
//
//   k_preprocess_fast  render.py:159-190, 193-250, 271-273, 292-302 -> RecF/RecB
//   k_blend_fast       _kernels.py:59-132 (decisions: skip alpha<1/255 :103,
//                      T<1e-4 stop :121, pixel count w>1/255 :112)
//   k_fixup_fwd        exact replay (same arithmetic as k_blend_exact) of flagged pixels
//   k_blend_bwd_fast   _kernels.py:181-318 back to front from the saved last contributor
//
// Decision guard band.  r = phi/phi_s is evaluated in fp64 from fp64 edge
// coefficients (error ~1e-12 vs the reference's fp64 phi/phi_s), so the skip
// test r >= r* is exact outside the fp32-rounded band [r_lo, r_hi]; inside
// it the decision is taken with the reference's fp64 arithmetic.  Alpha is
// then computed in fp32 with a per-fragment relative error bound eps_a, and
// the transmittance carries its accumulated relative error bound eps_T; a
// T<1e-4 or w>1/255 test whose operands lie within their error bound of the
// threshold flags the pixel, which stops here and is recomputed exactly by
// k_fixup_fwd.
#include "ts_kernels.cuh"

namespace ts {

constexpr float T_MIN_F = 1e-4f;
constexpr float ALPHA_CLAMP_F = 0.99f;

__device__ __forceinline__ float fast_lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fast_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---------------------------------------------------------------------------
// preprocess (fast records)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_preprocess_fast(Cam cam, Opts opt, const T* __restrict__ verts,
                                                         const T* __restrict__ opacity,
                                                         const T* __restrict__ sigma,
                                                         const T* __restrict__ sh, long long n,
                                                         FastPreOut out) {
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
            const T* shp = sh + i * 48;
#pragma unroll 8
            for (int k = 0; k < 48; k++) fs &= isfinite((double)shp[k]);
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
            int x0 = (int)E.bb[0], x1 = (int)E.bb[1], y0 = (int)E.bb[2], y1 = (int)E.bb[3];
            bb = make_short4((short)x0, (short)x1, (short)y0, (short)y1);
            tcount = (unsigned)tiles_touched(x0, x1, y0, y1);
            if (tcount) {
                RecF r;
                int ox = (x0 + x1) >> 1, oy = (y0 + y1) >> 1;
                double inv = 1.0 / p.phis;
                double dmax = 0.0;
#pragma unroll
                for (int e = 0; e < 3; e++) {
                    r.a[e * 3 + 0] = E.nx[e] * inv;
                    r.a[e * 3 + 1] = E.ny[e] * inv;
                    r.a[e * 3 + 2] = E.d[e] * inv;
                    dmax = fmax(dmax, fabs(E.d[e]));
                }
                // |r_fast - r_ref| bound: both are O(1e-16) x (sum of |terms| / |phi_s|)
                double mag = (fabs(p.q[0]) + fabs(p.q[1]) + fabs(p.q[2]) + fabs(p.q[3]) + fabs(p.q[4]) +
                              fabs(p.q[5]) + 4.0 * (cam.width + cam.height) + dmax) / fabs(p.phis);
                double delta = 1e-13 * mag + 1e-300;
                double rstar;  // contribution threshold on r (alpha >= 1/255)
                if (opt.mode == 0) {
                    rstar = o > ALPHA_MIN ? pow(ALPHA_MIN / o, 1.0 / sg) : 1e30;
                    if (rstar > 1.0) rstar = 1e30;
                    r.f0 = (float)sg;
                    r.f1 = (float)log2(o);
                } else {
                    double q = 255.0 * o - 1.0;
                    rstar = q > 0.0 ? sg * log(q) / p.phis : 1e30;
                    r.f0 = (float)(p.phis * 1.4426950408889634 / sg);
                    r.f1 = (float)o;
                }
                r.r_lo = rstar - delta - fabs(rstar) * 1e-12;
                r.r_hi = rstar + delta + fabs(rstar) * 1e-12;
                // view-dependent colour, render.py:292-302
                double u[3];
#pragma unroll
                for (int b = 0; b < 3; b++) u[b] = (v[b] + v[3 + b] + v[6 + b]) / 3.0 - cam.cc[b];
                double un = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
                un = un > 1e-12 ? un : 1e-12;
                double basis[16];
                sh_basis16(u[0] / un, u[1] / un, u[2] / un, basis);
                const T* shp = sh + i * 48;
                double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
                for (int c = 0; c < opt.ncoef; c++) {
                    acc0 += basis[c] * (double)shp[c * 3 + 0];
                    acc1 += basis[c] * (double)shp[c * 3 + 1];
                    acc2 += basis[c] * (double)shp[c * 3 + 2];
                }
                r.rgb[0] = (float)fmin(fmax(acc0 + 0.5, 0.0), 1.0);
                r.rgb[1] = (float)fmin(fmax(acc1 + 0.5, 0.0), 1.0);
                r.rgb[2] = (float)fmin(fmax(acc2 + 0.5, 0.0), 1.0);
                r.x0 = (short)x0; r.x1 = (short)x1; r.y0 = (short)y0; r.y1 = (short)y1;
                r.ox = (short)ox; r.oy = (short)oy;
                r.phis = p.phis;
                out.rec[i] = r;
                if (out.recb) {
                    RecB b;
#pragma unroll
                    for (int e = 0; e < 3; e++) {
                        b.qx[e] = (float)(p.q[e * 2] - ox);
                        b.qy[e] = (float)(p.q[e * 2 + 1] - oy);
                    }
                    b.phis = (float)p.phis;
                    b.opa = (float)o;
                    b.sig = (float)sg;
                    b.esign = E.esign;
                    b.pad[0] = b.pad[1] = 0.f;
                    out.recb[i] = b;
                }
            }
            key = (unsigned long long)__double_as_longlong(p.z);
        }
        out.bbox[i] = bb;
        out.flag[i] = ok ? 1u : 0u;
        out.tcount[i] = tcount;
        out.key[i] = key;
    }
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

void launch_preprocess_fast(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                            const FastPreOut& out, cudaStream_t st) {
    long long n = soup.n;
    if (n <= 0) return;
    unsigned grid = (unsigned)((n + 255) / 256);
    if (dtype == 1)
        k_preprocess_fast<double><<<grid, 256, 0, st>>>(cam, opt, (const double*)soup.vertices,
                                                        (const double*)soup.opacity,
                                                        (const double*)soup.sigma,
                                                        (const double*)soup.sh, n, out);
    else
        k_preprocess_fast<float><<<grid, 256, 0, st>>>(cam, opt, (const float*)soup.vertices,
                                                       (const float*)soup.opacity,
                                                       (const float*)soup.sigma,
                                                       (const float*)soup.sh, n, out);
}

// ---------------------------------------------------------------------------
// shared per-fragment evaluation
// ---------------------------------------------------------------------------
__device__ __forceinline__ double edge_r(const RecF& r, double pcx, double pcy, int& arg) {
    const double dx = pcx, dy = pcy;
    double l0 = fma(r.a[0], dx, fma(r.a[1], dy, r.a[2]));
    double l1 = fma(r.a[3], dx, fma(r.a[4], dy, r.a[5]));
    double l2 = fma(r.a[6], dx, fma(r.a[7], dy, r.a[8]));
    // argmax of phi = argmin of phi/phi_s (phi_s < 0); ties -> lowest edge (strict >, _kernels.py:36-42)
    double m = l0;
    arg = 0;
    if (l1 < m) { m = l1; arg = 1; }
    if (l2 < m) { m = l2; arg = 2; }
    return m;
}

__device__ __forceinline__ double edge_r(const RecF& r, double pcx, double pcy) {
    const double dx = pcx, dy = pcy;
    double l0 = fma(r.a[0], dx, fma(r.a[1], dy, r.a[2]));
    double l1 = fma(r.a[3], dx, fma(r.a[4], dy, r.a[5]));
    double l2 = fma(r.a[6], dx, fma(r.a[7], dy, r.a[8]));
    return fmin(l0, fmin(l1, l2));
}

// fp32 alpha (unclamped) and its relative error bound, given r above the band
__device__ __forceinline__ float alpha_fast(const RecF& r, double rr, int mode, float& eps) {
    if (mode == 0) {
        float rf = (float)fmin(rr, 1.0);
        float lg = fast_lg2(rf);
        float arg = fmaf(r.f0, lg, r.f1);
        float a = fast_ex2(arg);
        eps = 5e-7f + r.f0 * (6e-7f + 2.4e-7f * fabsf(lg)) + 1.2e-7f * fabsf(arg);
        return a;
    } else {
        float x = (float)rr * r.f0;  // phi/sigma * log2(e)
        float ex = fast_ex2(fminf(x, 1009.9f));
        float a = __fdividef(r.f1, 1.0f + ex);
        eps = 8e-7f + 1.2e-7f * fabsf(x);
        return a;
    }
}

// fp64 alpha from the fp64 r (the reference's fragment_alpha, _kernels.py:43-56,
// with phi = r * phi_s); used for decisions inside the guard band.  Opacity and
// sigma are read from the caller's parameter arrays so they are exact for
// fp32 and fp64 parameters alike.
template <typename T>
__device__ __forceinline__ double alpha_exact_r(const RecF& r, double rr, int mode, const Opts& opt,
                                                const T* __restrict__ opacity, const T* __restrict__ sigma,
                                                unsigned src) {
    const double o = opt.solid ? 1.0 : (double)opacity[src];
    const double sg = (double)sigma[src];
    double window;
    if (mode == 0) {
        if (rr <= 0.0) return 0.0;  // phi >= 0
        window = pow(fmin(rr, 1.0), sg);
    } else {
        double x = rr * r.phis / sg;
        if (x > 700.0) x = 700.0;
        window = 1.0 / (1.0 + exp(x));
    }
    return o * window;
}

// ---------------------------------------------------------------------------
// k_blend_fast: CTA per 16x16 tile, two balanced phases per batch of FB
// depth-ordered tile entries (render.py:349-361 order):
//
//  B. dense evaluation -- the batch's (entry, pixel) pairs with the pixel in
//     the entry's bbox (the reference's per-pixel bbox test, _kernels.py:87-95)
//     are enumerated as one flat range; each thread takes a contiguous slice
//     (merge-path split, record cached in registers while the entry repeats),
//     evaluates phi/phi_s in fp64 and, for contributing fragments, alpha in
//     fp32; results go to small per-pixel slot lists in shared memory.
//  C. compositing -- thread = pixel, walks only its slots in entry order
//     (front to back, _kernels.py:96-123): weight, colour, transmittance,
//     early stop, per-entry statistics, and the decision guard band.
//
// A pixel whose slot list overflows, or whose decision lands inside the guard
// band, is flagged and recomputed exactly by k_fixup_fwd.
// ---------------------------------------------------------------------------
constexpr int FB = 64;       // entries staged per batch
constexpr int PMAX = 4096;   // (entry, pixel) pairs per batch
constexpr int NSLOT = 12;    // contributing fragments per pixel per batch
constexpr int SREC_W = 36;   // staged record stride in 32-bit words (144 B: conflict-free broadcasts)

__global__ void __launch_bounds__(256) k_blend_fast(Cam cam, Opts opt, const RecF* __restrict__ rec,
                                                    const short4* __restrict__ bbox,
                                                    const int* __restrict__ tile_start,
                                                    const unsigned* __restrict__ ent_src,
                                                    FastBlendOut out) {
    (void)bbox;
    __shared__ __align__(16) unsigned s_rec[FB * SREC_W];
    __shared__ unsigned s_src[FB];
    __shared__ int s_geo[FB];                 // cx0 | w << 8 | ry0 << 16
    __shared__ int s_pre[FB + 1];             // exclusive prefix of pair counts
    extern __shared__ __align__(16) unsigned char s_dyn[];
    float* s_wr = reinterpret_cast<float*>(s_dyn);                                  // [PMAX] r, NaN: band
    float (*s_sa)[TILE_PIX] = reinterpret_cast<float (*)[TILE_PIX]>(s_wr + PMAX);   // [NSLOT][256] alpha
    float (*s_se)[TILE_PIX] = s_sa + NSLOT;                                         // [NSLOT][256] eps
    unsigned short* s_wl = reinterpret_cast<unsigned short*>(s_se + NSLOT);        // [PMAX] candidates
    unsigned char* s_pe = reinterpret_cast<unsigned char*>(s_wl + PMAX);           // [PMAX] pair -> entry
    unsigned char* s_pp = s_pe + PMAX;                                              // [PMAX] pair -> pixel
    unsigned char (*s_sj)[TILE_PIX] = reinterpret_cast<unsigned char (*)[TILE_PIX]>(s_pp + PMAX);
    __shared__ int s_wn, s_nbe;
    __shared__ unsigned s_maxw[FB];
    __shared__ int s_pix[FB];
    __shared__ unsigned char s_done[TILE_PIX];
    __shared__ unsigned char s_ovf[TILE_PIX];
    __shared__ int s_cnt[TILE_PIX];

    const int t = blockIdx.x;
    const int tx = t % cam.ntx, ty = t / cam.ntx;
    const int TX0 = tx * TILE, TY0 = ty * TILE;
    const int tid = threadIdx.x;
    const unsigned lane = tid & 31;
    const int px = TX0 + (tid & 15), py = TY0 + (tid >> 4);
    const bool inside = px < cam.width && py < cam.height;
    float T = 1.f, C0 = 0.f, C1 = 0.f, C2 = 0.f, epsT = 0.f;
    int last = -1, cnt = 0, flag_pos = -1;
    bool done = !inside;
    s_done[tid] = done ? 1 : 0;
    s_ovf[tid] = 0;
    s_cnt[tid] = 0;
    const int s = tile_start[t], e = tile_start[t + 1];
    const float tau = (float)opt.tau_contrib;
    if (tid < FB) {
        s_maxw[tid] = 0u;
        s_pix[tid] = 0;
    }
    int b = s;
    while (b < e) {
        if (__syncthreads_count(!done) == 0) break;
        const int nb0 = min(FB, e - b);
        // ---- stage up to FB records (144-byte stride) ----
        for (int c = tid; c < nb0 * 8; c += 256) {
            const int j = c >> 3, q = c & 7;
            const unsigned src = __ldg(ent_src + b + j);
            const float4 v = __ldg(reinterpret_cast<const float4*>(rec + src) + q);
            *reinterpret_cast<float4*>(&s_rec[j * SREC_W + q * 4]) = v;
            if (q == 7) {
                s_src[j] = src;
                const int xx = __float_as_int(v.y), yy = __float_as_int(v.z);
                const int cx0 = max((int)(short)(xx & 0xffff) - TX0, 0), cx1 = min((int)(short)(xx >> 16) - TX0, TILE);
                const int ry0 = max((int)(short)(yy & 0xffff) - TY0, 0), ry1 = min((int)(short)(yy >> 16) - TY0, TILE);
                const int w = max(cx1 - cx0, 0), h = max(ry1 - ry0, 0);
                s_geo[j] = cx0 | (w << 8) | (ry0 << 16);
                s_pre[j + 1] = w * h;
            }
        }
        if (tid == 0) s_wn = 0;
        __syncthreads();
        if (tid < 32) {
            const int c0 = tid * 2 < nb0 ? s_pre[tid * 2 + 1] : 0;
            const int c1 = tid * 2 + 1 < nb0 ? s_pre[tid * 2 + 2] : 0;
            int x = c0 + c1;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, off);
                if ((int)lane >= off) x += y;
            }
            const int ex = x - c0 - c1;
            __syncwarp();
            s_pre[tid * 2] = ex;
            s_pre[tid * 2 + 1] = ex + c0;
            if (tid == 31) s_pre[FB] = x;
            __syncwarp();
            // entries of this batch: as many as fit in PMAX pairs (at least one; one entry <= 256)
            const unsigned fits = __ballot_sync(0xffffffffu, s_pre[tid * 2 + 1] <= PMAX && tid * 2 < nb0);
            const unsigned fits2 = __ballot_sync(0xffffffffu, s_pre[tid * 2 + 2] <= PMAX && tid * 2 + 1 < nb0);
            if (tid == 0) {
                // number of leading entries j with pre[j+1] <= PMAX
                const int n1 = __popc(fits), n2 = __popc(fits2);
                s_nbe = max(1, min(nb0, n1 + n2));
            }
        }
        __syncthreads();
        const int nb = s_nbe;
        const int P = s_pre[nb];
        // ---- B0: pair -> (entry, pixel) map, contiguous slice per thread ----
        {
            const int per = (P + 255) >> 8;
            int q = tid * per;
            const int qend = min(q + per, P);
            if (q < qend) {
                int lo = 0, hi = nb - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_pre[mid] <= q) lo = mid; else hi = mid - 1;
                }
                int j = lo, jend = s_pre[j + 1], geo = s_geo[j], w = (geo >> 8) & 0xff;
                int tt = q - s_pre[j];
                int col = tt % w, row = tt / w;
                for (; q < qend; q++) {
                    while (q >= jend) {
                        j++;
                        jend = s_pre[j + 1];
                        geo = s_geo[j];
                        w = (geo >> 8) & 0xff;
                        col = 0;
                        row = 0;
                    }
                    s_pe[q] = (unsigned char)j;
                    s_pp[q] = (unsigned char)((((geo >> 16) + row) << 4) + (geo & 0xff) + col);
                    if (++col == w) { col = 0; row++; }
                }
            }
        }
        __syncthreads();
        // ---- B1: dense fp64 evaluation of all pairs; candidates -> work list ----
        for (int q0 = 0; q0 < P; q0 += 256) {
            const int q = q0 + tid;
            bool cand = false;
            float rf = 0.f;
            if (q < P) {
                const int pidx = s_pp[q];
                if (!s_done[pidx]) {
                    const double* r = reinterpret_cast<const double*>(&s_rec[s_pe[q] * SREC_W]);
                    const double pcx = TX0 + (pidx & 15) + 0.5, pcy = TY0 + (pidx >> 4) + 0.5;
                    const double rlo = r[10];
                    const double l0 = fma(r[0], pcx, fma(r[1], pcy, r[2]));
                    const double l1 = fma(r[3], pcx, fma(r[4], pcy, r[5]));
                    const double l2 = fma(r[6], pcx, fma(r[7], pcy, r[8]));
                    if (l0 >= rlo && l1 >= rlo && l2 >= rlo) {
                        const double rr = l0 < l1 ? (l0 < l2 ? l0 : l2) : (l1 < l2 ? l1 : l2);
                        cand = true;
                        // r for alpha, or NaN: inside the guard band, resolved by the fix-up
                        rf = rr > r[11] ? (float)(opt.mode == 0 ? fmin(rr, 1.0) : rr) : __int_as_float(0x7fc00000);
                    }
                }
            }
            const unsigned m = __ballot_sync(0xffffffffu, cand);
            if (m) {
                int base = 0;
                if (lane == 0) base = atomicAdd(&s_wn, __popc(m));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (cand) {
                    const int idx = base + __popc(m & lanemask_lt());
                    s_wl[idx] = (unsigned short)q;
                    s_wr[idx] = rf;
                }
            }
        }
        __syncthreads();
        // ---- B2: alpha for the candidates (dense), append to per-pixel slots ----
        {
            const int wn = s_wn;
            for (int i = tid; i < wn; i += 256) {
                const int q = s_wl[i];
                const int j = s_pe[q], pidx = s_pp[q];
                const float* rf32 = reinterpret_cast<const float*>(&s_rec[j * SREC_W + 24]);  // f0 f1 rgb...
                float a = -1.f, ea = 0.f;
                const float rr = s_wr[i];
                const bool band = isnan(rr);
                if (!band) {
                    if (opt.mode == 0) {
                        const float lg = fast_lg2(rr);
                        const float arg = fmaf(rf32[0], lg, rf32[1]);
                        a = fast_ex2(arg);
                        ea = 5e-7f + rf32[0] * (6e-7f + 2.4e-7f * fabsf(lg)) + 1.2e-7f * fabsf(arg);
                    } else {
                        const float x = rr * rf32[0];
                        a = __fdividef(rf32[1], 1.0f + fast_ex2(fminf(x, 1009.9f)));
                        ea = 8e-7f + 1.2e-7f * fabsf(x);
                    }
                    a = fminf(a, ALPHA_CLAMP_F);
                }
                const int k = atomicAdd(&s_cnt[pidx], 1);
                if (k < NSLOT) {
                    s_sa[k][pidx] = a;
                    s_se[k][pidx] = ea;
                    s_sj[k][pidx] = (unsigned char)j;
                } else {
                    s_ovf[pidx] = 1;
                }
            }
        }
        __syncthreads();
        // ---- C: per-pixel compositing in entry order ----
        if (!done) {
            const int n = s_cnt[tid];
            if (s_ovf[tid]) {
                flag_pos = b;  // conservative: nothing of this batch was committed for this pixel
                done = true;
            } else if (n > 0) {
                for (int i = 1; i < n; i++) {
                    const unsigned char jj = s_sj[i][tid];
                    const float aa = s_sa[i][tid], ee = s_se[i][tid];
                    int k = i - 1;
                    while (k >= 0 && s_sj[k][tid] > jj) {
                        s_sj[k + 1][tid] = s_sj[k][tid];
                        s_sa[k + 1][tid] = s_sa[k][tid];
                        s_se[k + 1][tid] = s_se[k][tid];
                        k--;
                    }
                    s_sj[k + 1][tid] = jj;
                    s_sa[k + 1][tid] = aa;
                    s_se[k + 1][tid] = ee;
                }
                for (int i = 0; i < n; i++) {
                    const int j = s_sj[i][tid];
                    const float a = s_sa[i][tid];
                    if (a < 0.f) {  // r inside the contribution guard band
                        flag_pos = b + j;
                        done = true;
                        break;
                    }
                    const float ea = s_se[i][tid];
                    const float w = T * a;
                    const float tn = fmaf(-T, a, T);
                    const float en = fmaf(ea * a, __frcp_rn(1.f - a), epsT + 2.4e-7f);
                    const float ew = epsT + ea + 1.2e-7f;
                    if (fabsf(tn - T_MIN_F) <= fmaf(2.f * en, tn, 1e-11f) ||
                        fabsf(w - tau) <= fmaf(2.f * ew, w, 1e-9f)) {
                        flag_pos = b + j;
                        done = true;
                        break;
                    }
                    const float* rgb = reinterpret_cast<const float*>(&s_rec[j * SREC_W + 26]);
                    C0 = fmaf(w, rgb[0], C0);
                    C1 = fmaf(w, rgb[1], C1);
                    C2 = fmaf(w, rgb[2], C2);
                    last = b + j;
                    cnt++;
                    T = tn;
                    epsT = en;
                    atomicMax(&s_maxw[j], __float_as_uint(w));
                    if (w > tau) atomicAdd(&s_pix[j], 1);
                    if (T < T_MIN_F) {
                        done = true;
                        break;
                    }
                }
            }
            s_done[tid] = done ? 1 : 0;
        }
        s_cnt[tid] = 0;
        s_ovf[tid] = 0;
        __syncthreads();
        if (tid < nb) {
            const unsigned src = s_src[tid];
            if (s_maxw[tid] && out.max_weight) atomicMax((unsigned*)out.max_weight + src, s_maxw[tid]);
            if (s_pix[tid] && out.pixel_count) atomicAdd(out.pixel_count + src, s_pix[tid]);
        }
        if (tid < FB) {
            s_maxw[tid] = 0u;
            s_pix[tid] = 0;
        }
        b += nb;
    }
    if (inside) {
        const int p = py * cam.width + px;
        if (flag_pos >= 0) {
            unsigned long long k = atomicAdd(&out.ctr->n_flagged, 1ull);
            out.flags[k] = make_int2(p, flag_pos);
        } else {
            if (out.image) {
                out.image[p * 3 + 0] = fminf(fmaxf(fmaf(T, (float)opt.bg[0], C0), 0.f), 1.f);
                out.image[p * 3 + 1] = fminf(fmaxf(fmaf(T, (float)opt.bg[1], C1), 0.f), 1.f);
                out.image[p * 3 + 2] = fminf(fmaxf(fmaf(T, (float)opt.bg[2], C2), 0.f), 1.f);
            }
            if (out.alpha_map) out.alpha_map[p] = 1.f - T;
            out.t_final[p] = T;
            out.last_pos[p] = last;
            if (out.n_frag) out.n_frag[p] = cnt;
            if (out.last_src) out.last_src[p] = last >= 0 ? (int)ent_src[last] : -1;
        }
    }
}

// ---------------------------------------------------------------------------
// k_fixup_fwd: exact (fp64) replay of flagged pixels, one warp per pixel:
// lanes evaluate 32 consecutive tile entries in parallel, then the warp
// composites the contributing ones in entry order.  Entries before the flag
// position already committed their statistics in k_blend_fast (their
// decisions were certain); from the flag position on the fix-up commits them.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_fixup_fwd(Cam cam, Opts opt, const T* __restrict__ opacity,
                                                   const T* __restrict__ sigma, const RecF* __restrict__ rec,
                                                   const int* __restrict__ tile_start,
                                                   const unsigned* __restrict__ ent_src, FastBlendOut out) {
    const unsigned lane = threadIdx.x & 31;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long nflag = (long long)out.ctr->n_flagged;
    for (long long k = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nflag; k += nw) {
        const int2 f = out.flags[k];
        const int p = f.x, fpos = f.y;
        const int px = p % cam.width, py = p / cam.width;
        const int t = (py / TILE) * cam.ntx + px / TILE;
        double Tt = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
        int last = -1, cnt = 0;
        bool done = false;
        const int s = tile_start[t], e = tile_start[t + 1];
        for (int base = s; base < e && !done; base += 32) {
            const int pos = base + (int)lane;
            double a = 0.0;
            unsigned src = 0;
            float cr = 0.f, cg = 0.f, cb = 0.f;
            if (pos < e) {
                src = ent_src[pos];
                const RecF& r = rec[src];
                if (px >= r.x0 && px < r.x1 && py >= r.y0 && py < r.y1) {
                    double rr = edge_r(r, px + 0.5, py + 0.5);
                    a = alpha_exact_r<T>(r, rr, opt.mode, opt, opacity, sigma, src);
                    if (a > ALPHA_CLAMP) a = ALPHA_CLAMP;
                    if (a < ALPHA_MIN) a = 0.0;
                    cr = r.rgb[0];
                    cg = r.rgb[1];
                    cb = r.rgb[2];
                }
            }
            unsigned m = __ballot_sync(0xffffffffu, a > 0.0);
            while (m && !done) {
                const int j = __ffs(m) - 1;
                m &= m - 1;
                const double aj = __shfl_sync(0xffffffffu, a, j);
                const double w = Tt * aj;
                C0 += w * (double)__shfl_sync(0xffffffffu, cr, j);
                C1 += w * (double)__shfl_sync(0xffffffffu, cg, j);
                C2 += w * (double)__shfl_sync(0xffffffffu, cb, j);
                const int posj = base + j;
                if ((int)lane == j && posj >= fpos) {
                    if (out.max_weight) atomicMax((unsigned*)out.max_weight + src, __float_as_uint((float)w));
                    if (w > opt.tau_contrib && out.pixel_count) atomicAdd(out.pixel_count + src, 1);
                }
                last = posj;
                cnt++;
                Tt = TS_M(Tt, TS_S(1.0, aj));
                if (Tt < T_MIN) done = true;
            }
        }
        if (lane == 0) {
            if (out.image) {
                out.image[p * 3 + 0] = (float)fmin(fmax(C0 + Tt * opt.bg[0], 0.0), 1.0);
                out.image[p * 3 + 1] = (float)fmin(fmax(C1 + Tt * opt.bg[1], 0.0), 1.0);
                out.image[p * 3 + 2] = (float)fmin(fmax(C2 + Tt * opt.bg[2], 0.0), 1.0);
            }
            if (out.alpha_map) out.alpha_map[p] = (float)(1.0 - Tt);
            out.t_final[p] = (float)Tt;
            out.last_pos[p] = last;
            if (out.n_frag) out.n_frag[p] = cnt;
            if (out.last_src) out.last_src[p] = last >= 0 ? (int)ent_src[last] : -1;
        }
    }
}

constexpr size_t BLEND_DYN_SMEM = PMAX * 4 + 2 * NSLOT * TILE_PIX * 4 + PMAX * 2 + 2 * PMAX + NSLOT * TILE_PIX;

void launch_blend_fast(const Cam& cam, const Opts& opt, const RecF* rec, const short4* bbox,
                       const int* tile_start, const unsigned* ent_src, const FastBlendOut& out,
                       cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_blend_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BLEND_DYN_SMEM);
        attr = true;
    }
    int ntiles = cam.ntx * cam.nty;
    k_blend_fast<<<ntiles, 256, BLEND_DYN_SMEM, st>>>(cam, opt, rec, bbox, tile_start, ent_src, out);
}

void launch_fixup_fwd(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype, const RecF* rec,
                      const int* tile_start, const unsigned* ent_src, const FastBlendOut& out,
                      cudaStream_t st) {
    const int grid = 148 * 4;
    if (dtype == 1)
        k_fixup_fwd<double><<<grid, 256, 0, st>>>(cam, opt, (const double*)soup.opacity,
                                                  (const double*)soup.sigma, rec, tile_start, ent_src, out);
    else
        k_fixup_fwd<float><<<grid, 256, 0, st>>>(cam, opt, (const float*)soup.opacity,
                                                 (const float*)soup.sigma, rec, tile_start, ent_src, out);
}

// ---------------------------------------------------------------------------
// k_blend_bwd_fast: back to front from the saved last contributor, fp32
// gradients, warp-reduced before fp32 atomics into the per-source buffer.
// Decisions inside the guard band (skip, clamp) and near-tied argmax edges
// are resolved with the reference fp64 arithmetic.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_blend_bwd_fast(Cam cam, Opts opt, const T* __restrict__ verts,
                                                        const T* __restrict__ opacity,
                                                        const T* __restrict__ sigma,
                                                        const RecF* __restrict__ rec,
                                                        const RecB* __restrict__ recb,
                                                        const int* __restrict__ tile_start,
                                                        const unsigned* __restrict__ ent_src,
                                                        const float* __restrict__ t_final,
                                                        const int* __restrict__ last_pos,
                                                        const float* __restrict__ d_image,
                                                        float* __restrict__ sgrad) {
    __shared__ RecF s_rec[FB];
    __shared__ RecB s_rb[FB];
    __shared__ unsigned s_src[FB];
    __shared__ int s_hi;
    const int t = blockIdx.x;
    const int tx = t % cam.ntx, ty = t / cam.ntx;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int px = tx * TILE + (lane & 15);
    const int py = ty * TILE + 2 * warp + (lane >> 4);
    const int wy0 = ty * TILE + 2 * warp;
    const bool inside = px < cam.width && py < cam.height;
    const int s = tile_start[t];
    int my_last = -1;
    float Tc = 1.f, d0 = 0.f, d1 = 0.f, d2 = 0.f;
    if (inside) {
        const int p = py * cam.width + px;
        my_last = last_pos[p];
        Tc = t_final[p];
        d0 = d_image[p * 3 + 0];
        d1 = d_image[p * 3 + 1];
        d2 = d_image[p * 3 + 2];
    }
    float S0 = Tc * (float)opt.bg[0], S1 = Tc * (float)opt.bg[1], S2 = Tc * (float)opt.bg[2];
    if (threadIdx.x == 0) s_hi = -1;
    __syncthreads();
    if (my_last >= 0) atomicMax(&s_hi, my_last);
    __syncthreads();
    const int hi = s_hi;
    const float fpx = (float)(px) + 0.5f, fpy = (float)(py) + 0.5f;
    for (int bend = hi + 1; bend > s; bend -= FB) {
        const int bstart = max(s, bend - FB);
        const int nb = bend - bstart;
        __syncthreads();
        for (int c = threadIdx.x; c < nb * 11; c += blockDim.x) {
            int j = c / 11, q = c - j * 11;
            unsigned src = __ldg(ent_src + bstart + j);
            if (q == 0) s_src[j] = src;
            if (q < 8)
                reinterpret_cast<float4*>(&s_rec[j])[q] = __ldg(reinterpret_cast<const float4*>(rec + src) + q);
            else
                reinterpret_cast<float4*>(&s_rb[j])[q - 8] = __ldg(reinterpret_cast<const float4*>(recb + src) + (q - 8));
        }
        __syncthreads();
        for (int jb = ((nb - 1) / 32) * 32; jb >= 0; jb -= 32) {
            int jl = jb + (int)lane;
            bool ov = jl < nb && s_rec[jl].y0 <= wy0 + 1 && s_rec[jl].y1 > wy0;
            unsigned mask = __ballot_sync(0xffffffffu, ov);
            while (mask) {
                const int j = jb + 31 - __clz(mask);
                mask &= ~(1u << (j - jb));
                const RecF& r = s_rec[j];
                const int pos = bstart + j;
                float g[12];
#pragma unroll
                for (int k = 0; k < 12; k++) g[k] = 0.f;
                bool act = false;
                if (pos <= my_last && px >= r.x0 && px < r.x1 && py >= r.y0 && py < r.y1) {
                    const RecB& rb = s_rb[j];
                    int edge;
                    double rr = edge_r(r, px + 0.5, py + 0.5, edge);
                    bool contributes = rr > (double)r.r_hi;
                    float alpha = 0.f;
                    bool clamped = false, exact_done = false;
                    if (!contributes && rr >= (double)r.r_lo) {
                        double ae = alpha_exact_r<T>(r, rr, opt.mode, opt, opacity, sigma, s_src[j]);
                        clamped = ae > ALPHA_CLAMP;
                        if (clamped) ae = ALPHA_CLAMP;
                        contributes = ae >= ALPHA_MIN;
                        alpha = (float)ae;
                        exact_done = true;
                    }
                    if (contributes) {
                        if (!exact_done) {
                            float ea;
                            alpha = alpha_fast(r, rr, opt.mode, ea);
                            if (fabsf(alpha - ALPHA_CLAMP_F) <= 2.f * ea * alpha + 1e-7f) {
                                double ae = alpha_exact_r<T>(r, rr, opt.mode, opt, opacity, sigma, s_src[j]);
                                clamped = ae > ALPHA_CLAMP;
                                alpha = clamped ? ALPHA_CLAMP_F : (float)ae;
                            } else {
                                clamped = alpha > ALPHA_CLAMP_F;
                                if (clamped) alpha = ALPHA_CLAMP_F;
                            }
                        }
                        act = true;
                        const float one_m = 1.f - alpha;
                        const float tb = Tc / one_m;
                        const float w = tb * alpha;
                        const float* c = r.rgb;
                        g[SG_GRGB + 0] = w * d0;
                        g[SG_GRGB + 1] = w * d1;
                        g[SG_GRGB + 2] = w * d2;
                        const float inv1m = 1.f / one_m;
                        float ga = d0 * (tb * c[0] - S0 * inv1m) + d1 * (tb * c[1] - S1 * inv1m) +
                                   d2 * (tb * c[2] - S2 * inv1m);
                        S0 = fmaf(w, c[0], S0);
                        S1 = fmaf(w, c[1], S1);
                        S2 = fmaf(w, c[2], S2);
                        Tc = tb;
                        if (!clamped) {
                            const float o = rb.opa, sg = rb.sig, phis = rb.phis;
                            g[SG_GO] = ga * (alpha / o);
                            const float g_win = o * ga;
                            const float window = alpha / o;
                            const float rf = (float)rr;
                            const float phi = rf * phis;
                            float g_phi;
                            if (opt.mode == 0) {
                                const float rc = fminf(rf, 1.f);
                                g[SG_GSIG] = g_win * window * __logf(rc);
                                const float g_r = g_win * sg * window / rc;
                                if (rr >= 1.0) {
                                    g_phi = 0.f;
                                } else {
                                    g_phi = g_r / phis;
                                    g[SG_GPHIS] = -g_r * rf / phis;
                                }
                            } else {
                                // window*(1-window) = E/(1+E)^2 with E = exp(phi/sigma): no cancellation
                                const float E = fast_ex2(fminf(rf * r.f0, 126.f));
                                const float inv = 1.f / (1.f + E);
                                const float ww = E * inv * inv;
                                g[SG_GSIG] = g_win * ww * phi / (sg * sg);
                                g_phi = -g_win * ww / sg;
                            }
                            // edge line L = s*(n.p)... derivative wrt its endpoints (_kernels.py:296-318)
                            const int ia = edge, ib = edge == 2 ? 0 : edge + 1;
                            const float ax = rb.qx[ia], ay = rb.qy[ia], bx = rb.qx[ib], by = rb.qy[ib];
                            const float pxr = (float)(px - r.ox) + 0.5f, pyr = (float)(py - r.oy) + 0.5f;
                            const float ex = bx - ax, ey = by - ay;
                            const float inv_l = rsqrtf(ex * ex + ey * ey);
                            const float inv_l2 = inv_l * inv_l;
                            const float sgn = ((rb.esign >> edge) & 1) ? -1.f : 1.f;
                            const float gax = sgn * (pyr - by) * inv_l - phi * (ax - bx) * inv_l2;
                            const float gay = sgn * (bx - pxr) * inv_l - phi * (ay - by) * inv_l2;
                            const float gbx = sgn * (ay - pyr) * inv_l - phi * (bx - ax) * inv_l2;
                            const float gby = sgn * (pxr - ax) * inv_l - phi * (by - ay) * inv_l2;
                            g[SG_GQ + ia * 2] = g_phi * gax;
                            g[SG_GQ + ia * 2 + 1] = g_phi * gay;
                            g[SG_GQ + ib * 2] = g_phi * gbx;
                            g[SG_GQ + ib * 2 + 1] = g_phi * gby;
                        }
                    }
                }
                if (__any_sync(0xffffffffu, act)) {
#pragma unroll
                    for (int k = 0; k < 12; k++) {
                        float v = g[k];
#pragma unroll
                        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                        g[k] = v;
                    }
                    if (lane < 12) {
                        float v = g[0];
#pragma unroll
                        for (int k = 1; k < 12; k++) v = (lane == (unsigned)k) ? g[k] : v;
                        if (v != 0.f) atomicAdd(sgrad + (size_t)s_src[j] * SG_STRIDE + lane, v);
                    }
                }
            }
        }
    }
    (void)fpx;
    (void)fpy;
}

void launch_blend_bwd_fast(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype, const RecF* rec,
                           const RecB* recb, const int* tile_start, const unsigned* ent_src,
                           const float* t_final, const int* last_pos, const float* d_image, float* sgrad,
                           cudaStream_t st) {
    int ntiles = cam.ntx * cam.nty;
    if (dtype == 1)
        k_blend_bwd_fast<double><<<ntiles, 256, 0, st>>>(cam, opt, (const double*)soup.vertices,
                                                         (const double*)soup.opacity,
                                                         (const double*)soup.sigma, rec, recb, tile_start,
                                                         ent_src, t_final, last_pos, d_image, sgrad);
    else
        k_blend_bwd_fast<float><<<ntiles, 256, 0, st>>>(cam, opt, (const float*)soup.vertices,
                                                        (const float*)soup.opacity,
                                                        (const float*)soup.sigma, rec, recb, tile_start,
                                                        ent_src, t_final, last_pos, d_image, sgrad);
}

}  // namespace ts
