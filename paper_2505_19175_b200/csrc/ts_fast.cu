// ts_fast.cu -- the fast (default) path: fp64 edge functions, fp32 alpha and
// compositing, with a guard band around every discrete decision of the
// reference compositor and an exact fp64 fix-up for the rare pixels whose
// decision falls inside it.
//
//   k_preprocess_fast  render.py:159-190, 193-250, 271-273, 292-302 -> RecF/RecB
//   k_blend_fast       _kernels.py:59-132 with fragment emission (collect_fragments,
//                      _kernels.py:107-116): fp64 re-composite of a training forward
//   k_fixup_fwd        exact replay (same arithmetic as k_blend_exact) of flagged pixels
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
#include <algorithm>
#include <type_traits>

#include "ts_kernels.cuh"

namespace ts {

constexpr float T_MIN_F = 1e-4f;
constexpr float ALPHA_CLAMP_F = 0.99f;

// ---------------------------------------------------------------------------
// preprocess (fast records).  Only the quantities that decide the
// reference's discrete outputs are computed with its exact fp64 arithmetic
// (explicit _rn intrinsics, same operation order): the depth key (sort
// order), the cull tests (render.py:165-174, 271-273) and the tight bbox
// (render.py:216-250, tile lists).  Edge functions, the contribution band and
// the SH colour only need to be accurate and use fast math.
// ---------------------------------------------------------------------------
// SH colour sum (fp64 basis and accumulation) over 16-byte vector loads
// (fp32 params) / scalar loads (fp64)
template <typename T>
__device__ __forceinline__ void sh_colour(const T* __restrict__ p, const double* bs, int ncoef, double& c0,
                                          double& c1, double& c2);
template <>
__device__ __forceinline__ void sh_colour<float>(const float* __restrict__ p, const double* bs, int ncoef,
                                                 double& c0, double& c1, double& c2) {
    const float4* q = reinterpret_cast<const float4*>(p);
    const int nv = (ncoef * 3 + 3) >> 2;
    // two partial sums per channel (even / odd coefficient): halves the
    // dependent fp64 FMA chain
    double acc[2][3] = {{c0, c1, c2}, {0.0, 0.0, 0.0}};
#pragma unroll
    for (int k = 0; k < 12; k++) {
        if (k < nv) {
            const float4 v = q[k];
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int idx = k * 4 + u;  // coefficient idx / 3, channel idx % 3
                const int co = idx / 3;
                if (co < ncoef) acc[co & 1][idx % 3] = fma(bs[co], (double)vv[u], acc[co & 1][idx % 3]);
            }
        }
    }
    c0 = acc[0][0] + acc[1][0]; c1 = acc[0][1] + acc[1][1]; c2 = acc[0][2] + acc[1][2];
}
template <>
__device__ __forceinline__ void sh_colour<double>(const double* __restrict__ p, const double* bs, int ncoef,
                                                  double& c0, double& c1, double& c2) {
    double acc[3] = {c0, c1, c2};
    for (int idx = 0; idx < ncoef * 3; idx++) acc[idx % 3] = fma(bs[idx / 3], p[idx], acc[idx % 3]);
    c0 = acc[0]; c1 = acc[1]; c2 = acc[2];
}

// soup.py:67-77 check of the 48 SH coefficients: x*0 is NaN for +-inf and NaN
template <typename T>
__device__ __forceinline__ bool sh_finite(const T* __restrict__ p);
template <>
__device__ __forceinline__ bool sh_finite<float>(const float* __restrict__ p) {
    const float4* q = reinterpret_cast<const float4*>(p);
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < 12; k++) {
        const float4 v = q[k];
        ss = fmaf(v.x, 0.f, ss);
        ss = fmaf(v.y, 0.f, ss);
        ss = fmaf(v.z, 0.f, ss);
        ss = fmaf(v.w, 0.f, ss);
    }
    return ss == 0.f;
}
template <>
__device__ __forceinline__ bool sh_finite<double>(const double* __restrict__ p) {
    double ss = 0.0;
    for (int k = 0; k < 48; k++) ss = fma(p[k], 0.0, ss);
    return ss == 0.0;
}

// One triangle of the fast preprocess: v = its 9 vertex coordinates, shp = its
// 48 SH coefficients (shared-memory copy for fp32 parameters).
template <typename T>
__device__ __forceinline__ bool pre_tri(const Cam& cam, const Opts& opt, long long i, const double* v,
                                        double o_raw, double sg, const T* shp, const FastPreOut& out,
                                        unsigned long long& key, unsigned& tcount) {
    bool ok = false;
    if (opt.validate) {
        // x*0 is NaN for +-inf and NaN
        double sv = 0.0;
#pragma unroll
        for (int k = 0; k < 9; k++) sv = fma(v[k], 0.0, sv);
        if (sv != 0.0) atomicMin(&out.ctr->err[0], i);
        if (!isfinite(o_raw)) atomicMin(&out.ctr->err[1], i);
        if (!isfinite(sg)) atomicMin(&out.ctr->err[2], i);
    }
    // ---- exact: _project_kernel, render.py:159-190 ----
    double xc2[3], q[6];
    bool z_ok = true;
#pragma unroll
    for (int k = 0; k < 3; k++) {
        double xk[3];
#pragma unroll
        for (int a = 0; a < 3; a++) {
            double t = TS_A(TS_M(v[k * 3 + 0], cam.R[a * 3 + 0]), TS_M(v[k * 3 + 1], cam.R[a * 3 + 1]));
            t = TS_A(t, TS_M(v[k * 3 + 2], cam.R[a * 3 + 2]));
            xk[a] = TS_A(t, cam.t[a]);
        }
        if (xk[2] < 1e-12) z_ok = false;
        xc2[k] = xk[2];
        q[k * 2 + 0] = TS_A(TS_D(TS_M(cam.fx, xk[0]), xk[2]), cam.cx);
        q[k * 2 + 1] = TS_A(TS_D(TS_M(cam.fy, xk[1]), xk[2]), cam.cy);
    }
    const double z = TS_D(TS_A(TS_A(xc2[0], xc2[1]), xc2[2]), 3.0);
    if (z < cam.z_near) z_ok = false;
    const double e1x = TS_S(q[2], q[0]), e1y = TS_S(q[3], q[1]);
    const double e2x = TS_S(q[4], q[0]), e2y = TS_S(q[5], q[1]);
    const double area = TS_M(fabs(TS_S(TS_M(e1x, e2y), TS_M(e1y, e2x))), 0.5);  // == /2.0
    double d0x = TS_S(q[2], q[4]), d0y = TS_S(q[3], q[5]);
    double d1x = TS_S(q[4], q[0]), d1y = TS_S(q[5], q[1]);
    double d2x = TS_S(q[0], q[2]), d2y = TS_S(q[1], q[3]);
    const double s0 = __dsqrt_rn(TS_A(TS_M(d0x, d0x), TS_M(d0y, d0y)));
    const double s1 = __dsqrt_rn(TS_A(TS_M(d1x, d1x), TS_M(d1y, d1y)));
    const double s2 = __dsqrt_rn(TS_A(TS_M(d2x, d2x), TS_M(d2y, d2y)));
    const double perim = TS_A(TS_A(s0, s1), s2);
    const double phis = TS_D(TS_M(-2.0, area), perim > 1e-300 ? perim : 1e-300);
    if (out.area) out.area[i] = z_ok ? (float)area : 0.0f;
    ok = z_ok && (area >= DEGENERATE_AREA) && (fabs(phis) >= DEGENERATE_INRADIUS);
    short4 bb = make_short4(0, 0, 0, 0);
    if (ok) {
        const double o = opt.solid ? 1.0 : o_raw;
        // ---- exact: incenter + tight bbox, render.py:216-250 ----
        const double sx = TS_D(TS_A(TS_A(TS_M(s0, q[0]), TS_M(s1, q[2])), TS_M(s2, q[4])), perim);
        const double sy = TS_D(TS_A(TS_A(TS_M(s0, q[1]), TS_M(s1, q[3])), TS_M(s2, q[5])), perim);
        double f;
        if (opt.mode == 0) {
            if (o > opt.tau_cutoff) {
                const double ratio = TS_D(opt.tau_cutoff, o);
                // pow(x, 1.0) == x exactly (glibc and CUDA)
                f = TS_S(1.0, sg == 1.0 ? ratio : pow(ratio, TS_D(1.0, sg)));
            } else {
                f = 0.0;
            }
        } else {
            const double ratio = TS_D(opt.tau_cutoff, o);
            f = ratio < 1.0 ? TS_S(1.0, TS_D(TS_M(sg, log(TS_D(ratio, TS_S(1.0, ratio)))), fabs(phis))) : 0.0;
        }
        int x0 = 0, x1 = 0, y0 = 0, y1 = 0;
        if (f > 0.0) {
            double xmin = 1e300, ymin = 1e300, xmax = -1e300, ymax = -1e300;
#pragma unroll
            for (int k = 0; k < 3; k++) {
                const double pxk = TS_A(sx, TS_M(TS_S(q[k * 2], sx), f));
                const double pyk = TS_A(sy, TS_M(TS_S(q[k * 2 + 1], sy), f));
                xmin = pxk < xmin ? pxk : xmin;
                xmax = pxk > xmax ? pxk : xmax;
                ymin = pyk < ymin ? pyk : ymin;
                ymax = pyk > ymax ? pyk : ymax;
            }
            const long long W = cam.width, H = cam.height;
            long long X0 = floor_i64(TS_S(xmin, 0.5)); X0 = X0 > 0 ? X0 : 0; X0 = X0 < W ? X0 : W;
            long long X1 = floor_i64(TS_S(xmax, 0.5)) + 1; X1 = X1 > 0 ? X1 : 0; X1 = X1 < W ? X1 : W;
            long long Y0 = floor_i64(TS_S(ymin, 0.5)); Y0 = Y0 > 0 ? Y0 : 0; Y0 = Y0 < H ? Y0 : H;
            long long Y1 = floor_i64(TS_S(ymax, 0.5)) + 1; Y1 = Y1 > 0 ? Y1 : 0; Y1 = Y1 < H ? Y1 : H;
            x0 = (int)X0; x1 = (int)(X1 > X0 ? X1 : X0); y0 = (int)Y0; y1 = (int)(Y1 > Y0 ? Y1 : Y0);
        }
        bb = make_short4((short)x0, (short)x1, (short)y0, (short)y1);
        tcount = (unsigned)tiles_touched(x0, x1, y0, y1);
        if (tcount) {
            // ---- accurate (not bit-exact): edge functions, orientation, band ----
            RecF r;
            const double ccx = (q[0] + q[2] + q[4]) * (1.0 / 3.0), ccy = (q[1] + q[3] + q[5]) * (1.0 / 3.0);
            const double inv = 1.0 / phis;
            double dmax = 0.0;
            int esign = 0;
            float qf[6];
#pragma unroll
            for (int e = 0; e < 3; e++) {
                const int bi = e == 2 ? 0 : e + 1;
                const double ax = q[e * 2], ay = q[e * 2 + 1];
                const double evx = q[bi * 2] - ax, evy = q[bi * 2 + 1] - ay;
                const double il = rsqrt(evx * evx + evy * evy);
                double nx = evy * il, ny = -evx * il;
                if (nx * (ccx - ax) + ny * (ccy - ay) > 0) {
                    nx = -nx;
                    ny = -ny;
                    esign |= 1 << e;
                }
                const double d = -(nx * ax + ny * ay);
                r.a[e * 3 + 0] = nx * inv;
                r.a[e * 3 + 1] = ny * inv;
                r.a[e * 3 + 2] = d * inv;
                dmax = fmax(dmax, fabs(d));
            }
            const double mag = (fabs(q[0]) + fabs(q[1]) + fabs(q[2]) + fabs(q[3]) + fabs(q[4]) + fabs(q[5]) +
                                4.0 * (cam.width + cam.height) + dmax) * fabs(inv);
            const double delta = 1e-13 * mag + 1e-300;
            double rstar;
            if (opt.mode == 0) {
                rstar = o > ALPHA_MIN ? (sg == 1.0 ? ALPHA_MIN / o : pow(ALPHA_MIN / o, 1.0 / sg)) : 1e30;
                if (rstar > 1.0) rstar = 1e30;
                r.f0 = (float)sg;
                r.f1 = log2f((float)o);
            } else {
                const double qq = 255.0 * o - 1.0;
                rstar = qq > 0.0 ? sg * log(qq) / phis : 1e30;
                r.f0 = (float)(phis * 1.4426950408889634 / sg);
                r.f1 = (float)o;
            }
            r.r_lo = rstar - delta - fabs(rstar) * 1e-12;
            r.r_hi = rstar + delta + fabs(rstar) * 1e-12;
            r.phis = phis;
            // view-dependent SH colour (render.py:292-302) in fp64 (rounded once to
            // fp32: the backward's colour differences cancel, fp32 sums cost ~1e-4)
            double u0 = (v[0] + v[3] + v[6]) * (1.0 / 3.0) - cam.cc[0];
            double u1 = (v[1] + v[4] + v[7]) * (1.0 / 3.0) - cam.cc[1];
            double u2 = (v[2] + v[5] + v[8]) * (1.0 / 3.0) - cam.cc[2];
            const double iu = rsqrt(fmax(u0 * u0 + u1 * u1 + u2 * u2, 1e-48));
            u0 *= iu; u1 *= iu; u2 *= iu;
            const double xx = u0 * u0, yy = u1 * u1, zz = u2 * u2;
            double bs[16];
            bs[0] = 0.28209479177387814;
            bs[1] = -0.4886025119029199 * u1;
            bs[2] = 0.4886025119029199 * u2;
            bs[3] = -0.4886025119029199 * u0;
            bs[4] = 1.0925484305920792 * u0 * u1;
            bs[5] = -1.0925484305920792 * u1 * u2;
            bs[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
            bs[7] = -1.0925484305920792 * u0 * u2;
            bs[8] = 0.5462742152960396 * (xx - yy);
            bs[9] = -0.5900435899266435 * u1 * (3.0 * xx - yy);
            bs[10] = 2.890611442640554 * u0 * u1 * u2;
            bs[11] = -0.4570457994644658 * u1 * (4.0 * zz - xx - yy);
            bs[12] = 0.3731763325901154 * u2 * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            bs[13] = -0.4570457994644658 * u0 * (4.0 * zz - xx - yy);
            bs[14] = 1.445305721320277 * u2 * (xx - yy);
            bs[15] = -0.5900435899266435 * u0 * (xx - 3.0 * yy);
            double d0 = 0.5, d1 = 0.5, d2 = 0.5;
            sh_colour<T>(shp, bs, opt.ncoef, d0, d1, d2);
            const float c0 = (float)d0, c1 = (float)d1, c2 = (float)d2;
            r.rgb[0] = fminf(fmaxf(c0, 0.f), 1.f);
            r.rgb[1] = fminf(fmaxf(c1, 0.f), 1.f);
            r.rgb[2] = fminf(fmaxf(c2, 0.f), 1.f);
            const int ox = (x0 + x1) >> 1, oy = (y0 + y1) >> 1;
            r.x0 = (short)x0; r.x1 = (short)x1; r.y0 = (short)y0; r.y1 = (short)y1;
            r.ox = (short)ox; r.oy = (short)oy;
            out.rec[i] = r;
            if (out.recb) {
                RecB rb;
#pragma unroll
                for (int e = 0; e < 3; e++) rb.q[e] = make_double2(q[e * 2] - ox, q[e * 2 + 1] - oy);
                rb.inv_phis = 1.0 / phis;
                rb.esign = (unsigned)esign;
                rb.pad = 0u;
                out.recb[i] = rb;
            }
            if (out.recc) {
                RecC rc;
                rc.rgb[0] = fmin(fmax(d0, 0.0), 1.0);
                rc.rgb[1] = fmin(fmax(d1, 0.0), 1.0);
                rc.rgb[2] = fmin(fmax(d2, 0.0), 1.0);
                rc.opa = o;
                rc.sig = sg;
                rc.inv_opa = 1.0 / o;
                out.recc[i] = rc;
            }
            (void)qf;
        }
        key = (unsigned long long)__double_as_longlong(z);
    }
    if (opt.validate && !sh_finite<T>(shp)) atomicMin(&out.ctr->err[3], i);
    out.bbox[i] = bb;
    out.flag[i] = ok ? 1u : 0u;
    out.tcount[i] = tcount;
    if (out.max_weight) out.max_weight[i] = 0.f;
    if (out.pixel_count) out.pixel_count[i] = 0;
    out.key[i] = key;
    return ok;
}

// Warp-reduce the per-triangle counters and publish them (one atomic set per warp).
__device__ __forceinline__ void pre_publish(Counters* ctr, unsigned long long kmin, unsigned long long kmax,
                                            unsigned cnt, unsigned long long tc) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, off);
        const unsigned long long bq = __shfl_xor_sync(0xffffffffu, kmax, off);
        kmin = a < kmin ? a : kmin;
        kmax = bq > kmax ? bq : kmax;
        cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        tc += __shfl_xor_sync(0xffffffffu, tc, off);
    }
    if ((threadIdx.x & 31) == 0 && cnt) {
        atomicMin(&ctr->key_min, kmin);
        atomicMax(&ctr->key_max, kmax);
        atomicAdd(&ctr->m, (unsigned long long)cnt);
        atomicAdd(&ctr->e, tc);
    }
}

// fp64 parameters (drop-in parity path): one thread per triangle, direct loads.
__global__ void __launch_bounds__(128) k_preprocess_fast64(Cam cam, Opts opt, const double* __restrict__ verts,
                                                           const double* __restrict__ opacity,
                                                           const double* __restrict__ sigma,
                                                           const double* __restrict__ sh, long long n,
                                                           FastPreOut out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long key = 0;
    unsigned tcount = 0;
    bool ok = false;
    if (i < n) {
        double v[9];
#pragma unroll
        for (int k = 0; k < 9; k++) v[k] = verts[i * 9 + k];
        ok = pre_tri<double>(cam, opt, i, v, opacity[i], sigma[i], sh + i * 48, out, key, tcount);
    }
    pre_publish(out.ctr, ok ? key : ~0ull, ok ? key : 0ull, ok ? 1u : 0u, tcount);
}

// fp32 parameters: persistent CTAs walk blocks of 128 triangles; the next
// block's vertices, opacity, sigma and SH rows are copied to shared memory
// (cp.async, double-buffered, SH rows padded to 13 float4 so per-thread row
// reads are bank-conflict free) while the current block is computed.
#ifndef TS_PRE_BLK
#define TS_PRE_BLK 32  // (one warp x 16 CTAs per SM: more independent stages in flight; 64 x 8 and 128 x 4 slower)
#endif
constexpr int PRE_BLK = TS_PRE_BLK;  // triangles (threads) per CTA stage
#ifndef TS_PRE_MINB
#define TS_PRE_MINB 16  // CTAs per SM of the staged preprocess
#endif
struct PreStage {
    float4 sh[PRE_BLK * 13];
    float v[PRE_BLK * 9];
    float o[PRE_BLK], sg[PRE_BLK];
};

template <int NBUF, int MINB, int PF = 0>
__global__ void __launch_bounds__(PRE_BLK, MINB) k_preprocess_fast32(Cam cam, Opts opt, const float* __restrict__ verts,
                                                               const float* __restrict__ opacity,
                                                               const float* __restrict__ sigma,
                                                               const float* __restrict__ sh, long long n,
                                                               FastPreOut out) {
    TS_PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char s_pre[];
    PreStage* stage = reinterpret_cast<PreStage*>(s_pre);  // [NBUF]
    const long long nblk = (n + PRE_BLK - 1) / PRE_BLK;
    const int tid = threadIdx.x;
    auto issue = [&](long long blk, int buf) {
        const long long i0 = blk * PRE_BLK;
        const int nt = (int)min((long long)PRE_BLK, n - i0);
        PreStage& S = stage[buf];
        const float4* g = reinterpret_cast<const float4*>(sh + i0 * 48);
        for (int c = tid; c < nt * 12; c += PRE_BLK) {
            const int tri = c / 12;
            cp_async16(&S.sh[tri * 13 + (c - tri * 12)], g + c);
        }
        const float* gv = verts + i0 * 9;
        if (nt == PRE_BLK) {
            for (int c = tid; c < PRE_BLK * 9 / 4; c += PRE_BLK)
                cp_async16(reinterpret_cast<float4*>(S.v) + c, reinterpret_cast<const float4*>(gv) + c);
            if (tid < PRE_BLK / 4) {
                cp_async16(reinterpret_cast<float4*>(S.o) + tid, reinterpret_cast<const float4*>(opacity + i0) + tid);
                cp_async16(reinterpret_cast<float4*>(S.sg) + tid, reinterpret_cast<const float4*>(sigma + i0) + tid);
            }
        } else {
            for (int c = tid; c < nt * 9; c += PRE_BLK) cp_async4(S.v + c, gv + c);
            if (tid < nt) {
                cp_async4(S.o + tid, opacity + i0 + tid);
                cp_async4(S.sg + tid, sigma + i0 + tid);
            }
        }
    };
    unsigned long long kmin = ~0ull, kmax = 0ull, tc = 0;
    unsigned cnt = 0;
    long long blk = blockIdx.x;
    if (NBUF == 2 && blk < nblk) issue(blk, 0);
    cp_async_commit();
    for (int it = 0; blk < nblk; blk += gridDim.x, it++) {
        const int buf = NBUF == 2 ? (it & 1) : 0;
        if constexpr (NBUF == 2) {
            if (blk + gridDim.x < nblk) issue(blk + gridDim.x, buf ^ 1);
            cp_async_commit();
            cp_async_wait_group1();
        } else {  // single stage: other CTAs of the SM overlap its load
            issue(blk, 0);
            cp_async_commit();
            cp_async_wait_all();
        }
        __syncthreads();
        if (PF > 0 && tid < 4 * PF) {  // later stages' rows on their way to L2 while this one computes
            const int d = (it == 0 ? 1 + (tid >> 2) : PF);  // first pass: distances 1..PF, then PF
            const long long nx = blk + (long long)d * gridDim.x;
            if ((it == 0 || tid < 4) && nx < nblk && (nx + 1) * PRE_BLK <= n) {
                const long long i0 = nx * PRE_BLK;
                const int f = tid & 3;
                if (f == 0) prefetch_l2_bulk(sh + i0 * 48, PRE_BLK * 48 * 4);
                if (f == 1) prefetch_l2_bulk(verts + i0 * 9, PRE_BLK * 9 * 4);
                if (f == 2) prefetch_l2_bulk(opacity + i0, PRE_BLK * 4);
                if (f == 3) prefetch_l2_bulk(sigma + i0, PRE_BLK * 4);
            }
        }
        const long long i = blk * PRE_BLK + tid;
        if (i < n) {
            const PreStage& S = stage[buf];
            double v[9];
#pragma unroll
            for (int k = 0; k < 9; k++) v[k] = (double)S.v[tid * 9 + k];
            unsigned long long key = 0;
            unsigned tcount = 0;
            const bool ok = pre_tri<float>(cam, opt, i, v, (double)S.o[tid], (double)S.sg[tid],
                                           reinterpret_cast<const float*>(&S.sh[tid * 13]), out, key, tcount);
            if (ok) {
                kmin = key < kmin ? key : kmin;
                kmax = key > kmax ? key : kmax;
                cnt++;
            }
            tc += tcount;
        }
        __syncthreads();
    }
    cp_async_wait_all();
    pre_publish(out.ctr, kmin, kmax, cnt, tc);
}

void launch_preprocess_fast(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype,
                            const FastPreOut& out, cudaStream_t st) {
    long long n = soup.n;
    if (n <= 0) return;
    if (dtype == 1) {
        unsigned grid = (unsigned)((n + 127) / 128);
        k_preprocess_fast64<<<grid, 128, 0, st>>>(cam, opt, (const double*)soup.vertices, (const double*)soup.opacity,
                                                  (const double*)soup.sigma, (const double*)soup.sh, n, out);
    } else {
        // single-buffered stage, 4 CTAs per SM (the other CTAs overlap each one's
        // loads; 126 registers), the CTA's next stage bulk-prefetched into L2 while
        // it computes (measured against double buffering at 3 CTAs / 5 CTAs / no
        // prefetch: DESIGN.md section 6)
        const int sms = sm_count();
        const int smem = (int)sizeof(PreStage);
        smem_optin((const void*)k_preprocess_fast32<1, TS_PRE_MINB, 1>, smem);
        const long long nblk = (n + PRE_BLK - 1) / PRE_BLK;
        const long long grid = std::min<long long>(nblk, (long long)sms * TS_PRE_MINB);
        launch_pdl(k_preprocess_fast32<1, TS_PRE_MINB, 1>, dim3((unsigned)grid), dim3(PRE_BLK), smem, st, cam, opt,
                   (const float*)soup.vertices, (const float*)soup.opacity, (const float*)soup.sigma,
                   (const float*)soup.sh, n, out);
    }
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
        window = sg == 1.0 ? fmin(rr, 1.0) : pow(fmin(rr, 1.0), sg);  // pow(x, 1) == x
    } else {
        double x = rr * r.phis / sg;
        if (x > 700.0) x = 700.0;
        window = 1.0 / (1.0 + exp(x));
    }
    return o * window;
}

// ---------------------------------------------------------------------------
// k_blend_fast: CTA per 16x16 tile, lane = pixel.  Warp w owns the 2x16
// column strip x in [2w, 2w+2) of the tile, split into 8 groups of 4 lanes
// (2x2 pixel quads).  Each group walks its OWN list of the batch's entries
// whose bbox overlaps its quad (the reference's per-pixel bbox test,
// _kernels.py:87-95, hoisted to quad level), so lanes stay busy even though
// the triangles are a few pixels wide.  Edge functions in fp64, alpha and
// compositing in fp32 with the decision guard band.
// ---------------------------------------------------------------------------
constexpr int FB = 64;

struct __align__(16) SRec {
    RecF r;
    float4 pad;  // 144-byte stride: groups reading different records hit different banks
};

// ACC64 (training forward, keep_backward=1): alpha with the reference formula
// in fp64 and fp64 transmittance, so the saved T_final and every decision are
// exact up to the ~1e-13 difference of r; the backward then reconstructs the
// transmittances the reference uses.
template <typename PT, bool ACC64>
__global__ void __launch_bounds__(256) k_blend_fast(Cam cam, Opts opt, const RecF* __restrict__ rec,
                                                    const short4* __restrict__ bbox,
                                                    const int* __restrict__ tile_start,
                                                    const unsigned* __restrict__ ent_src,
                                                    const PT* __restrict__ opacity,
                                                    const PT* __restrict__ sigma,
                                                    FastBlendOut out) {
    using Real = typename std::conditional<ACC64, double, float>::type;
    __shared__ SRec s_rec[FB];
    __shared__ double2 s_os[ACC64 ? FB : 1];  // exact (opacity, sigma)
    __shared__ short4 s_bb[FB];
    __shared__ unsigned s_src[FB];
    __shared__ unsigned s_maxw[FB];
    __shared__ int s_pix[FB];
    const int t = blockIdx.x;
    const int tx = t % cam.ntx, ty = t / cam.ntx;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned grp = lane >> 2;
    const int X0 = tx * TILE + 2 * (int)warp;  // strip columns [X0, X0+2)
    const int Y0 = ty * TILE;
    const int px = X0 + (int)(lane & 1);
    const int py = Y0 + 2 * (int)grp + (int)((lane >> 1) & 1);
    const double pcx = px + 0.5, pcy = py + 0.5;
    const bool inside = px < cam.width && py < cam.height;
    Real T = 1, C0 = 0, C1 = 0, C2 = 0;
    float epsT = 0.f;
    int last = -1, cnt = 0, flag_pos = -1;
    bool done = !inside;
    const int s = tile_start[t], e = tile_start[t + 1];
    const float tau = (float)opt.tau_contrib;
    if (threadIdx.x < FB) {
        s_maxw[threadIdx.x] = 0u;
        s_pix[threadIdx.x] = 0;
    }
    for (int b = s; b < e; b += FB) {
        if (__syncthreads_count(!done) == 0) break;
        const int nb = min(FB, e - b);
        for (int c = threadIdx.x; c < nb * 8; c += blockDim.x) {
            const int j = c >> 3, q = c & 7;
            const unsigned src = __ldg(ent_src + b + j);
            if (q == 0) {
                s_src[j] = src;
                s_bb[j] = __ldg(bbox + src);
                if constexpr (ACC64)
                    s_os[j] = make_double2(opt.solid ? 1.0 : (double)opacity[src], (double)sigma[src]);
            }
            reinterpret_cast<float4*>(&s_rec[j].r)[q] = __ldg(reinterpret_cast<const float4*>(rec + src) + q);
        }
        __syncthreads();
        for (int jb = 0; jb < nb; jb += 32) {
            if (!__any_sync(0xffffffffu, !done)) break;
            // lane l builds, for entry jb+l, the 32-bit mask of this warp's pixels inside
            // its bbox: bits [4g, 4g+4) = quad g (column bit = lane&1, row bit = lane>>1&1)
            unsigned W = 0u;
            const int jl = jb + (int)lane;
            if (jl < nb) {
                const short4 bb = s_bb[jl];
                const unsigned cb = (unsigned)(X0 >= bb.x && X0 < bb.y) | ((unsigned)(X0 + 1 >= bb.x && X0 + 1 < bb.y) << 1);
                const int r0 = max((int)bb.z - Y0, 0), r1 = min((int)bb.w - Y0, TILE);
                if (cb && r1 > r0) {
                    unsigned x = ((1u << (r1 - r0)) - 1u) << r0;  // rows of the tile, 16 bits
                    x = (x | (x << 8)) & 0x00FF00FFu;
                    x = (x | (x << 4)) & 0x0F0F0F0Fu;
                    x = (x | (x << 2)) & 0x33333333u;
                    x = (x | (x << 1)) & 0x55555555u;                // row r -> bit 2r
                    W = x * cb;                                       // row r -> bits 2r, 2r+1 = cb
                }
            }
            unsigned gmask = 0u;
#pragma unroll
            for (int g = 0; g < 8; g++) {
                const unsigned bm = __ballot_sync(0xffffffffu, ((W >> (4 * g)) & 0xFu) != 0u);
                if ((int)grp == g) gmask = bm;
            }
            if (done) gmask = 0u;
            const unsigned mybit = 4u * grp + (lane & 3u);
            while (__any_sync(0xffffffffu, gmask != 0u)) {
                const int jo = __ffs(gmask) - 1;
                gmask &= gmask - 1;
                const int j = jb + jo;
                bool contrib = false;
                float w = 0.f;
                const unsigned Wj = __shfl_sync(0xffffffffu, W, jo & 31);
                if (jo >= 0 && !done) {
                    if ((Wj >> mybit) & 1u) {
                        const RecF& r = s_rec[j].r;
                        const double l0 = fma(r.a[0], pcx, fma(r.a[1], pcy, r.a[2]));
                        const double l1 = fma(r.a[3], pcx, fma(r.a[4], pcy, r.a[5]));
                        const double l2 = fma(r.a[6], pcx, fma(r.a[7], pcy, r.a[8]));
                        if (l0 >= r.r_lo && l1 >= r.r_lo && l2 >= r.r_lo) {
                            const double rr = l0 < l1 ? (l0 < l2 ? l0 : l2) : (l1 < l2 ? l1 : l2);
                            bool flag = rr <= r.r_hi;
                            if (!flag) {
                                if constexpr (ACC64) {
                                    const double2 os = s_os[j];
                                    double a;
                                    if (opt.mode == 0) {
                                        const double rc = fmin(rr, 1.0);
                                        a = os.x * (os.y == 1.0 ? rc : pow(rc, os.y));
                                    } else {
                                        double x = rr * r.phis / os.y;
                                        if (x > 700.0) x = 700.0;
                                        a = os.x * (1.0 / (1.0 + exp(x)));
                                    }
                                    if (a > ALPHA_CLAMP) a = ALPHA_CLAMP;
                                    const double wd = TS_M(T, a);
                                    const double tn = TS_M(T, TS_S(1.0, a));
                                    // r differs from the reference's by ~1e-13 relative
                                    flag = fabs(tn - T_MIN) <= 1e-9 * tn || fabs(wd - opt.tau_contrib) <= 1e-9 * wd;
                                    if (!flag) {
                                        C0 += wd * r.rgb[0];
                                        C1 += wd * r.rgb[1];
                                        C2 += wd * r.rgb[2];
                                        w = (float)wd;
                                        contrib = true;
                                        last = b + j;
                                        if (out.frag_tri) {
                                            const long long fi = out.frag_off[py * cam.width + px] + cnt;
                                            const unsigned src = s_src[j];
                                            out.frag_tri[fi] = (int)src;
                                            out.frag_w[fi] = wd;
                                            out.frag_z[fi] = __longlong_as_double((long long)out.zkey[src]);
                                        }
                                        cnt++;
                                        T = tn;
                                        done = tn < T_MIN;
                                        // pixel count uses the fp64 weight
                                        if (wd > opt.tau_contrib) red_add_shared(&s_pix[j], 1);
                                    }
                                } else {
                                    float ea;
                                    const float a = fminf(alpha_fast(r, rr, opt.mode, ea), ALPHA_CLAMP_F);
                                    w = (float)T * a;
                                    const float tn = fmaf(-(float)T, a, (float)T);
                                    const float en = fmaf(ea * a, __frcp_rn(1.f - a), epsT + 2.4e-7f);
                                    const float ew = epsT + ea + 1.2e-7f;
                                    flag = fabsf(tn - T_MIN_F) <= fmaf(2.f * en, tn, 1e-11f) ||
                                           fabsf(w - tau) <= fmaf(2.f * ew, w, 1e-9f);
                                    if (!flag) {
                                        C0 = fmaf(w, r.rgb[0], (float)C0);
                                        C1 = fmaf(w, r.rgb[1], (float)C1);
                                        C2 = fmaf(w, r.rgb[2], (float)C2);
                                        contrib = true;
                                        last = b + j;
                                        cnt++;
                                        T = tn;
                                        epsT = en;
                                        done = tn < T_MIN_F;
                                        if (w > tau) red_add_shared(&s_pix[j], 1);
                                    }
                                }
                            }
                            if (flag) {
                                flag_pos = b + j;
                                done = true;
                            }
                        }
                    }
                }
                if (done) gmask = 0u;
                if (contrib) red_max_shared(&s_maxw[j], __float_as_uint(w));
            }
        }
        __syncthreads();
        if (threadIdx.x < nb) {
            const unsigned src = s_src[threadIdx.x];
            if (s_maxw[threadIdx.x] && out.max_weight)
                red_gmax_u32((unsigned*)out.max_weight + src, s_maxw[threadIdx.x]);
            if (s_pix[threadIdx.x] && out.pixel_count) red_gadd_s32(out.pixel_count + src, s_pix[threadIdx.x]);
            s_maxw[threadIdx.x] = 0u;
            s_pix[threadIdx.x] = 0;
        }
    }
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
            out.last_pos[p] = last;
            if (out.n_frag) out.n_frag[p] = cnt;
            if (out.last_src) out.last_src[p] = last >= 0 ? (int)ent_src[last] : -1;
        }
    }
    // this tile's flags are published: count the CTA (k_fixup_fwd ends when all have)
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(&out.ctr->blend_done, 1ull);
}

// ---------------------------------------------------------------------------
// k_fixup_fwd: exact (fp64) replay of flagged pixels, one CTA per pixel.
// The CTA evaluates alpha for FXC consecutive tile entries in parallel
// (shared memory), then warp 0 composites the contributing ones in entry
// order; repeat until the pixel saturates or the tile's list ends.  Entries
// before the flag position already committed their statistics in
// k_blend_fast (their decisions were certain); from it on the fix-up does.
// ---------------------------------------------------------------------------
constexpr int FXC = 1024;
constexpr int FX_T = 512, FX_PER = FXC / FX_T;  // threads per CTA, entries per thread

template <typename T>
__global__ void __launch_bounds__(FX_T, 2) k_fixup_fwd(Cam cam, Opts opt, const T* __restrict__ opacity,
                                                   const T* __restrict__ sigma, const RecF* __restrict__ rec,
                                                   const int* __restrict__ tile_start,
                                                   const unsigned* __restrict__ ent_src, FastBlendOut out) {
    TS_PDL_LAUNCH_ONLY();
    __shared__ double s_a[FXC];
    __shared__ double s_c[3][FXC];     // colour (training forwards: the fp64 RecC colour)
    __shared__ unsigned s_s[FXC];
    __shared__ int s_done;
    __shared__ short s_idx[FXC];        // render path: passing entries of the chunk, in order
    __shared__ double s_tb[FXC];        // ... and the transmittance in front of each
    __shared__ int s_np, s_used;
    __shared__ int2 s_flag;
    __shared__ double s_red[3][FX_T / 32];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // render forwards (no records / fragments / fp64 colour totals): only the
    // transmittance chain is sequential (one lane); weights, colour sums and
    // statistics of the chunk's fragments are computed in parallel
    const bool fastc = out.frec == nullptr && out.frag_tri == nullptr && out.c_total64 == nullptr;
    // flagged pixel k is published by the blend CTA that stopped on it (pixel >= 0
    // in flags[k]); the list ends when every blend CTA has finished and entry k is
    // still empty.  Entries are consumed (reset to -1) for the next frame.
    const unsigned long long nblend = (unsigned long long)cam.ntx * cam.nty;
    const long long kcap = (long long)cam.width * cam.height;
    for (long long k = blockIdx.x; k < kcap; k += gridDim.x) {
        if (threadIdx.x == 0) {
            volatile int2* fv = reinterpret_cast<volatile int2*>(out.flags + k);
            volatile unsigned long long* dv = &out.ctr->blend_done;
            int2 g;
            for (long long spin = 0;; spin++) {
                g.x = fv->x;
                if (g.x >= 0) break;
                if (*dv >= nblend) {
                    __threadfence();
                    g.x = fv->x;
                    break;
                }
                if (spin > (1ll << 25)) __trap();  // (seconds: the blend never finished -- fail, do not hang)
                __nanosleep(200);
            }
            __threadfence();
            g.y = fv->y;
            s_flag = g;
        }
        __syncthreads();
        const int2 f = s_flag;
        if (f.x < 0) break;
        const int p = f.x, fpos = f.y;
        const int px = p % cam.width, py = p / cam.width;
        const int t = (py / TILE) * cam.ntx + px / TILE;
        double Tt = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0;
        int last = -1, cnt = 0;
        const int s = tile_start[t], e = tile_start[t + 1];
        if (threadIdx.x == 0) s_done = 0;
        __syncthreads();
        for (int base = s; base < e; base += FXC) {
            const int nb = min(FXC, e - base);
            // FX_PER entries per thread, their source ids and bboxes loaded up front
            unsigned srcs[FX_PER];
            short4 bbs[FX_PER];
#pragma unroll
            for (int u = 0; u < FX_PER; u++) {
                const int i = (int)threadIdx.x + u * FX_T;
                srcs[u] = i < nb ? __ldg(ent_src + base + i) : 0u;
            }
#pragma unroll
            for (int u = 0; u < FX_PER; u++) {
                const int i = (int)threadIdx.x + u * FX_T;
                bbs[u] = make_short4(0, 0, 0, 0);
                if (i < nb) {  // x0..y1 sit at byte 116 of the record (4-byte aligned)
                    const int xx = __ldg(reinterpret_cast<const int*>(&rec[srcs[u]].x0));
                    const int yy = __ldg(reinterpret_cast<const int*>(&rec[srcs[u]].y0));
                    bbs[u] = make_short4((short)(xx & 0xffff), (short)(xx >> 16), (short)(yy & 0xffff), (short)(yy >> 16));
                }
            }
#pragma unroll
            for (int u = 0; u < FX_PER; u++) {
                const int i = (int)threadIdx.x + u * FX_T;
                if (i >= nb) break;
                const unsigned src = srcs[u];
                const RecF& r = rec[src];
                double a = 0.0;
                if (px >= bbs[u].x && px < bbs[u].y && py >= bbs[u].z && py < bbs[u].w) {
                    const double rr = edge_r(r, px + 0.5, py + 0.5);
                    a = alpha_exact_r<T>(r, rr, opt.mode, opt, opacity, sigma, src);
                    if (a > ALPHA_CLAMP) a = ALPHA_CLAMP;
                    if (a < ALPHA_MIN) a = 0.0;
                    if (out.recc) {
                        const RecC& rc = out.recc[src];
                        s_c[0][i] = rc.rgb[0];
                        s_c[1][i] = rc.rgb[1];
                        s_c[2][i] = rc.rgb[2];
                    } else {
                        s_c[0][i] = r.rgb[0];
                        s_c[1][i] = r.rgb[1];
                        s_c[2][i] = r.rgb[2];
                    }
                }
                s_a[i] = a;
                s_s[i] = src;
            }
            __syncthreads();
            if (fastc) {
                if (warp == 0) {  // compaction of the passing entries (entry order)
                    int np = 0;
                    for (int i0 = 0; i0 < nb; i0 += 32) {
                        const int i = i0 + (int)lane;
                        const bool pz = i < nb && s_a[i] > 0.0;
                        const unsigned m = __ballot_sync(0xffffffffu, pz);
                        if (pz) s_idx[np + __popc(m & ((1u << lane) - 1u))] = (short)i;
                        np += __popc(m);
                    }
                    __syncwarp();
                    if (lane == 0) {  // the reference's sequential fp64 transmittance
                        int used = np;
                        double tt = Tt;
                        for (int q = 0; q < np; q++) {
                            s_tb[q] = tt;
                            tt = TS_M(tt, TS_S(1.0, s_a[s_idx[q]]));
                            if (tt < T_MIN) {
                                used = q + 1;
                                s_done = 1;
                                break;
                            }
                        }
                        s_np = np;
                        s_used = used;
                    }
                }
                __syncthreads();
                const int used = s_used;
                double c0 = 0.0, c1 = 0.0, c2 = 0.0;
                for (int q = threadIdx.x; q < used; q += FX_T) {
                    const int j = s_idx[q];
                    const double w = s_tb[q] * s_a[j];
                    c0 += w * s_c[0][j];
                    c1 += w * s_c[1][j];
                    c2 += w * s_c[2][j];
                    if (base + j >= fpos) {
                        if (out.max_weight) red_gmax_u32((unsigned*)out.max_weight + s_s[j], __float_as_uint((float)w));
                        if (w > opt.tau_contrib && out.pixel_count) red_gadd_s32(out.pixel_count + s_s[j], 1);
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    c0 += __shfl_xor_sync(0xffffffffu, c0, off);
                    c1 += __shfl_xor_sync(0xffffffffu, c1, off);
                    c2 += __shfl_xor_sync(0xffffffffu, c2, off);
                }
                if (lane == 0) {
                    s_red[0][warp] = c0;
                    s_red[1][warp] = c1;
                    s_red[2][warp] = c2;
                }
                __syncthreads();
#pragma unroll
                for (int w2 = 0; w2 < FX_T / 32; w2++) {
                    C0 += s_red[0][w2];
                    C1 += s_red[1][w2];
                    C2 += s_red[2][w2];
                }
                if (used > 0) {
                    last = base + s_idx[used - 1];
                    // transmittance after the chunk: continue the chain from the last stored value
                    Tt = TS_M(s_tb[used - 1], TS_S(1.0, s_a[s_idx[used - 1]]));
                }
                cnt += used;
                __syncthreads();
                if (s_done) break;
                continue;
            }
            if (threadIdx.x < 32) {
                for (int i0 = 0; i0 < nb && !s_done; i0 += 32) {
                    const int i = i0 + (int)lane;
                    unsigned m = __ballot_sync(0xffffffffu, i < nb && s_a[i] > 0.0);
                    while (m) {
                        const int j = i0 + __ffs(m) - 1;
                        m &= m - 1;
                        const double aj = s_a[j];
                        const double w = Tt * aj;
                        if (lane == 0 && out.frec && base + j >= fpos) {
                            // training forward: record of the exactly replayed fragment
                            const unsigned long long fi = atomicAdd(&out.ctr->n_frec, 1ull);
                            if (fi < out.frec_cap) {
                                FragRec& fr = out.frec[fi];
                                fr.T = Tt;
                                fr.C[0] = C0;
                                fr.C[1] = C1;
                                fr.C[2] = C2;
                                fr.pix = (unsigned)p;
                                fr.src = s_s[j];
                                fr.ord = (unsigned)cnt;
                            } else {
                                out.ctr->frec_over = 1ull;
                            }
                        }
                        C0 += w * s_c[0][j];
                        C1 += w * s_c[1][j];
                        C2 += w * s_c[2][j];
                        const int posj = base + j;
                        if (lane == 0 && out.frag_tri) {
                            const long long fi = out.frag_off[p] + cnt;
                            out.frag_tri[fi] = (int)s_s[j];
                            out.frag_w[fi] = w;
                            out.frag_z[fi] = __longlong_as_double((long long)out.zkey[s_s[j]]);
                        }
                        if (lane == 0 && posj >= fpos) {
                            if (out.max_weight) red_gmax_u32((unsigned*)out.max_weight + s_s[j], __float_as_uint((float)w));
                            if (w > opt.tau_contrib && out.pixel_count) red_gadd_s32(out.pixel_count + s_s[j], 1);
                        }
                        last = posj;
                        cnt++;
                        Tt = TS_M(Tt, TS_S(1.0, aj));
                        if (Tt < T_MIN) {
                            if (lane == 0) s_done = 1;
                            break;
                        }
                    }
                    __syncwarp();
                }
            }
            __syncthreads();
            if (s_done) break;
        }
        if (threadIdx.x == 0) {
            if (out.image) {
                out.image[p * 3 + 0] = (float)fmin(fmax(C0 + Tt * opt.bg[0], 0.0), 1.0);
                out.image[p * 3 + 1] = (float)fmin(fmax(C1 + Tt * opt.bg[1], 0.0), 1.0);
                out.image[p * 3 + 2] = (float)fmin(fmax(C2 + Tt * opt.bg[2], 0.0), 1.0);
            }
            if (out.alpha_map) out.alpha_map[p] = (float)(1.0 - Tt);
            out.t_final[p] = (float)Tt;
            if (out.t_final64) out.t_final64[p] = Tt;
            if (out.c_total64) {
                out.c_total64[p * 3 + 0] = C0 + Tt * opt.bg[0];
                out.c_total64[p * 3 + 1] = C1 + Tt * opt.bg[1];
                out.c_total64[p * 3 + 2] = C2 + Tt * opt.bg[2];
            }
            out.last_pos[p] = last;
            if (out.n_frag) out.n_frag[p] = cnt;
            if (out.last_src) out.last_src[p] = last >= 0 ? (int)ent_src[last] : -1;
            out.flags[k] = make_int2(-1, -1);  // consumed
        }
        __syncthreads();
    }
}

// fragment collection (ts_collect_fragments): fp64 re-composite of the last
// training forward that emits every composited fragment
void launch_blend_fast(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype, const RecF* rec,
                       const short4* bbox, const int* tile_start, const unsigned* ent_src, const FastBlendOut& out,
                       cudaStream_t st) {
    const int ntiles = cam.ntx * cam.nty;
    if (dtype == 1)
        k_blend_fast<double, true><<<ntiles, 256, 0, st>>>(cam, opt, rec, bbox, tile_start, ent_src,
                                                           (const double*)soup.opacity, (const double*)soup.sigma, out);
    else
        k_blend_fast<float, true><<<ntiles, 256, 0, st>>>(cam, opt, rec, bbox, tile_start, ent_src,
                                                          (const float*)soup.opacity, (const float*)soup.sigma, out);
}

void launch_fixup_fwd(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype, const RecF* rec,
                      const int* tile_start, const unsigned* ent_src, const FastBlendOut& out,
                      cudaStream_t st) {
    // 2 entries per thread of a 1024-entry chunk: the dependent record loads of
    // the whole chunk are in flight at once
    const int grid = sm_count() * 2;
    if (dtype == 1)
        launch_pdl(k_fixup_fwd<double>, dim3(grid), dim3(FX_T), 0, st, cam, opt, (const double*)soup.opacity,
                   (const double*)soup.sigma, rec, tile_start, ent_src, out);
    else
        launch_pdl(k_fixup_fwd<float>, dim3(grid), dim3(FX_T), 0, st, cam, opt, (const float*)soup.opacity,
                   (const float*)soup.sigma, rec, tile_start, ent_src, out);
}


}  // namespace ts
