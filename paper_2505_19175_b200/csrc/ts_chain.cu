// ts_chain.cu -- screen-space gradients -> the 59 parameter gradients of every
// triangle (backward.py:59-90 _phis_q_grad, backward.py:158-210 projection
// Jacobian and SH colour path, sh.py:55-100 basis gradient), fp32 parameters.
//
// CTA = 64 triangles, thread = triangle.  The CTA's SH block, vertices and
// screen-space gradient rows are copied to shared memory with coalesced
// cp.async (rows padded against bank conflicts); d_sh is written in place over
// the thread's own SH row and every output block leaves with coalesced 16-byte
// stores (read-add-write when accumulating).  Geometry and the view-direction
// chain are fp64; the 48 SH gradients are basis * dL/draw (fp64, stored fp32).
#include "ts_kernels.cuh"

namespace ts {

namespace {
constexpr int CB = 64;      // triangles per CTA (8 CTAs per SM: independent load / compute phases overlap)
constexpr int SGW = 18;     // doubles per staged gradient row (16 used; 144 B keeps 16-B chunks aligned)

struct ChainStage {
    float4 sh[CB * 13];     // SH rows (12 float4, padded to 13); overwritten with d_sh
    float v[CB * 9];        // vertices; overwritten with d_vertices
    double sg[CB * SGW];    // screen-space gradient rows
    float os[2][CB];        // d_opacity, d_sigma
    // accumulating calls: the gradients already in the output, prefetched with the inputs
    float4 ash[CB * 12];
    float av[CB * 9];
    float aos[2][CB];
};

// sum_c s_c * grad(Y_c)(x, y, z) for the 16 real SH basis functions (sh.py:55-100)
__device__ __forceinline__ void sh_weighted_grad(double x, double y, double z, const double* s, double* g) {
    const double C1 = 0.4886025119029199;
    const double C20 = 1.0925484305920792, C21 = -1.0925484305920792, C22 = 0.31539156525252005,
                 C23 = -1.0925484305920792, C24 = 0.5462742152960396;
    const double C30 = -0.5900435899266435, C31 = 2.890611442640554, C32 = -0.4570457994644658,
                 C33 = 0.3731763325901154, C34 = -0.4570457994644658, C35 = 1.445305721320277,
                 C36 = -0.5900435899266435;
    double gx = 0.0, gy = 0.0, gz = 0.0;
    gy += s[1] * -C1;
    gz += s[2] * C1;
    gx += s[3] * -C1;
    gx += s[4] * (C20 * y);
    gy += s[4] * (C20 * x);
    gy += s[5] * (C21 * z);
    gz += s[5] * (C21 * y);
    gx += s[6] * (C22 * (-2.0 * x));
    gy += s[6] * (C22 * (-2.0 * y));
    gz += s[6] * (C22 * 4.0 * z);
    gx += s[7] * (C23 * z);
    gz += s[7] * (C23 * x);
    gx += s[8] * (C24 * 2.0 * x);
    gy += s[8] * (C24 * (-2.0 * y));
    gx += s[9] * (C30 * 6.0 * x * y);
    gy += s[9] * (C30 * (3.0 * x * x - 3.0 * y * y));
    gx += s[10] * (C31 * y * z);
    gy += s[10] * (C31 * x * z);
    gz += s[10] * (C31 * x * y);
    gx += s[11] * (C32 * (-2.0 * x * y));
    gy += s[11] * (C32 * (4.0 * z * z - x * x - 3.0 * y * y));
    gz += s[11] * (C32 * 8.0 * y * z);
    gx += s[12] * (C33 * (-6.0 * x * z));
    gy += s[12] * (C33 * (-6.0 * y * z));
    gz += s[12] * (C33 * (6.0 * z * z - 3.0 * x * x - 3.0 * y * y));
    gx += s[13] * (C34 * (4.0 * z * z - 3.0 * x * x - y * y));
    gy += s[13] * (C34 * (-2.0 * x * y));
    gz += s[13] * (C34 * 8.0 * x * z);
    gx += s[14] * (C35 * 2.0 * x * z);
    gy += s[14] * (C35 * (-2.0 * y * z));
    gz += s[14] * (C35 * (x * x - y * y));
    gx += s[15] * (C36 * (3.0 * x * x - 3.0 * y * y));
    gy += s[15] * (C36 * (-6.0 * x * y));
    g[0] = gx;
    g[1] = gy;
    g[2] = gz;
}
}  // namespace

// One view's chain for one triangle the view's forward kept (flag set): its
// screen-space gradient row sg -> dv += d_vertices, dop += d_opacity, dsig +=
// d_sigma, and d_sh = basis * dL/draw, written over the SH row (IN_PLACE: one
// view) or added to dsh (several views against the same SH row).
template <bool IN_PLACE>
__device__ __forceinline__ void chain_tri(const Cam& cam, const Opts& opt, const double* v, float4* shrow,
                                          float4* dsh, const double* sg, double* dv, double& dop, double& dsig) {
    double gq[6];
#pragma unroll
    for (int k = 0; k < 6; k++) gq[k] = sg[SG_GQ + k];
    dop += sg[SG_GO];
    dsig += sg[SG_GSIG];
    const double grgb[3] = {sg[SG_GRGB], sg[SG_GRGB + 1], sg[SG_GRGB + 2]};
    const double gphis = sg[SG_GPHIS], gzz = sg[SG_GZ];
    // camera-space vertices and their projections; the gradient only needs them
    // accurate (not bit-exact): one reciprocal per vertex instead of two quotients
    double xc[9], iz[3], q[6];
#pragma unroll
    for (int k = 0; k < 3; k++) {
#pragma unroll
        for (int a = 0; a < 3; a++)
            xc[k * 3 + a] = fma(v[k * 3 + 0], cam.R[a * 3 + 0],
                                fma(v[k * 3 + 1], cam.R[a * 3 + 1], fma(v[k * 3 + 2], cam.R[a * 3 + 2], cam.t[a])));
        iz[k] = 1.0 / xc[k * 3 + 2];
        q[k * 2 + 0] = fma(cam.fx * xc[k * 3 + 0], iz[k], cam.cx);
        q[k * 2 + 1] = fma(cam.fy * xc[k * 3 + 1], iz[k], cam.cy);
    }
    if (opt.mode == 0) {
        // _phis_q_grad, backward.py:59-90: phi_s = -2 area / perimeter
        const double e1x = q[2] - q[0], e1y = q[3] - q[1];
        const double e2x = q[4] - q[0], e2y = q[5] - q[1];
        const double cross = e1x * e2y - e1y * e2x;
        const double sgn = (cross > 0) - (cross < 0);
        double dperim[6] = {0, 0, 0, 0, 0, 0};
        double perim = 0.0;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            const int b = a == 2 ? 0 : a + 1;
            const double dx = q[a * 2] - q[b * 2], dy = q[a * 2 + 1] - q[b * 2 + 1];
            const double nn = dx * dx + dy * dy;
            const double ind = rsqrt(nn);
            perim += nn * ind;
            const double ux = dx * ind, uy = dy * ind;
            dperim[a * 2] += ux;
            dperim[a * 2 + 1] += uy;
            dperim[b * 2] -= ux;
            dperim[b * 2 + 1] -= uy;
        }
        const double area = fabs(cross) * 0.5;
        const double dcross[6] = {q[3] - q[5], q[4] - q[2], q[5] - q[1], q[0] - q[4], q[1] - q[3], q[2] - q[0]};
        const double ip = 1.0 / perim;
        const double coef_a = -2.0 * ip;
        const double coef_p = 2.0 * area * ip * ip;
#pragma unroll
        for (int k = 0; k < 6; k++) gq[k] += gphis * (coef_a * (0.5 * sgn * dcross[k]) + coef_p * dperim[k]);
    }
    // projection Jacobian, backward.py:181-190
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const double izk = iz[k];
        const double dx = cam.fx * gq[k * 2] * izk;
        const double dy = cam.fy * gq[k * 2 + 1] * izk;
        const double dz = (-cam.fx * xc[k * 3] * gq[k * 2] - cam.fy * xc[k * 3 + 1] * gq[k * 2 + 1]) * (izk * izk) +
                          gzz * (1.0 / 3.0);
#pragma unroll
        for (int b = 0; b < 3; b++) dv[k * 3 + b] += dx * cam.R[b] + dy * cam.R[3 + b] + dz * cam.R[6 + b];
    }
    // colour path, backward.py:192-205 (sh.py:30-52 basis, 55-100 gradient)
    double u[3];
#pragma unroll
    for (int b = 0; b < 3; b++) u[b] = (v[b] + v[3 + b] + v[6 + b]) * (1.0 / 3.0) - cam.cc[b];
    // 1 / max(|u|, 1e-12)
    const double uu2 = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    const double iun = uu2 > 1e-24 ? rsqrt(uu2) : 1e12;
    const double vx = u[0] * iun, vy = u[1] * iun, vz = u[2] * iun;
    double basis[16];
    sh_basis16(vx, vy, vz, basis);
    const int ncoef = opt.ncoef;
    double raw[3] = {0.5, 0.5, 0.5};
#pragma unroll
    for (int qd = 0; qd < 12; qd++) {
        const float4 c4 = shrow[qd];
        const float cv[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int uu = 0; uu < 4; uu++) {
            const int idx = qd * 4 + uu;
            if (idx / 3 < ncoef) raw[idx % 3] += basis[idx / 3] * (double)cv[uu];
        }
    }
    double d_raw[3];
#pragma unroll
    for (int ch = 0; ch < 3; ch++) d_raw[ch] = (raw[ch] > 0.0 && raw[ch] < 1.0) ? grgb[ch] : 0.0;
    // s_c = sum_ch d_raw[ch] * coef[c][ch]; d_sh[c][ch] = basis[c] * d_raw[ch] (IN_PLACE)
    double s[16];
#pragma unroll
    for (int c = 0; c < 16; c++) s[c] = 0.0;
#pragma unroll
    for (int qd = 0; qd < 12; qd++) {
        const float4 c4 = shrow[qd];
        const float cv[4] = {c4.x, c4.y, c4.z, c4.w};
        float o4[4];
#pragma unroll
        for (int uu = 0; uu < 4; uu++) {
            const int idx = qd * 4 + uu, c = idx / 3, ch = idx % 3;
            const bool on = c < ncoef;
            if (on) s[c] += d_raw[ch] * (double)cv[uu];
            o4[uu] = on ? (float)(basis[c] * d_raw[ch]) : 0.f;
        }
        if constexpr (IN_PLACE) {
            shrow[qd] = make_float4(o4[0], o4[1], o4[2], o4[3]);
        } else {
            float4 a4 = dsh[qd];
            a4.x += o4[0]; a4.y += o4[1]; a4.z += o4[2]; a4.w += o4[3];
            dsh[qd] = a4;
        }
    }
    double ddir[3];
    sh_weighted_grad(vx, vy, vz, s, ddir);
    const double dot = vx * ddir[0] + vy * ddir[1] + vz * ddir[2];
#pragma unroll
    for (int b = 0; b < 3; b++) {
        const double du = (ddir[b] - (b == 0 ? vx : b == 1 ? vy : vz) * dot) * (iun * (1.0 / 3.0));
#pragma unroll
        for (int k = 0; k < 3; k++) dv[k * 3 + b] += du;
    }
}

__global__ void __launch_bounds__(CB, 8) k_chain_bwd32(Cam cam, Opts opt, const float* __restrict__ verts,
                                                       const float* __restrict__ sh,
                                                       const unsigned* __restrict__ flag,
                                                       const double* __restrict__ sgrad, long long n,
                                                       ts_grads grads, int accumulate) {
    TS_PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char s_chain[];
    ChainStage& S = *reinterpret_cast<ChainStage*>(s_chain);
    const int tid = threadIdx.x;
    const long long i0 = (long long)blockIdx.x * CB;
    const int nt = (int)min((long long)CB, n - i0);
    // ---- stage (coalesced cp.async) ----
    {
        const float4* g = reinterpret_cast<const float4*>(sh + i0 * 48);
        for (int c = tid; c < nt * 12; c += CB) {
            const int tri = c / 12;
            cp_async16(&S.sh[tri * 13 + (c - tri * 12)], g + c);
        }
        const float* gv = verts + i0 * 9;
        if (nt == CB) {
            for (int c = tid; c < CB * 9 / 4; c += CB)
                cp_async16(reinterpret_cast<float4*>(S.v) + c, reinterpret_cast<const float4*>(gv) + c);
        } else {
            for (int c = tid; c < nt * 9; c += CB) cp_async4(S.v + c, gv + c);
        }
        const double2* gs = reinterpret_cast<const double2*>(sgrad + i0 * SG_STRIDE);
        for (int c = tid; c < nt * (SG_STRIDE / 2); c += CB) {
            const int tri = c / (SG_STRIDE / 2), q = c - tri * (SG_STRIDE / 2);
            cp_async16(reinterpret_cast<double2*>(&S.sg[tri * SGW]) + q, gs + c);
        }
        cp_async_commit();
        if (accumulate) {  // the output's current values, consumed only at the write-out
            const float4* ga = reinterpret_cast<const float4*>(grads.d_sh + i0 * 48);
            for (int c = tid; c < nt * 12; c += CB) cp_async16(&S.ash[c], ga + c);
            const float* gva = grads.d_vertices + i0 * 9;
            for (int c = tid; c < nt * 9; c += CB) cp_async4(&S.av[c], gva + c);
            if (tid < nt) {
                cp_async4(&S.aos[0][tid], grads.d_opacity + i0 + tid);
                cp_async4(&S.aos[1][tid], grads.d_sigma + i0 + tid);
            }
            cp_async_commit();
            cp_async_wait_group1();  // the inputs; the prefetch may still be in flight
        } else {
            cp_async_wait_all();
        }
        __syncthreads();
    }
    const long long i = i0 + tid;
    if (tid < nt) {
        float* vrow = &S.v[tid * 9];
        float4* shrow = &S.sh[tid * 13];
        double dv[9];
#pragma unroll
        for (int k = 0; k < 9; k++) dv[k] = 0.0;
        double dop = 0.0, dsig = 0.0;
        if (!flag[i]) {
#pragma unroll
            for (int q = 0; q < 12; q++) shrow[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            const double* sg = &S.sg[tid * SGW];
            double v[9];
#pragma unroll
            for (int k = 0; k < 9; k++) v[k] = (double)vrow[k];
            chain_tri<true>(cam, opt, v, shrow, nullptr, sg, dv, dop, dsig);
        }
#pragma unroll
        for (int k = 0; k < 9; k++) vrow[k] = (float)dv[k];
        S.os[0][tid] = (float)dop;
        S.os[1][tid] = (float)dsig;
    }
    cp_async_wait_all();
    __syncthreads();
    // ---- coalesced write-out ----
    {
        float4* g = reinterpret_cast<float4*>(grads.d_sh + i0 * 48);
        for (int c = tid; c < nt * 12; c += CB) {
            const int tri = c / 12;
            float4 v = S.sh[tri * 13 + (c - tri * 12)];
            if (accumulate) {
                const float4 o = S.ash[c];
                v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
            }
            g[c] = v;
        }
        float* gv = grads.d_vertices + i0 * 9;
        for (int c = tid; c < nt * 9; c += CB) gv[c] = accumulate ? S.av[c] + S.v[c] : S.v[c];
        if (tid < nt) {
            grads.d_opacity[i0 + tid] = accumulate ? S.aos[0][tid] + S.os[0][tid] : S.os[0][tid];
            grads.d_sigma[i0 + tid] = accumulate ? S.aos[1][tid] + S.os[1][tid] : S.os[1][tid];
        }
    }
}

// Deferred chain of several views of one scene (training steps over many
// views): each view's blend backward left its screen-space gradients in its
// own slot, and this kernel chains all of them per triangle against ONE read
// of the parameters and ONE read-add-write of the accumulated gradients
// (instead of one of each per view: 1.6 GB -> ~0.4 + 0.26 GB per view at
// 2M triangles).  Same stage / write-out scheme as k_chain_bwd32, with a
// padded d_sh accumulator instead of the in-place SH row.
struct ChainMultiStage {
    float4 sh[CB * 13];
    float4 dsh[CB * 13];    // d_sh accumulator (the output's values when accumulating)
    float v[CB * 9];
    float av[CB * 9];
    float aos[2][CB];
};

#ifndef TS_CHAIN_MULTI_MINB
#define TS_CHAIN_MULTI_MINB 6  // (8: 0.272 ms per view at 8 views, spilling; 6: 0.258; 4: 0.315)
#endif
__global__ void __launch_bounds__(CB, TS_CHAIN_MULTI_MINB) k_chain_multi32(ChainViews cv, Opts opt, const float* __restrict__ verts,
                                                         const float* __restrict__ sh, long long lo, long long n,
                                                         ts_grads grads, int accumulate) {
    TS_PDL_ENTRY();
    extern __shared__ __align__(16) unsigned char s_chain[];
    ChainMultiStage& S = *reinterpret_cast<ChainMultiStage*>(s_chain);
    const int tid = threadIdx.x;
    const long long i0 = (long long)blockIdx.x * CB;  // (relative to lo: every pointer below is offset)
    const int nt = (int)min((long long)CB, n - i0);
    {
        const float4* g = reinterpret_cast<const float4*>(sh + i0 * 48);
        for (int c = tid; c < nt * 12; c += CB) {
            const int tri = c / 12;
            cp_async16(&S.sh[tri * 13 + (c - tri * 12)], g + c);
        }
        const float* gv = verts + i0 * 9;
        if (nt == CB) {
            for (int c = tid; c < CB * 9 / 4; c += CB)
                cp_async16(reinterpret_cast<float4*>(S.v) + c, reinterpret_cast<const float4*>(gv) + c);
        } else {
            for (int c = tid; c < nt * 9; c += CB) cp_async4(S.v + c, gv + c);
        }
        if (accumulate) {
            const float4* ga = reinterpret_cast<const float4*>(grads.d_sh + i0 * 48);
            for (int c = tid; c < nt * 12; c += CB) {
                const int tri = c / 12;
                cp_async16(&S.dsh[tri * 13 + (c - tri * 12)], ga + c);
            }
            const float* gva = grads.d_vertices + i0 * 9;
            for (int c = tid; c < nt * 9; c += CB) cp_async4(&S.av[c], gva + c);
            if (tid < nt) {
                cp_async4(&S.aos[0][tid], grads.d_opacity + i0 + tid);
                cp_async4(&S.aos[1][tid], grads.d_sigma + i0 + tid);
            }
        } else {
            for (int c = tid; c < nt * 13; c += CB) S.dsh[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int c = tid; c < nt * 9; c += CB) S.av[c] = 0.f;
            if (tid < nt) S.aos[0][tid] = S.aos[1][tid] = 0.f;
        }
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();
    }
    const long long i = lo + i0 + tid;  // absolute triangle index (flags, screen-space rows)
    if (tid < nt) {
        float* vrow = &S.v[tid * 9];
        double v[9];
#pragma unroll
        for (int k = 0; k < 9; k++) v[k] = (double)vrow[k];
        double dv[9];
#pragma unroll
        for (int k = 0; k < 9; k++) dv[k] = 0.0;
        double dop = 0.0, dsig = 0.0;
        unsigned vis = 0u;  // the views that kept the triangle: all flags in flight at once
        for (int w = 0; w < cv.n; w++) vis |= (__ldg(cv.flag[w] + i) != 0u ? 1u : 0u) << w;
        for (int w = 0; w < cv.n; w++) {
            if (!((vis >> w) & 1u)) continue;
            const double2* row = reinterpret_cast<const double2*>(cv.sgrad[w] + (size_t)i * SG_STRIDE);
            double sg[14];
#pragma unroll
            for (int k = 0; k < 7; k++) {
                const double2 t = __ldg(row + k);
                sg[2 * k] = t.x;
                sg[2 * k + 1] = t.y;
            }
            chain_tri<false>(cv.cam[w], opt, v, &S.sh[tid * 13], &S.dsh[tid * 13], sg, dv, dop, dsig);
        }
#pragma unroll
        for (int k = 0; k < 9; k++) vrow[k] = (float)dv[k];
        S.aos[0][tid] += (float)dop;
        S.aos[1][tid] += (float)dsig;
    }
    __syncthreads();
    {
        float4* g = reinterpret_cast<float4*>(grads.d_sh + i0 * 48);
        for (int c = tid; c < nt * 12; c += CB) {
            const int tri = c / 12;
            g[c] = S.dsh[tri * 13 + (c - tri * 12)];
        }
        float* gv = grads.d_vertices + i0 * 9;
        for (int c = tid; c < nt * 9; c += CB) gv[c] = S.av[c] + S.v[c];
        if (tid < nt) {
            grads.d_opacity[i0 + tid] = S.aos[0][tid];
            grads.d_sigma[i0 + tid] = S.aos[1][tid];
        }
    }
}

bool chain_bwd_fast_ok(const ts_soup& soup, int dtype, const ts_grads& g) {
    // fp32 parameters, 16-byte vector access of the SH / gradient blocks
    return dtype == 0 && !(((uintptr_t)soup.sh | (uintptr_t)g.d_sh | (uintptr_t)soup.vertices) & 15);
}

bool launch_chain_bwd_fast(const Cam& cam, const Opts& opt, const ts_soup& soup, int dtype, const unsigned* flag,
                           const double* sgrad, const ts_grads& g, int accumulate, cudaStream_t st, long long lo,
                           long long hi) {
    if (!chain_bwd_fast_ok(soup, dtype, g)) return false;
    if (hi < 0) hi = soup.n;
    const long long n = hi - lo;
    if (n <= 0) return true;
    // triangles [lo, hi) (lo a multiple of 64: the offset blocks stay 16-byte aligned)
    const float* verts = (const float*)soup.vertices + 9 * lo;
    const float* sh = (const float*)soup.sh + 48 * lo;
    ts_grads gr = g;
    gr.d_vertices += 9 * lo;
    gr.d_opacity += lo;
    gr.d_sigma += lo;
    gr.d_sh += 48 * lo;
    const int smem = (int)sizeof(ChainStage);
    smem_optin((const void*)k_chain_bwd32, smem);
    const unsigned grid = (unsigned)((n + CB - 1) / CB);
    launch_pdl(k_chain_bwd32, dim3(grid), dim3(CB), smem, st, cam, opt, verts, sh, flag + lo,
               sgrad + (size_t)SG_STRIDE * lo, n, gr, accumulate);
    return true;
}

void launch_chain_multi(const ChainViews& cv, const Opts& opt, const ts_soup& soup, const ts_grads& g,
                        int accumulate, cudaStream_t st, long long lo, long long hi) {
    if (hi < 0) hi = soup.n;
    const long long n = hi - lo;
    if (n <= 0) return;
    const float* verts = (const float*)soup.vertices + 9 * lo;
    const float* sh = (const float*)soup.sh + 48 * lo;
    ts_grads gr = g;
    gr.d_vertices += 9 * lo;
    gr.d_opacity += lo;
    gr.d_sigma += lo;
    gr.d_sh += 48 * lo;
    const int smem = (int)sizeof(ChainMultiStage);
    smem_optin((const void*)k_chain_multi32, smem);
    launch_pdl(k_chain_multi32, dim3((unsigned)((n + CB - 1) / CB)), dim3(CB), smem, st, cv, opt, verts, sh, lo, n,
               gr, accumulate);
}

}  // namespace ts
