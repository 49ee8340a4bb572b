// ts_common.cuh -- shared definitions for the B200 triangle-splat rasterizer.
//
// fp64 device functions here restate the reference arithmetic operation for
// operation (numba, no fastmath => every product and sum rounded separately),
// written with explicit round-to-nearest intrinsics so that no translation
// unit can contract them into FMAs.  Citations are to /root/reference/pkg/src/trisplat.
#pragma once
#include <cuda_runtime.h>

// Bounds / invariant checks compiled into the checked build only
// (python -m paper_2505_19175_b200.build --checked): a failing check traps the
// kernel (device assert) and the next ts_* call returns TS_ERR_CUDA.
#ifdef TS_CHECKED
#include <cassert>
#define TS_ASSERT(cond) assert(cond)
#else
#define TS_ASSERT(cond) ((void)0)
#endif
#include <stdint.h>

#include "../../include/trisplat_b200.h"

namespace ts {

constexpr double ALPHA_CLAMP = 0.99;         // _kernels.py:18
constexpr double ALPHA_MIN = 1.0 / 255.0;    // _kernels.py:19
constexpr double T_MIN = 1e-4;               // _kernels.py:20
constexpr double DEGENERATE_AREA = 1e-8;     // geometry.py:18
constexpr double DEGENERATE_INRADIUS = 1e-6; // geometry.py:19
constexpr int TILE = 16;                     // render.py:26
constexpr int TILE_PIX = TILE * TILE;

// Camera in device-friendly form (POD, passed by value as a kernel argument).
struct Cam {
    double fx, fy, cx, cy, z_near;
    double R[9];
    double t[3];
    double cc[3];  // camera centre -R^T t (geometry.py:72-74)
    int width, height;
    int ntx, nty;
};

struct Opts {
    int mode, sh_degree, ncoef, solid, validate;
    double tau_cutoff, tau_contrib;
    double bg[3];
};

// Per-source fp64 record consumed by the exact blend / backward kernels.
// 208 B, 16-byte aligned.
struct __align__(16) Rec64 {
    double nx[3], ny[3], d[3];  // outward unit edge normals and offsets (render.py:200-214)
    double phis, sig, opa;      // incenter SDF (<0), window sharpness, opacity
    double rgb[3];              // clamped SH colour (render.py:301-302)
    double qx[3], qy[3];        // projected vertices (needed by backward edge chain)
    int bx0, bx1, by0, by1;     // half-open clipped pixel bbox (render.py:243-250)
    int esign;                  // bit e set <=> esign[e] == -1
    int pad[3];
};
static_assert(sizeof(Rec64) == 208, "Rec64 layout");

// Per-source record of the fast blend (128 B = one cache line).  Edge
// functions are stored pre-divided by phi_s, in fp64, as functions of the
// absolute pixel centre: r = phi/phi_s = min_e(a0*pcx + a1*pcy + a2), which
// matches the reference's fp64 phi/phi_s to ~1e-13 * (W+H)/|phi_s|.  The
// contribution decision alpha >= 1/255 (_kernels.py:103) is r >= r*,
// decided outside the band [r_lo, r_hi] and resolved in fp64 inside it.
struct __align__(16) RecF {
    double a[9];           // (a0,a1,a2) per edge
    double phis;           // phi(s) < 0
    double r_lo, r_hi;     // contribution threshold band
    float f0, f1;          // normalized: sigma, log2(opacity); sigmoid: phis*log2(e)/sigma, opacity
    float rgb[3];
    short x0, x1, y0, y1;  // clipped half-open pixel bbox
    short ox, oy;          // origin of the backward record's relative coordinates
};
static_assert(sizeof(RecF) == 128, "RecF layout");

// Backward-only per-source data (64 B): vertices relative to the record origin,
// 1 / phi_s and the orientation bits of the edges.  The constants of an edge's
// endpoint derivative (_kernels.py:296-318) -- sl = s/l, ul = (b-a)_x/l^2,
// vl = (b-a)_y/l^2 with s the edge's outward sign -- are derived from the
// vertices where they are used (rb_edge), in fp64: edge lengths of
// near-degenerate triangles are ill-conditioned.
struct __align__(16) RecB {
    double2 q[3];     // (x, y) per vertex (one 16-byte load each)
    double inv_phis;  // 1 / phi_s (the backward multiplies instead of dividing)
    unsigned esign;   // bit e: edge e's normal was flipped (s = -1)
    unsigned pad;
};
static_assert(sizeof(RecB) == 64, "RecB layout");

// the derivative constants of edge e = (a -> b) of a RecB
__device__ __forceinline__ void rb_edge(double2 a, double2 b, unsigned esign, int e, double& sl, double& ul,
                                        double& vl) {
    const double ex = b.x - a.x, ey = b.y - a.y;
    const double il = rsqrt(ex * ex + ey * ey);
    sl = ((esign >> e) & 1) ? -il : il;
    ul = ex * il * il;
    vl = ey * il * il;
}

// Training-only per-source fp64 data (48 B): the SH colour before its fp32
// rounding (clipped, render.py:302) and the exact opacity (1 for solid soups)
// and sigma.  The training forward composites and the backward differentiates
// with these, so the suffix colours S_k and dL/dalpha (_kernels.py:250-277)
// carry the reference's fp64 colour, not a rounded copy.
struct __align__(16) RecC {
    double opa, sig;  // (16-byte aligned pairs: one double2 load each)
    double rgb[3];
    double inv_opa;   // 1 / opacity (the backward multiplies instead of dividing)
};
static_assert(sizeof(RecC) == 48, "RecC layout");
// (the streaming backward reads (a[8], phis), (rgb[2], inv_opa) and (ox, oy) as pairs)
static_assert(offsetof(RecF, phis) == offsetof(RecF, a) + 64 + 8 && offsetof(RecF, oy) == offsetof(RecF, ox) + 2 &&
                  offsetof(RecF, ox) % 4 == 0 && offsetof(RecC, inv_opa) == offsetof(RecC, rgb) + 24 &&
                  offsetof(RecC, rgb) % 16 == 0,
              "record layouts of the paired loads");

// Shared-memory images of a RecF for the dense blend kernels: the evaluation
// part (first 96 B) and the tail (last 32 B), copied with 16-byte cp.async.
struct __align__(16) EvalRec {
    double a[9];
    double phis, r_lo, r_hi;
};
static_assert(sizeof(EvalRec) == 96, "EvalRec layout");
struct __align__(16) TailRec {
    float f0, f1, rgb[3];
    short x0, x1, y0, y1, ox, oy;
};
static_assert(sizeof(TailRec) == 32, "TailRec layout");

// Screen-space gradient accumulator per source triangle (backward), fp64.
// gq[6] (q0x,q0y,q1x,q1y,q2x,q2y), go, gsig, grgb[3], gphis, gz, pad
constexpr int SG_STRIDE = 16;
enum { SG_GQ = 0, SG_GO = 6, SG_GSIG = 7, SG_GRGB = 8, SG_GPHIS = 11, SG_GZ = 12 };

#define TS_M(a, b) __dmul_rn((a), (b))
#define TS_A(a, b) __dadd_rn((a), (b))
#define TS_S(a, b) __dsub_rn((a), (b))
#define TS_D(a, b) __ddiv_rn((a), (b))

// numba np.int64(np.floor(x)) on x86-64 (cvttsd2si): INT64_MIN when out of range.
__device__ __forceinline__ long long floor_i64(double x) {
    double f = floor(x);
    if (!(f >= -9223372036854775808.0 && f < 9223372036854775808.0)) return (long long)0x8000000000000000LL;
    return (long long)f;
}

// _project_kernel, render.py:159-190.
struct Proj64 {
    double xc[9];
    double q[6];
    double z, area, phis;
    bool valid_z;
};

__device__ __forceinline__ void project64(const double* v, const Cam& c, Proj64& p) {
    bool z_ok = true;
#pragma unroll
    for (int k = 0; k < 3; k++) {
#pragma unroll
        for (int a = 0; a < 3; a++) {
            double s = TS_A(TS_M(v[k * 3 + 0], c.R[a * 3 + 0]), TS_M(v[k * 3 + 1], c.R[a * 3 + 1]));
            s = TS_A(s, TS_M(v[k * 3 + 2], c.R[a * 3 + 2]));
            p.xc[k * 3 + a] = TS_A(s, c.t[a]);
        }
        if (p.xc[k * 3 + 2] < 1e-12) z_ok = false;
    }
    p.z = TS_D(TS_A(TS_A(p.xc[2], p.xc[5]), p.xc[8]), 3.0);
    if (p.z < c.z_near) z_ok = false;
    p.valid_z = z_ok;
#pragma unroll
    for (int k = 0; k < 3; k++) {
        p.q[k * 2 + 0] = TS_A(TS_D(TS_M(c.fx, p.xc[k * 3 + 0]), p.xc[k * 3 + 2]), c.cx);
        p.q[k * 2 + 1] = TS_A(TS_D(TS_M(c.fy, p.xc[k * 3 + 1]), p.xc[k * 3 + 2]), c.cy);
    }
    double e1x = TS_S(p.q[2], p.q[0]), e1y = TS_S(p.q[3], p.q[1]);
    double e2x = TS_S(p.q[4], p.q[0]), e2y = TS_S(p.q[5], p.q[1]);
    p.area = TS_D(fabs(TS_S(TS_M(e1x, e2y), TS_M(e1y, e2x))), 2.0);
    double perim = 0.0;
#pragma unroll
    for (int e = 0; e < 3; e++) {
        int j = (e + 1) % 3, k = (e + 2) % 3;
        double dx = TS_S(p.q[j * 2], p.q[k * 2]), dy = TS_S(p.q[j * 2 + 1], p.q[k * 2 + 1]);
        perim = TS_A(perim, __dsqrt_rn(TS_A(TS_M(dx, dx), TS_M(dy, dy))));
    }
    p.phis = TS_D(TS_M(-2.0, p.area), perim > 1e-300 ? perim : 1e-300);
}

__device__ __forceinline__ bool accepted(const Proj64& p) {
    // render.py:271-273
    return p.valid_z && (p.area >= DEGENERATE_AREA) && (fabs(p.phis) >= DEGENERATE_INRADIUS);
}

// _edge_bbox_kernel, render.py:193-250.  Writes edges, esign bits, bbox.
struct Edge64 {
    double nx[3], ny[3], d[3];
    int esign;
    long long bb[4];  // x0, x1, y0, y1
};

__device__ __forceinline__ void edge_bbox64(const double* q, double phis, double opa, double sig,
                                            int mode, double tau, int width, int height,
                                            Edge64& E) {
    double ccx = TS_D(TS_A(TS_A(q[0], q[2]), q[4]), 3.0);
    double ccy = TS_D(TS_A(TS_A(q[1], q[3]), q[5]), 3.0);
    E.esign = 0;
#pragma unroll
    for (int e = 0; e < 3; e++) {
        int b = (e + 1) % 3;
        double ax = q[e * 2], ay = q[e * 2 + 1], bx = q[b * 2], by = q[b * 2 + 1];
        double evx = TS_S(bx, ax), evy = TS_S(by, ay);
        double ell = __dsqrt_rn(TS_A(TS_M(evx, evx), TS_M(evy, evy)));
        double nx = TS_D(evy, ell), ny = TS_D(-evx, ell);
        double side = TS_A(TS_M(nx, TS_S(ccx, ax)), TS_M(ny, TS_S(ccy, ay)));
        double s = side > 0 ? -1.0 : 1.0;
        if (side > 0) E.esign |= (1 << e);
        double snx = TS_M(s, nx), sny = TS_M(s, ny);
        E.nx[e] = snx;
        E.ny[e] = sny;
        E.d[e] = -TS_A(TS_M(snx, ax), TS_M(sny, ay));
    }
    double d, t;
    d = TS_S(q[2], q[4]); t = TS_M(d, d); d = TS_S(q[3], q[5]);
    double s0 = __dsqrt_rn(TS_A(t, TS_M(d, d)));
    d = TS_S(q[4], q[0]); t = TS_M(d, d); d = TS_S(q[5], q[1]);
    double s1 = __dsqrt_rn(TS_A(t, TS_M(d, d)));
    d = TS_S(q[0], q[2]); t = TS_M(d, d); d = TS_S(q[1], q[3]);
    double s2 = __dsqrt_rn(TS_A(t, TS_M(d, d)));
    double perim = TS_A(TS_A(s0, s1), s2);
    double sx = TS_D(TS_A(TS_A(TS_M(s0, q[0]), TS_M(s1, q[2])), TS_M(s2, q[4])), perim);
    double sy = TS_D(TS_A(TS_A(TS_M(s0, q[1]), TS_M(s1, q[3])), TS_M(s2, q[5])), perim);
    double f;
    if (mode == 0) {
        f = opa > tau ? TS_S(1.0, pow(TS_D(tau, opa), TS_D(1.0, sig))) : 0.0;
    } else {
        double ratio = TS_D(tau, opa);
        f = ratio < 1.0 ? TS_S(1.0, TS_D(TS_M(sig, log(TS_D(ratio, TS_S(1.0, ratio)))), fabs(phis)))
                        : 0.0;
    }
    E.bb[0] = E.bb[1] = E.bb[2] = E.bb[3] = 0;
    if (!(f > 0.0)) return;
    double xmin = 1e300, ymin = 1e300, xmax = -1e300, ymax = -1e300;
#pragma unroll
    for (int k = 0; k < 3; k++) {
        double px = TS_A(sx, TS_M(TS_S(q[k * 2], sx), f));
        double py = TS_A(sy, TS_M(TS_S(q[k * 2 + 1], sy), f));
        xmin = px < xmin ? px : xmin;
        xmax = px > xmax ? px : xmax;
        ymin = py < ymin ? py : ymin;
        ymax = py > ymax ? py : ymax;
    }
    long long W = width, H = height;
    long long x0 = floor_i64(TS_S(xmin, 0.5)); x0 = x0 > 0 ? x0 : 0; x0 = x0 < W ? x0 : W;
    long long x1 = floor_i64(TS_S(xmax, 0.5)) + 1; x1 = x1 > 0 ? x1 : 0; x1 = x1 < W ? x1 : W;
    long long y0 = floor_i64(TS_S(ymin, 0.5)); y0 = y0 > 0 ? y0 : 0; y0 = y0 < H ? y0 : H;
    long long y1 = floor_i64(TS_S(ymax, 0.5)) + 1; y1 = y1 > 0 ? y1 : 0; y1 = y1 < H ? y1 : H;
    E.bb[0] = x0;
    E.bb[1] = x1 > x0 ? x1 : x0;
    E.bb[2] = y0;
    E.bb[3] = y1 > y0 ? y1 : y0;
}

// sh.py:1-52 constants and basis
__device__ __forceinline__ void sh_basis16(double x, double y, double z, double* out) {
    const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
    const double C20 = 1.0925484305920792, C21 = -1.0925484305920792, C22 = 0.31539156525252005,
                 C23 = -1.0925484305920792, C24 = 0.5462742152960396;
    const double C30 = -0.5900435899266435, C31 = 2.890611442640554, C32 = -0.4570457994644658,
                 C33 = 0.3731763325901154, C34 = -0.4570457994644658, C35 = 1.445305721320277,
                 C36 = -0.5900435899266435;
    double xx = TS_M(x, x), yy = TS_M(y, y), zz = TS_M(z, z);
    out[0] = C0;
    out[1] = TS_M(-C1, y);
    out[2] = TS_M(C1, z);
    out[3] = TS_M(-C1, x);
    out[4] = TS_M(TS_M(C20, x), y);
    out[5] = TS_M(TS_M(C21, y), z);
    out[6] = TS_M(C22, TS_S(TS_S(TS_M(2.0, zz), xx), yy));
    out[7] = TS_M(TS_M(C23, x), z);
    out[8] = TS_M(C24, TS_S(xx, yy));
    out[9] = TS_M(TS_M(C30, y), TS_S(TS_M(3.0, xx), yy));
    out[10] = TS_M(TS_M(TS_M(C31, x), y), z);
    out[11] = TS_M(TS_M(C32, y), TS_S(TS_S(TS_M(4.0, zz), xx), yy));
    out[12] = TS_M(TS_M(C33, z), TS_S(TS_S(TS_M(2.0, zz), TS_M(3.0, xx)), TS_M(3.0, yy)));
    out[13] = TS_M(TS_M(C34, x), TS_S(TS_S(TS_M(4.0, zz), xx), yy));
    out[14] = TS_M(TS_M(C35, z), TS_S(xx, yy));
    out[15] = TS_M(TS_M(C36, x), TS_S(xx, TS_M(3.0, yy)));
}

// sh.py:55-100: d(basis)/d(x,y,z)
__device__ __forceinline__ void sh_basis_grad16(double x, double y, double z, double g[16][3]) {
    const double C1 = 0.4886025119029199;
    const double C20 = 1.0925484305920792, C21 = -1.0925484305920792, C22 = 0.31539156525252005,
                 C23 = -1.0925484305920792, C24 = 0.5462742152960396;
    const double C30 = -0.5900435899266435, C31 = 2.890611442640554, C32 = -0.4570457994644658,
                 C33 = 0.3731763325901154, C34 = -0.4570457994644658, C35 = 1.445305721320277,
                 C36 = -0.5900435899266435;
#pragma unroll
    for (int i = 0; i < 16; i++) g[i][0] = g[i][1] = g[i][2] = 0.0;
    g[1][1] = -C1;
    g[2][2] = C1;
    g[3][0] = -C1;
    g[4][0] = C20 * y;
    g[4][1] = C20 * x;
    g[5][1] = C21 * z;
    g[5][2] = C21 * y;
    g[6][0] = C22 * (-2.0 * x);
    g[6][1] = C22 * (-2.0 * y);
    g[6][2] = C22 * 4.0 * z;
    g[7][0] = C23 * z;
    g[7][2] = C23 * x;
    g[8][0] = C24 * 2.0 * x;
    g[8][1] = C24 * (-2.0 * y);
    g[9][0] = C30 * 6.0 * x * y;
    g[9][1] = C30 * (3.0 * x * x - 3.0 * y * y);
    g[10][0] = C31 * y * z;
    g[10][1] = C31 * x * z;
    g[10][2] = C31 * x * y;
    g[11][0] = C32 * (-2.0 * x * y);
    g[11][1] = C32 * (4.0 * z * z - x * x - 3.0 * y * y);
    g[11][2] = C32 * 8.0 * y * z;
    g[12][0] = C33 * (-6.0 * x * z);
    g[12][1] = C33 * (-6.0 * y * z);
    g[12][2] = C33 * (6.0 * z * z - 3.0 * x * x - 3.0 * y * y);
    g[13][0] = C34 * (4.0 * z * z - 3.0 * x * x - y * y);
    g[13][1] = C34 * (-2.0 * x * y);
    g[13][2] = C34 * 8.0 * x * z;
    g[14][0] = C35 * 2.0 * x * z;
    g[14][1] = C35 * (-2.0 * y * z);
    g[14][2] = C35 * (x * x - y * y);
    g[15][0] = C36 * (3.0 * x * x - 3.0 * y * y);
    g[15][1] = C36 * (-6.0 * x * y);
}

// _fragment_alpha, _kernels.py:26-56 (fp64, exact op order).
// Returns unclamped alpha; r, phi, edge as the reference.
__device__ __forceinline__ double fragment_alpha64(double pcx, double pcy, const Rec64& r,
                                                   int mode, double& rr, double& phi_out,
                                                   int& edge_out) {
    double phi = TS_A(TS_A(TS_M(r.nx[0], pcx), TS_M(r.ny[0], pcy)), r.d[0]);
    int edge = 0;
    double v1 = TS_A(TS_A(TS_M(r.nx[1], pcx), TS_M(r.ny[1], pcy)), r.d[1]);
    if (v1 > phi) { phi = v1; edge = 1; }
    double v2 = TS_A(TS_A(TS_M(r.nx[2], pcx), TS_M(r.ny[2], pcy)), r.d[2]);
    if (v2 > phi) { phi = v2; edge = 2; }
    phi_out = phi;
    edge_out = edge;
    double window;
    if (mode == 0) {
        if (phi >= 0.0) { rr = 0.0; return 0.0; }
        double q = TS_D(phi, r.phis);
        if (q > 1.0) q = 1.0;
        rr = q;
        window = pow(q, r.sig);
    } else {
        double x = TS_D(phi, r.sig);
        if (x > 700.0) x = 700.0;
        window = TS_D(1.0, TS_A(1.0, exp(x)));
        rr = window;
    }
    return TS_M(r.opa, window);
}

// Tile-span of a bbox, render.py:322-325.
__device__ __forceinline__ int tiles_touched(int x0, int x1, int y0, int y1) {
    if (x1 <= x0 || y1 <= y0) return 0;
    int tx0 = x0 / TILE, tx1 = (x1 - 1) / TILE + 1, ty0 = y0 / TILE, ty1 = (y1 - 1) / TILE + 1;
    return (tx1 - tx0) * (ty1 - ty0);
}

template <typename T>
__device__ __forceinline__ bool finite_t(T x) { return isfinite((double)x); }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// fast MUFU math and shared-memory reductions used by the blend kernels
__device__ __forceinline__ float fast_lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void red_max_shared(unsigned* p, unsigned v) {
    asm volatile("red.shared.max.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_shared(int* p, int v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ float fast_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// fire-and-forget global reductions (RED: no value returns to a register)
__device__ __forceinline__ void red_gmax_u32(unsigned* a, unsigned v) {
    asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_gadd_s32(int* a, int v) {
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

// asynchronous global -> shared copies (LDGSTS)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
// bulk prefetch of [p, p + bytes) into L2 (p and bytes multiples of 16)
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}


}  // namespace ts

// Programmatic dependent launch of the per-frame kernel chain: each kernel waits
// for its predecessor grid to complete (griddepcontrol.wait) before touching its
// outputs, then lets its own successor launch, so successor CTAs are scheduled
// while this grid's last wave drains.  A no-op for kernels launched without the
// attribute.
#define TS_PDL_ENTRY() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")
// (the fix-up: its CTAs start while the blend's last wave runs and take each
// flagged pixel as soon as the blend publishes it; no grid-wide wait)
#define TS_PDL_LAUNCH_ONLY() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")
#ifndef __CUDACC_RTC__
#include <mutex>
#include <utility>
namespace ts {
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Per-device launch facts: the SM count and the dynamic shared-memory opt-in of
// each kernel are properties of the current device, cached per device ordinal
// (a process may drive several GPUs, one context each).
constexpr int TS_MAX_DEVICES = 64;
inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev < 0 || dev >= TS_MAX_DEVICES ? 0 : dev;
}
inline int sm_count() {
    static int cache[TS_MAX_DEVICES] = {};
    const int dev = current_device();
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 148;
    }
    return cache[dev];
}
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, size)
inline void smem_optin(const void* kernel, int bytes) {
    struct Entry { const void* k; int dev; int bytes; };
    static std::mutex mu;
    static Entry done[256];
    static int n = 0;
    if (bytes <= 48 * 1024) return;
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < n; i++)
        if (done[i].k == kernel && done[i].dev == dev && done[i].bytes >= bytes) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (n < 256) done[n++] = Entry{kernel, dev, bytes};
}
}  // namespace ts
#endif
