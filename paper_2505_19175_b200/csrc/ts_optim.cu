// ts_optim.cu -- fused Adam step on the device: the
// reference's adam_step (trisplat/training.py:81-110) over the 59 fp32
// parameters of every triangle, with per-group learning rates and the opacity
// / sigma clamps, moments kept in fp32 on the device.
//
//   k_adam_check  -- thread per parameter element: a non-finite gradient
//                    records the smallest offending triangle of its group
//                    (the reference raises before touching any state); thread
//                    0 turns the device step counter t into this step's bias
//                    corrections (step t + 1);
//   k_adam_update -- thread per element, skipped entirely if any group was
//                    flagged: m, v in fp64 arithmetic, the bias-corrected step in
//                    fp32 (fp64 below the fp32 normal range), clamps; t += 1 only
//                    when the update ran (the step count stays the reference's
//                    even when the host does not read the flags).
// Element e of the flat 59 N space (the DeviceGrads / moment layout
// [vertices 9N | opacity N | sigma N | sh 48N]) reads the parameter tensors
// in place, so one grid covers all groups with coalesced accesses.
#include <algorithm>

#include "ts_kernels.cuh"

namespace ts {

namespace {
constexpr double ADAM_B1 = 0.9, ADAM_B2 = 0.999, ADAM_EPS = 1e-15;

struct AdamGroups {
    float* p[4];
    const float* g[4];
    long long off[5];  // element offsets of the groups; off[4] = 59 N
    int width[4];      // elements per triangle
    double lr[4];
};

__device__ __forceinline__ int group_of(const AdamGroups& a, long long e) {
    return e < a.off[1] ? 0 : (e < a.off[2] ? 1 : (e < a.off[3] ? 2 : 3));
}
// selects instead of a dynamically indexed parameter array (which would be
// copied to local memory)
template <typename T>
__device__ __forceinline__ T pick(int k, T a0, T a1, T a2, T a3) {
    return k == 0 ? a0 : (k == 1 ? a1 : (k == 2 ? a2 : a3));
}
}  // namespace

__global__ void __launch_bounds__(256) k_adam_check(AdamGroups a, unsigned long long* __restrict__ bad,
                                                    const long long* __restrict__ t, double* __restrict__ ibc) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e == 0) {
        const double tt = (double)(*t + 1);
        ibc[0] = 1.0 / (1.0 - pow(ADAM_B1, tt));
        ibc[1] = 1.0 / (1.0 - pow(ADAM_B2, tt));
    }
    if (e >= a.off[4]) return;
    const int k = group_of(a, e);
    const long long local = e - pick(k, a.off[0], a.off[1], a.off[2], a.off[3]);
    const float* g = pick(k, a.g[0], a.g[1], a.g[2], a.g[3]);
    if (!isfinite(g[local])) atomicMin(bad + k, (unsigned long long)(local / pick(k, 9, 1, 1, 48)));
}

__global__ void __launch_bounds__(256) k_adam_update(AdamGroups a, float* __restrict__ m, float* __restrict__ v,
                                                     const double* __restrict__ ibc, long long* __restrict__ t,
                                                     const unsigned long long* __restrict__ bad) {
    if ((bad[0] & bad[1] & bad[2] & bad[3]) != ~0ull) return;  // some group flagged
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e == 0) *t += 1;  // (no thread of this grid reads t)
    if (e >= a.off[4]) return;
    const double ibc1 = ibc[0], ibc2 = ibc[1];
    const int k = group_of(a, e);
    const long long local = e - pick(k, a.off[0], a.off[1], a.off[2], a.off[3]);
    const double g = (double)pick(k, a.g[0], a.g[1], a.g[2], a.g[3])[local];
    float* pp = pick(k, a.p[0], a.p[1], a.p[2], a.p[3]);
    const double lr = pick(k, a.lr[0], a.lr[1], a.lr[2], a.lr[3]);
    const double mm = ADAM_B1 * (double)m[e] + (1.0 - ADAM_B1) * g;
    const double vv = ADAM_B2 * (double)v[e] + (1.0 - ADAM_B2) * g * g;
    m[e] = (float)mm;
    v[e] = (float)vv;
    // the step in fp32 (the parameter is fp32; ~1e-7 relative) unless the
    // second moment is below the fp32 normal range (then fp64 as the reference)
    const double mh = mm * ibc1, vh = vv * ibc2;
    const float step = vh > 1e-30 ? (float)lr * (float)mh / (sqrtf((float)vh) + 1e-15f)
                                  : (float)(lr * mh / (sqrt(vh) + ADAM_EPS));
    float p = pp[local] - step;
    if (k == 1) p = fminf(fmaxf(p, 1e-4f), 1.0f - 1e-4f);  // opacity clamp
    if (k == 2) p = fminf(fmaxf(p, 1e-3f), 1e3f);          // sigma clamp
    pp[local] = p;
}

// The same two passes over four consecutive elements per thread (16-byte loads
// and stores; n % 4 == 0, so a group boundary never splits a quad and every
// group's offset stays 16-byte aligned), grid-stride over one wave of CTAs.
__global__ void __launch_bounds__(256) k_adam_check4(AdamGroups a, unsigned long long* __restrict__ bad,
                                                     const long long* __restrict__ t, double* __restrict__ ibc) {
    const long long nq = a.off[4] >> 2;
    const long long q0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q0 == 0) {
        const double tt = (double)(*t + 1);
        ibc[0] = 1.0 / (1.0 - pow(ADAM_B1, tt));
        ibc[1] = 1.0 / (1.0 - pow(ADAM_B2, tt));
    }
    for (long long q = q0; q < nq; q += (long long)gridDim.x * blockDim.x) {
        const long long e = q << 2;
        const int k = group_of(a, e);
        const long long local = e - pick(k, a.off[0], a.off[1], a.off[2], a.off[3]);
        const float4 g = __ldg(reinterpret_cast<const float4*>(pick(k, a.g[0], a.g[1], a.g[2], a.g[3]) + local));
        const bool f0 = isfinite(g.x), f1 = isfinite(g.y), f2 = isfinite(g.z), f3 = isfinite(g.w);
        if (!(f0 && f1 && f2 && f3)) {
            const long long bad_local = local + (f0 ? (f1 ? (f2 ? 3 : 2) : 1) : 0);  // first non-finite of the quad
            atomicMin(bad + k, (unsigned long long)(bad_local / pick(k, 9, 1, 1, 48)));
        }
    }
}

__global__ void __launch_bounds__(256) k_adam_update4(AdamGroups a, float* __restrict__ m, float* __restrict__ v,
                                                      const double* __restrict__ ibc, long long* __restrict__ t,
                                                      const unsigned long long* __restrict__ bad) {
    if ((bad[0] & bad[1] & bad[2] & bad[3]) != ~0ull) return;  // some group flagged
    const long long q0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q0 == 0) *t += 1;  // (no thread of this grid reads t)
    const double ibc1 = ibc[0], ibc2 = ibc[1];
    const long long nq = a.off[4] >> 2;
    for (long long q = q0; q < nq; q += (long long)gridDim.x * blockDim.x) {
        const long long e = q << 2;
        const int k = group_of(a, e);
        const long long local = e - pick(k, a.off[0], a.off[1], a.off[2], a.off[3]);
        const float4 g4 = __ldg(reinterpret_cast<const float4*>(pick(k, a.g[0], a.g[1], a.g[2], a.g[3]) + local));
        float* pp = pick(k, a.p[0], a.p[1], a.p[2], a.p[3]) + local;
        const double lr = pick(k, a.lr[0], a.lr[1], a.lr[2], a.lr[3]);
        float4 m4 = reinterpret_cast<const float4*>(m)[q], v4 = reinterpret_cast<const float4*>(v)[q];
        float4 p4 = *reinterpret_cast<const float4*>(pp);
        const float gs[4] = {g4.x, g4.y, g4.z, g4.w};
        float ms[4] = {m4.x, m4.y, m4.z, m4.w}, vs[4] = {v4.x, v4.y, v4.z, v4.w};
        float ps[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const double g = (double)gs[u];
            const double mm = ADAM_B1 * (double)ms[u] + (1.0 - ADAM_B1) * g;
            const double vv = ADAM_B2 * (double)vs[u] + (1.0 - ADAM_B2) * g * g;
            ms[u] = (float)mm;
            vs[u] = (float)vv;
            const double mh = mm * ibc1, vh = vv * ibc2;
            const float step = vh > 1e-30 ? (float)lr * (float)mh / (sqrtf((float)vh) + 1e-15f)
                                          : (float)(lr * mh / (sqrt(vh) + ADAM_EPS));
            float p = ps[u] - step;
            if (k == 1) p = fminf(fmaxf(p, 1e-4f), 1.0f - 1e-4f);  // opacity clamp
            if (k == 2) p = fminf(fmaxf(p, 1e-3f), 1e3f);          // sigma clamp
            ps[u] = p;
        }
        reinterpret_cast<float4*>(m)[q] = make_float4(ms[0], ms[1], ms[2], ms[3]);
        reinterpret_cast<float4*>(v)[q] = make_float4(vs[0], vs[1], vs[2], vs[3]);
        *reinterpret_cast<float4*>(pp) = make_float4(ps[0], ps[1], ps[2], ps[3]);
    }
}

void launch_adam_step(float* const params[4], const float* const grads[4], long long n, float* m, float* v,
                      long long* t, const double lrs[4], long long* bad, double* ibc, cudaStream_t st) {
    AdamGroups a;
    const int width[4] = {9, 1, 1, 48};
    long long off = 0;
    for (int k = 0; k < 4; k++) {
        a.p[k] = params[k];
        a.g[k] = grads[k];
        a.width[k] = width[k];
        a.lr[k] = lrs[k];
        a.off[k] = off;
        off += (long long)width[k] * n;
    }
    a.off[4] = off;
    unsigned long long* b = (unsigned long long*)bad;
    cudaMemsetAsync(b, 0xff, 4 * sizeof(unsigned long long), st);  // "none" = all bits set (-1 as int64)
    bool quads = n > 0 && n % 4 == 0 && !(((uintptr_t)m | (uintptr_t)v) & 15);
    for (int k = 0; k < 4; k++) quads = quads && !(((uintptr_t)params[k] | (uintptr_t)grads[k]) & 15);
    if (quads) {
        const long long nq = off / 4;
        const unsigned grid = (unsigned)std::min<long long>((nq + 255) / 256, (long long)sm_count() * 8);
        k_adam_check4<<<grid, 256, 0, st>>>(a, b, t, ibc);
        k_adam_update4<<<grid, 256, 0, st>>>(a, m, v, ibc, t, b);
        return;
    }
    // (n == 0: one thread still advances the step count, like the reference)
    const unsigned grid = (unsigned)((off + 255) / 256) + (off == 0 ? 1u : 0u);
    k_adam_check<<<grid, 256, 0, st>>>(a, b, t, ibc);
    k_adam_update<<<grid, 256, 0, st>>>(a, m, v, ibc, t, b);
}

}  // namespace ts
