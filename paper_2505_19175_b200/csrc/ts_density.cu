// ts_density.cu -- adaptive density control on the device:
// the array work of the reference's ViewStats / prune / sample_candidates /
// midpoint_subdivide / clone_with_noise (trisplat/density.py:27-171) over
// triangles resident in HBM.  The sequential pick loop of densify_step
// (density.py:209-245) is only a prefix sum over the picks' costs and stays on
// the host (density.py in this package), which also draws the random numbers
// from the caller's numpy Generator in the reference's order.
//
//   k_stats_accum    -- one view's (max weight, pixel count, area) folded into
//                       the aggregates: max, count of pixel_count >= min_pixels,
//                       fp64 area sum (density.py:42-71, views in insertion order)
//   k_prune_mark     -- per-triangle low-weight / few-views / dead-opacity bits
//                       (density.py:74-94); the survivors are compacted in order
//                       by the scan in ts_sort.cu
//   k_sample_weights -- inverse-sigma or opacity weights of the pool and their
//                       fp64 sum / NaN flag (density.py:97-100, 111-115)
//   k_sample_keys    -- exponential / max(w, 1e-300) as fp64 bits (all ones when
//                       the weight sum is not finite and positive); a stable LSD
//                       radix sort on those bits is np.argsort(kind="stable")
//   k_pick_info      -- per pick: source triangle, mean area, degenerate flag
//   k_gather_rows    -- row gather by an origin array (-1: zeros), used for the
//                       new soup and for AdamState.remap (training.py:64-78)
//   k_child_vertices -- subdivision corners / in-plane jitter of the children
//                       (density.py:123-171)
#include "ts_kernels.cuh"

namespace ts {

namespace {
constexpr int DT = 256;

__global__ void __launch_bounds__(DT) k_stats_accum(long long n, const float* __restrict__ maxw,
                                                    const int* __restrict__ pixcnt, const float* __restrict__ area,
                                                    int min_pixels, int first, double* __restrict__ acc_maxw,
                                                    int* __restrict__ acc_views, double* __restrict__ acc_area) {
    long long i = (long long)blockIdx.x * DT + threadIdx.x;
    if (i >= n) return;
    const double w = (double)maxw[i];
    const int cov = pixcnt[i] >= min_pixels ? 1 : 0;
    const double a = (double)area[i];
    if (first) {
        // np.maximum(zeros, w): NaN propagates, like the reference
        acc_maxw[i] = (w > 0.0 || isnan(w)) ? w : 0.0;
        acc_views[i] = cov;
        acc_area[i] = 0.0 + a;
    } else {
        const double m = acc_maxw[i];
        acc_maxw[i] = (isnan(m) || isnan(w)) ? (isnan(m) ? m : w) : (w > m ? w : m);
        acc_views[i] += cov;
        acc_area[i] += a;
    }
}

template <typename T>
__global__ void __launch_bounds__(DT) k_prune_mark(long long n, const double* __restrict__ acc_maxw,
                                                   const int* __restrict__ acc_views, const T* __restrict__ opacity,
                                                   double tau_prune, int min_views, double opacity_dead,
                                                   unsigned char* __restrict__ flags) {
    long long i = (long long)blockIdx.x * DT + threadIdx.x;
    if (i >= n) return;
    unsigned f = 0;
    if (acc_maxw[i] < tau_prune) f |= 1u;
    if (acc_views[i] < min_views) f |= 2u;
    if ((double)opacity[i] < opacity_dead) f |= 4u;
    flags[i] = (unsigned char)f;
}

__device__ __forceinline__ long long source_of(long long k, const long long* pool, const long long* kept) {
    long long s = pool ? pool[k] : k;
    return kept ? kept[s] : s;
}

template <typename T>
__global__ void __launch_bounds__(DT) k_sample_weights(long long n, const long long* __restrict__ pool,
                                                       const long long* __restrict__ kept, const T* __restrict__ param,
                                                       int inverse, double* __restrict__ w, double* __restrict__ sum,
                                                       unsigned* __restrict__ nan_flag) {
    long long k = (long long)blockIdx.x * DT + threadIdx.x;
    double x = 0.0;
    if (k < n) {
        const double p = (double)param[source_of(k, pool, kept)];
        // np.maximum propagates NaN
        x = inverse ? 1.0 / (isnan(p) ? p : fmax(p, 1e-12)) : (isnan(p) ? p : fmax(p, 0.0));
        w[k] = x;
    }
    const bool bad = isnan(x);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nan_flag, 1u);
    double s = bad ? 0.0 : x;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    __shared__ double sh[DT / 32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < DT / 32; q++) t += sh[q];
        atomicAdd(sum, t);
    }
}

__global__ void __launch_bounds__(DT) k_sample_keys(long long n, const double* __restrict__ e,
                                                    const double* __restrict__ w, const double* __restrict__ sum,
                                                    const unsigned* __restrict__ nan_flag,
                                                    unsigned long long* __restrict__ keys, unsigned* __restrict__ vals) {
    long long k = (long long)blockIdx.x * DT + threadIdx.x;
    if (k >= n) return;
    const double tot = *sum;
    const bool uniform = *nan_flag != 0u || !isfinite(tot) || !(tot > 0.0);
    const double wk = uniform ? 1.0 : w[k];
    const double key = e[k] / fmax(wk, 1e-300);
    // keys are >= 0 (exponential draws over positive weights): the IEEE bits
    // order like the values; +0.0 for a zero draw
    keys[k] = (unsigned long long)__double_as_longlong(key == 0.0 ? 0.0 : key);
    vals[k] = (unsigned)k;
}

__global__ void k_take(long long count, const unsigned* __restrict__ vals, long long* __restrict__ out) {
    long long k = (long long)blockIdx.x * DT + threadIdx.x;
    if (k < count) out[k] = (long long)vals[k];
}

template <typename T>
__device__ __forceinline__ void load_tri(const T* v, long long i, double p[3][3]) {
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) p[a][b] = (double)v[9 * i + 3 * a + b];
}

// np.cross / np.linalg.norm without contractions
__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
    c[0] = __dsub_rn(__dmul_rn(a[1], b[2]), __dmul_rn(a[2], b[1]));
    c[1] = __dsub_rn(__dmul_rn(a[2], b[0]), __dmul_rn(a[0], b[2]));
    c[2] = __dsub_rn(__dmul_rn(a[0], b[1]), __dmul_rn(a[1], b[0]));
}
__device__ __forceinline__ double norm3(const double* a) {
    return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(a[0], a[0]), __dmul_rn(a[1], a[1])), __dmul_rn(a[2], a[2])));
}

template <typename T>
__global__ void __launch_bounds__(DT) k_pick_info(long long count, const long long* __restrict__ picked,
                                                  const long long* __restrict__ pool, const long long* __restrict__ kept,
                                                  const double* __restrict__ acc_area, double views_div,
                                                  const T* __restrict__ vertices, long long* __restrict__ src,
                                                  double* __restrict__ mean_area, unsigned char* __restrict__ degen) {
    long long k = (long long)blockIdx.x * DT + threadIdx.x;
    if (k >= count) return;
    const long long o = source_of(picked[k], pool, kept);
    src[k] = o;
    mean_area[k] = acc_area[o] / views_div;  // out / max(n_views, 1)
    double p[3][3];
    load_tri(vertices, o, p);
    double a[3], b[3], c[3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
        a[q] = __dsub_rn(p[1][q], p[0][q]);
        b[q] = __dsub_rn(p[2][q], p[0][q]);
    }
    cross3(a, b, c);
    degen[k] = norm3(c) < 1e-12 ? 1 : 0;
}

template <typename T>
__global__ void __launch_bounds__(DT) k_gather_rows(long long n_out, const long long* __restrict__ origin,
                                                    const T* __restrict__ src, T* __restrict__ dst, int width) {
    long long e = (long long)blockIdx.x * DT + threadIdx.x;
    if (e >= n_out * width) return;
    const long long r = e / width;
    const int c = (int)(e - r * width);
    const long long o = origin[r];
    dst[e] = o >= 0 ? src[o * width + c] : (T)0;
}

// code: 0..3 subdivision corner (density.py:130-142), 4 + r clone jittered with
// uniforms[6r .. 6r+5] (angle, radius per vertex; density.py:146-171)
template <typename T>
__global__ void __launch_bounds__(DT) k_child_vertices(long long n_child, const long long* __restrict__ parent,
                                                       const int* __restrict__ code, const double* __restrict__ uni,
                                                       double max_noise_factor, const T* __restrict__ src,
                                                       T* __restrict__ dst) {
    long long k = (long long)blockIdx.x * DT + threadIdx.x;
    if (k >= n_child) return;
    const int cd = code[k];
    if (cd < 0) return;  // plain copy, already gathered
    double v[3][3];
    load_tri(src, parent[k], v);
    double out[3][3];
    if (cd < 4) {
        double m01[3], m12[3], m20[3];
#pragma unroll
        for (int q = 0; q < 3; q++) {
            m01[q] = __dadd_rn(v[0][q], v[1][q]) / 2.0;
            m12[q] = __dadd_rn(v[1][q], v[2][q]) / 2.0;
            m20[q] = __dadd_rn(v[2][q], v[0][q]) / 2.0;
        }
#pragma unroll
        for (int q = 0; q < 3; q++) {
            const double c0[3] = {v[0][q], m01[q], m20[q]};
            const double c1[3] = {m01[q], v[1][q], m12[q]};
            const double c2[3] = {m20[q], m12[q], v[2][q]};
            const double c3[3] = {m01[q], m12[q], m20[q]};
            const double* cc = cd == 0 ? c0 : (cd == 1 ? c1 : (cd == 2 ? c2 : c3));
            out[0][q] = cc[0];
            out[1][q] = cc[1];
            out[2][q] = cc[2];
        }
    } else {
        const double* u = uni + 6 * (long long)(cd - 4);
        double e0[3], e1[3], e2[3], a[3], b[3], nrm[3];
#pragma unroll
        for (int q = 0; q < 3; q++) {
            e0[q] = __dsub_rn(v[1][q], v[0][q]);
            e1[q] = __dsub_rn(v[2][q], v[1][q]);
            e2[q] = __dsub_rn(v[0][q], v[2][q]);
            a[q] = e0[q];
            b[q] = __dsub_rn(v[2][q], v[0][q]);
        }
        const double mean_edge = __dadd_rn(__dadd_rn(norm3(e0), norm3(e1)), norm3(e2)) / 3.0;
        cross3(a, b, nrm);
        const double nn = norm3(nrm);
        double b1[3], b2[3], nh[3];
        const double la = norm3(a);
#pragma unroll
        for (int q = 0; q < 3; q++) {
            nh[q] = nrm[q] / nn;
            b1[q] = a[q] / la;
        }
        cross3(nh, b1, b2);
        const double cap = max_noise_factor * mean_edge;
#pragma unroll
        for (int i = 0; i < 3; i++) {
            const double ang = 2.0 * M_PI * u[2 * i];
            const double rad = cap * u[2 * i + 1];
            double s, c;
            sincos(ang, &s, &c);
#pragma unroll
            for (int q = 0; q < 3; q++)
                out[i][q] = __dadd_rn(v[i][q], __dmul_rn(rad, __dadd_rn(__dmul_rn(c, b1[q]), __dmul_rn(s, b2[q]))));
        }
    }
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) dst[9 * k + 3 * a + b] = (T)out[a][b];
}

inline unsigned grid_of(long long n) { return (unsigned)((n + DT - 1) / DT); }
}  // namespace

void launch_stats_accum(long long n, const float* maxw, const int* pixcnt, const float* area, int min_pixels,
                        int first, double* acc_maxw, int* acc_views, double* acc_area, cudaStream_t st) {
    if (n > 0) k_stats_accum<<<grid_of(n), DT, 0, st>>>(n, maxw, pixcnt, area, min_pixels, first, acc_maxw,
                                                         acc_views, acc_area);
}

void launch_prune_mark(long long n, const double* acc_maxw, const int* acc_views, const void* opacity, int is_f64,
                       double tau_prune, int min_views, double opacity_dead, unsigned char* flags,
                       cudaStream_t st) {
    if (n <= 0) return;
    if (is_f64)
        k_prune_mark<double><<<grid_of(n), DT, 0, st>>>(n, acc_maxw, acc_views, (const double*)opacity, tau_prune,
                                                          min_views, opacity_dead, flags);
    else
        k_prune_mark<float><<<grid_of(n), DT, 0, st>>>(n, acc_maxw, acc_views, (const float*)opacity, tau_prune,
                                                         min_views, opacity_dead, flags);
}

size_t sample_scratch_bytes(long long n) {
    return (size_t)n * (8 + 8 + 8 + 4 + 4) + 64;
}

// scratch: [w f64 n | keys u64 n | keys_alt u64 n | vals u32 n | vals_alt u32 n | sum f64 | flag u32]
void launch_sample_candidates(long long n, const long long* pool, const long long* kept, const void* param,
                              int is_f64, int inverse, const double* expo, long long count, long long* picked,
                              void* scratch, const SortScratch& ss, cudaStream_t st) {
    if (n <= 0 || count <= 0) return;
    char* p = (char*)scratch;
    double* w = (double*)p;
    unsigned long long* keys = (unsigned long long*)(p + 8 * n);
    unsigned long long* keys_alt = keys + n;
    unsigned* vals = (unsigned*)(keys_alt + n);
    unsigned* vals_alt = vals + n;
    double* sum = (double*)(((size_t)(vals_alt + n) + 15) & ~(size_t)15);
    unsigned* flag = (unsigned*)(sum + 1);
    cudaMemsetAsync(sum, 0, 16, st);
    if (is_f64)
        k_sample_weights<double><<<grid_of(n), DT, 0, st>>>(n, pool, kept, (const double*)param, inverse, w, sum,
                                                             flag);
    else
        k_sample_weights<float><<<grid_of(n), DT, 0, st>>>(n, pool, kept, (const float*)param, inverse, w, sum,
                                                            flag);
    k_sample_keys<<<grid_of(n), DT, 0, st>>>(n, expo, w, sum, flag, keys, vals);
    const int parity = radix_sort_u64(n, keys, vals, keys_alt, vals_alt, 0, 64, ss, st);
    k_take<<<grid_of(count), DT, 0, st>>>(count, parity ? vals_alt : vals, picked);
}

void launch_pick_info(long long count, const long long* picked, const long long* pool, const long long* kept,
                      const double* acc_area, long long n_views, const void* vertices, int is_f64, long long* src,
                      double* mean_area, unsigned char* degen, cudaStream_t st) {
    if (count <= 0) return;
    const double div = (double)(n_views > 1 ? n_views : 1);
    if (is_f64)
        k_pick_info<double><<<grid_of(count), DT, 0, st>>>(count, picked, pool, kept, acc_area, div,
                                                            (const double*)vertices, src, mean_area, degen);
    else
        k_pick_info<float><<<grid_of(count), DT, 0, st>>>(count, picked, pool, kept, acc_area, div,
                                                           (const float*)vertices, src, mean_area, degen);
}

void launch_gather_rows(long long n_out, const long long* origin, const void* src, void* dst, int width,
                        int elem_bytes, cudaStream_t st) {
    if (n_out <= 0 || width <= 0) return;
    const long long tot = n_out * width;
    if (elem_bytes == 8)
        k_gather_rows<double><<<grid_of(tot), DT, 0, st>>>(n_out, origin, (const double*)src, (double*)dst, width);
    else
        k_gather_rows<float><<<grid_of(tot), DT, 0, st>>>(n_out, origin, (const float*)src, (float*)dst, width);
}

void launch_child_vertices(long long n_child, const long long* parent, const int* code, const double* uni,
                           double max_noise_factor, const void* src, void* dst, int is_f64, cudaStream_t st) {
    if (n_child <= 0) return;
    if (is_f64)
        k_child_vertices<double><<<grid_of(n_child), DT, 0, st>>>(n_child, parent, code, uni, max_noise_factor,
                                                                  (const double*)src, (double*)dst);
    else
        k_child_vertices<float><<<grid_of(n_child), DT, 0, st>>>(n_child, parent, code, uni, max_noise_factor,
                                                                 (const float*)src, (float*)dst);
}

}  // namespace ts
