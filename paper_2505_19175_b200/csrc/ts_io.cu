// ts_io.cu -- model I/O byte work on the device: the binary
// PLY body of the reference's export_mesh / import_ply
// (trisplat/scene_io.py:365-455) packed and unpacked next to the resident
// parameters, so a 2M-triangle soup leaves / enters HBM as one contiguous byte
// buffer per element instead of per-field numpy passes.
//
// Body layout (binary_little_endian 1.0, scene_io.py:382-414):
//   vertex element: 3 N records of 15 bytes {float x, y, z; uchar r, g, b},
//                   the triangle's three vertices in order, colour = quantised
//                   degree-0 SH colour clip(C0 sh0 + 0.5, 0, 1) (:356-363)
//   face element:   N records of 16 bytes {int 3; int 3i, 3i+1, 3i+2}
// The two elements are produced in separate device buffers (the face buffer
// stays 16-byte aligned for vector stores) and concatenated by the host copy.
//
//   k_ply_pack   -- CTA of 256 triangles: the 11,520-byte vertex chunk is
//                   assembled in shared memory and written with 16-byte
//                   coalesced stores; faces as one int4 per triangle
//   k_ply_unpack -- thread per face: count / index validation, positions and
//                   the first vertex's colour gathered by the face indices,
//                   SH DC = (rgb / 255 - 0.5) / C0, opacity 1, sigma given
#include "ts_kernels.cuh"

namespace ts {

namespace {
constexpr int PT = 256;               // triangles per CTA
constexpr int VREC = 15;              // bytes per vertex record
constexpr int VCHUNK = PT * 3 * VREC;  // 11,520 bytes (a multiple of 16)
constexpr double SH_C0 = 0.28209479177387814;

__device__ __forceinline__ unsigned char quantise(double sh0) {
    // np.floor(np.clip(C0 * sh + 0.5, 0, 1) * 255 + 0.5), no contractions
    double c = __dadd_rn(__dmul_rn(SH_C0, sh0), 0.5);
    c = c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);  // NaN passes through like np.clip
    const double q = floor(__dadd_rn(__dmul_rn(c, 255.0), 0.5));
    return (unsigned char)(int)q;
}

template <typename T>
__global__ void __launch_bounds__(PT) k_ply_pack(long long n, const T* __restrict__ vertices,
                                                 const T* __restrict__ sh, unsigned char* __restrict__ vout,
                                                 int4* __restrict__ fout) {
    __shared__ __align__(16) unsigned char s[VCHUNK];
    const long long t0 = (long long)blockIdx.x * PT;
    const long long t = t0 + threadIdx.x;
    if (t < n) {
        unsigned char rgb[3];
#pragma unroll
        for (int c = 0; c < 3; c++) rgb[c] = quantise((double)sh[t * 48 + c]);
        unsigned char* rec = s + threadIdx.x * 3 * VREC;
#pragma unroll
        for (int v = 0; v < 3; v++) {
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const float f = (float)vertices[t * 9 + 3 * v + c];
                const unsigned u = __float_as_uint(f);
#pragma unroll
                for (int b = 0; b < 4; b++) rec[v * VREC + 4 * c + b] = (unsigned char)(u >> (8 * b));
            }
#pragma unroll
            for (int c = 0; c < 3; c++) rec[v * VREC + 12 + c] = rgb[c];
        }
        const int i = (int)(3 * t);
        fout[t] = make_int4(3, i, i + 1, i + 2);
    }
    __syncthreads();
    const long long cnt = n - t0 < PT ? n - t0 : PT;
    const long long bytes = cnt * 3 * VREC;
    unsigned char* dst = vout + t0 * 3 * VREC;
    const long long nvec = bytes / 16;
    for (long long k = threadIdx.x; k < nvec; k += PT)
        reinterpret_cast<uint4*>(dst)[k] = reinterpret_cast<const uint4*>(s)[k];
    for (long long k = nvec * 16 + threadIdx.x; k < bytes; k += PT) dst[k] = s[k];
}

__device__ __forceinline__ float load_f32(const unsigned char* p) {
    const unsigned u = (unsigned)p[0] | ((unsigned)p[1] << 8) | ((unsigned)p[2] << 16) | ((unsigned)p[3] << 24);
    return __uint_as_float(u);
}

template <typename T>
__global__ void __launch_bounds__(PT) k_ply_unpack(long long n_face, long long n_vertex,
                                                   const unsigned char* __restrict__ vin,
                                                   const int4* __restrict__ fin, double sigma,
                                                   T* __restrict__ vertices, T* __restrict__ opacity,
                                                   T* __restrict__ sig, T* __restrict__ sh,
                                                   unsigned long long* __restrict__ bad) {
    const long long t = (long long)blockIdx.x * PT + threadIdx.x;
    if (t >= n_face) return;
    const int4 f = fin[t];
    const int idx[3] = {f.y, f.z, f.w};
    bool ok = f.x == 3;
    for (int v = 0; v < 3; v++) ok = ok && idx[v] >= 0 && (long long)idx[v] < n_vertex;
    if (!ok) {
        // (count mismatch -> 1, index out of range -> 2) in the top bits, first face in the rest
        const unsigned long long code = (f.x != 3 ? 1ull : 2ull) << 62;
        atomicMin(bad, code | (unsigned long long)t);
        return;
    }
#pragma unroll
    for (int v = 0; v < 3; v++) {
        const unsigned char* rec = vin + (long long)idx[v] * VREC;
#pragma unroll
        for (int c = 0; c < 3; c++) vertices[t * 9 + 3 * v + c] = (T)(double)load_f32(rec + 4 * c);
    }
    const unsigned char* rec0 = vin + (long long)idx[0] * VREC;
#pragma unroll
    for (int c = 0; c < 3; c++) {
        const double rgb = (double)rec0[12 + c] / 255.0;
        sh[t * 48 + c] = (T)(__dsub_rn(rgb, 0.5) / SH_C0);
    }
    for (int k = 3; k < 48; k++) sh[t * 48 + k] = (T)0;
    opacity[t] = (T)1;
    sig[t] = (T)sigma;
}

inline unsigned grid_of(long long n) { return (unsigned)((n + PT - 1) / PT); }
}  // namespace

void launch_ply_pack(long long n, const void* vertices, const void* sh, int is_f64, unsigned char* vout,
                     void* fout, cudaStream_t st) {
    if (n <= 0) return;
    if (is_f64)
        k_ply_pack<double><<<grid_of(n), PT, 0, st>>>(n, (const double*)vertices, (const double*)sh, vout,
                                                      (int4*)fout);
    else
        k_ply_pack<float><<<grid_of(n), PT, 0, st>>>(n, (const float*)vertices, (const float*)sh, vout,
                                                     (int4*)fout);
}

void launch_ply_unpack(long long n_face, long long n_vertex, const unsigned char* vin, const void* fin,
                       double sigma, int is_f64, void* vertices, void* opacity, void* sig, void* sh,
                       unsigned long long* bad, cudaStream_t st) {
    cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st);
    if (n_face <= 0) return;
    if (is_f64)
        k_ply_unpack<double><<<grid_of(n_face), PT, 0, st>>>(n_face, n_vertex, vin, (const int4*)fin, sigma,
                                                             (double*)vertices, (double*)opacity, (double*)sig,
                                                             (double*)sh, bad);
    else
        k_ply_unpack<float><<<grid_of(n_face), PT, 0, st>>>(n_face, n_vertex, vin, (const int4*)fin, sigma,
                                                            (float*)vertices, (float*)opacity, (float*)sig,
                                                            (float*)sh, bad);
}

}  // namespace ts
