// ts_loss.cu -- on-device photometric loss: the
// reference's (1-lam) L1 + lam (1-SSIM)/2 and its gradient w.r.t. the
// rendered image (trisplat/losses.py:46-142), fp64 statistics.
//
//   k_ssim_stats  -- CTA = 16x16 valid 11x11 windows of one channel: the
//                    26x26 input patch of x and y in shared memory, separable
//                    Gaussian sums of x, y, x^2, xy, y^2 (horizontal pass over
//                    26 rows, vertical pass per window), the SSIM map value and
//                    its partials w.r.t. the window statistics (losses.py:
//                    76-100), written as three fp32 gradient maps; the map sum
//                    per channel by one fp64 atomic per CTA;
//   k_ssim_grad   -- CTA = 16x16 pixels of one channel: the adjoint (same,
//                    zero-embedded) correlations of the three maps (:69-73,
//                    :101-106) combined with x and y, plus the L1 term's sign
//                    gradient and |diff| sum (:130-132), into d_image;
//   k_loss_final  -- the scalar loss and mean SSIM (:133-142).
#include "ts_kernels.cuh"

namespace ts {

namespace {
constexpr int LW = 11, LH = 5, LT = 16, LP = LT + LW - 1;  // window, half, tile, patch
constexpr double LK1 = 0.01, LK2 = 0.03;

__device__ __forceinline__ double gw(int k) {  // normalised Gaussian, sigma 1.5 (losses.py:48-52)
    const double x = (double)(k - LH);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < LW; i++) {
        const double t = (double)(i - LH);
        s += exp(-t * t / 4.5);
    }
    return exp(-x * x / 4.5) / s;
}

__device__ __forceinline__ double block_sum_256(double v, double* s_red) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int tid = threadIdx.y * LT + threadIdx.x;
    if ((tid & 31) == 0) s_red[tid >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (tid == 0)
        for (int w = 0; w < 8; w++) t += s_red[w];
    return t;
}
}  // namespace

__global__ void __launch_bounds__(256) k_ssim_stats(const float* __restrict__ x, const float* __restrict__ y, int H,
                                                    int W, float* __restrict__ gmap, double* __restrict__ sums) {
    __shared__ double s_x[LP][LP + 1], s_y[LP][LP + 1];
    __shared__ double s_h[5][LP][LT];
    __shared__ double s_w[LW];
    __shared__ double s_red[8];
    const int c = blockIdx.z, Hv = H - 2 * LH, Wv = W - 2 * LH;
    const int v0 = blockIdx.y * LT, u0 = blockIdx.x * LT;  // first valid window (row, col)
    const int tid = threadIdx.y * LT + threadIdx.x;
    if (tid < LW) s_w[tid] = gw(tid);
    for (int k = tid; k < LP * LP; k += 256) {
        const int r = k / LP, q = k % LP, i = v0 + r, j = u0 + q;
        const bool in = i < H && j < W;
        s_x[r][q] = in ? (double)x[((size_t)i * W + j) * 3 + c] : 0.0;
        s_y[r][q] = in ? (double)y[((size_t)i * W + j) * 3 + c] : 0.0;
    }
    __syncthreads();
    for (int k = tid; k < LP * LT; k += 256) {  // horizontal pass
        const int r = k / LT, q = k % LT;
        double a = 0, b = 0, aa = 0, ab = 0, bb = 0;
#pragma unroll
        for (int t = 0; t < LW; t++) {
            const double w = s_w[t], xv = s_x[r][q + t], yv = s_y[r][q + t];
            a = fma(w, xv, a);
            b = fma(w, yv, b);
            aa = fma(w, xv * xv, aa);
            ab = fma(w, xv * yv, ab);
            bb = fma(w, yv * yv, bb);
        }
        s_h[0][r][q] = a; s_h[1][r][q] = b; s_h[2][r][q] = aa; s_h[3][r][q] = ab; s_h[4][r][q] = bb;
    }
    __syncthreads();
    const int vi = v0 + threadIdx.y, vj = u0 + threadIdx.x;
    double smap = 0.0;
    if (vi < Hv && vj < Wv) {
        double st[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int t = 0; t < LW; t++) {
            const double w = s_w[t];
#pragma unroll
            for (int m = 0; m < 5; m++) st[m] = fma(w, s_h[m][threadIdx.y + t][threadIdx.x], st[m]);
        }
        const double mx = st[0], my = st[1];
        const double c1 = LK1 * LK1, c2 = LK2 * LK2;
        const double vx = st[2] - mx * mx, vy = st[4] - my * my, cxy = st[3] - mx * my;
        const double a1 = 2.0 * mx * my + c1, a2 = 2.0 * cxy + c2;
        const double b1 = mx * mx + my * my + c1, b2 = vx + vy + c2;
        const double bb = b1 * b2;
        smap = (a1 * a2) / bb;
        const double da1 = a2 / bb, da2 = a1 / bb, db1 = -smap / b1, db2 = -smap / b2;
        const double s = 1.0 / ((double)Hv * (double)Wv);
        const double g_mu = 2.0 * my * da1 + 2.0 * mx * db1 - 2.0 * my * da2 - 2.0 * mx * db2;
        const size_t plane = (size_t)Hv * Wv, o = (size_t)vi * Wv + vj;
        float* g = gmap + (size_t)c * 3 * plane;
        g[o] = (float)(g_mu * s);
        g[plane + o] = (float)(db2 * s);
        g[2 * plane + o] = (float)(2.0 * da2 * s);
    }
    const double t = block_sum_256(smap, s_red);
    if (tid == 0) atomicAdd(sums + 1 + c, t);
}

__global__ void __launch_bounds__(256) k_ssim_grad(const float* __restrict__ x, const float* __restrict__ y, int H,
                                                   int W, const float* __restrict__ gmap, int with_ssim, double lam,
                                                   float* __restrict__ d_image, double* __restrict__ sums) {
    __shared__ float s_g[3][LP][LP + 1];
    __shared__ double s_h[3][LP][LT];
    __shared__ double s_w[LW];
    __shared__ double s_red[8];
    const int c = blockIdx.z, Hv = H - 2 * LH, Wv = W - 2 * LH;
    const int i0 = blockIdx.y * LT, j0 = blockIdx.x * LT;
    const int tid = threadIdx.y * LT + threadIdx.x;
    const int i = i0 + threadIdx.y, j = j0 + threadIdx.x;
    double dssim = 0.0;
    if (with_ssim) {
        if (tid < LW) s_w[tid] = gw(tid);
        // zero-embedded maps: pixel (i, j) of the same correlation reads map
        // (i + a - 2 LH, j + b - 2 LH) for taps a, b in [0, LW)
        const size_t plane = (size_t)Hv * Wv;
        const float* g = gmap + (size_t)c * 3 * plane;
        for (int k = tid; k < LP * LP; k += 256) {
            const int r = k / LP, q = k % LP, vi = i0 + r - 2 * LH, vj = j0 + q - 2 * LH;
            const bool in = vi >= 0 && vi < Hv && vj >= 0 && vj < Wv;
            const size_t o = in ? (size_t)vi * Wv + vj : 0;
            s_g[0][r][q] = in ? g[o] : 0.f;
            s_g[1][r][q] = in ? g[plane + o] : 0.f;
            s_g[2][r][q] = in ? g[2 * plane + o] : 0.f;
        }
        __syncthreads();
        for (int k = tid; k < LP * LT; k += 256) {
            const int r = k / LT, q = k % LT;
            double a = 0, b = 0, d = 0;
#pragma unroll
            for (int t = 0; t < LW; t++) {
                const double w = s_w[t];
                a = fma(w, (double)s_g[0][r][q + t], a);
                b = fma(w, (double)s_g[1][r][q + t], b);
                d = fma(w, (double)s_g[2][r][q + t], d);
            }
            s_h[0][r][q] = a; s_h[1][r][q] = b; s_h[2][r][q] = d;
        }
        __syncthreads();
        if (i < H && j < W) {
            double am = 0, ae = 0, ax = 0;
#pragma unroll
            for (int t = 0; t < LW; t++) {
                const double w = s_w[t];
                am = fma(w, s_h[0][threadIdx.y + t][threadIdx.x], am);
                ae = fma(w, s_h[1][threadIdx.y + t][threadIdx.x], ae);
                ax = fma(w, s_h[2][threadIdx.y + t][threadIdx.x], ax);
            }
            const double xv = x[((size_t)i * W + j) * 3 + c], yv = y[((size_t)i * W + j) * 3 + c];
            dssim = am + 2.0 * xv * ae + yv * ax;
        }
    }
    double ad = 0.0;
    if (i < H && j < W) {
        const size_t o = ((size_t)i * W + j) * 3 + c;
        const double d = (double)x[o] - (double)y[o];
        ad = fabs(d);
        const double sgn = (double)((d > 0.0) - (d < 0.0));
        const double n = 3.0 * (double)H * (double)W;
        if (d_image) {
            const double gl = lam == 0.0 ? sgn / n : (1.0 - lam) * sgn / n - (lam / 2.0) * dssim / 3.0;
            d_image[o] = (float)gl;
        }
    }
    const double t = block_sum_256(ad, s_red);
    if (tid == 0) atomicAdd(sums, t);
}

__global__ void k_loss_final(int H, int W, int with_ssim, double lam, const double* __restrict__ sums,
                             double* __restrict__ out) {
    const double l1 = sums[0] / (3.0 * (double)H * (double)W);
    double sv = 1.0;
    if (with_ssim) {
        const double np = (double)(H - 2 * LH) * (double)(W - 2 * LH);
        sv = (sums[1] + sums[2] + sums[3]) / (3.0 * np);
    }
    out[0] = lam == 0.0 ? l1 : (1.0 - lam) * l1 + lam * (1.0 - sv) / 2.0;
    out[1] = sv;
}

size_t photometric_scratch_bytes(int H, int W) {
    const size_t hv = H > 2 * LH ? (size_t)(H - 2 * LH) : 0, wv = W > 2 * LH ? (size_t)(W - 2 * LH) : 0;
    return 64 + sizeof(float) * 9 * hv * wv;
}

// scratch: photometric_scratch_bytes(H, W), 16-byte aligned
void launch_photometric_loss(const float* x, const float* y, int H, int W, double lam, double* out, float* d_image,
                             void* scratch, bool ssim_only, cudaStream_t st) {
    double* sums = (double*)scratch;  // |diff| sum, 3 SSIM map sums
    float* gmap = (float*)((char*)scratch + 64);
    cudaMemsetAsync(sums, 0, 4 * sizeof(double), st);
    const bool with_ssim = (lam != 0.0 || ssim_only) && H >= LW && W >= LW;
    if (with_ssim) {
        const dim3 g((W - 2 * LH + LT - 1) / LT, (H - 2 * LH + LT - 1) / LT, 3);
        k_ssim_stats<<<g, dim3(LT, LT), 0, st>>>(x, y, H, W, gmap, sums);
    }
    if (!ssim_only || !with_ssim) {
        const dim3 g((W + LT - 1) / LT, (H + LT - 1) / LT, 3);
        k_ssim_grad<<<g, dim3(LT, LT), 0, st>>>(x, y, H, W, gmap, with_ssim && !ssim_only, lam, d_image, sums);
    }
    k_loss_final<<<1, 1, 0, st>>>(H, W, with_ssim ? 1 : 0, ssim_only ? 1.0 : lam, sums, out);
}

}  // namespace ts
