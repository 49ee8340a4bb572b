// ts_loss.cu -- on-device photometric loss: the
// reference's (1-lam) L1 + lam (1-SSIM)/2 and its gradient w.r.t. the
// rendered image (trisplat/losses.py:46-142).  The separable window sums run
// in fp32 (the SSIM stabilisers c1 = 1e-4, c2 = 9e-4 dominate the fp32
// cancellation error of E[x^2] - E[x]^2 ~ 1e-8); the per-window SSIM value and
// its partials are evaluated in fp64.
//
//   k_ssim_stats  -- CTA = 32x16 valid 11x11 windows of the three channels: the
//                    42x26 input patch of x and y in shared memory, separable
//                    Gaussian sums of x, y, x^2, xy, y^2 (fp32; horizontal pass over
//                    26 rows, vertical pass per window), the SSIM map value and
//                    its partials w.r.t. the window statistics (losses.py:
//                    76-100), written as three fp32 gradient maps; the map sum
//                    per CTA as an fp64 partial;
//   k_ssim_grad   -- CTA = 32x16 pixels of the three channels: the adjoint (same,
//                    zero-embedded) correlations of the three maps (:69-73,
//                    :101-106) combined with x and y, plus the L1 term's sign
//                    gradient and |diff| partial (:130-132), into d_image;
//   k_loss_final  -- the scalar loss and mean SSIM (:133-142).
#include "ts_kernels.cuh"

namespace ts {

namespace {
constexpr int LW = 11, LH = 5;  // window, half width
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
    const int tid = threadIdx.x;
    if ((tid & 31) == 0) s_red[tid >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (tid == 0)
        for (int w = 0; w < 8; w++) t += s_red[w];
    return t;
}
}  // namespace

// CTA = TX x TY outputs (windows or pixels) of all three channels; 256
// threads = TX x (TY / 2), two output rows per thread.  The interleaved RGB
// patch arrives with coalesced row loads and is split into channel planes in
// shared memory.
constexpr int TX = 32, TY = 16, PX = TX + LW - 1, PY = TY + LW - 1;

__global__ void __launch_bounds__(256) k_ssim_stats(const float* __restrict__ x, const float* __restrict__ y, int H,
                                                    int W, float* __restrict__ gmap, double* __restrict__ part) {
    __shared__ float s_x[3][PY][PX + 1], s_y[3][PY][PX + 1];
    __shared__ float s_h[5][PY][TX];
    __shared__ float s_w[LW];
    __shared__ double s_red[8];
    const int Hv = H - 2 * LH, Wv = W - 2 * LH;
    const int v0 = blockIdx.y * TY, u0 = blockIdx.x * TX;  // first valid window (row, col)
    const int tid = threadIdx.x, tx = tid & (TX - 1), ty = tid / TX;
    if (tid < LW) s_w[tid] = (float)gw(tid);
    for (int k = tid; k < PY * PX * 3; k += 256) {  // patch rows are 3 PX contiguous floats
        const int r = k / (3 * PX), rem = k - r * 3 * PX, q = rem / 3, c = rem - q * 3;
        const int i = v0 + r, j = u0 + q;
        const bool in = i < H && j < W;
        const size_t o = ((size_t)i * W + j) * 3 + c;
        s_x[c][r][q] = in ? x[o] : 0.f;
        s_y[c][r][q] = in ? y[o] : 0.f;
    }
    __syncthreads();
    const double s = 1.0 / ((double)Hv * (double)Wv);
    const size_t plane = (size_t)Hv * Wv;
    double smap_sum = 0.0;
    for (int c = 0; c < 3; c++) {
        for (int k = tid; k < PY * TX; k += 256) {  // horizontal pass
            const int r = k / TX, q = k % TX;
            float a = 0, b = 0, aa = 0, ab = 0, bb = 0;
#pragma unroll
            for (int t = 0; t < LW; t++) {
                const float w = s_w[t], xv = s_x[c][r][q + t], yv = s_y[c][r][q + t];
                const float wx = w * xv, wy = w * yv;
                a += wx;
                b += wy;
                aa = fmaf(wx, xv, aa);
                ab = fmaf(wx, yv, ab);
                bb = fmaf(wy, yv, bb);
            }
            s_h[0][r][q] = a; s_h[1][r][q] = b; s_h[2][r][q] = aa; s_h[3][r][q] = ab; s_h[4][r][q] = bb;
        }
        __syncthreads();
#pragma unroll
        for (int rr = 0; rr < 2; rr++) {
            const int oy = ty + rr * (TY / 2);
            const int vi = v0 + oy, vj = u0 + tx;
            if (vi < Hv && vj < Wv) {
                float sf[5] = {0, 0, 0, 0, 0};
#pragma unroll
                for (int t = 0; t < LW; t++) {
                    const float w = s_w[t];
#pragma unroll
                    for (int m = 0; m < 5; m++) sf[m] = fmaf(w, s_h[m][oy + t][tx], sf[m]);
                }
                const double mx = sf[0], my = sf[1];
                const double c1 = LK1 * LK1, c2 = LK2 * LK2;
                const double vx = (double)sf[2] - mx * mx, vy = (double)sf[4] - my * my;
                const double cxy = (double)sf[3] - mx * my;
                const double a1 = 2.0 * mx * my + c1, a2 = 2.0 * cxy + c2;
                const double b1 = mx * mx + my * my + c1, b2 = vx + vy + c2;
                const double ib = 1.0 / (b1 * b2);  // one division: 1/b1 = b2 ib, 1/b2 = b1 ib
                const double smap = a1 * a2 * ib;
                const double da1 = a2 * ib, da2 = a1 * ib, db1 = -smap * b2 * ib, db2 = -smap * b1 * ib;
                const double g_mu = 2.0 * my * da1 + 2.0 * mx * db1 - 2.0 * my * da2 - 2.0 * mx * db2;
                const size_t o = (size_t)vi * Wv + vj;
                float* g = gmap + (size_t)c * 3 * plane;
                g[o] = (float)(g_mu * s);
                g[plane + o] = (float)(db2 * s);
                g[2 * plane + o] = (float)(2.0 * da2 * s);
                smap_sum += smap;
            }
        }
        __syncthreads();
    }
    const double t = block_sum_256(smap_sum, s_red);  // per-CTA partial (no contended atomics)
    if (tid == 0) part[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
}

__global__ void __launch_bounds__(256) k_ssim_grad(const float* __restrict__ x, const float* __restrict__ y, int H,
                                                   int W, const float* __restrict__ gmap, int with_ssim, double lam,
                                                   float* __restrict__ d_image, double* __restrict__ part) {
    __shared__ float s_g[3][PY][PX + 1];
    __shared__ float s_h[3][PY][TX];
    __shared__ float s_w[LW];
    __shared__ double s_red[8];
    const int Hv = H - 2 * LH, Wv = W - 2 * LH;
    const int i0 = blockIdx.y * TY, j0 = blockIdx.x * TX;
    const int tid = threadIdx.x, tx = tid & (TX - 1), ty = tid / TX;
    const double n = 3.0 * (double)H * (double)W;
    const size_t plane = (size_t)Hv * Wv;
    double ad = 0.0;
    if (with_ssim && tid < LW) s_w[tid] = (float)gw(tid);
    for (int c = 0; c < 3; c++) {
        double dss[2] = {0.0, 0.0};
        if (with_ssim) {
            // zero-embedded maps: pixel (i, j) of the same correlation reads map
            // (i + a - 2 LH, j + b - 2 LH) for taps a, b in [0, LW)
            const float* g = gmap + (size_t)c * 3 * plane;
            for (int k = tid; k < PY * PX; k += 256) {
                const int r = k / PX, q = k % PX, vi = i0 + r - 2 * LH, vj = j0 + q - 2 * LH;
                const bool in = vi >= 0 && vi < Hv && vj >= 0 && vj < Wv;
                const size_t o = in ? (size_t)vi * Wv + vj : 0;
                s_g[0][r][q] = in ? g[o] : 0.f;
                s_g[1][r][q] = in ? g[plane + o] : 0.f;
                s_g[2][r][q] = in ? g[2 * plane + o] : 0.f;
            }
            __syncthreads();
            for (int k = tid; k < PY * TX; k += 256) {
                const int r = k / TX, q = k % TX;
                float a = 0, b = 0, d = 0;
#pragma unroll
                for (int t = 0; t < LW; t++) {
                    const float w = s_w[t];
                    a = fmaf(w, s_g[0][r][q + t], a);
                    b = fmaf(w, s_g[1][r][q + t], b);
                    d = fmaf(w, s_g[2][r][q + t], d);
                }
                s_h[0][r][q] = a; s_h[1][r][q] = b; s_h[2][r][q] = d;
            }
            __syncthreads();
#pragma unroll
            for (int rr = 0; rr < 2; rr++) {
                const int oy = ty + rr * (TY / 2), i = i0 + oy, j = j0 + tx;
                if (i < H && j < W) {
                    float am = 0, ae = 0, ax = 0;
#pragma unroll
                    for (int t = 0; t < LW; t++) {
                        const float w = s_w[t];
                        am = fmaf(w, s_h[0][oy + t][tx], am);
                        ae = fmaf(w, s_h[1][oy + t][tx], ae);
                        ax = fmaf(w, s_h[2][oy + t][tx], ax);
                    }
                    const size_t o = ((size_t)i * W + j) * 3 + c;
                    dss[rr] = (double)am + 2.0 * (double)x[o] * ae + (double)y[o] * ax;  // (fp64: the terms cancel)
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int rr = 0; rr < 2; rr++) {
            const int i = i0 + ty + rr * (TY / 2), j = j0 + tx;
            if (i < H && j < W) {
                const size_t o = ((size_t)i * W + j) * 3 + c;
                const double d = (double)x[o] - (double)y[o];
                ad += fabs(d);
                const double sgn = (double)((d > 0.0) - (d < 0.0));
                if (d_image) {
                    const double gl = lam == 0.0 ? sgn / n
                                                 : (1.0 - lam) * sgn / n - (lam / 2.0) * dss[rr] / 3.0;
                    d_image[o] = (float)gl;
                }
            }
        }
    }
    const double t = block_sum_256(ad, s_red);
    if (tid == 0) part[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
}

// one CTA: sums of the per-CTA partials (|diff| and SSIM map), the loss
__global__ void __launch_bounds__(256) k_loss_final(int H, int W, int with_ssim, double lam,
                                                    const double* __restrict__ pl1, int nl1,
                                                    const double* __restrict__ pss, int nss,
                                                    double* __restrict__ out) {
    __shared__ double s_red[8];
    double a = 0.0, b = 0.0;
    for (int k = threadIdx.x; k < nl1; k += 256) a += pl1[k];
    for (int k = threadIdx.x; k < nss; k += 256) b += pss[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, off);
        b += __shfl_xor_sync(0xffffffffu, b, off);
    }
    __shared__ double s_b[8];
    if ((threadIdx.x & 31) == 0) {
        s_red[threadIdx.x >> 5] = a;
        s_b[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sa = 0.0, sb = 0.0;
        for (int w = 0; w < 8; w++) {
            sa += s_red[w];
            sb += s_b[w];
        }
        const double l1 = sa / (3.0 * (double)H * (double)W);
        double sv = 1.0;
        if (with_ssim) sv = sb / (3.0 * (double)(H - 2 * LH) * (double)(W - 2 * LH));
        out[0] = lam == 0.0 ? l1 : (1.0 - lam) * l1 + lam * (1.0 - sv) / 2.0;
        out[1] = sv;
    }
}

static inline size_t tiles_x(int n) { return (size_t)((n + TX - 1) / TX); }
static inline size_t tiles_y(int n) { return (size_t)((n + TY - 1) / TY); }

size_t photometric_scratch_bytes(int H, int W) {
    const size_t hv = H > 2 * LH ? (size_t)(H - 2 * LH) : 0, wv = W > 2 * LH ? (size_t)(W - 2 * LH) : 0;
    const size_t parts = tiles_x(W) * tiles_y(H) + tiles_x((int)wv) * tiles_y((int)hv);
    return sizeof(double) * parts + sizeof(float) * 9 * hv * wv + 256;
}

// scratch: photometric_scratch_bytes(H, W), 16-byte aligned
void launch_photometric_loss(const float* x, const float* y, int H, int W, double lam, double* out, float* d_image,
                             void* scratch, bool ssim_only, cudaStream_t st) {
    const bool with_ssim = (lam != 0.0 || ssim_only) && H >= LW && W >= LW;
    const int Hv = H - 2 * LH, Wv = W - 2 * LH;
    const int nl1 = (int)(tiles_x(W) * tiles_y(H));
    const int nss = with_ssim ? (int)(tiles_x(Wv) * tiles_y(Hv)) : 0;
    double* pl1 = (double*)scratch;  // per-CTA |diff| partials
    double* pss = pl1 + nl1;          // per-CTA SSIM map partials
    float* gmap = (float*)(((uintptr_t)(pss + nss) + 15) & ~(uintptr_t)15);
    if (with_ssim)
        k_ssim_stats<<<dim3((unsigned)tiles_x(Wv), (unsigned)tiles_y(Hv)), 256, 0, st>>>(x, y, H, W, gmap, pss);
    int nl = 0;
    if (!ssim_only || !with_ssim) {
        k_ssim_grad<<<dim3((unsigned)tiles_x(W), (unsigned)tiles_y(H)), 256, 0, st>>>(
            x, y, H, W, gmap, with_ssim && !ssim_only, lam, d_image, pl1);
        nl = nl1;
    }
    k_loss_final<<<1, 256, 0, st>>>(H, W, with_ssim ? 1 : 0, ssim_only ? 1.0 : lam, pl1, nl, pss, nss, out);
}

// ---------------------------------------------------------------------------
// Distortion loss (losses.py:153-203): per pixel, sum over ordered fragment
// pairs of w_i w_j |z_i - z_j|, averaged over image_size pixels, with its
// gradients w.r.t. every fragment's weight and depth, over the CSR fragment runs.
// ---------------------------------------------------------------------------
// Eight lanes per pixel (four pixels per warp), each lane holding four consecutive
// fragments of a 32-fragment chunk: the prefix sums are a serial sum inside the lane
// and a 3-step exclusive scan across the group, so a warp spends its instructions on
// four pixels instead of one (most lists are far shorter than 32).  Lists longer than
// one chunk are read twice (totals, then prefixes with a carry).  As in the reference
// (losses.py:178-203) the form is chosen for the whole fragment set: the prefix-sum
// form when every run is depth sorted, else the pairwise form for every run
// (_distortion_pairwise :153-166) -- the two differ on depth ties (d_depth).  The
// prefix pass checks the order as it reads the runs; the pairwise kernel after it
// exits at once unless a run was out of order, and then rewrites every output.
constexpr int DIST_PW_BLOCKS = 148 * 8;  // grid of the pairwise redo (grid-stride)
constexpr int DIST_SUM_BLOCKS = 256;     // first level of the deterministic loss sum

__global__ void __launch_bounds__(256, 4) k_distortion_g8(long long npix, const long long* __restrict__ off,
                                                          const double* __restrict__ w, const double* __restrict__ z,
                                                          double scale, unsigned* __restrict__ unsorted,
                                                          double* __restrict__ d_w, double* __restrict__ d_z,
                                                          double* __restrict__ wpart) {
    const unsigned lane = threadIdx.x & 31, gl = lane & 7;
    const unsigned gmask = 0xffu << (lane & 24);
    const long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    double tot = 0.0;
    bool bad = false;
    if (p < npix) {
        const long long lo = off[p], hi = off[p + 1];
        if (hi - lo < 2) {
            if (gl == 0 && hi > lo) {
                if (d_w) d_w[lo] = 0.0;
                if (d_z) d_z[lo] = 0.0;
            }
        } else {
            const bool multi = hi - lo > 32;
            double wv[4], zv[4];
            auto load = [&](long long c0) {
#pragma unroll
                for (int r = 0; r < 4; r++) {
                    const long long k = c0 + 4 * gl + r;
                    wv[r] = k < hi ? w[k] : 0.0;
                    zv[r] = k < hi ? z[k] : 0.0;
                }
            };
            // pass 1: the run's totals and its depth order
            double tw = 0.0, ts = 0.0, zc = 0.0;
            for (long long c0 = lo; c0 < hi; c0 += 32) {
                load(c0);
                const long long kf = c0 + 4 * gl;
#pragma unroll
                for (int r = 0; r < 4; r++) {
                    tw += wv[r];
                    ts += wv[r] * zv[r];
                    if (r > 0) bad |= kf + r < hi && zv[r] < zv[r - 1];
                }
                const double zl = __shfl_up_sync(gmask, zv[3], 1, 8);  // the previous lane's last
                bad |= kf < hi && kf > lo && zv[0] < (gl > 0 ? zl : zc);
                zc = __shfl_sync(gmask, zv[3], 7, 8);  // the next chunk's predecessor
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                tw += __shfl_xor_sync(gmask, tw, o, 8);
                ts += __shfl_xor_sync(gmask, ts, o, 8);
            }
            // pass 2: weight / weighted depth in front of each fragment
            double cw = 0.0, cs = 0.0;  // carried from earlier chunks
            for (long long c0 = lo; c0 < hi; c0 += 32) {
                if (multi) load(c0);
                double aw = 0.0, as = 0.0;  // the lane's totals
#pragma unroll
                for (int r = 0; r < 4; r++) {
                    aw += wv[r];
                    as += wv[r] * zv[r];
                }
                double iw = aw, is = as;  // inclusive scan of the lane totals
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
                    const double yw = __shfl_up_sync(gmask, iw, o, 8), ys = __shfl_up_sync(gmask, is, o, 8);
                    if ((int)gl >= o) {
                        iw += yw;
                        is += ys;
                    }
                }
                double wb = cw + (iw - aw), sb = cs + (is - as);  // in front of the lane's first
                const long long kf = c0 + 4 * gl;
#pragma unroll
                for (int r = 0; r < 4; r++) {
                    if (kf + r >= hi) break;
                    const double wk = wv[r], zk = zv[r];
                    const double wa = tw - wb - wk, sa = ts - sb - wk * zk;
                    const double fwd = zk * wb - sb;
                    tot += wk * fwd;
                    if (d_w) d_w[kf + r] = 2.0 * (fwd + (sa - zk * wa)) * scale;
                    if (d_z) d_z[kf + r] = 2.0 * wk * (wb - wa) * scale;
                    wb += wk;
                    sb += wk * zk;
                }
                cw += __shfl_sync(gmask, iw, 7, 8);
                cs += __shfl_sync(gmask, is, 7, 8);
            }
            tot *= 2.0;
        }
    }
    // per-warp partial (no block barrier: a warp with short runs retires early)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(unsorted, 1u);
    if (lane == 0) wpart[((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5] = tot;
}

// the pairwise form for every run when any run is out of depth order
__global__ void __launch_bounds__(256) k_distortion_pairwise(long long npix, const long long* __restrict__ off,
                                                             const double* __restrict__ w,
                                                             const double* __restrict__ z, double scale,
                                                             const unsigned* __restrict__ unsorted,
                                                             double* __restrict__ d_w, double* __restrict__ d_z,
                                                             double* __restrict__ fpart) {
    __shared__ double s_red[8];
    if (*unsorted == 0u) return;
    const unsigned gl = threadIdx.x & 7;
    double tot = 0.0;
    for (long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 3; p < npix;
         p += (long long)gridDim.x * (blockDim.x >> 3)) {
        const long long lo = off[p], hi = off[p + 1];
        if (hi - lo < 2) continue;
        for (long long i = lo + gl; i < hi; i += 8) {
            double gw_ = 0.0, gz = 0.0;
            const double zi = z[i], wi = w[i];
            for (long long j = lo; j < hi; j++) {
                const double dz = zi - z[j];
                tot += wi * fabs(dz) * w[j];
                gw_ += fabs(dz) * w[j];
                gz += (double)((dz > 0.0) - (dz < 0.0)) * w[j];
            }
            if (d_w) d_w[i] = 2.0 * gw_ * scale;
            if (d_z) d_z[i] = 2.0 * gz * wi * scale;
        }
    }
    const double t = block_sum_256(tot, s_red);
    if (threadIdx.x == 0) fpart[blockIdx.x] = t;
}

// first level of the loss sum over the partials of whichever form ran (fixed
// slices: the sum is deterministic)
__global__ void __launch_bounds__(256) k_distortion_sum(const double* __restrict__ wpart, long long nw,
                                                        const double* __restrict__ fpart,
                                                        const unsigned* __restrict__ unsorted,
                                                        double* __restrict__ p2) {
    __shared__ double s_red[8];
    const bool pw = *unsorted != 0u;
    const double* src = pw ? fpart : wpart;
    const long long n = pw ? DIST_PW_BLOCKS : nw;
    double a = 0.0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        a += src[k];
    const double t = block_sum_256(a, s_red);
    if (threadIdx.x == 0) p2[blockIdx.x] = t;
}

__global__ void __launch_bounds__(256) k_sum_scaled(const double* __restrict__ part, int n, double scale,
                                                    double* __restrict__ out) {
    __shared__ double s_red[8];
    double a = 0.0;
    for (int k = threadIdx.x; k < n; k += 256) a += part[k];
    const double t = block_sum_256(a, s_red);
    if (threadIdx.x == 0) out[0] = t * scale;
}

// depth_from_fragments (losses.py:206-216): blend-weight-normalised depth per pixel;
// eight lanes per pixel over fragments l, l+8, ... (coalesced run reads)
__global__ void __launch_bounds__(256) k_fragment_depth(long long npix, const long long* __restrict__ off,
                                                        const double* __restrict__ w, const double* __restrict__ z,
                                                        double* __restrict__ depth) {
    const unsigned gl = threadIdx.x & 7, lane = threadIdx.x & 31;
    const unsigned gmask = 0xffu << (lane & 24);
    const long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    if (p >= npix) return;  // whole groups leave together
    double a = 0.0, b = 0.0;
    for (long long k = off[p] + gl, k1 = off[p + 1]; k < k1; k += 8) {
        const double wk = w[k];
        a += wk * z[k];
        b += wk;
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
        a += __shfl_xor_sync(gmask, a, o, 8);
        b += __shfl_xor_sync(gmask, b, o, 8);
    }
    if (gl == 0) depth[p] = a / fmax(b, 1e-8);
}

// ---------------------------------------------------------------------------
// Normal loss (losses.py:219-292): blend-weighted misalignment of the
// camera-facing triangle normals with the normals of the depth map.
//   k_depth_normals -- per pixel: backprojected points, central differences
//                      with border replication, unit normal facing the camera,
//                      rotated into the world frame (n @ R);
//   k_tri_normals   -- per triangle: c = (v1-v0) x (v2-v0), |c| (floored), the
//                      unit normal and its camera-facing sign;
//   k_normal_frag   -- eight lanes per pixel over its fragments: w (1 - n.N), the
//                      weight gradient, and dL/dc per triangle (fp64 atomics);
//   k_normal_chain  -- per triangle: the cross-product chain into d_vertices.
// ---------------------------------------------------------------------------
#ifndef TS_NORMAL_U
#define TS_NORMAL_U 1  // fragments per lane per step of k_normal_frag
#endif
constexpr int NORMAL_SUM_BLOCKS = 256;
struct NCam {
    double fx, fy, cx, cy, R[9], t[3];
};

__global__ void __launch_bounds__(256) k_depth_normals(const double* __restrict__ depth, int H, int W, NCam cm,
                                                       double* __restrict__ nmap) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= H * W) return;
    const int y = p / W, x = p % W;
    auto pt = [&](int yy, int xx, double* o) {  // edge-replicated backprojection
        yy = min(max(yy, 0), H - 1);
        xx = min(max(xx, 0), W - 1);
        const double d = depth[(size_t)yy * W + xx];
        o[0] = d * ((xx + 0.5 - cm.cx) / cm.fx);
        o[1] = d * ((yy + 0.5 - cm.cy) / cm.fy);
        o[2] = d;
    };
    double xp[3], xm[3], yp[3], ym[3];
    pt(y, x + 1, xp);
    pt(y, x - 1, xm);
    pt(y + 1, x, yp);
    pt(y - 1, x, ym);
    double dx[3], dy[3];
    for (int k = 0; k < 3; k++) {
        dx[k] = (xp[k] - xm[k]) / 2.0;
        dy[k] = (yp[k] - ym[k]) / 2.0;
    }
    double n[3] = {dx[1] * dy[2] - dx[2] * dy[1], dx[2] * dy[0] - dx[0] * dy[2], dx[0] * dy[1] - dx[1] * dy[0]};
    const double nn = fmax(sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]), 1e-12);
    for (int k = 0; k < 3; k++) n[k] /= nn;
    if (n[2] > 0.0)
        for (int k = 0; k < 3; k++) n[k] = -n[k];
    // world frame: m = n @ R  (m_j = sum_i n_i R[i][j])
    for (int j = 0; j < 3; j++)
        nmap[(size_t)p * 3 + j] = n[0] * cm.R[0 * 3 + j] + n[1] * cm.R[1 * 3 + j] + n[2] * cm.R[2 * 3 + j];
}

// tri[4 per triangle]: chat xyz, flip / |c| (one 32-byte sector per gather; the sign
// is the flip: |c| is floored above zero)
// the CTA's 256 vertex rows (9 floats each) staged through shared memory with
// coalesced loads; the odd row stride reads them back without bank conflicts
__device__ __forceinline__ void stage_vertex_rows(const float* __restrict__ v, long long n, float* s_v) {
    const long long base = (long long)blockIdx.x * 256;
    const int cnt = (int)min(256LL, n - base) * 9;
    for (int k = threadIdx.x; k < cnt; k += 256) s_v[k] = v[base * 9 + k];
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_tri_normals(const float* __restrict__ v, long long n, NCam cm,
                                                     double* __restrict__ tri, double* __restrict__ gc) {
    __shared__ float s_v[256 * 9];
    stage_vertex_rows(v, n, s_v);
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double p[9];
    for (int k = 0; k < 9; k++) p[k] = (double)s_v[threadIdx.x * 9 + k];
    const double a[3] = {p[3] - p[0], p[4] - p[1], p[5] - p[2]};
    const double b[3] = {p[6] - p[0], p[7] - p[1], p[8] - p[2]};
    const double c[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
    const double cn = fmax(sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]), 1e-12);
    const double ch[3] = {c[0] / cn, c[1] / cn, c[2] / cn};
    // camera-facing orientation: centroid_cam = mean(v) @ R^T + t, n_cam = chat @ R^T
    double facing = 0.0;
    for (int r = 0; r < 3; r++) {
        const double cc = ((p[0] + p[3] + p[6]) / 3.0) * cm.R[r * 3 + 0] + ((p[1] + p[4] + p[7]) / 3.0) * cm.R[r * 3 + 1] +
                          ((p[2] + p[5] + p[8]) / 3.0) * cm.R[r * 3 + 2] + cm.t[r];
        const double nc = ch[0] * cm.R[r * 3 + 0] + ch[1] * cm.R[r * 3 + 1] + ch[2] * cm.R[r * 3 + 2];
        facing += nc * cc;
    }
    double* o = tri + i * 4;
    o[0] = ch[0]; o[1] = ch[1]; o[2] = ch[2]; o[3] = (facing > 0.0 ? -1.0 : 1.0) / cn;
    gc[i * 3 + 0] = gc[i * 3 + 1] = gc[i * 3 + 2] = 0.0;
}

// Eight lanes per pixel (four pixels per warp): lane l of a pixel's group takes
// fragments l, l+8, ... -- the source ids, weights and d_weight stores are
// coalesced, and a warp has up to eight triangle-row gathers in flight per pixel.
__global__ void __launch_bounds__(256) k_normal_frag(long long npix, const long long* __restrict__ off,
                                                     const int* __restrict__ ftri, const double* __restrict__ w,
                                                     const double* __restrict__ nmap, const double* __restrict__ tri,
                                                     double inv_nf, double* __restrict__ d_w, double* __restrict__ gc,
                                                     double* __restrict__ part) {
    const unsigned gl = threadIdx.x & 7;
    const long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    double sum = 0.0;
    if (p < npix) {
        const double m0 = nmap[p * 3 + 0], m1 = nmap[p * 3 + 1], m2 = nmap[p * 3 + 2];
        const long long k0 = off[p], k1 = off[p + 1];
        constexpr int U = TS_NORMAL_U;  // fragments per lane in flight at once
        for (long long kb = k0 + gl; kb < k1; kb += 8 * U) {
            long long t[U];
            double wk[U], c[U][4];
#pragma unroll
            for (int u = 0; u < U; u++) t[u] = kb + 8 * u < k1 ? (long long)ftri[kb + 8 * u] : -1;
#pragma unroll
            for (int u = 0; u < U; u++) {
                wk[u] = 0.0;
                if (t[u] >= 0) {
                    const double* o = tri + t[u] * 4;
                    const double2 a = *reinterpret_cast<const double2*>(o);
                    const double2 b = *reinterpret_cast<const double2*>(o + 2);
                    c[u][0] = a.x; c[u][1] = a.y; c[u][2] = b.x; c[u][3] = b.y;
                    wk[u] = w[kb + 8 * u];
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (t[u] < 0) continue;
                const long long k = kb + 8 * u;
                const double c0 = c[u][0], c1 = c[u][1], c2 = c[u][2], fc = c[u][3];
                const double fl = fc < 0.0 ? -1.0 : 1.0;
                const double cm = c0 * m0 + c1 * m1 + c2 * m2;
                const double dot = cm * fl;
                sum += wk[u] * (1.0 - dot);
                if (d_w) d_w[k] = (1.0 - dot) * inv_nf;
                const double coef = -wk[u] * inv_nf * fc;
                atomicAdd(gc + t[u] * 3 + 0, coef * (m0 - c0 * cm));
                atomicAdd(gc + t[u] * 3 + 1, coef * (m1 - c1 * cm));
                atomicAdd(gc + t[u] * 3 + 2, coef * (m2 - c2 * cm));
            }
        }
    }
    // per-warp partial (no block barrier: a warp with short runs retires early)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) part[((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5] = sum;
}

// first level of a deterministic sum of n partials (fixed slices per CTA)
__global__ void __launch_bounds__(256) k_sum_level1(const double* __restrict__ src, long long n,
                                                    double* __restrict__ p2) {
    __shared__ double s_red[8];
    double a = 0.0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        a += src[k];
    const double t = block_sum_256(a, s_red);
    if (threadIdx.x == 0) p2[blockIdx.x] = t;
}

__global__ void __launch_bounds__(256) k_normal_chain(const float* __restrict__ v, long long n,
                                                      const double* __restrict__ gc, double* __restrict__ dv) {
    __shared__ float s_v[256 * 9];
    __shared__ double s_o[256 * 9];
    stage_vertex_rows(v, n, s_v);
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long base = (long long)blockIdx.x * 256;
    const int cnt = (int)min(256LL, n - base) * 9;
    double p[9];
    for (int k = 0; k < 9; k++) p[k] = (double)s_v[threadIdx.x * 9 + k];
    const double a[3] = {p[3] - p[0], p[4] - p[1], p[5] - p[2]};
    const double b[3] = {p[6] - p[0], p[7] - p[1], p[8] - p[2]};
    const double g[3] = {i < n ? gc[i * 3] : 0.0, i < n ? gc[i * 3 + 1] : 0.0, i < n ? gc[i * 3 + 2] : 0.0};
    const double da[3] = {b[1] * g[2] - b[2] * g[1], b[2] * g[0] - b[0] * g[2], b[0] * g[1] - b[1] * g[0]};
    const double db[3] = {g[1] * a[2] - g[2] * a[1], g[2] * a[0] - g[0] * a[2], g[0] * a[1] - g[1] * a[0]};
    double* o = s_o + threadIdx.x * 9;  // staged for coalesced row stores
    for (int k = 0; k < 3; k++) {
        o[3 + k] = da[k];
        o[6 + k] = db[k];
        o[k] = -(da[k] + db[k]);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += 256) dv[base * 9 + k] = s_o[k];
}

size_t normal_scratch_bytes(long long n, long long npix) {
    return sizeof(double) * (size_t)(4 * n + 3 * n + 3 * npix + (npix + 3) / 4 + NORMAL_SUM_BLOCKS + 8);
}

void launch_normal_loss(const float* v, long long n, const long long* off, const int* ftri, const double* w,
                        long long nfrag, const double* depth, int H, int W, const double cam[16], double* out,
                        double* d_vertices, double* d_w, void* scratch, cudaStream_t st) {
    NCam cm;
    cm.fx = cam[0]; cm.fy = cam[1]; cm.cx = cam[2]; cm.cy = cam[3];
    for (int k = 0; k < 9; k++) cm.R[k] = cam[4 + k];
    for (int k = 0; k < 3; k++) cm.t[k] = cam[13 + k];
    const long long npix = (long long)H * W;
    double* tri = (double*)scratch;
    double* gc = tri + 4 * n;
    double* nmap = gc + 3 * n;
    double* part = nmap + 3 * npix;
    double* p2 = part + (npix + 3) / 4;  // after the per-warp partials
    const int nb = (int)((npix + 31) / 32);  // eight lanes per pixel
    if (n > 0) k_tri_normals<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(v, n, cm, tri, gc);
    if (npix > 0) {
        k_depth_normals<<<(unsigned)((npix + 255) / 256), 256, 0, st>>>(depth, H, W, cm, nmap);
        k_normal_frag<<<nb, 256, 0, st>>>(npix, off, ftri, w, nmap, tri, nfrag > 0 ? 1.0 / (double)nfrag : 0.0, d_w,
                                          gc, part);
    }
    k_sum_level1<<<NORMAL_SUM_BLOCKS, 256, 0, st>>>(part, npix > 0 ? (long long)nb * 8 : 0, p2);
    k_sum_scaled<<<1, 256, 0, st>>>(p2, NORMAL_SUM_BLOCKS, nfrag > 0 ? 1.0 / (double)nfrag : 0.0, out);
    if (n > 0 && d_vertices) k_normal_chain<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(v, n, gc, d_vertices);
}

// per-warp partials (or the pairwise kernel's per-CTA partials), the first-level sums
// and the order flag
size_t distortion_scratch_bytes(long long npix) {
    return sizeof(double) * (size_t)((npix + 7) / 8 + (npix + 3) / 4 + DIST_PW_BLOCKS + DIST_SUM_BLOCKS + 1);
}

void launch_distortion_loss(long long npix, const long long* off, const double* w, const double* z,
                            long long image_size, double* out, double* d_w, double* d_z, void* scratch,
                            cudaStream_t st) {
    const double scale = 1.0 / (double)(image_size > 1 ? image_size : 1);
    double* part = (double*)scratch;
    const int nb = (int)((npix + 31) / 32);  // eight lanes per pixel, 32 pixels per CTA
    double* fpart = part + (npix + 3) / 4;
    double* p2 = fpart + DIST_PW_BLOCKS;
    unsigned* unsorted = (unsigned*)(p2 + DIST_SUM_BLOCKS);
    cudaMemsetAsync(unsorted, 0, sizeof(unsigned), st);
    if (nb > 0) {
        k_distortion_g8<<<nb, 256, 0, st>>>(npix, off, w, z, scale, unsorted, d_w, d_z, part);
        k_distortion_pairwise<<<DIST_PW_BLOCKS, 256, 0, st>>>(npix, off, w, z, scale, unsorted, d_w, d_z, fpart);
    }
    k_distortion_sum<<<DIST_SUM_BLOCKS, 256, 0, st>>>(part, nb > 0 ? (long long)nb * 8 : 0, fpart, unsorted, p2);
    k_sum_scaled<<<1, 256, 0, st>>>(p2, DIST_SUM_BLOCKS, scale, out);
}

void launch_fragment_depth(long long npix, const long long* off, const double* w, const double* z, double* depth,
                           cudaStream_t st) {
    if (npix > 0) k_fragment_depth<<<(unsigned)((npix + 31) / 32), 256, 0, st>>>(npix, off, w, z, depth);
}

}  // namespace ts
