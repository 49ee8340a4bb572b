// ts_bin.cu -- tile-first binning: the per-tile entry lists of the reference
// (render.py:275-277 depth order np.lexsort((idx, z)), then 315-361
// duplicate / stable sort by tile / ranges) built without a global sort.
//
// The reference sorts all triangles by (z, idx), duplicates each into the
// tiles its bbox touches and stable-sorts the duplicates by tile id, so a
// tile's list is its triangles in (z, idx) order.  Here:
//   k_bin_count  -- CTA per chunk of triangles: per-tile counts in shared
//                   memory (no global atomics), one row of the chunk x tile
//                   count matrix;
//   k_bin_cols   -- per tile: prefix over the chunks (the chunk's first slot
//                   within the tile) and the tile total;
//   k_tile_scan  -- one CTA: exclusive scan of the totals -> tile_start (all
//                   tiles empty and the sticky overflow flag raised if the total
//                   exceeds the entry capacity);
//   k_bin_fill   -- CTA per chunk: shared-memory cursors from the matrix, one
//                   slot per (triangle, tile); the bucket holds the tile's
//                   triangles (and their depth keys) in arbitrary order;
//   k_tile_sort  -- CTA per tile: the depth keys (fp64 bit patterns of the
//                   positive centroid depth, monotone) are range-reduced to 32
//                   bits, counting-sorted on their top 11 bits in shared memory,
//                   and every run of equal 12-bit keys is ordered by the exact
//                   (z, idx) pair.  Tiles longer than the shared-memory
//                   capacity, or with long runs (equal or clustered depths), take
//                   a stable LSD radix path (by idx, then by all 64 key bits).
// The result is bit-identical to the global sort's tile lists.
#include "ts_kernels.cuh"

namespace ts {

namespace {
constexpr int BT = 256;       // threads per CTA
constexpr int BW = BT / 32;   // warps
constexpr int RUN_SHORT = 48; // runs up to this length are insertion-sorted by one thread
constexpr int RUN_LONG = 64;  // buckets up to this length are ranked item by item

__device__ __forceinline__ unsigned excl_scan_256(unsigned v, unsigned* s_w, unsigned& total) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= (unsigned)off) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned w = lane < BW ? s_w[lane] : 0u;
#pragma unroll
        for (int off = 1; off < BW; off <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= (unsigned)off) w += y;
        }
        if (lane < BW) s_w[lane] = w;
    }
    __syncthreads();
    const unsigned pre = warp ? s_w[warp - 1] : 0u;
    total = s_w[BW - 1];
    __syncthreads();
    return pre + x - v;
}
}  // namespace

// tile blend-order class: longest lists first, two classes per octave of the length
__device__ __forceinline__ int tile_class(unsigned c) {
    const int l = 31 - __clz(c + 1);                               // floor(log2(c + 1))
    const int h = l > 0 ? (int)(((c + 1) >> (l - 1)) & 1u) : 0;    // upper half of the octave
    return 63 - min(63, 2 * l + h);
}

__global__ void __launch_bounds__(1024) k_tile_scan(int ntiles, unsigned* __restrict__ tcnt, int* __restrict__ tile_start,
                                                    long long cap, unsigned* overflow, int small_cap,
                                                    int* __restrict__ big_list, int* __restrict__ n_big,
                                                    int* __restrict__ order) {
    TS_PDL_ENTRY();
    __shared__ unsigned s_w[32];
    __shared__ unsigned long long s_total;
    __shared__ int s_nbig;
    __shared__ int s_ccnt[64];
    if (threadIdx.x == 0) s_nbig = 0;
    if (threadIdx.x < 64) s_ccnt[threadIdx.x] = 0;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long carry = 0;
    for (int b0 = 0; b0 < ntiles; b0 += 1024) {
        const int i = b0 + (int)threadIdx.x;
        const unsigned v = i < ntiles ? tcnt[i] : 0u;
        unsigned x = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= (unsigned)off) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            unsigned w = s_w[lane];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, w, off);
                if (lane >= (unsigned)off) w += y;
            }
            s_w[lane] = w;
        }
        __syncthreads();
        const unsigned long long ex = carry + (warp ? s_w[warp - 1] : 0u) + x - v;
        if (i < ntiles) {
            tile_start[i] = (int)ex;
            if ((int)v > small_cap) big_list[atomicAdd(&s_nbig, 1)] = i;  // long tiles, any order
            if (order) atomicAdd(&s_ccnt[tile_class(v)], 1);
        }
        carry += s_w[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) s_total = carry;
    __syncthreads();
    if (s_total > (unsigned long long)cap) {
        // over capacity: every tile empty, the forward is redone with larger buffers
        for (int i = threadIdx.x; i <= ntiles; i += 1024) tile_start[i] = 0;
        if (threadIdx.x == 0) {
            if (overflow) *overflow = 1u;
            *n_big = 0;
        }
    } else if (threadIdx.x == 0) {
        tile_start[ntiles] = (int)s_total;
        *n_big = s_nbig;
    }
    if (order) {
        // blend order of the tiles: longest lists first (any order within a class),
        // so the frame's tail is not a long tile that happened to come last
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = 0;
            for (int k = 0; k < 64; k++) {
                const int c = s_ccnt[k];
                s_ccnt[k] = run;
                run += c;
            }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < ntiles; t += 1024) order[atomicAdd(&s_ccnt[tile_class(tcnt[t])], 1)] = t;
    }
}

// ---------------------------------------------------------------------------
// Two-level counting (chunk x tile matrix): no contended global atomics.
constexpr int BIN_CT = 1024;               // threads per chunk CTA
constexpr int BIN_PER = 8;                 // triangles per thread
constexpr int BIN_CHUNK = BIN_CT * BIN_PER;
constexpr int BIN_MAX_TILES = 12288;       // shared-memory counters per CTA (48 KB): tile range per blockIdx.y

__global__ void __launch_bounds__(BIN_CT) k_bin_count(long long n, const short4* __restrict__ bbox, int ntx,
                                                      int ntiles, unsigned* __restrict__ mat) {
    TS_PDL_ENTRY();
    extern __shared__ unsigned s_cnt[];
    const int t0 = blockIdx.y * BIN_MAX_TILES, nt = min(BIN_MAX_TILES, ntiles - t0);  // this CTA's tile range
    for (int t = threadIdx.x; t < nt; t += BIN_CT) s_cnt[t] = 0u;
    __syncthreads();
    const long long c0 = (long long)blockIdx.x * BIN_CHUNK;
    short4 bb[BIN_PER];  // all loads in flight before the first use
#pragma unroll
    for (int k = 0; k < BIN_PER; k++) {
        const long long i = c0 + k * BIN_CT + threadIdx.x;
        bb[k] = i < n ? __ldg(bbox + i) : make_short4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < BIN_PER; k++) {
        if (bb[k].y <= bb[k].x || bb[k].w <= bb[k].z) continue;
        const int tx0 = bb[k].x / TILE, tx1 = (bb[k].y - 1) / TILE + 1;
        const int ty0 = bb[k].z / TILE, ty1 = (bb[k].w - 1) / TILE + 1;
        for (int ty = ty0; ty < ty1; ty++)
            for (int tx = tx0; tx < tx1; tx++) {
                const int t = ty * ntx + tx - t0;
                if ((unsigned)t < (unsigned)nt) atomicAdd(&s_cnt[t], 1u);
            }
    }
    __syncthreads();
    unsigned* row = mat + (size_t)blockIdx.x * ntiles + t0;
    for (int t = threadIdx.x; t < nt; t += BIN_CT) row[t] = s_cnt[t];
}

// per tile: exclusive prefix over the chunks in place, totals into tcnt.  CTA =
// 32 consecutive tiles (lane) x 8 chunk ranges (warp): coalesced 128-byte rows.
__global__ void __launch_bounds__(256) k_bin_cols(int nchunk, int ntiles, unsigned* __restrict__ mat,
                                                  unsigned* __restrict__ tcnt) {
    TS_PDL_ENTRY();
    __shared__ unsigned s_part[8][33];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + (int)lane;
    const int per = (nchunk + 7) / 8;
    const int b0 = (int)warp * per, b1 = min(nchunk, b0 + per);
    unsigned sum = 0;
    if (t < ntiles)
        for (int b = b0; b < b1; b++) sum += mat[(size_t)b * ntiles + t];
    s_part[warp][lane] = sum;
    __syncthreads();
    unsigned run = 0;
    for (int w = 0; w < (int)warp; w++) run += s_part[w][lane];
    if (t < ntiles) {
        for (int b = b0; b < b1; b++) {
            const unsigned v = mat[(size_t)b * ntiles + t];
            mat[(size_t)b * ntiles + t] = run;
            run += v;
        }
        if (warp == 7) tcnt[t] = run;
    }
}

__global__ void __launch_bounds__(BIN_CT) k_bin_fill(long long n, const short4* __restrict__ bbox, int ntx,
                                                     int ntiles, const unsigned* __restrict__ mat,
                                                     const int* __restrict__ tile_start,
                                                     const unsigned long long* __restrict__ key64,
                                                     const Counters* __restrict__ ctr, uint2* __restrict__ bucket) {
    TS_PDL_ENTRY();
    extern __shared__ unsigned s_cur[];
    if (tile_start[ntiles] == 0) return;  // empty (or over capacity)
    const int t0 = blockIdx.y * BIN_MAX_TILES, nt = min(BIN_MAX_TILES, ntiles - t0);  // this CTA's tile range
    // 32-bit depth keys, range-reduced over the accepted triangles (monotone in
    // the fp64 key; ties of the reduced key are broken exactly by the tile sort)
    const unsigned long long kmin = ctr->key_min, krange = ctr->key_max - kmin;
    const int kbits = krange ? 64 - __clzll((long long)krange) : 0;
    const int gshift = kbits > 32 ? kbits - 32 : 0;
    const unsigned* row = mat + (size_t)blockIdx.x * ntiles + t0;
    for (int t = threadIdx.x; t < nt; t += BIN_CT) s_cur[t] = (unsigned)tile_start[t0 + t] + row[t];
    __syncthreads();
    const long long c0 = (long long)blockIdx.x * BIN_CHUNK;
    short4 bb[BIN_PER];
    unsigned long long key[BIN_PER];
#pragma unroll
    for (int k = 0; k < BIN_PER; k++) {
        const long long i = c0 + k * BIN_CT + threadIdx.x;
        bb[k] = i < n ? __ldg(bbox + i) : make_short4(0, 0, 0, 0);
        key[k] = i < n ? __ldg(key64 + i) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < BIN_PER; k++) {
        if (bb[k].y <= bb[k].x || bb[k].w <= bb[k].z) continue;
        const long long i = c0 + k * BIN_CT + threadIdx.x;
        const int tx0 = bb[k].x / TILE, tx1 = (bb[k].y - 1) / TILE + 1;
        const int ty0 = bb[k].z / TILE, ty1 = (bb[k].w - 1) / TILE + 1;
        for (int ty = ty0; ty < ty1; ty++)
            for (int tx = tx0; tx < tx1; tx++) {
                const int t = ty * ntx + tx - t0;
                if ((unsigned)t >= (unsigned)nt) continue;
                const unsigned pos = atomicAdd(&s_cur[t], 1u);
                bucket[pos] = make_uint2((unsigned)((key[k] - kmin) >> gshift), (unsigned)i);
            }
    }
}

// ---------------------------------------------------------------------------
// Stable LSD pass over items [0, cnt): warp w owns the contiguous segment
// [w*seg, (w+1)*seg), visited in rounds of 32 (so (round, lane) order is item
// order); per-warp digit counters, ranked with __match_any_sync.
template <class Dig>
__device__ __forceinline__ void radix_pass(int cnt, const unsigned* kin, const unsigned* vin, unsigned* kout,
                                           unsigned* vout, Dig dig, unsigned (*wc)[256], unsigned* s_w) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int seg = (cnt + BW - 1) / BW;
    const int s0 = (int)warp * seg, s1 = min(cnt, s0 + seg);
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int w = 0; w < BW; w++) wc[w][threadIdx.x] = 0u;
    __syncthreads();
    for (int r0 = s0; r0 < s1; r0 += 32) {
        const int i = r0 + (int)lane;
        const bool valid = i < s1;
        const unsigned d = valid ? dig(kin[i], vin[i]) : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (valid && (peers & lt) == 0u) wc[warp][d] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    unsigned tot = 0;
#pragma unroll
    for (int w = 0; w < BW; w++) tot += wc[w][threadIdx.x];
    unsigned all;
    unsigned run = excl_scan_256(tot, s_w, all);
#pragma unroll
    for (int w = 0; w < BW; w++) {
        const unsigned c = wc[w][threadIdx.x];
        wc[w][threadIdx.x] = run;
        run += c;
    }
    __syncthreads();
    for (int r0 = s0; r0 < s1; r0 += 32) {
        const int i = r0 + (int)lane;
        const bool valid = i < s1;
        unsigned k = 0u, v = 0u;
        if (valid) {
            k = kin[i];
            v = vin[i];
        }
        const unsigned d = valid ? dig(k, v) : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned b = valid ? wc[warp][d] : 0u;
        __syncwarp();
        if (valid && (peers & lt) == 0u) wc[warp][d] = b + __popc(peers);
        __syncwarp();
        if (valid) {
            const unsigned pos = b + __popc(peers & lt);
            kout[pos] = k;
            vout[pos] = v;
        }
    }
    __syncthreads();
}

// (z, idx) order of two sources (key64 = fp64 bits of the positive depth)
__device__ __forceinline__ bool zidx_less(const unsigned long long* key64, unsigned a, unsigned b) {
    const unsigned long long ka = key64[a], kb = key64[b];
    return ka < kb || (ka == kb && a < b);
}

// Sorts the tile list [base, base + cnt) of bucket into out (exact (z, idx) order).
// k0/v0/k1/v1: working arrays of cnt items (shared memory or global scratch).
__device__ __forceinline__ void sort_tile(int cnt, const uint2* bucket, const unsigned long long* key64,
                                          unsigned* out, unsigned* k0, unsigned* v0, unsigned* k1, unsigned* v1,
                                          int srcbits, unsigned (*wc)[256], unsigned* s_w,
                                          unsigned long long* s_red, int* s_flag) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // depth-key range of the tile
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int i = threadIdx.x; i < cnt; i += BT) {
        const unsigned src = bucket[i].y;
        const unsigned long long k = key64[src];  // (the bucket's key is the 32-bit reduced one)
        lo = k < lo ? k : lo;
        hi = k > hi ? k : hi;
        v0[i] = src;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, off);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi, off);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if (lane == 0) {
        s_red[warp] = lo;
        s_red[BW + warp] = hi;
    }
    if (threadIdx.x == 0) *s_flag = 0;
    __syncthreads();
    lo = s_red[0];
    hi = s_red[BW];
#pragma unroll
    for (int w = 1; w < BW; w++) {
        lo = s_red[w] < lo ? s_red[w] : lo;
        hi = s_red[BW + w] > hi ? s_red[BW + w] : hi;
    }
    const unsigned long long range = hi - lo;
    const int nbits = range ? 64 - __clzll((long long)range) : 0;
    const int shift = nbits > 16 ? nbits - 16 : 0;
    const int passes = ((nbits < 16 ? nbits : 16) + 7) / 8;
    for (int i = threadIdx.x; i < cnt; i += BT) k0[i] = (unsigned)((key64[v0[i]] - lo) >> shift);
    __syncthreads();
    for (int p = 0; p < passes; p++) {
        const int sh = 8 * p;
        radix_pass(cnt, k0, v0, k1, v1, [sh](unsigned k, unsigned) { return (k >> sh) & 0xffu; }, wc, s_w);
        unsigned* t = k0; k0 = k1; k1 = t;
        t = v0; v0 = v1; v1 = t;
    }
    // runs of equal reduced keys: exact (z, idx) order
    for (int i = threadIdx.x; i < cnt; i += BT) {
        if (i > 0 && k0[i] == k0[i - 1]) continue;
        int j = i + 1;
        while (j < cnt && k0[j] == k0[i] && j - i <= RUN_SHORT) j++;
        if (j - i > RUN_SHORT) {
            *s_flag = 1;
            continue;
        }
        for (int a = i + 1; a < j; a++) {
            const unsigned x = v0[a];
            int b = a - 1;
            while (b >= i && zidx_less(key64, x, v0[b])) {
                v0[b + 1] = v0[b];
                b--;
            }
            v0[b + 1] = x;
        }
    }
    __syncthreads();
    if (*s_flag) {
        // long runs (clustered or equal depths): stable LSD by idx, then by all 64 key bits
        for (int p = 0; p < (srcbits + 7) / 8; p++) {
            const int sh = 8 * p;
            radix_pass(cnt, k0, v0, k1, v1, [sh](unsigned, unsigned v) { return (v >> sh) & 0xffu; }, wc, s_w);
            unsigned* t = k0; k0 = k1; k1 = t;
            t = v0; v0 = v1; v1 = t;
        }
        for (int p = 0; p < 8; p++) {
            const int sh = 8 * p;
            radix_pass(cnt, k0, v0, k1, v1,
                       [sh, key64](unsigned, unsigned v) { return (unsigned)(key64[v] >> sh) & 0xffu; }, wc, s_w);
            unsigned* t = k0; k0 = k1; k1 = t;
            t = v0; v0 = v1; v1 = t;
        }
    }
    for (int i = threadIdx.x; i < cnt; i += BT) out[i] = v0[i];
}

// exact (z, idx) order of two packed items (reduced key << 32 | src)
__device__ __forceinline__ bool item_less(const unsigned long long* key64, unsigned long long a,
                                          unsigned long long b) {
    if ((a >> 32) != (b >> 32)) return (a >> 32) < (b >> 32);
    return zidx_less(key64, (unsigned)a, (unsigned)b);
}

template <int CAP, int NB>
__global__ void __launch_bounds__(BT) k_tile_sort(int ntiles, const int* __restrict__ tile_start,
                                                  const uint2* __restrict__ bucket,
                                                  const unsigned long long* __restrict__ key64,
                                                  unsigned* __restrict__ ent_src, unsigned* gk0, unsigned* gv0,
                                                  unsigned* gk1, unsigned* gv1, int srcbits,
                                                  const int* __restrict__ order) {
    constexpr int IPT = CAP / BT;
    __shared__ unsigned long long s_item[CAP];   // reduced key << 32 | src
    __shared__ unsigned s_hist[NB];
    __shared__ unsigned s_wc[BW][256];
    __shared__ unsigned s_w[32];
    __shared__ unsigned long long s_red[2 * BW];
    __shared__ int s_flag;
    // the long-tile kernel (independent tiles) may launch while this grid drains
    TS_PDL_ENTRY();
    const int t = order ? order[blockIdx.x] : (int)blockIdx.x;  // (longest lists first)
    const int base = tile_start[t], cnt = tile_start[t + 1] - base;
    if (cnt <= 0 || cnt > CAP) return;  // (longer tiles: k_tile_sort_big)
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long kk[IPT];
    unsigned src[IPT];
    unsigned long long lo = ~0ull, hi = 0ull;
#pragma unroll
    for (int q = 0; q < IPT; q++) {
        const int i = q * BT + threadIdx.x;
        kk[q] = 0ull;
        src[q] = 0u;
        if (i < cnt) {
            const uint2 r = bucket[base + i];
            kk[q] = r.x;
            src[q] = r.y;
            lo = kk[q] < lo ? kk[q] : lo;
            hi = kk[q] > hi ? kk[q] : hi;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, off);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi, off);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if (lane == 0) {
        s_red[warp] = lo;
        s_red[BW + warp] = hi;
    }
    for (int b = threadIdx.x; b < NB; b += BT) s_hist[b] = 0u;
    __syncthreads();
    lo = s_red[0];
    hi = s_red[BW];
#pragma unroll
    for (int w = 1; w < BW; w++) {
        lo = s_red[w] < lo ? s_red[w] : lo;
        hi = s_red[BW + w] > hi ? s_red[BW + w] : hi;
    }
    const unsigned long long range = hi - lo;
    const int nbits = range ? 64 - __clzll((long long)range) : 0;
    const int s32 = nbits > 32 ? nbits - 32 : 0;                       // 64 -> 32-bit reduced key
    const int b32 = nbits < 32 ? nbits : 32;
    constexpr int LB = NB == 4096 ? 12 : (NB == 2048 ? 11 : 10);
    const int s12 = b32 > LB ? b32 - LB : 0;                            // 32-bit key -> bucket
    unsigned kr[IPT];
#pragma unroll
    for (int q = 0; q < IPT; q++) {
        kr[q] = (unsigned)((kk[q] - lo) >> s32);
        if (q * BT + (int)threadIdx.x < cnt) atomicAdd(&s_hist[kr[q] >> s12], 1u);
    }
    __syncthreads();
    {  // exclusive scan of the NB bucket counts (NB / BT consecutive per thread)
        constexpr int PT = NB / BT;
        unsigned v[PT], sum = 0;
#pragma unroll
        for (int u = 0; u < PT; u++) {
            v[u] = s_hist[threadIdx.x * PT + u];
            sum += v[u];
        }
        unsigned all;
        unsigned run = excl_scan_256(sum, s_w, all);
#pragma unroll
        for (int u = 0; u < PT; u++) {
            s_hist[threadIdx.x * PT + u] = run;
            run += v[u];
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < IPT; q++) {
        if (q * BT + (int)threadIdx.x < cnt) {
            const unsigned pos = atomicAdd(&s_hist[kr[q] >> s12], 1u);
            s_item[pos] = ((unsigned long long)kr[q] << 32) | src[q];
        }
    }
    __syncthreads();
    // exact (z, idx) order inside every bucket: an item's final position is
    // its bucket's start plus the number of bucket items ordered before it
    // (s_hist[b] now holds the end of bucket b); long buckets -> fallback
    int longb = 0;
    for (int i = threadIdx.x; i < cnt; i += BT) {
        const unsigned long long x = s_item[i];
        const unsigned b = (unsigned)(x >> 32) >> s12;
        const int be = (int)s_hist[b], bs = b ? (int)s_hist[b - 1] : 0;
        if (be - bs > RUN_LONG) {
            longb = 1;
            continue;
        }
        int rank = 0;
        for (int j = bs; j < be; j++) {
            const unsigned long long y = s_item[j];
            if (y != x) rank += item_less(key64, y, x);
        }
        TS_ASSERT(bs + rank < be && be <= cnt);
        ent_src[base + bs + rank] = (unsigned)x;
    }
    if (__syncthreads_or(longb))
        sort_tile(cnt, bucket + base, key64, ent_src + base, gk0 + base, gv0 + base, gk1 + base, gv1 + base,
                  srcbits, s_wc, s_w, s_red, &s_flag);
}


// Tiles of (SMALL, CAP] entries (listed by k_tile_scan): the same bucket sort
// with the bucket re-read from L2 instead of staged in registers, the sorted
// items in dynamic shared memory (8 x CAP bytes); longer tiles take the stable
// LSD path on global scratch.  Persistent CTAs walk the list.
template <int CAP, int NB>
__global__ void __launch_bounds__(BT) k_tile_sort_big(const int* __restrict__ big_list, const int* __restrict__ n_big,
                                                      const int* __restrict__ tile_start,
                                                      const uint2* __restrict__ bucket,
                                                      const unsigned long long* __restrict__ key64,
                                                      unsigned* __restrict__ ent_src, unsigned* gk0, unsigned* gv0,
                                                      unsigned* gk1, unsigned* gv1, int srcbits) {
    // waits for k_tile_sort (PDL chain: the blend after this grid waits only on it)
    TS_PDL_ENTRY();
    extern __shared__ __align__(16) unsigned long long s_item[];  // [CAP]
    __shared__ unsigned s_hist[NB];
    __shared__ unsigned s_wc[BW][256];
    __shared__ unsigned s_w[32];
    __shared__ unsigned long long s_red[2 * BW];
    __shared__ int s_flag;
    const int nbig = *n_big;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = blockIdx.x; k < nbig; k += gridDim.x) {
        const int t = big_list[k];
        const int base = tile_start[t], cnt = tile_start[t + 1] - base;
        if (cnt > CAP) {
            sort_tile(cnt, bucket + base, key64, ent_src + base, gk0 + base, gv0 + base, gk1 + base, gv1 + base,
                      srcbits, s_wc, s_w, s_red, &s_flag);
            __syncthreads();
            continue;
        }
        unsigned lo = ~0u, hi = 0u;
        for (int i = threadIdx.x; i < cnt; i += BT) {
            const unsigned x = bucket[base + i].x;
            lo = x < lo ? x : lo;
            hi = x > hi ? x : hi;
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if (lane == 0) {
            s_red[warp] = lo;
            s_red[BW + warp] = hi;
        }
        for (int b = threadIdx.x; b < NB; b += BT) s_hist[b] = 0u;
        __syncthreads();
        lo = (unsigned)s_red[0];
        hi = (unsigned)s_red[BW];
#pragma unroll
        for (int w = 1; w < BW; w++) {
            lo = (unsigned)s_red[w] < lo ? (unsigned)s_red[w] : lo;
            hi = (unsigned)s_red[BW + w] > hi ? (unsigned)s_red[BW + w] : hi;
        }
        const unsigned range = hi - lo;
        const int nbits = range ? 32 - __clz((int)range) : 0;
        constexpr int LB = NB == 4096 ? 12 : (NB == 2048 ? 11 : 10);
        const int s12 = nbits > LB ? nbits - LB : 0;
        for (int i = threadIdx.x; i < cnt; i += BT) atomicAdd(&s_hist[(bucket[base + i].x - lo) >> s12], 1u);
        __syncthreads();
        {
            constexpr int PT = NB / BT;
            unsigned v[PT], sum = 0;
#pragma unroll
            for (int u = 0; u < PT; u++) {
                v[u] = s_hist[threadIdx.x * PT + u];
                sum += v[u];
            }
            unsigned all;
            unsigned run = excl_scan_256(sum, s_w, all);
#pragma unroll
            for (int u = 0; u < PT; u++) {
                s_hist[threadIdx.x * PT + u] = run;
                run += v[u];
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += BT) {
            const uint2 r = bucket[base + i];
            const unsigned kr = r.x - lo;
            const unsigned pos = atomicAdd(&s_hist[kr >> s12], 1u);
            s_item[pos] = ((unsigned long long)kr << 32) | r.y;
        }
        __syncthreads();
        int longb = 0;
        for (int i = threadIdx.x; i < cnt; i += BT) {
            const unsigned long long x = s_item[i];
            const unsigned b = (unsigned)(x >> 32) >> s12;
            const int be = (int)s_hist[b], bs = b ? (int)s_hist[b - 1] : 0;
            if (be - bs > RUN_LONG) {
                longb = 1;
                continue;
            }
            int rank = 0;
            for (int j = bs; j < be; j++) {
                const unsigned long long y = s_item[j];
                if (y != x) rank += item_less(key64, y, x);
            }
            TS_ASSERT(bs + rank < be && be <= cnt);
        ent_src[base + bs + rank] = (unsigned)x;
        }
        if (__syncthreads_or(longb))
            sort_tile(cnt, bucket + base, key64, ent_src + base, gk0 + base, gv0 + base, gk1 + base, gv1 + base,
                      srcbits, s_wc, s_w, s_red, &s_flag);
        __syncthreads();
    }
}

constexpr int SORT_SMALL = 2048, SORT_BIG = 8192;

void bin_tiles_fill(long long n, const short4* bbox, const unsigned long long* key64, int ntx, int ntiles,
                    unsigned* tcnt, unsigned* mat, int* tile_start, uint2* bucket, const Counters* ctr,
                    long long cap, unsigned* overflow, int* big_list, cudaStream_t st, int* tile_order) {
    const int nchunk = (int)((n + BIN_CHUNK - 1) / BIN_CHUNK);
    const int nrange = (ntiles + BIN_MAX_TILES - 1) / BIN_MAX_TILES;  // tile ranges (grid y)
    const int smem = (nrange > 1 ? BIN_MAX_TILES : ntiles) * (int)sizeof(unsigned);
    smem_optin((const void*)k_bin_count, 4 * BIN_MAX_TILES);
    smem_optin((const void*)k_bin_fill, 4 * BIN_MAX_TILES);
    if (n > 0) {
        launch_pdl(k_bin_count, dim3(nchunk, nrange), dim3(BIN_CT), smem, st, n, bbox, ntx, ntiles, mat);
        launch_pdl(k_bin_cols, dim3((ntiles + 31) / 32), dim3(256), 0, st, nchunk, ntiles, mat, tcnt);
    } else {
        cudaMemsetAsync(tcnt, 0, sizeof(unsigned) * ntiles, st);
    }
    // big_list[ntiles]: tiles longer than SORT_SMALL; its count at big_list[ntiles]
    launch_pdl(k_tile_scan, dim3(1), dim3(1024), 0, st, ntiles, tcnt, tile_start, cap, overflow, SORT_SMALL, big_list,
                                    big_list + ntiles, tile_order);
    if (n > 0)
        launch_pdl(k_bin_fill, dim3(nchunk, nrange), dim3(BIN_CT), smem, st, n, bbox, ntx, ntiles, mat, tile_start, key64, ctr,
                                                              bucket);
}

size_t bin_matrix_bytes(long long n, int ntiles) {
    const long long nchunk = (n + BIN_CHUNK - 1) / BIN_CHUNK;
    return sizeof(unsigned) * (size_t)(nchunk > 0 ? nchunk : 1) * (size_t)ntiles;
}

int bin_max_tiles() { return 1 << 22; }  // (any view: larger tile counts use several tile ranges)

void bin_tiles_sort(long long n, int ntiles, const int* tile_start, const uint2* bucket,
                    const unsigned long long* key64, unsigned* ent_src, unsigned* const scratch[4],
                    const int* big_list, cudaStream_t st, const int* tile_order) {
    const int srcbits = n > 1 ? 64 - __builtin_clzll((unsigned long long)(n - 1)) : 1;
    launch_pdl(k_tile_sort<SORT_SMALL, 2048>, dim3(ntiles), dim3(BT), 0, st, ntiles, tile_start, bucket, key64, ent_src, scratch[0],
                                                        scratch[1], scratch[2], scratch[3], srcbits, tile_order);
    // tiles above SORT_SMALL entries (dense views), listed by k_tile_scan
    const int sms = sm_count();
    const int smem = SORT_BIG * (int)sizeof(unsigned long long);
    smem_optin((const void*)k_tile_sort_big<SORT_BIG, 4096>, smem);
    // programmatic dependent launch: its CTAs are scheduled during k_tile_sort's last
    // wave and wait for that grid (TS_PDL_ENTRY), so the blend after it may rely on both
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * sms);
    cfg.blockDim = dim3(BT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int* n_big = big_list + ntiles;
    cudaLaunchKernelEx(&cfg, k_tile_sort_big<SORT_BIG, 4096>, big_list, n_big, tile_start, bucket, key64, ent_src,
                       scratch[0], scratch[1], scratch[2], scratch[3], srcbits);
}

}  // namespace ts
