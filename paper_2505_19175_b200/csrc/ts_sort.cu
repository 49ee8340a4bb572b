// ts_sort.cu -- device-wide scans, compaction, stable LSD radix sort, tile
// duplication and tile ranges.
//
// Replaces the host side of the reference's binning (render.py:271-283 cull +
// np.lexsort((idx, z)) and render.py:315-361 _tile_counts/_tile_fill): the
// accepted triangles are compacted in source order, stably radix-sorted on the
// fp64 depth bits (a stable sort of idx-ordered items reproduces the index
// tie-break of np.lexsort), duplicated per touched tile in depth-rank order and
// stably sorted by tile id, which yields exactly the reference CSR order.
#include "ts_kernels.cuh"

namespace ts {

constexpr int SB = 256;  // threads per block for scan / sort kernels
constexpr int RADIX = 256;

size_t sort_scratch_bytes(int max_blocks) {
    return sizeof(unsigned) * ((size_t)RADIX * max_blocks + max_blocks + 1 + 64);
}

int sort_grid(long long count, int max_blocks) {
    long long g = (count + SB * 8 - 1) / (SB * 8);  // >= 8 rounds of 256 per block
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (int)g;
}

static inline long long chunk_of(long long count, int g) {
    long long c = (count + g - 1) / g;
    return (c + SB - 1) / SB * SB;
}

__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned& total) {
    __shared__ unsigned s_warp[SB / 32];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= (unsigned)off) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned w = lane < SB / 32 ? s_warp[lane] : 0u;
#pragma unroll
        for (int off = 1; off < SB / 32; off <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= (unsigned)off) w += y;
        }
        if (lane < SB / 32) s_warp[lane] = w;
    }
    __syncthreads();
    unsigned pre = warp ? s_warp[warp - 1] : 0u;
    total = s_warp[SB / 32 - 1];
    __syncthreads();
    return pre + x - v;
}

// ---------------- generic reduce-then-scan over a functor ----------------
template <class F>
__global__ void __launch_bounds__(SB) k_scan_reduce(long long n, long long chunk, F f, unsigned* bsums) {
    long long lo = (long long)blockIdx.x * chunk, hi = min(n, lo + chunk);
    unsigned acc = 0;
    for (long long i = lo + threadIdx.x; i < hi; i += SB) acc += f.load(i);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    __shared__ unsigned s[SB / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = 0;
        for (int w = 0; w < SB / 32; w++) t += s[w];
        bsums[blockIdx.x] = t;
    }
}

// single-block exclusive scan of a[0..len) in place; a[len] = total
__global__ void __launch_bounds__(1024) k_scan_single(unsigned* a, long long len) {
    __shared__ unsigned s_warp[32];
    long long per = (len + 1023) / 1024;
    long long lo = threadIdx.x * per, hi = min(len, lo + per);
    unsigned acc = 0;
    for (long long i = lo; i < hi; i++) acc += a[i];
    // block exclusive scan of acc (1024 threads)
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = acc;
    for (int off = 1; off < 32; off <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= (unsigned)off) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned w = s_warp[lane];
        for (int off = 1; off < 32; off <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= (unsigned)off) w += y;
        }
        s_warp[lane] = w;
    }
    __syncthreads();
    unsigned run = (warp ? s_warp[warp - 1] : 0u) + x - acc;
    for (long long i = lo; i < hi; i++) {
        unsigned v = a[i];
        a[i] = run;
        run += v;
    }
    if (threadIdx.x == 1023) a[len] = s_warp[31];
}

template <class F>
__global__ void __launch_bounds__(SB) k_scan_apply(long long n, long long chunk, F f, const unsigned* bsums) {
    long long lo = (long long)blockIdx.x * chunk, hi = min(n, lo + chunk);
    unsigned run = bsums[blockIdx.x];
    for (long long base = lo; base < hi; base += SB) {
        long long i = base + threadIdx.x;
        unsigned v = i < hi ? f.load(i) : 0u;
        unsigned tot;
        unsigned ex = block_excl_scan(v, tot);
        if (i < hi) f.store(i, run + ex, v);
        run += tot;
    }
}

template <class F>
static void scan_functor(long long n, F f, const SortScratch& s, cudaStream_t st) {
    if (n <= 0) return;
    int g = sort_grid(n, s.max_blocks);
    long long chunk = chunk_of(n, g);
    g = (int)((n + chunk - 1) / chunk);
    k_scan_reduce<<<g, SB, 0, st>>>(n, chunk, f, s.bsums);
    k_scan_single<<<1, 1024, 0, st>>>(s.bsums, g);
    k_scan_apply<<<g, SB, 0, st>>>(n, chunk, f, s.bsums);
}

struct CompactF {
    const unsigned* flag;
    const unsigned long long* key;
    unsigned long long* keys_c;
    unsigned* vals_c;
    __device__ unsigned load(long long i) const { return flag[i]; }
    __device__ void store(long long i, unsigned ex, unsigned v) const {
        if (v) {
            keys_c[ex] = key[i];
            vals_c[ex] = (unsigned)i;
        }
    }
};

void compact_accepted(long long n, const unsigned* flag, const unsigned long long* key,
                      unsigned long long* keys_c, unsigned* vals_c, const SortScratch& s,
                      cudaStream_t st) {
    scan_functor(n, CompactF{flag, key, keys_c, vals_c}, s, st);
}

struct KeptF {
    const unsigned char* flags;
    long long n;
    long long* kept;
    long long* n_kept;
    __device__ unsigned load(long long i) const { return flags[i] == 0 ? 1u : 0u; }
    __device__ void store(long long i, unsigned ex, unsigned v) const {
        if (v) kept[ex] = i;
        if (i == n - 1) *n_kept = (long long)ex + v;
    }
};

void compact_unflagged(long long n, const unsigned char* flags, long long* kept, long long* n_kept,
                       const SortScratch& s, cudaStream_t st) {
    if (n <= 0) {
        cudaMemsetAsync(n_kept, 0, sizeof(long long), st);
        return;
    }
    scan_functor(n, KeptF{flags, n, kept, n_kept}, s, st);
}

struct RankF {
    const unsigned* sorted_src;
    const unsigned* tcount;
    unsigned* offs;
    int* rank_of;  // nullable (debug dumps only)
    __device__ unsigned load(long long m) const { return tcount[sorted_src[m]]; }
    __device__ void store(long long m, unsigned ex, unsigned) const {
        offs[m] = ex;
        if (rank_of) rank_of[sorted_src[m]] = (int)m;
    }
};

void rank_offsets(long long m, const unsigned* sorted_src, const unsigned* tcount, unsigned* offs,
                  int* rank_of, const SortScratch& s, cudaStream_t st) {
    scan_functor(m, RankF{sorted_src, tcount, offs, rank_of}, s, st);
}

// ---------------- stable LSD radix sort ----------------
template <typename K>
__global__ void __launch_bounds__(SB) k_radix_hist(long long count, long long chunk, const K* __restrict__ keys,
                                                   int shift, unsigned mask, unsigned* hist, int g) {
    __shared__ unsigned s_h[RADIX];
    s_h[threadIdx.x] = 0;
    __syncthreads();
    long long lo = (long long)blockIdx.x * chunk, hi = min(count, lo + chunk);
    for (long long i = lo + threadIdx.x; i < hi; i += SB) {
        unsigned d = (unsigned)(keys[i] >> shift) & mask;
        atomicAdd(&s_h[d], 1u);
    }
    __syncthreads();
    hist[(size_t)threadIdx.x * g + blockIdx.x] = s_h[threadIdx.x];
}

template <typename K>
__global__ void __launch_bounds__(SB) k_radix_scatter(long long count, long long chunk,
                                                      const K* __restrict__ kin, const unsigned* __restrict__ vin,
                                                      K* __restrict__ kout, unsigned* __restrict__ vout,
                                                      int shift, unsigned mask, const unsigned* hist, int g) {
    __shared__ unsigned s_base[RADIX];
    __shared__ unsigned s_wcnt[SB / 32][RADIX];
    const unsigned warp = threadIdx.x >> 5;
    s_base[threadIdx.x] = hist[(size_t)threadIdx.x * g + blockIdx.x];
    long long lo = (long long)blockIdx.x * chunk, hi = min(count, lo + chunk);
    const unsigned lt = lanemask_lt();
    for (long long base = lo; base < hi; base += SB) {
        long long i = base + threadIdx.x;
        bool valid = i < hi;
        K k = valid ? kin[i] : (K)0;
        unsigned v = valid ? vin[i] : 0u;
        unsigned d = valid ? ((unsigned)(k >> shift) & mask) : RADIX;
#pragma unroll
        for (int w = 0; w < SB / 32; w++) s_wcnt[w][threadIdx.x] = 0;
        __syncthreads();
        unsigned peers = __match_any_sync(0xffffffffu, d);
        unsigned rank = __popc(peers & lt);
        if (valid && rank == 0) s_wcnt[warp][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            unsigned pre = s_base[d] + rank;
            for (unsigned w = 0; w < warp; w++) pre += s_wcnt[w][d];
            kout[pre] = k;
            vout[pre] = v;
        }
        __syncthreads();
        unsigned tot = 0;
#pragma unroll
        for (int w = 0; w < SB / 32; w++) tot += s_wcnt[w][threadIdx.x];
        s_base[threadIdx.x] += tot;
        __syncthreads();
    }
}

template <typename K>
static int radix_sort_impl(long long count, K* keys, unsigned* vals, K* keys_alt, unsigned* vals_alt,
                           int bit_lo, int bit_hi, const SortScratch& s, cudaStream_t st) {
    if (count <= 1 || bit_hi <= bit_lo) return 0;
    int g = sort_grid(count, s.max_blocks);
    long long chunk = chunk_of(count, g);
    g = (int)((count + chunk - 1) / chunk);
    K* kin = keys;
    unsigned* vin = vals;
    K* kout = keys_alt;
    unsigned* vout = vals_alt;
    int parity = 0;
    for (int shift = bit_lo; shift < bit_hi; shift += 8) {
        int nb = bit_hi - shift < 8 ? bit_hi - shift : 8;
        unsigned mask = (1u << nb) - 1u;
        k_radix_hist<K><<<g, SB, 0, st>>>(count, chunk, kin, shift, mask, s.hist, g);
        k_scan_single<<<1, 1024, 0, st>>>(s.hist, (long long)RADIX * g);
        k_radix_scatter<K><<<g, SB, 0, st>>>(count, chunk, kin, vin, kout, vout, shift, mask, s.hist, g);
        K* tk = kin; kin = kout; kout = tk;
        unsigned* tv = vin; vin = vout; vout = tv;
        parity ^= 1;
    }
    return parity;
}

int radix_sort_u64(long long count, unsigned long long* keys, unsigned* vals,
                   unsigned long long* keys_alt, unsigned* vals_alt, int bit_lo, int bit_hi,
                   const SortScratch& s, cudaStream_t st) {
    return radix_sort_impl<unsigned long long>(count, keys, vals, keys_alt, vals_alt, bit_lo, bit_hi, s, st);
}

int radix_sort_u32(long long count, unsigned* keys, unsigned* vals, unsigned* keys_alt,
                   unsigned* vals_alt, int bit_lo, int bit_hi, const SortScratch& s,
                   cudaStream_t st) {
    return radix_sort_impl<unsigned>(count, keys, vals, keys_alt, vals_alt, bit_lo, bit_hi, s, st);
}

// ---------------- duplication / ranges ----------------
__global__ void __launch_bounds__(256) k_duplicate(long long m, const unsigned* __restrict__ sorted_src,
                                                   const short4* __restrict__ bbox, const unsigned* __restrict__ offs,
                                                   int ntx, unsigned* __restrict__ tkey,
                                                   unsigned* __restrict__ tval, long long cap, unsigned* overflow) {
    long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    unsigned src = sorted_src[k];
    const short4 bb = bbox[src];
    int x0 = bb.x, x1 = bb.y, y0 = bb.z, y1 = bb.w;
    if (x1 <= x0 || y1 <= y0) return;
    int tx0 = x0 / TILE, tx1 = (x1 - 1) / TILE + 1, ty0 = y0 / TILE, ty1 = (y1 - 1) / TILE + 1;
    unsigned pos = offs[k];
    for (int ty = ty0; ty < ty1; ty++)
        for (int tx = tx0; tx < tx1; tx++) {
            if (pos < cap) {
                tkey[pos] = (unsigned)(ty * ntx + tx);
                tval[pos] = src;
            } else if (overflow) {
                *overflow = 1u;  // sticky until ts_forward_status
            }
            pos++;
        }
}

void duplicate_entries(long long m, const unsigned* sorted_src, const short4* bbox, const unsigned* offs,
                       int ntx, unsigned* tkey, unsigned* tval, long long cap, unsigned* overflow,
                       cudaStream_t st) {
    if (m <= 0) return;
    k_duplicate<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, sorted_src, bbox, offs, ntx, tkey, tval, cap,
                                                              overflow);
}

__global__ void k_ranges(long long e, const unsigned long long* de, const unsigned* __restrict__ tkey, int ntiles,
                         int* __restrict__ start) {
    if (de) e = min(e, (long long)*de);
    long long pos = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e <= 0) {
        if (pos <= ntiles) start[pos] = 0;
        return;
    }
    if (pos >= e) return;
    int k = (int)tkey[pos];
    int kp = pos > 0 ? (int)tkey[pos - 1] : -1;
    for (int t = kp + 1; t <= k; t++) start[t] = (int)pos;
    if (pos == e - 1)
        for (int t = k + 1; t <= ntiles; t++) start[t] = (int)e;
}

void tile_ranges(long long e, const unsigned* tkey, int ntiles, int* tile_start, cudaStream_t st) {
    tile_ranges_dev(e, nullptr, tkey, ntiles, tile_start, st);
}

void tile_ranges_dev(long long cap, const unsigned long long* de, const unsigned* tkey, int ntiles, int* tile_start,
                     cudaStream_t st) {
    const long long g = (cap > ntiles + 1 ? cap : ntiles + 1);
    k_ranges<<<(unsigned)((g + 255) / 256), 256, 0, st>>>(cap, de, tkey, ntiles, tile_start);
}

__global__ void k_entries_to_rank(long long e, const unsigned* ent_src, const int* rank_of, int* out) {
    long long pos = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos < e) out[pos] = rank_of[ent_src[pos]];
}

void entries_to_rank(long long e, const unsigned* ent_src, const int* rank_of, int* out, cudaStream_t st) {
    if (e <= 0) return;
    k_entries_to_rank<<<(unsigned)((e + 255) / 256), 256, 0, st>>>(e, ent_src, rank_of, out);
}

__global__ void k_bbox_dump(long long n, const short4* bbox, int* out) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const short4 b = bbox[i];
    out[i * 4 + 0] = b.x;
    out[i * 4 + 1] = b.y;
    out[i * 4 + 2] = b.z;
    out[i * 4 + 3] = b.w;
}

void bbox_dump(long long n, const short4* bbox, int* out, cudaStream_t st) {
    if (n <= 0) return;
    k_bbox_dump<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, bbox, out);
}

}  // namespace ts

// ===========================================================================
// Onesweep LSD radix sort (single kernel per 8-bit pass, decoupled look-back),
// 32-bit keys + 32-bit values, stable.  Tile = 4096 items per CTA; each warp
// owns a contiguous 512-item segment loaded warp-striped so (item, lane)
// order equals input order, which keeps the sort stable.
// ===========================================================================
namespace ts {

constexpr int OS_THREADS = 256;
constexpr int OS_ITEMS = 8;
constexpr int OS_TILE = OS_THREADS * OS_ITEMS;  // 4096

size_t onesweep_scratch_bytes(long long max_count, int max_passes) {
    long long tiles = (max_count + OS_TILE - 1) / OS_TILE + 1;
    return sizeof(unsigned) * ((size_t)max_passes * tiles * RADIX + (size_t)max_passes * RADIX + 64);
}

// per-tile digit counts of one pass, digit-major: cnt[d * tiles + tile]
__global__ void __launch_bounds__(OS_THREADS) k_os_count(long long count, const unsigned long long* dcount,
                                                         const unsigned* __restrict__ keys,
                                                         int shift, unsigned* __restrict__ cnt, int tiles) {
    if (dcount) count = min(count, (long long)*dcount);
    if ((long long)blockIdx.x * OS_TILE >= count) return;
    __shared__ unsigned s_h[RADIX];
    s_h[threadIdx.x] = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * OS_TILE;
    if (base + OS_TILE <= count && (((size_t)(keys + base)) & 15) == 0) {
        const uint4* k4 = reinterpret_cast<const uint4*>(keys + base);
        uint4 v[OS_ITEMS / 4];
#pragma unroll
        for (int i = 0; i < OS_ITEMS / 4; i++) v[i] = __ldg(k4 + i * OS_THREADS + threadIdx.x);
#pragma unroll
        for (int i = 0; i < OS_ITEMS / 4; i++) {
            atomicAdd(&s_h[(v[i].x >> shift) & 0xffu], 1u);
            atomicAdd(&s_h[(v[i].y >> shift) & 0xffu], 1u);
            atomicAdd(&s_h[(v[i].z >> shift) & 0xffu], 1u);
            atomicAdd(&s_h[(v[i].w >> shift) & 0xffu], 1u);
        }
    } else {
        for (int i = 0; i < OS_ITEMS; i++) {
            const long long idx = base + i * OS_THREADS + threadIdx.x;
            if (idx < count) atomicAdd(&s_h[(__ldg(keys + idx) >> shift) & 0xffu], 1u);
        }
    }
    __syncthreads();
    cnt[(size_t)threadIdx.x * tiles + blockIdx.x] = s_h[threadIdx.x];
}

// per digit (one block each): exclusive scan over tiles in place; tot[d] = column total
__global__ void __launch_bounds__(1024) k_os_scan(unsigned* __restrict__ cnt, int stride, long long count,
                                                  const unsigned long long* dcount, unsigned* __restrict__ tot) {
    __shared__ unsigned s_w[32];
    if (dcount) count = min(count, (long long)*dcount);
    const int tiles = (int)((count + OS_TILE - 1) / OS_TILE);
    unsigned* row = cnt + (size_t)blockIdx.x * stride;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned carry = 0;
    for (int b0 = 0; b0 < tiles; b0 += 1024) {
        const int i = b0 + threadIdx.x;
        const unsigned v = i < tiles ? row[i] : 0u;
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
        const unsigned ex = carry + (warp ? s_w[warp - 1] : 0u) + x - v;
        if (i < tiles) row[i] = ex;
        carry += s_w[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) tot[blockIdx.x] = carry;
}

// Stable scatter of one 8-bit pass: items are ranked with warp match +
// per-warp counters, staged in shared memory in tile-local sorted order and
// written out in coalesced runs at cnt_scanned[d][tile] + global digit start.
__global__ void __launch_bounds__(OS_THREADS) k_os_scatter(long long count, const unsigned long long* dcount,
                                                           const unsigned* __restrict__ kin,
                                                           const unsigned* __restrict__ vin,
                                                           unsigned* __restrict__ kout, unsigned* __restrict__ vout,
                                                           int shift, const unsigned* __restrict__ cnt, int tiles,
                                                           const unsigned* __restrict__ tot) {
    __shared__ unsigned s_wc[OS_THREADS / 32][RADIX];
    __shared__ unsigned s_lstart[RADIX];
    __shared__ unsigned s_gbase[RADIX];
    __shared__ unsigned s_k[OS_TILE];
    __shared__ unsigned s_v[OS_TILE];
    if (dcount) count = min(count, (long long)*dcount);
    if ((long long)blockIdx.x * OS_TILE >= count) return;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned tile = blockIdx.x;
    for (int w = 0; w < OS_THREADS / 32; w++) s_wc[w][threadIdx.x] = 0;
    unsigned tsum;
    const unsigned gstart = block_excl_scan(tot[threadIdx.x], tsum);  // has __syncthreads
    s_gbase[threadIdx.x] = gstart + cnt[(size_t)threadIdx.x * tiles + tile];
    const long long base = (long long)tile * OS_TILE + (long long)warp * (OS_TILE / (OS_THREADS / 32));
    const unsigned lt = lanemask_lt();
    unsigned key[OS_ITEMS], val[OS_ITEMS], off[OS_ITEMS];
#pragma unroll
    for (int i = 0; i < OS_ITEMS; i++) {
        const long long idx = base + i * 32 + lane;
        const bool valid = idx < count;
        key[i] = valid ? __ldg(kin + idx) : 0u;
        val[i] = valid ? __ldg(vin + idx) : 0u;
    }
#pragma unroll
    for (int i = 0; i < OS_ITEMS; i++) {
        const long long idx = base + i * 32 + lane;
        const bool valid = idx < count;
        const unsigned d = valid ? ((key[i] >> shift) & 0xffu) : 0x100u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned rank = __popc(peers & lt);
        const unsigned b = valid ? s_wc[warp][d] : 0u;
        __syncwarp();
        if (valid && rank == 0) s_wc[warp][d] = b + __popc(peers);
        __syncwarp();
        off[i] = b + rank;
    }
    __syncthreads();
    unsigned run = 0;
#pragma unroll
    for (int w = 0; w < OS_THREADS / 32; w++) {
        const unsigned c = s_wc[w][threadIdx.x];
        s_wc[w][threadIdx.x] = run;
        run += c;
    }
    unsigned tot2;
    const unsigned lstart = block_excl_scan(run, tot2);  // has __syncthreads
    s_lstart[threadIdx.x] = lstart;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < OS_ITEMS; i++) {
        const long long idx = base + i * 32 + lane;
        if (idx < count) {
            const unsigned dd = (key[i] >> shift) & 0xffu;
            const unsigned lp = s_lstart[dd] + s_wc[warp][dd] + off[i];
            s_k[lp] = key[i];
            s_v[lp] = val[i];
        }
    }
    __syncthreads();
    const long long n_here = min((long long)OS_TILE, count - (long long)tile * OS_TILE);
    for (int lp = threadIdx.x; lp < n_here; lp += OS_THREADS) {
        const unsigned k = s_k[lp];
        const unsigned dd = (k >> shift) & 0xffu;
        const unsigned pos = s_gbase[dd] + (lp - s_lstart[dd]);
        kout[pos] = k;
        vout[pos] = s_v[lp];
    }
}

// Sorts (keys, vals) by bits [0, nbits).  Returns 1 if the result is in the alt buffers.
int onesweep_sort_u32(long long count, unsigned* keys, unsigned* vals, unsigned* keys_alt,
                      unsigned* vals_alt, int nbits, void* scratch, cudaStream_t st) {
    return onesweep_sort_u32_dev(count, nullptr, keys, vals, keys_alt, vals_alt, nbits, scratch, st);
}

// count = min(cap, *dcount) when dcount is given (read on the device: no host sync)
int onesweep_sort_u32_dev(long long cap, const unsigned long long* dcount, unsigned* keys, unsigned* vals,
                          unsigned* keys_alt, unsigned* vals_alt, int nbits, void* scratch, cudaStream_t st) {
    const long long count = cap;
    if (count <= 1 || nbits <= 0) return 0;
    int npass = (nbits + 7) / 8;
    const int tiles = (int)((count + OS_TILE - 1) / OS_TILE);
    unsigned* cnt = (unsigned*)scratch;  // [256][tiles]
    unsigned* tot = cnt + (size_t)RADIX * tiles;
    unsigned *kin = keys, *vin = vals, *kout = keys_alt, *vout = vals_alt;
    int parity = 0;
    for (int p = 0; p < npass; p++) {
        k_os_count<<<tiles, OS_THREADS, 0, st>>>(count, dcount, kin, 8 * p, cnt, tiles);
        k_os_scan<<<RADIX, 1024, 0, st>>>(cnt, tiles, count, dcount, tot);
        k_os_scatter<<<tiles, OS_THREADS, 0, st>>>(count, dcount, kin, vin, kout, vout, 8 * p, cnt, tiles, tot);
        unsigned* t = kin; kin = kout; kout = t;
        t = vin; vin = vout; vout = t;
        parity ^= 1;
    }
    return parity;
}

// ---------------------------------------------------------------------------
// Depth-key helpers: 32-bit range-reduced keys, then exact (z64, idx) order
// restored inside runs of equal reduced keys.
// ---------------------------------------------------------------------------
struct CompactKey32F {
    const unsigned* flag;
    const unsigned long long* key;
    unsigned long long kmin;
    int shift;
    unsigned* keys_c;
    unsigned* vals_c;
    __device__ unsigned load(long long i) const { return flag[i]; }
    __device__ void store(long long i, unsigned ex, unsigned v) const {
        if (v) {
            keys_c[ex] = (unsigned)((key[i] - kmin) >> shift);
            vals_c[ex] = (unsigned)i;
        }
    }
};

void compact_accepted32(long long n, const unsigned* flag, const unsigned long long* key,
                        unsigned long long kmin, int shift, unsigned* keys_c, unsigned* vals_c,
                        const SortScratch& s, cudaStream_t st) {
    scan_functor(n, CompactKey32F{flag, key, kmin, shift, keys_c, vals_c}, s, st);
}

// Depth keys of all n triangles without compaction: accepted triangles get
// their range-reduced key, clamped below kmax_key; culled ones get kmax_key and
// therefore sort after every accepted triangle (stable: source order within).
// The reduction (key_min, shift) comes from the preprocess counters on the
// device, so the sort is enqueued without a host round trip.
__global__ void k_depth_keys(long long n, const unsigned* __restrict__ flag, const unsigned long long* __restrict__ key,
                             const Counters* __restrict__ ctr, int kbits_cap, unsigned* __restrict__ k32,
                             unsigned* __restrict__ vals) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned kmax_key = (1u << kbits_cap) - 1u;
    const unsigned long long kmin = ctr->key_min;
    const unsigned long long range = ctr->m ? ctr->key_max - kmin : 0ull;
    const int kb = range ? 64 - __clzll((long long)range) : 0;
    const int shift = kb > kbits_cap ? kb - kbits_cap : 0;
    unsigned v = kmax_key;
    if (flag[i]) {
        const unsigned long long r = (key[i] - kmin) >> shift;
        v = r < kmax_key ? (unsigned)r : kmax_key - 1u;
    }
    k32[i] = v;
    vals[i] = (unsigned)i;
}

void depth_keys(long long n, const unsigned* flag, const unsigned long long* key, const Counters* ctr, int kbits_cap,
                unsigned* k32, unsigned* vals, cudaStream_t st) {
    if (n <= 0) return;
    k_depth_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, flag, key, ctr, kbits_cap, k32, vals);
}

// Restore exact order inside runs of equal reduced keys: insertion sort on
// (key64[src], src) -- runs are short in practice and already in src order.
// Keys >= skip_key (culled triangles) are left alone.
__global__ void k_fix_runs(long long m, const unsigned* __restrict__ k32, unsigned* __restrict__ vals,
                           const unsigned long long* __restrict__ key64, unsigned skip_key) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= m) return;
    unsigned k = k32[p];
    if (k >= skip_key) return;
    if (p > 0 && k32[p - 1] == k) return;
    if (p + 1 >= m || k32[p + 1] != k) return;
    long long end = p + 1;
    while (end < m && k32[end] == k) end++;
    for (long long i = p + 1; i < end; i++) {
        unsigned v = vals[i];
        unsigned long long kv = key64[v];
        long long j = i - 1;
        while (j >= p) {
            unsigned u = vals[j];
            unsigned long long ku = key64[u];
            if (ku < kv || (ku == kv && u < v)) break;
            vals[j + 1] = u;
            j--;
        }
        vals[j + 1] = v;
    }
}

void fix_depth_runs(long long m, const unsigned* k32, unsigned* vals, const unsigned long long* key64,
                    cudaStream_t st, unsigned skip_key) {
    if (m <= 1) return;
    k_fix_runs<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, k32, vals, key64, skip_key);
}


// ---------------------------------------------------------------------------
// exclusive scan of per-pixel int32 counts into int64 CSR offsets (P+1):
// per-block totals, one-block scan of the totals, block scan + offset.
// ---------------------------------------------------------------------------
constexpr int CS_T = 512, CS_PER = 8, CS_CHUNK = CS_T * CS_PER;

__device__ __forceinline__ long long cs_block_excl(long long v, long long* s_w, long long& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        long long w = lane < CS_T / 32 ? s_w[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < CS_T / 32) s_w[lane] = w;
    }
    __syncthreads();
    total = s_w[CS_T / 32 - 1];
    const long long before = warp ? s_w[warp - 1] : 0;
    __syncthreads();
    return before + x - v;
}

__global__ void __launch_bounds__(CS_T) k_cs_totals(long long n, const int* __restrict__ cnt, long long* __restrict__ bt) {
    __shared__ long long s_w[CS_T / 32];
    const long long base = (long long)blockIdx.x * CS_CHUNK + (long long)threadIdx.x * CS_PER;
    long long v = 0;
#pragma unroll
    for (int k = 0; k < CS_PER; k++)
        if (base + k < n) v += cnt[base + k];
    long long tot;
    cs_block_excl(v, s_w, tot);
    if (threadIdx.x == 0) bt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(CS_T) k_cs_scan_totals(long long nb, long long* __restrict__ bt) {
    __shared__ long long s_w[CS_T / 32];
    long long carry = 0;
    for (long long b0 = 0; b0 < nb; b0 += CS_T) {
        const long long i = b0 + threadIdx.x;
        const long long v = i < nb ? bt[i] : 0;
        long long tot;
        const long long ex = cs_block_excl(v, s_w, tot);
        if (i < nb) bt[i] = carry + ex;
        carry += tot;
    }
}

__global__ void __launch_bounds__(CS_T) k_cs_apply(long long n, const int* __restrict__ cnt, const long long* __restrict__ bt,
                                                   long long* __restrict__ off) {
    __shared__ long long s_w[CS_T / 32];
    const long long base = (long long)blockIdx.x * CS_CHUNK + (long long)threadIdx.x * CS_PER;
    int c[CS_PER];
    long long v = 0;
#pragma unroll
    for (int k = 0; k < CS_PER; k++) {
        c[k] = base + k < n ? cnt[base + k] : 0;
        v += c[k];
    }
    long long tot;
    long long run = bt[blockIdx.x] + cs_block_excl(v, s_w, tot);
#pragma unroll
    for (int k = 0; k < CS_PER; k++) {
        if (base + k < n) off[base + k] = run;
        run += c[k];
    }
    if (base < n && base + CS_PER >= n) off[n] = run;
}

size_t count_scan_scratch_bytes(long long n) { return sizeof(long long) * (size_t)((n + CS_CHUNK - 1) / CS_CHUNK + 1); }

void count_scan_i64(long long n, const int* cnt, long long* off, void* scratch, cudaStream_t st) {
    if (n <= 0) {
        cudaMemsetAsync(off, 0, sizeof(long long), st);
        return;
    }
    const long long nb = (n + CS_CHUNK - 1) / CS_CHUNK;
    long long* bt = (long long*)scratch;
    k_cs_totals<<<(unsigned)nb, CS_T, 0, st>>>(n, cnt, bt);
    k_cs_scan_totals<<<1, CS_T, 0, st>>>(nb, bt);
    k_cs_apply<<<(unsigned)nb, CS_T, 0, st>>>(n, cnt, bt, off);
}

__global__ void k_offsets_mismatch(long long n, const long long* __restrict__ a, const long long* __restrict__ b,
                                   unsigned long long* bad) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (long long)gridDim.x * blockDim.x)
        if (a[i] != b[i]) atomicAdd(bad, 1ull);
}

void offsets_mismatch(long long n, const long long* a, const long long* b, unsigned long long* bad, cudaStream_t st) {
    k_offsets_mismatch<<<592, 256, 0, st>>>(n, a, b, bad);
}

// ---------------- build_tile_lists for any tile size (render.py:315-361) ----------------
// Parity dump path: per-triangle tile counts, an int64 scan, (tile, rank) pairs
// emitted in rank order, a stable radix sort on the tile, then CSR offsets.
__global__ void k_tl_count(long long m, const long long* __restrict__ bbox, int ts, int* __restrict__ cnt) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const long long x0 = bbox[4 * i], x1 = bbox[4 * i + 1], y0 = bbox[4 * i + 2], y1 = bbox[4 * i + 3];
    if (x1 <= x0 || y1 <= y0) {
        cnt[i] = 0;
        return;
    }
    cnt[i] = (int)(((x1 - 1) / ts + 1 - x0 / ts) * ((y1 - 1) / ts + 1 - y0 / ts));
}

__global__ void k_tl_emit(long long m, const long long* __restrict__ bbox, int ts, int ntx,
                          const long long* __restrict__ off, unsigned* __restrict__ key, unsigned* __restrict__ val) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const long long x0 = bbox[4 * i], x1 = bbox[4 * i + 1], y0 = bbox[4 * i + 2], y1 = bbox[4 * i + 3];
    if (x1 <= x0 || y1 <= y0) return;
    long long pos = off[i];
    for (long long ty = y0 / ts; ty < (y1 - 1) / ts + 1; ty++)
        for (long long tx = x0 / ts; tx < (x1 - 1) / ts + 1; tx++) {
            key[pos] = (unsigned)(ty * ntx + tx);
            val[pos] = (unsigned)i;
            pos++;
        }
}

__global__ void k_tl_out(long long e, int ntiles, const unsigned* __restrict__ key, const unsigned* __restrict__ val,
                         long long* __restrict__ start, long long* __restrict__ entry) {
    const long long pos = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e <= 0) {
        if (pos <= ntiles) start[pos] = 0;
        return;
    }
    if (pos >= e) return;
    entry[pos] = (long long)val[pos];
    const int k = (int)key[pos];
    const int kp = pos > 0 ? (int)key[pos - 1] : -1;
    for (int t = kp + 1; t <= k; t++) start[t] = pos;
    if (pos == e - 1)
        for (int t = k + 1; t <= ntiles; t++) start[t] = e;
}

void tile_lists_count(long long m, const long long* bbox, int ts, int* cnt, long long* off, void* cs_scratch,
                      cudaStream_t st) {
    if (m > 0) k_tl_count<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, bbox, ts, cnt);
    count_scan_i64(m, cnt, off, cs_scratch, st);
}

void tile_lists_fill(long long m, long long e, const long long* bbox, int ts, int ntx, int ntiles,
                     const long long* off, unsigned* const kv[4], const SortScratch& s, long long* start,
                     long long* entry, cudaStream_t st) {
    if (m > 0 && e > 0) k_tl_emit<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, bbox, ts, ntx, off, kv[0], kv[1]);
    int bits = 1;
    while ((1ll << bits) < (long long)ntiles) bits++;
    const int alt = radix_sort_u32(e, kv[0], kv[1], kv[2], kv[3], 0, bits, s, st);
    const unsigned* key = alt ? kv[2] : kv[0];
    const unsigned* val = alt ? kv[3] : kv[1];
    const long long g = e > ntiles + 1 ? e : ntiles + 1;
    k_tl_out<<<(unsigned)((g + 255) / 256), 256, 0, st>>>(e, ntiles, key, val, start, entry);
}

}  // namespace ts
