// ts_host.cpp -- host side of the drop-in upload (render() with the reference's
// fp64 soup): fp64 -> fp32 conversion into the caller's page-locked staging
// chunk on a small persistent pool of host threads, with the exactness test of
// every value.  A soup whose values are all fp32 values (the reference's
// synthetic scenes round every parameter to fp32) then crosses PCIe
// at half the bytes and renders through the fp32-parameter kernels with the
// very same values.  Compiled by the host compiler (g++ -O3): AVX2 conversion
// with streaming stores where the CPU has it, scalar otherwise.
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include <map>

#include "trisplat_b200.h"

namespace {

class HostPool {
  public:
    explicit HostPool(int n) {
        for (int i = 0; i < n; i++) th_.emplace_back([this, i] { loop(i + 1); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return (int)th_.size() + 1; }
    // f(part) for part in [0, parts), parts <= size(); part 0 on the calling thread
    void run(int parts, const std::function<void(int)>& f) {
        std::lock_guard<std::mutex> call(call_m_);
        {
            std::lock_guard<std::mutex> g(m_);
            f_ = &f;
            parts_ = parts;
            pending_ = parts - 1;
            gen_++;
        }
        cv_.notify_all();
        f(0);
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [this] { return pending_ == 0; });
        f_ = nullptr;
    }

  private:
    void loop(int id) {
        unsigned long long seen = 0;
        for (;;) {
            const std::function<void(int)>* f;
            int parts;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                f = f_;
                parts = parts_;
            }
            if (id < parts) {
                (*f)(id);
                std::lock_guard<std::mutex> g(m_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_, call_m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* f_ = nullptr;
    int parts_ = 0, pending_ = 0;
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

HostPool& host_pool() {
    static HostPool pool(std::max(0, std::min<int>((int)std::thread::hardware_concurrency(), 16) - 1));
    return pool;
}

int pack_scalar(const double* __restrict__ s, float* __restrict__ d, int64_t n) {
    int ok = 1;
    for (int64_t i = 0; i < n; i++) {
        const float f = (float)s[i];
        d[i] = f;
        ok &= (double)f == s[i];  // (NaN != NaN: a non-finite value is not "exact")
    }
    return ok;
}

// 8 values per step; streaming (non-temporal) stores: the staging chunk is read
// next by the DMA engine, not by this core
template <bool STREAM>
__attribute__((target("avx2"))) int pack_avx2(const double* __restrict__ s, float* __restrict__ d, int64_t n) {
    int64_t i = 0;
    int ok = 1;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); i++) {
        const float f = (float)s[i];
        d[i] = f;
        ok &= (double)f == s[i];
    }
    __m256d all = _mm256_castsi256_pd(_mm256_set1_epi64x(-1));
    for (; i + 8 <= n; i += 8) {
        const __m256d a = _mm256_loadu_pd(s + i), b = _mm256_loadu_pd(s + i + 4);
        const __m128 fa = _mm256_cvtpd_ps(a), fb = _mm256_cvtpd_ps(b);
        if constexpr (STREAM)
            _mm256_stream_ps(d + i, _mm256_set_m128(fb, fa));
        else
            _mm256_store_ps(d + i, _mm256_set_m128(fb, fa));
        const __m256d ea = _mm256_cmp_pd(_mm256_cvtps_pd(fa), a, _CMP_EQ_OQ);
        const __m256d eb = _mm256_cmp_pd(_mm256_cvtps_pd(fb), b, _CMP_EQ_OQ);
        all = _mm256_and_pd(all, _mm256_and_pd(ea, eb));
    }
    if constexpr (STREAM) _mm_sfence();
    ok &= _mm256_movemask_pd(all) == 0xF;
    for (; i < n; i++) {
        const float f = (float)s[i];
        d[i] = f;
        ok &= (double)f == s[i];
    }
    return ok;
}

}  // namespace

extern "C" int ts_pack_f32(const double* src, float* dst, int64_t n, int threads) {
    if (n < 0 || (n > 0 && (!src || !dst))) return TS_ERR_INVALID_ARG;
    static const bool avx2 = __builtin_cpu_supports("avx2");
    HostPool& pool = host_pool();
    int parts = threads > 0 ? std::min(threads, pool.size()) : pool.size();
    if (n < (1 << 16)) parts = 1;
    std::atomic<int> exact{1};
    // slices in whole 64-byte lines of the output
    const int64_t per = ((n + parts - 1) / parts + 15) / 16 * 16;
    pool.run(parts, [&](int k) {
        const int64_t lo = std::min<int64_t>(n, k * per), hi = std::min<int64_t>(n, lo + per);
        const int ok = avx2 ? pack_avx2<true>(src + lo, dst + lo, hi - lo) : pack_scalar(src + lo, dst + lo, hi - lo);
        if (!ok) exact.store(0, std::memory_order_relaxed);
    });
    return exact.load();
}

// ---------------------------------------------------------------------------
// Whole upload in one call: chunks of the fp64 array are converted into a small
// ring of page-locked slots (small enough to stay in the host's last-level cache
// between the conversion and the DMA that reads it) and copied to dst on
// `stream`; the conversion of chunk i+1 overlaps the DMA of chunk i.  Returns 1
// when every value was an fp32 value (dst complete once the stream reaches the
// copies), 0 when one was not (the copies issued so far have finished; dst is
// incomplete), < 0 on a CUDA error.
// ---------------------------------------------------------------------------
namespace {
struct UploadRing {
    std::vector<float*> slot;
    std::vector<cudaEvent_t> ev;
    int64_t slot_floats = 0;
};
std::mutex g_ring_m;
std::map<int, UploadRing> g_rings;  // per device

int ring_for(int dev, int64_t slot_floats, int nslot, UploadRing** out) {
    UploadRing& r = g_rings[dev];
    if (r.slot_floats != slot_floats || (int)r.slot.size() != nslot) {
        for (size_t k = 0; k < r.slot.size(); k++) {
            cudaEventSynchronize(r.ev[k]);
            cudaEventDestroy(r.ev[k]);
            cudaFreeHost(r.slot[k]);
        }
        r.slot.assign(nslot, nullptr);
        r.ev.assign(nslot, nullptr);
        r.slot_floats = slot_floats;
        for (int k = 0; k < nslot; k++) {
            if (cudaHostAlloc((void**)&r.slot[k], sizeof(float) * slot_floats, cudaHostAllocPortable) != cudaSuccess ||
                cudaEventCreateWithFlags(&r.ev[k], cudaEventDisableTiming) != cudaSuccess) {
                r.slot_floats = 0;
                return TS_ERR_OOM;
            }
        }
    }
    *out = &r;
    return TS_OK;
}
}  // namespace

extern "C" int ts_upload_f32(const double* src, int64_t n, float* dst, void* stream, int64_t chunk_bytes,
                             int nslot, int flags) {
    if (n < 0 || (n > 0 && (!src || !dst))) return TS_ERR_INVALID_ARG;
    if (n == 0) return 1;
    const int64_t cb = chunk_bytes > 0 ? chunk_bytes : (4ll << 20);
    const int64_t step = std::max<int64_t>(1024, cb / 4 / 64 * 64);
    nslot = nslot > 1 ? nslot : 4;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TS_ERR_CUDA;
    std::lock_guard<std::mutex> lock(g_ring_m);
    UploadRing* r = nullptr;
    int rc = ring_for(dev, step, nslot, &r);
    if (rc) return rc;
    HostPool& pool = host_pool();
    static const bool avx2 = __builtin_cpu_supports("avx2");
    const bool stream_stores = (flags & 1) != 0;
    cudaStream_t st = (cudaStream_t)stream;
    int exact = 1;
    int64_t i = 0;
    for (int64_t off = 0; off < n; off += step, i++) {
        const int k = (int)(i % nslot);
        const int64_t c = std::min(step, n - off);
        if (cudaEventSynchronize(r->ev[k]) != cudaSuccess) return TS_ERR_CUDA;  // the slot's last DMA is done
        float* slot = r->slot[k];
        const int parts = c < (1 << 16) ? 1 : pool.size();
        const int64_t per = ((c + parts - 1) / parts + 15) / 16 * 16;
        std::atomic<int> ok{1};
        pool.run(parts, [&](int p) {
            const int64_t lo = std::min<int64_t>(c, p * per), hi = std::min<int64_t>(c, lo + per);
            int good;
            if (!avx2)
                good = pack_scalar(src + off + lo, slot + lo, hi - lo);
            else if (stream_stores)
                good = pack_avx2<true>(src + off + lo, slot + lo, hi - lo);
            else
                good = pack_avx2<false>(src + off + lo, slot + lo, hi - lo);
            if (!good) ok.store(0, std::memory_order_relaxed);
        });
        if (!ok.load()) {
            exact = 0;
            break;
        }
        if (cudaMemcpyAsync(dst + off, slot, sizeof(float) * c, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaEventRecord(r->ev[k], st) != cudaSuccess)
            return TS_ERR_CUDA;
    }
    if (!exact && cudaStreamSynchronize(st) != cudaSuccess) return TS_ERR_CUDA;
    return exact;
}
