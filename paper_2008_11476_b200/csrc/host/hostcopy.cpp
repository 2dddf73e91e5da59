#include "hostcopy.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#if defined(__x86_64__)
#include <emmintrin.h>
#endif

namespace gvx::dev {

namespace {

/// memcpy with non-temporal stores for the 16-byte-aligned body.
void stream_copy(char* d, const char* s, std::size_t n) {
#if defined(__x86_64__)
    const std::size_t head = std::min(n, static_cast<std::size_t>((16 - (reinterpret_cast<std::uintptr_t>(d) & 15)) & 15));
    std::memcpy(d, s, head);
    d += head, s += head, n -= head;
    const std::size_t body = n & ~static_cast<std::size_t>(63);
    for (std::size_t i = 0; i < body; i += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
        const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
    }
    std::memcpy(d + body, s + body, n - body);
    _mm_sfence();
#else
    std::memcpy(d, s, n);
#endif
}

class CopyPool {
public:
    explicit CopyPool(int workers) {
        for (int i = 0; i < workers; ++i) threads_.emplace_back([this] { work(); });
    }
    int lanes() const { return static_cast<int>(threads_.size()) + 1; }

    void copy(char* dst, const char* src, std::size_t n, bool streaming) {
        std::unique_lock<std::mutex> call(call_mu_); // one job at a time
        std::unique_lock<std::mutex> l(mu_);
        streaming_ = streaming;
        dst_ = dst;
        src_ = src;
        n_ = n;
        parts_ = lanes();
        next_ = 0;
        remaining_ = parts_;
        ++gen_;
        cv_.notify_all();
        run_parts(l);
        done_.wait(l, [&] { return remaining_ == 0; });
    }

private:
    void run_parts(std::unique_lock<std::mutex>& l) {
        while (next_ < parts_) {
            const int p = next_++;
            const std::size_t per = (n_ + static_cast<std::size_t>(parts_) - 1) / static_cast<std::size_t>(parts_);
            const std::size_t a = std::min(n_, per * static_cast<std::size_t>(p));
            const std::size_t b = std::min(n_, a + per);
            char* d = dst_;
            const char* s = src_;
            const bool nt = streaming_;
            l.unlock();
            if (b > a) {
                if (nt) stream_copy(d + a, s + a, b - a);
                else std::memcpy(d + a, s + a, b - a);
            }
            l.lock();
            if (--remaining_ == 0) done_.notify_all();
        }
    }
    void work() {
        unsigned long long seen = 0;
        std::unique_lock<std::mutex> l(mu_);
        while (true) {
            cv_.wait(l, [&] { return gen_ != seen; });
            seen = gen_;
            run_parts(l);
        }
    }

    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_;
    std::vector<std::thread> threads_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    std::size_t n_ = 0;
    int parts_ = 0, next_ = 0, remaining_ = 0;
    bool streaming_ = false;
    unsigned long long gen_ = 0;
};

CopyPool& pool() {
    // leaked on purpose: worker threads never join at process exit
    static CopyPool* p = [] {
        const unsigned hw = std::thread::hardware_concurrency();
        const int workers = static_cast<int>(std::clamp(hw / 2u, 1u, 8u)) - 1;
        return new CopyPool(workers);
    }();
    return *p;
}

} // namespace

void parallel_copy(void* dst, const void* src, std::size_t n, bool streaming) {
    static const std::size_t min_bytes = [] {
        const char* e = std::getenv("GVX_COPY_MIN_KB"); // tuning experiments
        return static_cast<std::size_t>(e ? std::atoi(e) : 256) << 10; // pooled from 256 KB: 1080p run_plan 0.63 -> 0.32 ms
    }();
    if (n < min_bytes || pool().lanes() == 1) {
        if (streaming) stream_copy(static_cast<char*>(dst), static_cast<const char*>(src), n);
        else std::memcpy(dst, src, n);
        return;
    }
    pool().copy(static_cast<char*>(dst), static_cast<const char*>(src), n, streaming);
}

} // namespace gvx::dev
