// host_pool.h — a small persistent pool of host threads for parallel host
// copies (zsvd_api.cu: pageable rows into pinned bounce buffers).
#pragma once

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace zsvd {

class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool* pool = new CopyPool();  // never destroyed: its workers are detached
        return *pool;
    }
    // Runs fn(0 .. parts-1) on the workers and the calling thread; returns when done.
    void run(int parts, const std::function<void(int)>& fn) {
        std::unique_lock<std::mutex> lk(mu_);
        job_ = &fn;
        parts_ = parts;
        next_ = 0;
        pending_ = parts;
        ++gen_;
        cv_.notify_all();
        lk.unlock();
        work();
        lk.lock();
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }
    int threads() const { return (int)th_.size() + 1; }

private:
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        const int n = (int)std::max(1u, std::min(11u, hw > 2 ? hw - 2 : 1u));
        for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
        for (auto& t : th_) t.detach();  // process-lifetime workers
    }
    void work() {
        for (;;) {
            int i;
            const std::function<void(int)>* f;
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (!job_ || next_ >= parts_) return;
                i = next_++;
                f = job_;
            }
            (*f)(i);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen && job_ && next_ < parts_; });
                seen = gen_;
            }
            work();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<std::thread> th_;
    const std::function<void(int)>* job_ = nullptr;
    int parts_ = 0, next_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
};


}  // namespace zsvd
