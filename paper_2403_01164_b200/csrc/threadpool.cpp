// threadpool.cpp -- persistent host-thread pool for the CPU lane.
//
// The paper runs its CPU share "using multithreading" with at most 16
// cores.  Here the pool is persistent (created with the context), each
// worker optionally pinned to one core, and a dispatch is a generation-counter
// bump: workers spin briefly (microsecond wake-up between linears) and then
// sleep on a futex so an idle library does not burn the host.
#include <linux/futex.h>
#include <pthread.h>
#include <sched.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <thread>
#include <vector>

#include "hg_internal.h"

namespace hg {

class ThreadPool {
   public:
    ThreadPool(int n, int first_core) : n_(n < 1 ? 1 : n) {
        for (int i = 1; i < n_; ++i) {
            threads_.emplace_back([this, i, first_core] {
                if (first_core >= 0) pin(first_core + i);
                loop(i);
            });
        }
    }
    ThreadPool(int n, const std::vector<int> &cpus) : n_(n < 1 ? 1 : n) {
        for (int i = 1; i < n_; ++i) {
            const int core = cpus.empty() ? -1 : cpus[(size_t)i % cpus.size()];
            threads_.emplace_back([this, i, core] {
                if (core >= 0) pin(core);
                loop(i);
            });
        }
    }
    ~ThreadPool() {
        stop_.store(true, std::memory_order_release);
        gen_.fetch_add(1, std::memory_order_acq_rel);
        futex_wake();
        for (auto &t : threads_) t.join();
    }
    int size() const { return n_; }

    // Start fn(arg, i) on workers 1..n-1 and return at once (the caller may enqueue GPU
    // work meanwhile); join() then runs fn(arg, 0) on the caller and waits for all.
    void post(void (*fn)(void *, int), void *arg) {
        fn_ = fn;
        arg_ = arg;
        done_.store(0, std::memory_order_relaxed);
        gen_.fetch_add(1, std::memory_order_acq_rel);
        if (sleepers_.load(std::memory_order_acquire) > 0) futex_wake();
    }
    void join() {
        fn_(arg_, 0);
        while (done_.load(std::memory_order_acquire) != n_ - 1) _mm_pause();
    }
    void run(void (*fn)(void *, int), void *arg) {
        post(fn, arg);
        join();
    }

   private:
    static void pin(int core) {
        int ncpu = (int)sysconf(_SC_NPROCESSORS_ONLN);
        if (ncpu <= 0) return;
        cpu_set_t set;
        CPU_ZERO(&set);
        CPU_SET(core % ncpu, &set);
        pthread_setaffinity_np(pthread_self(), sizeof set, &set);
    }
    void futex_wake() {
        syscall(SYS_futex, reinterpret_cast<uint32_t *>(&gen_), FUTEX_WAKE_PRIVATE, INT32_MAX, 0,
                0, 0);
    }
    void loop(int idx) {
        uint32_t seen = 0;  // generation at construction: a job posted before this thread ran is not missed
        for (;;) {
            // spin ~2 ms, then sleep until the generation changes
            auto t0 = std::chrono::steady_clock::now();
            uint32_t g;
            int spins = 0;
            while ((g = gen_.load(std::memory_order_acquire)) == seen) {
                _mm_pause();
                if (++spins == 4096) {
                    spins = 0;
                    if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(2)) {
                        sleepers_.fetch_add(1, std::memory_order_acq_rel);
                        if (gen_.load(std::memory_order_acquire) == seen)
                            syscall(SYS_futex, reinterpret_cast<uint32_t *>(&gen_),
                                    FUTEX_WAIT_PRIVATE, seen, 0, 0, 0);
                        sleepers_.fetch_sub(1, std::memory_order_acq_rel);
                        t0 = std::chrono::steady_clock::now();
                    }
                }
            }
            seen = g;
            if (stop_.load(std::memory_order_acquire)) return;
            fn_(arg_, idx);
            done_.fetch_add(1, std::memory_order_acq_rel);
        }
    }

    int n_;
    std::vector<std::thread> threads_;
    std::atomic<uint32_t> gen_{0};
    std::atomic<int> done_{0};
    std::atomic<int> sleepers_{0};
    std::atomic<bool> stop_{false};
    void (*fn_)(void *, int) = nullptr;
    void *arg_ = nullptr;
};

static_assert(sizeof(std::atomic<uint32_t>) == 4, "futex word");

ThreadPool *pool_create(int nthreads, int first_core) { return new ThreadPool(nthreads, first_core); }
ThreadPool *pool_create_cpus(int nthreads, const std::vector<int> &cpus) { return new ThreadPool(nthreads, cpus); }
void pool_destroy(ThreadPool *p) { delete p; }
int pool_size(const ThreadPool *p) { return p->size(); }
void pool_run(ThreadPool *p, void (*fn)(void *, int), void *arg) { p->run(fn, arg); }
void pool_post(ThreadPool *p, void (*fn)(void *, int), void *arg) { p->post(fn, arg); }
void pool_join(ThreadPool *p) { p->join(); }

}  // namespace hg
