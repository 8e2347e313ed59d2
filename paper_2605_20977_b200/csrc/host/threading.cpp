// pswa/threading.h: a persistent worker pool (the reference spawns and joins
// threads on every parallel_for call, proj/src/threading.cpp:45-72). Work is
// handed out in dynamic index chunks; each index runs exactly once, so the
// bytes written do not depend on the worker count or the schedule.
#include "pswa/threading.h"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace pswa {
namespace {

// set on pool threads (and the caller while it runs a loop): a parallel_for
// nested inside fn runs serially on that thread instead of deadlocking
thread_local bool in_pool = false;

class Pool {
 public:
  ~Pool() { resize(0); }

  void resize(int helpers) {
    std::unique_lock<std::mutex> lk(m_);
    if (static_cast<int>(threads_.size()) == helpers) return;
    stop_ = true;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    for (auto& t : threads_) t.join();
    lk.lock();
    threads_.clear();
    stop_ = false;
    // a helper starts from the generation current at its creation, so a run
    // published before it first takes the lock is not missed
    for (int i = 0; i < helpers; ++i) threads_.emplace_back([this, g = gen_] { loop(g); });
  }

  void run(int helpers, int64_t begin, int64_t end, int64_t chunk,
           const std::function<void(int64_t)>* fn) {
    std::unique_lock<std::mutex> run_lk(run_m_);  // one parallel_for at a time
    resize(helpers);
    in_pool = true;
    struct Reset {
      ~Reset() { in_pool = false; }
    } reset;
    {
      std::lock_guard<std::mutex> lk(m_);
      next_.store(begin);
      end_ = end;
      chunk_ = chunk;
      fn_ = fn;
      active_ = static_cast<int>(threads_.size());
      ++gen_;
    }
    cv_.notify_all();
    work();  // the calling thread is worker 0
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [&] { return active_ == 0; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      const int64_t i0 = next_.fetch_add(chunk_);
      if (i0 >= end_) return;
      const int64_t i1 = std::min(end_, i0 + chunk_);
      for (int64_t i = i0; i < i1; ++i) (*fn_)(i);
    }
  }
  void loop(uint64_t seen) {
    in_pool = true;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      work();
      std::lock_guard<std::mutex> lk(m_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }

  std::mutex m_, run_m_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> threads_;
  std::atomic<int64_t> next_{0};
  int64_t end_ = 0, chunk_ = 1;
  const std::function<void(int64_t)>* fn_ = nullptr;
  int active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

std::atomic<int> g_workers{0};

Pool& pool() {
  static Pool* p = new Pool();  // never destroyed: helpers may outlive static destructors
  return *p;
}

int default_workers() {
  if (const char* env = std::getenv("PSWA_THREADS")) {
    const int n = std::atoi(env);
    if (n >= 1) return n;
  }
  return 1;
}

}  // namespace

void set_workers(int n) { g_workers.store(n >= 1 ? n : 1); }

int workers() {
  int w = g_workers.load();
  if (w == 0) {
    w = default_workers();
    g_workers.store(w);
  }
  return w;
}

void parallel_for(int64_t begin, int64_t end, const std::function<void(int64_t)>& fn) {
  const int64_t n = end - begin;
  if (n <= 0) return;
  int w = workers();
  if (w == 1 || n == 1 || in_pool) {
    for (int64_t i = begin; i < end; ++i) fn(i);
    return;
  }
  if (static_cast<int64_t>(w) > n) w = static_cast<int>(n);
  pool().run(workers() - 1, begin, end, std::max<int64_t>(1, n / (static_cast<int64_t>(w) * 8)), &fn);
}

}  // namespace pswa
