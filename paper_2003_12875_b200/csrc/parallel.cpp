#include "parallel.hpp"

#include <algorithm>
#include <cstdlib>

namespace ffb {

ThreadPool& ThreadPool::instance() {
  static ThreadPool* pool = [] {
    int n = static_cast<int>(std::thread::hardware_concurrency());
    if (const char* v = std::getenv("FFB_HOST_THREADS")) n = std::atoi(v);
    n = std::clamp(n, 1, 64);
    return new ThreadPool(n - 1);  // process lifetime; the caller is the n-th thread
  }();
  return *pool;
}

ThreadPool::ThreadPool(int nworkers) {
  for (int i = 0; i < nworkers; ++i) workers_.emplace_back([this] { run_worker(); });
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

void ThreadPool::drain() {
  // take indices until none are left (caller holds no lock)
  for (;;) {
    int i;
    const std::function<void(int)>* job;
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (!job_ || next_ >= n_) return;
      i = next_++;
      job = job_;
      ++active_;
    }
    try {
      (*job)(i);
    } catch (...) {
      std::lock_guard<std::mutex> lk(mu_);
      if (!error_ || i < error_index_) {  // the lowest index's error, as a serial loop raises
        error_ = std::current_exception();
        error_index_ = i;
      }
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      --active_;
      if (next_ >= n_ && active_ == 0) done_cv_.notify_all();
    }
  }
}

void ThreadPool::run_worker() {
  unsigned long long seen = 0;
  for (;;) {
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || generation_ != seen; });
      if (stop_) return;
      seen = generation_;
    }
    drain();
  }
}

void ThreadPool::parallel_for(int n, const std::function<void(int)>& f) {
  if (n <= 0) return;
  if (n == 1 || workers_.empty()) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::lock_guard<std::mutex> call(call_mu_);
  {
    std::lock_guard<std::mutex> lk(mu_);
    job_ = &f;
    n_ = n;
    next_ = 0;
    active_ = 0;
    error_ = nullptr;
    ++generation_;
  }
  cv_.notify_all();
  drain();
  std::exception_ptr err;
  {
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return next_ >= n_ && active_ == 0; });
    job_ = nullptr;
    err = error_;
    error_ = nullptr;
  }
  if (err) std::rethrow_exception(err);
}

}  // namespace ffb
