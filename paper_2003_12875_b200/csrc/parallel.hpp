// A small persistent host thread pool for the per-point host work of a launch (the
// constant rows: normalisation integrals, which for Simpson-normalised pdfs -- ChiSquare,
// JohnsonSU, Expression -- cost ~70 us each, i.e. 14 ms for a 200-point launch on one
// thread while the kernel itself takes ~8 ms).
#pragma once

#include <condition_variable>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace ffb {

class ThreadPool {
 public:
  static ThreadPool& instance();

  // Runs f(i) for i in [0, n) on the pool and the calling thread; after all calls
  // finished, rethrows the exception of the lowest index that raised one (what a serial
  // loop would have raised first).
  void parallel_for(int n, const std::function<void(int)>& f);
  int size() const { return static_cast<int>(workers_.size()) + 1; }

 private:
  explicit ThreadPool(int nworkers);
  ~ThreadPool();
  void run_worker();
  void drain();

  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0, next_ = 0, active_ = 0;
  unsigned long long generation_ = 0;
  bool stop_ = false;
  std::exception_ptr error_;
  int error_index_ = 0;
  std::mutex call_mu_;  // one parallel_for at a time
};

}  // namespace ffb
