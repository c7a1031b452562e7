// loopback_group.h — shared state of t in-process ranks on one GPU (the
// loopback backend of comm.cu and the local peer backend of peer.cu).
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

namespace memo {

struct LoopbackGroup {
  explicit LoopbackGroup(int n) : size(n), send(n), ready(n), done(n) {
    for (int k = 0; k < n; ++k) {
      cudaEventCreateWithFlags(&ready[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming);
    }
  }
  ~LoopbackGroup() {
    for (int k = 0; k < size; ++k) {
      cudaEventDestroy(ready[k]);
      cudaEventDestroy(done[k]);
    }
    for (auto& kv : chan)
      for (cudaEvent_t e : kv.second) cudaEventDestroy(e);
    for (cudaEvent_t e : free_events) cudaEventDestroy(e);
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long gen = generation;
    if (++arrived == size) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
  int size;
  std::vector<const void*> send;
  std::vector<cudaEvent_t> ready, done;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long generation = 0;

  // ---- local peer backend: attached bases and (src, dst, channel) signal queues
  std::vector<char*> base = std::vector<char*>(8, nullptr);
  std::vector<size_t> bytes = std::vector<size_t>(8, 0);
  std::map<std::tuple<int, int, int>, std::deque<cudaEvent_t>> chan;
  std::vector<cudaEvent_t> free_events;
};

}  // namespace memo
