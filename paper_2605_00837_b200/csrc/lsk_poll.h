// Host-side early exit for the enqueue-only solve loops (lsk_points_solve.cu,
// lsk_dense_loop.cu): after each check the loop snapshots the device's
// per-problem active flags into pinned memory; once a completed snapshot shows
// every problem stopped, the host stops enqueueing (the kernels of a stopped
// problem would exit at once, but tens of thousands of empty launches still
// cost wall time). Never blocks the stream; disabled under stream capture.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <string>

#include "../../include/lsk.h"

namespace lsk_host {
int32_t fail(int32_t code, const std::string& msg);
}

namespace lsk_poll {

#define POLL_CUDA(expr)                                                                                \
  do {                                                                                                 \
    cudaError_t e__ = (expr);                                                                          \
    if (e__ != cudaSuccess) return lsk_host::fail(LSK_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

// Host poll of the device stop flags: a pinned ring of snapshots, one per
// check. The buffer and events are per host thread and reused across solves
// (freeing pinned memory would synchronise the device); a new solve first
// waits for the previous solve's snapshots, which completed long ago.
struct PollRing {
  static constexpr int kSlots = 4;
  int* host = nullptr;
  size_t cap = 0;  // ints per slot
  cudaEvent_t ev[kSlots] = {};
  int device = -1;
};
inline thread_local PollRing t_ring;

struct StopPoll {
  PollRing* r = nullptr;
  int B = 0, issued = 0, done = 0;
  int32_t init(int B_, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    POLL_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) return LSK_OK;  // no host interaction under capture
    int dev = 0;
    POLL_CUDA(cudaGetDevice(&dev));
    PollRing& g = t_ring;
    for (auto& e : g.ev)
      if (e) POLL_CUDA(cudaEventSynchronize(e));
    if (g.device != dev) {  // events belong to a device context
      for (auto& e : g.ev) {
        if (e) cudaEventDestroy(e);
        e = nullptr;
      }
      g.device = dev;
    }
    for (auto& e : g.ev)
      if (!e) POLL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (g.cap < size_t(B_)) {
      if (g.host) POLL_CUDA(cudaFreeHost(g.host));
      g.host = nullptr;
      POLL_CUDA(cudaHostAlloc(&g.host, size_t(PollRing::kSlots) * B_ * 4, cudaHostAllocPortable));
      g.cap = size_t(B_);
    }
    B = B_;
    r = &g;
    return LSK_OK;
  }
  // after a check: snapshot the active flags; all_stopped once a completed
  // snapshot shows every problem stopped. Blocks only when kSlots-1 snapshots
  // are in flight, which bounds the host's run-ahead of the device.
  int32_t after_check(const int* act_dev, cudaStream_t s, bool& all_stopped) {
    all_stopped = false;
    if (!r) return LSK_OK;
    if (issued - done >= PollRing::kSlots - 1) {
      POLL_CUDA(cudaEventSynchronize(r->ev[done % PollRing::kSlots]));
      if (read(done++)) { all_stopped = true; return LSK_OK; }
    }
    const int k = issued % PollRing::kSlots;
    POLL_CUDA(cudaMemcpyAsync(r->host + size_t(k) * r->cap, act_dev, size_t(B) * 4, cudaMemcpyDeviceToHost, s));
    POLL_CUDA(cudaEventRecord(r->ev[k], s));
    ++issued;
    while (done < issued && cudaEventQuery(r->ev[done % PollRing::kSlots]) == cudaSuccess)
      if (read(done++)) { all_stopped = true; return LSK_OK; }
    return LSK_OK;
  }
  bool read(int i) const {
    const int* h = r->host + size_t(i % PollRing::kSlots) * r->cap;
    for (int b = 0; b < B; ++b)
      if (h[b]) return false;
    return true;
  }
};

}  // namespace lsk_poll
