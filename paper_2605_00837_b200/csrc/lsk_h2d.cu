// Host -> device staging of a cost matrix from pageable host memory (the
// reference's input: CostMatrix.values, an (n, m) float64 numpy array,
// types.py:60-86), with the one fp64 -> fp32 rounding of solver.py:253 done on
// the host while the previous chunk is in flight.
//
// A pageable cudaMemcpy is staged by the driver through its own pinned buffers
// by one thread (~10 GB/s) and moves 8 bytes per element. Here T worker
// threads each own two pinned row-chunk buffers and a stream: a worker rounds
// its rows to fp32 into the padded device layout (row stride ldd, zero tail),
// issues an async H2D of the chunk on its stream, and moves to its next chunk
// while the copy runs; a buffer is reused only after its previous copy's event
// completed. The caller's stream then waits on every worker stream, so the
// matrix is complete in stream order when the solve launches. Rounding on the
// CPU (cvtsd2ss, round-to-nearest-even, subnormals kept) is bit-identical to
// __double2float_rn.
#include <cuda_runtime.h>
#include <emmintrin.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lsk.h"

namespace lsk_host {
int32_t fail(int32_t code, const std::string& msg);
}

namespace {

// one row fp64 -> fp32 (round-to-nearest-even, as cvtsd2ss): 16-byte
// non-temporal stores into the pinned chunk (no read-for-ownership of the
// destination lines: ~1/4 less host memory traffic per call; the DMA reads the
// chunk after the worker's sfence). o must be 16-byte aligned.
void row_f64_to_f32_nt(const double* in, float* o, int m) {
  int j = 0;
  for (; j + 4 <= m; j += 4) {
    const __m128 lo = _mm_cvtpd_ps(_mm_loadu_pd(in + j));
    const __m128 hi = _mm_cvtpd_ps(_mm_loadu_pd(in + j + 2));
    _mm_stream_ps(o + j, _mm_movelh_ps(lo, hi));
  }
  for (; j < m; ++j) o[j] = static_cast<float>(in[j]);
}

struct Worker {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  float* buf[2] = {nullptr, nullptr};
  size_t cap = 0;  // floats per buffer
  bool used[2] = {false, false};
};

struct Pool {
  int device = -1;
  std::vector<Worker> w;
};
thread_local Pool t_pool;  // per caller thread: streams/events belong to a device context
std::mutex g_err_mu;

int32_t cfail(const char* what, cudaError_t e) {
  return lsk_host::fail(LSK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int32_t ensure(Pool& p, int dev, int T, size_t floats) {
  if (p.device != dev) {
    for (auto& w : p.w) {
      for (int k = 0; k < 2; ++k) {
        if (w.ev[k]) cudaEventDestroy(w.ev[k]);
        if (w.buf[k]) cudaFreeHost(w.buf[k]);
      }
      if (w.s) cudaStreamDestroy(w.s);
    }
    p.w.clear();
    p.device = dev;
  }
  while (int(p.w.size()) < T) {
    Worker w;
    cudaError_t e = cudaStreamCreateWithFlags(&w.s, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cfail("cudaStreamCreateWithFlags", e);
    for (int k = 0; k < 2; ++k) {
      e = cudaEventCreateWithFlags(&w.ev[k], cudaEventDisableTiming);
      if (e != cudaSuccess) return cfail("cudaEventCreate", e);
    }
    p.w.push_back(w);
  }
  for (int t = 0; t < T; ++t) {
    Worker& w = p.w[t];
    if (w.cap < floats) {
      for (int k = 0; k < 2; ++k) {
        if (w.used[k]) cudaEventSynchronize(w.ev[k]);
        if (w.buf[k]) cudaFreeHost(w.buf[k]);
        w.buf[k] = nullptr;
        w.used[k] = false;
        cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&w.buf[k]), floats * 4, cudaHostAllocPortable);
        if (e != cudaSuccess) return cfail("cudaHostAlloc", e);
      }
      w.cap = floats;
    }
  }
  return LSK_OK;
}

}  // namespace

extern "C" int32_t lsk_h2d_cost_f32(const void* src, int32_t src_is_f64, int64_t lds, int32_t n, int32_t m,
                                    float* dst, int64_t ldd, int32_t threads, void* stream) {
  if (!src || !dst) return lsk_host::fail(LSK_EINVAL, "null pointer");
  if (n < 1 || m < 1 || lds < m || ldd < m) return lsk_host::fail(LSK_EINVAL, "bad shape");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cfail("cudaGetDevice", e);
  const size_t row_bytes = size_t(ldd) * 4;
  // ~1 MB of fp32 per chunk: C2's 8192 x 8192 fp64 matrix stages in 8.5 ms vs 9.0 ms with
  // 4 MB and 12.3 ms with 16 MB chunks (tools/gpu_h2d.sh, 16 host cores; the pinned fp32
  // PCIe floor is 4.9 ms on that box); with the non-temporal stores 7.4 vs 8.2 ms on a box
  // whose floor is 6.05 ms. LSK_H2D_CHUNK_KB overrides it (experiments).
  size_t chunk_bytes = size_t(1) << 20;
  if (const char* v = getenv("LSK_H2D_CHUNK_KB")) chunk_bytes = std::max<size_t>(64, strtoull(v, nullptr, 10)) << 10;
  const int chunk_rows = int(std::max<size_t>(1, chunk_bytes / row_bytes));
  const int nchunks = (n + chunk_rows - 1) / chunk_rows;
  int T = threads > 0 ? threads : int(std::thread::hardware_concurrency());
  T = std::max(1, std::min({T, nchunks, 32}));
  Pool& p = t_pool;
  int32_t rc = ensure(p, dev, T, size_t(chunk_rows) * ldd);
  if (rc != LSK_OK) return rc;
  // the destination must not be written before prior work on `st` (e.g. a solve
  // still reading the previous matrix in the same buffer) is done
  cudaEvent_t start;
  e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  if (e != cudaSuccess) return cfail("cudaEventCreate", e);
  cudaEventRecord(start, st);
  for (int t = 0; t < T; ++t) cudaStreamWaitEvent(p.w[t].s, start, 0);
  // rows are 16-byte aligned in the pinned chunk when ldd % 4 == 0 (cudaHostAlloc is page aligned)
  const char* ntenv = getenv("LSK_H2D_NT");
  const bool nt = ldd % 4 == 0 && !(ntenv && ntenv[0] == '0');
  std::atomic<int> err{0};
  std::string err_msg;
  auto body = [&](int t) {
    Worker& w = p.w[t];
    int k = 0;
    for (int c = t; c < nchunks; c += T, k ^= 1) {
      if (w.used[k]) cudaEventSynchronize(w.ev[k]);
      const int r0 = c * chunk_rows, r1 = std::min(n, r0 + chunk_rows);
      float* out = w.buf[k];
      for (int r = r0; r < r1; ++r) {
        float* o = out + size_t(r - r0) * ldd;
        if (src_is_f64) {
          const double* in = static_cast<const double*>(src) + size_t(r) * lds;
          if (nt) row_f64_to_f32_nt(in, o, m);
          else
            for (int j = 0; j < m; ++j) o[j] = static_cast<float>(in[j]);
        } else {
          std::memcpy(o, static_cast<const float*>(src) + size_t(r) * lds, size_t(m) * 4);
        }
        for (int64_t j = m; j < ldd; ++j) o[j] = 0.f;
      }
      if (nt) _mm_sfence();
      cudaError_t ce = cudaMemcpyAsync(dst + size_t(r0) * ldd, out, size_t(r1 - r0) * row_bytes,
                                       cudaMemcpyHostToDevice, w.s);
      if (ce == cudaSuccess) ce = cudaEventRecord(w.ev[k], w.s);
      if (ce != cudaSuccess && !err.exchange(1)) {
        std::lock_guard<std::mutex> g(g_err_mu);
        err_msg = std::string("cudaMemcpyAsync: ") + cudaGetErrorString(ce);
      }
      w.used[k] = true;
    }
  };
  {
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back([&, t] {
      cudaSetDevice(dev);
      body(t);
    });
    body(0);
    for (auto& th : pool) th.join();
  }
  // the caller's stream waits for every worker's copies
  for (int t = 0; t < T; ++t) {
    Worker& w = p.w[t];
    cudaEvent_t done;
    cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    cudaEventRecord(done, w.s);
    cudaStreamWaitEvent(st, done, 0);
    cudaEventDestroy(done);
  }
  cudaEventDestroy(start);
  if (err.load()) return lsk_host::fail(LSK_ECUDA, err_msg);
  return LSK_OK;
}
