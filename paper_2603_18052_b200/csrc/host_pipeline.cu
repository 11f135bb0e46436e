// host_pipeline.cu — the end-to-end host-buffer evolve shared by
// lbg_evolve_shared_p and lbg_evolve_density (include/lbg.h): rho0 and out are
// the caller's HOST buffers, like lb::evolve's MatrixAoS arguments
// (proj/src/propagate.cpp:75-109; storage proj/include/lb/complex_matrix.hpp:15-31).
//
// Pipeline over chunks of the batch (sizes ramp 1, 2, 4, ..., 4, 2, 1 so only a
// small first H2D and a small last D2H are exposed):
//   stream H : H2D of chunk c;
//   stream K (highest priority): the rho0 validation (K6) of chunk c after its
//              H2D, and a 24-byte D2H of its result into pinned memory;
//   stream C0/C1 (alternating chunks, so one chunk's kernel tail overlaps the
//              next chunk's start): the steps of chunk c (in place), after its
//              H2D AND its validation (which reads the same buffer);
//   stream D : D2H of chunk c after its steps.
// Validation before output (propagate.cpp:79-80 throws before any work): the
// host waits for the validation of EVERY chunk (stream H only carries copies
// and the tiny check kernels, so this completes long before the stepping) and
// issues the D2H copies only when all of rho0 passed; on failure `out` is left
// untouched. The stepping already queued is drained (streams synchronised)
// before the error returns, so the pooled buffers are never reused while a
// kernel may still run — also on any other exception.
//
// Pageable caller buffers (lb::MatrixAoS is an aligned_vector, not pinned):
// cudaMemcpyAsync from / to pageable memory blocks the host, which would
// serialise the pipeline. Such buffers are staged through pinned buffers kept in
// the pool: a persistent pool of host threads copies chunk c of rho0 into
// pinned memory (while the GPU works on earlier chunks) before its H2D, and
// copies chunk c of the result out of pinned memory as soon as its D2H has
// landed (while later chunks still compute / copy). Pinned caller buffers
// (cudaHostAlloc / cudaHostRegister) are used directly.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace lbg {
namespace {

// Device buffers and streams reused across calls (grown on demand), so the
// end-to-end call pays no cudaMalloc / cudaFree / cudaHostAlloc per call.
struct Grow {
  void* ptr = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (ptr) check_cuda(cudaFree(ptr), "cudaFree");
    ptr = nullptr;
    check_cuda(cudaMalloc(&ptr, bytes), "cudaMalloc");
    cap = bytes;
  }
};
struct PinnedGrow {
  void* ptr = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (ptr) check_cuda(cudaFreeHost(ptr), "cudaFreeHost");
    ptr = nullptr;
    check_cuda(cudaHostAlloc(&ptr, bytes, cudaHostAllocDefault), "cudaHostAlloc");
    cap = bytes;
  }
};
constexpr int kMaxChunks = 16;
struct EvolvePool {
  std::mutex mu;
  Grow p, x, chk, w[2];
  PinnedGrow pin_in, pin_out, pin_chk;
  cudaStream_t st[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // H, C0, C1, D, K (checks)
  cudaEvent_t ev_x[kMaxChunks] = {}, ev_h[kMaxChunks] = {}, ev_c[kMaxChunks] = {}, ev_d[kMaxChunks] = {},
              ev_chk = nullptr;
  void ensure(size_t pb, size_t xb, size_t cb, size_t wb) {
    if (!st[0]) {
      for (int i = 0; i < 4; ++i) check_cuda(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking), "stream");
      // the rho0 checks run at the highest priority: their few blocks take the
      // next free SM slots ahead of the stepping kernels, so the validation of
      // every chunk completes early and the D2H copies overlap the stepping
      int lo = 0, hi = 0;
      check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
      check_cuda(cudaStreamCreateWithPriority(&st[4], cudaStreamNonBlocking, hi), "stream");
      for (int i = 0; i < kMaxChunks; ++i)
        for (cudaEvent_t* e : {&ev_x[i], &ev_h[i], &ev_c[i], &ev_d[i]})
          check_cuda(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
      check_cuda(cudaEventCreateWithFlags(&ev_chk, cudaEventDisableTiming), "event");
    }
    p.ensure(pb);
    x.ensure(xb);
    chk.ensure(cb);
    pin_chk.ensure(cb);
    w[0].ensure(wb);
    w[1].ensure(wb);
  }
  void drain() {  // error path: nothing may still run on the pooled buffers
    for (auto& s : st)
      if (s) (void)cudaStreamSynchronize(s);
    (void)cudaGetLastError();
  }
};
EvolvePool& evolve_pool() {  // one per device (buffers and streams belong to it)
  static std::mutex mu;
  static std::map<int, EvolvePool*>* pools = new std::map<int, EvolvePool*>;  // leaked: outlives CUDA teardown
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  EvolvePool*& p = (*pools)[dev];
  if (!p) p = new EvolvePool;
  return *p;
}

// Persistent host threads for the pageable <-> pinned staging copies (one
// memcpy thread moves ~5-10 GB/s; the calling thread takes a slice too).
// Hand-off by atomics with spinning: a worker that finished a slice polls for
// the next one for up to kSpin before it sleeps on the condition variable, and
// the caller polls the pending count — a condition-variable wake-up costs
// 0.05-0.3 ms on the GPU box, and a host-buffer call hands out ~20 copies.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* pool = new CopyPool;  // leaked: workers outlive static destruction
    return *pool;
  }
  void copy(void* dst, const void* src, size_t bytes) {
    if (bytes < (size_t(1) << 20) || workers_.empty()) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> one(call_mu_);  // one parallel copy at a time
    const size_t parts = workers_.size() + 1;
    size_t slice = (bytes + parts - 1) / parts;
    slice = (slice + 63) & ~size_t(63);
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    bytes_ = bytes;
    slice_ = slice;
    pending_.store(int(workers_.size()), std::memory_order_relaxed);
    gen_.fetch_add(1, std::memory_order_release);  // publishes the fields above
    { std::lock_guard<std::mutex> lk(mu_); }        // no lost wake-up for a worker about to sleep
    cv_.notify_all();
    copy_part(0);  // the caller's own slice
    while (pending_.load(std::memory_order_acquire) != 0) pause();
  }

 private:
  static constexpr std::chrono::microseconds kSpin{3000};
  static void pause() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned n = std::min(11u, hw > 1 ? hw - 1 : 0u);
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this, i] { run(int(i) + 1); });
    for (auto& t : workers_) t.detach();
  }
  void copy_part(int part) {
    const size_t b0 = std::min(bytes_, size_t(part) * slice_), b1 = std::min(bytes_, b0 + slice_);
    if (b1 > b0) std::memcpy(dst_ + b0, src_ + b0, b1 - b0);
  }
  void run(int part) {
    unsigned seen = 0;
    while (true) {
      const auto t0 = std::chrono::steady_clock::now();
      while (gen_.load(std::memory_order_acquire) == seen &&
             std::chrono::steady_clock::now() - t0 < kSpin)
        pause();
      if (gen_.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
      }
      seen = gen_.load(std::memory_order_acquire);
      copy_part(part);
      pending_.fetch_sub(1, std::memory_order_release);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0, slice_ = 0;
  std::atomic<int> pending_{0};
  std::atomic<unsigned> gen_{0};
};

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace

void host_evolve(const double* p, size_t d, const double* rho0, int64_t batch, double* out, bool single,
                 const ChunkWork& work_bytes, const ChunkStep& step) {
  if (d == 0) throw invalid_argument("evolve: state dimension must be positive");
  if (batch < 0) throw invalid_argument("evolve: negative batch or steps");
  if (batch == 0) return;
  if (!p || !rho0 || !out) throw invalid_argument("evolve: null pointer");
  const size_t n = d * d;
  const int64_t min_chunk = 32768;
  // measured at c1 (ms per call), equal chunks: 4 -> 21.1, 8 -> 20.4, 16 -> 21.6-27 (+ outliers); one
  // compute stream instead of two: 21.2 at 8 (kernel tails no longer overlap). Chunk sizes ramp
  // 1, 2, 4, ..., 4, 2, 1 (10 chunks) so only a small first H2D and a small last D2H are exposed:
  // 20.19 vs 20.48 ms for 8 equal chunks in the same run (1, 2, 4, 8 ramp over 12: no better).
  constexpr int64_t max_chunks = 10;
  static_assert(max_chunks <= kMaxChunks, "events per chunk");
  const int nchunks = (single || batch < 2 * min_chunk) ? 1 : int(std::min<int64_t>(max_chunks, batch / min_chunk));
  int64_t bounds[kMaxChunks + 1];
  {
    int64_t wsum = 0, wts[kMaxChunks];
    for (int c = 0; c < nchunks; ++c) {
      wts[c] = int64_t(1) << std::min(std::min(c, nchunks - 1 - c), 2);
      wsum += wts[c];
    }
    int64_t acc = 0;
    bounds[0] = 0;
    for (int c = 0; c < nchunks; ++c) {
      acc += wts[c];
      bounds[c + 1] = batch * acc / wsum;
    }
  }
  int64_t chunk = 0;
  for (int c = 0; c < nchunks; ++c) chunk = std::max(chunk, bounds[c + 1] - bounds[c]);
  const size_t total = size_t(batch) * n * 16;
  const bool in_pinned = is_pinned(rho0), out_pinned = is_pinned(out);
  EvolvePool& pool = evolve_pool();
  std::lock_guard<std::mutex> lk(pool.mu);
  pool.ensure(n * n * 16, total, size_t(nchunks) * 3 * 8, work_bytes(chunk));
  if (!in_pinned) pool.pin_in.ensure(total);
  if (!out_pinned) pool.pin_out.ensure(total);
  double* dp = static_cast<double*>(pool.p.ptr);
  double* dx = static_cast<double*>(pool.x.ptr);
  double* dchk = static_cast<double*>(pool.chk.ptr);
  double* hchk = static_cast<double*>(pool.pin_chk.ptr);
  char* pin_in = static_cast<char*>(pool.pin_in.ptr);
  char* pin_out = static_cast<char*>(pool.pin_out.ptr);
  cudaStream_t sh = pool.st[0], sd = pool.st[3], sk = pool.st[4];
  CopyPool& cp = CopyPool::get();
  // LBG_PIPELINE_TIMING (measurement only): device timestamps of each chunk's
  // H2D end, steps start / end and D2H end, printed relative to the call start
  static const bool timing = std::getenv("LBG_PIPELINE_TIMING") != nullptr;
  struct TimingEvents {
    cudaEvent_t e[4 * kMaxChunks + 1] = {};
    ~TimingEvents() {
      for (auto& x : e)
        if (x) (void)cudaEventDestroy(x);
    }
  } tev;
  cudaEvent_t* te = tev.e;
  if (timing)
    for (auto& e : tev.e) check_cuda(cudaEventCreate(&e), "event");
  auto mark = [&](int i, cudaStream_t st) {
    if (timing) check_cuda(cudaEventRecord(te[i], st), "event");
  };
  try {
    mark(4 * kMaxChunks, sh);
    check_cuda(cudaMemcpyAsync(dp, p, n * n * 16, cudaMemcpyHostToDevice, sh), "H2D P");
    for (int c = 0; c < nchunks; ++c) {
      const int64_t b0 = bounds[c], nb = bounds[c + 1] - bounds[c];
      double* xc = dx + size_t(b0) * n * 2;
      const size_t off = size_t(b0) * n * 16, bytes = size_t(nb) * n * 16;
      const void* src = reinterpret_cast<const char*>(rho0) + off;
      if (!in_pinned) {  // stage through pinned memory while the GPU works on earlier chunks
        cp.copy(pin_in + off, src, bytes);
        src = pin_in + off;
      }
      check_cuda(cudaMemcpyAsync(xc, src, bytes, cudaMemcpyHostToDevice, sh), "H2D rho0");
      mark(4 * c, sh);
      check_cuda(cudaEventRecord(pool.ev_x[c], sh), "event");
      // propagate.cpp:79 — every rho0 must pass check_state at 1e-8 (on the
      // check stream, so the copies never queue behind a check kernel); the
      // steps (in place) wait for the check, which reads the chunk
      check_cuda(cudaStreamWaitEvent(sk, pool.ev_x[c], 0), "wait");
      launch_check_state(xc, d, nb, dchk + 3 * c, sk);
      check_cuda(cudaEventRecord(pool.ev_h[c], sk), "event");
      check_cuda(cudaMemcpyAsync(hchk + 3 * c, dchk + 3 * c, 24, cudaMemcpyDeviceToHost, sk), "D2H check");
      cudaStream_t sc = pool.st[1 + (c & 1)];
      check_cuda(cudaStreamWaitEvent(sc, pool.ev_h[c], 0), "wait");
      mark(4 * c + 1, sc);
      step(dp, xc, nb, pool.w[c & 1].ptr, sc);
      mark(4 * c + 2, sc);
      check_cuda(cudaEventRecord(pool.ev_c[c], sc), "event");
    }
    check_cuda(cudaEventRecord(pool.ev_chk, sk), "event");
    sync_event_spin(pool.ev_chk, "sync check");
    for (int c = 0; c < nchunks; ++c)
      if (!(hchk[3 * c] <= 1e-8 && hchk[3 * c + 1] <= 1e-8 && hchk[3 * c + 2] >= -1e-8))
        throw invalid_argument("evolve: initial state fails physical-state checks");
    for (int c = 0; c < nchunks; ++c) {
      const int64_t b0 = bounds[c], nb = bounds[c + 1] - bounds[c];
      const size_t off = size_t(b0) * n * 16, bytes = size_t(nb) * n * 16;
      void* dst = out_pinned ? static_cast<void*>(reinterpret_cast<char*>(out) + off) : pin_out + off;
      check_cuda(cudaStreamWaitEvent(sd, pool.ev_c[c], 0), "wait");
      check_cuda(cudaMemcpyAsync(dst, dx + size_t(b0) * n * 2, bytes, cudaMemcpyDeviceToHost, sd), "D2H rho");
      mark(4 * c + 3, sd);
      check_cuda(cudaEventRecord(pool.ev_d[c], sd), "event");
    }
    if (!out_pinned)
      for (int c = 0; c < nchunks; ++c) {  // copy each chunk out as soon as it has landed
        const size_t off = size_t(bounds[c]) * n * 16, bytes = size_t(bounds[c + 1] - bounds[c]) * n * 16;
        sync_event_spin(pool.ev_d[c], "sync D2H");
        cp.copy(reinterpret_cast<char*>(out) + off, pin_out + off, bytes);
      }
    sync_stream_spin(sd, "sync");
    if (timing) {
      for (int c = 0; c < nchunks; ++c) {
        float t[4];
        for (int k = 0; k < 4; ++k) check_cuda(cudaEventElapsedTime(&t[k], te[4 * kMaxChunks], te[4 * c + k]), "t");
        std::fprintf(stderr, "chunk %d: h2d end %.3f  steps %.3f-%.3f  d2h end %.3f ms\n", c, t[0], t[1], t[2], t[3]);
      }
    }
  } catch (...) {
    pool.drain();
    throw;
  }
}

}  // namespace lbg
