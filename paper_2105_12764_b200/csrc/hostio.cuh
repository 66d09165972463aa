// hostio.cuh -- host side of the host-buffer C ABI (mgrg_*_host*).
//
// A reference caller hands the drop-in ordinary pageable memory: the
// values of a TensorGrid and the per-class std::vectors of RefactoredData
// (refactor.hpp:18-76).  cudaMemcpyAsync from pageable memory is staged by
// the driver through a small bounce buffer at 11-16 GB/s and serialises
// with the host thread; cudaHostRegister of a 4.3 GB vector costs 0.47 s +
// 0.11 s to unregister (profiles/r2/host_probe.json) -- more than the whole
// pinned transfer (78 ms).  So pageable buffers go through plan-owned pinned
// rings instead:
//   * uploads: the calling thread copies each <= 32 MiB chunk into a free
//     ring slot with the parallel copy pool (80+ GB/s with 8-16 host
//     threads) and issues the DMA from it; the next chunk's host copy
//     overlaps the previous chunk's DMA;
//   * downloads: a per-plan worker thread issues the DMA into a ring slot
//     after the producing kernel's event and copies finished slots out to
//     the caller's memory, so the calling thread keeps enqueuing kernels and
//     uploads while results stream back.
// Pinned buffers (cudaHostAlloc / registered) keep the direct async DMA.
//
// A HostView is the caller's buffer seen as the flat class-buffer element
// range [0, N): one pointer, or one pointer per class (class l covering
// [off[l], off[l+1]), the concatenation order of RefactoredData::classes),
// so the drop-in's per-class vectors are written in place -- no flat copy.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace mgrg {

// ---- parallel memcpy pool (process-wide, lazily started) -----------------
class CopyPool {
public:
  static CopyPool &get() {
    static CopyPool pool;
    return pool;
  }
  // dst <- src, n bytes, split over the pool; blocks until done (the caller
  // works on its own pieces meanwhile)
  void copy(void *dst, const void *src, size_t n) {
    constexpr size_t kMinPiece = size_t(1) << 20;
    const size_t parts = std::max<size_t>(1, std::min<size_t>(nthreads_ + 1, n / kMinPiece));
    if (parts == 1) {
      std::memcpy(dst, src, n);
      return;
    }
    Batch b;
    b.left = parts;
    const size_t per = (n + parts - 1) / parts;
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (size_t i = 1; i < parts; ++i) {
        const size_t a = std::min(n, i * per), e = std::min(n, (i + 1) * per);
        q_.push_back({static_cast<char *>(dst) + a, static_cast<const char *>(src) + a, e - a,
                      &b});
      }
    }
    cv_.notify_all();
    std::memcpy(dst, src, std::min(n, per));
    finish(&b);
    // help with queued pieces (ours or another caller's) while waiting
    for (;;) {
      Piece pc;
      {
        std::unique_lock<std::mutex> lk(mu_);
        if (b.left == 0)
          return;
        if (q_.empty()) {
          done_cv_.wait(lk, [&] { return b.left == 0 || !q_.empty(); });
          if (b.left == 0)
            return;
          if (q_.empty())
            continue;
        }
        pc = q_.front();
        q_.pop_front();
      }
      std::memcpy(pc.dst, pc.src, pc.n);
      finish(pc.b);
    }
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto &t : th_)
      t.join();
  }

private:
  struct Batch {
    size_t left = 0;
  };
  struct Piece {
    char *dst;
    const char *src;
    size_t n;
    Batch *b;
  };
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    nthreads_ = std::min(15u, hw > 1 ? hw - 1 : 1u);
    for (unsigned i = 0; i < nthreads_; ++i)
      th_.emplace_back([this] { run(); });
  }
  void finish(Batch *b) {
    std::lock_guard<std::mutex> lk(mu_);
    if (--b->left == 0)
      done_cv_.notify_all();
  }
  void run() {
    for (;;) {
      Piece pc;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
        if (stop_ && q_.empty())
          return;
        pc = q_.front();
        q_.pop_front();
      }
      std::memcpy(pc.dst, pc.src, pc.n);
      finish(pc.b);
    }
  }
  unsigned nthreads_ = 1;
  std::vector<std::thread> th_;
  std::deque<Piece> q_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  bool stop_ = false;
};

inline bool host_pinned(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}
// device memory passed where the host-buffer entry points expect host memory
inline bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice;
}

// ---- the caller's host buffer as a flat element range -------------------
struct HostView {
  size_t es = 0;                  // element size
  char *flat = nullptr;           // one buffer ...
  std::vector<char *> seg;        // ... or one per class
  std::vector<uint64_t> off;      // class offsets (seg.size() + 1 entries)
  bool pinned = false;
  bool device = false; // a device pointer: rejected by the entry points

  static HostView of(const void *p, size_t es) {
    HostView v;
    v.es = es;
    v.flat = static_cast<char *>(const_cast<void *>(p));
    v.pinned = host_pinned(p);
    v.device = !v.pinned && is_device_ptr(p);
    return v;
  }
  static HostView classes(const void *const *ptrs, const uint64_t *offs, int nclass, size_t es) {
    HostView v;
    v.es = es;
    v.pinned = true;
    for (int l = 0; l < nclass; ++l) {
      v.seg.push_back(static_cast<char *>(const_cast<void *>(ptrs[l])));
      v.off.push_back(offs[l]);
      if (offs[l + 1] > offs[l] && !host_pinned(ptrs[l])) {
        v.pinned = false;
        if (is_device_ptr(ptrs[l]))
          v.device = true;
      }
    }
    v.off.push_back(offs[nclass]);
    return v;
  }
  // fn(host pointer, element offset within [o, o + n), element count) for
  // each contiguous piece of [o, o + n)
  template <typename Fn> void pieces(uint64_t o, uint64_t n, Fn fn) const {
    if (flat) {
      if (n)
        fn(flat + o * es, uint64_t(0), n);
      return;
    }
    const uint64_t e = o + n;
    for (size_t l = 0; l < seg.size(); ++l) {
      const uint64_t a = std::max(o, off[l]), b = std::min(e, off[l + 1]);
      if (b > a)
        fn(seg[l] + (a - off[l]) * es, a - o, b - a);
    }
  }
};

// ---- per-plan pinned rings + download worker -----------------------------
class HostXfer {
public:
  static constexpr int kSlots = 4;

  explicit HostXfer(int device) : device_(device) {}
  ~HostXfer() {
    if (worker_.joinable()) {
      {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
      }
      cv_.notify_all();
      worker_.join();
    }
    for (int i = 0; i < kSlots; ++i) {
      if (up_[i])
        cudaFreeHost(up_[i]);
      if (dn_[i])
        cudaFreeHost(dn_[i]);
      if (up_ev_[i])
        cudaEventDestroy(up_ev_[i]);
      if (dn_ev_[i])
        cudaEventDestroy(dn_ev_[i]);
    }
  }
  // s_out: the download stream; slot size scales with the plan (1..32 MiB)
  void init(cudaStream_t s_out, uint64_t plan_bytes) {
    s_out_ = s_out;
    slot_ = size_t(std::min<uint64_t>(uint64_t(32) << 20,
                                      std::max<uint64_t>(uint64_t(1) << 20, plan_bytes / 16)));
  }

  // [o, o + n) of the view -> dev (elements), DMA on stream s.  Pinned views
  // go straight; pageable ones through the upload ring (the host copies
  // happen here, on the calling thread).
  cudaError_t upload(void *dev, const HostView &v, uint64_t o, uint64_t n, cudaStream_t s) {
    char *d = static_cast<char *>(dev);
    cudaError_t err = cudaSuccess;
    if (v.pinned) {
      v.pieces(o, n, [&](char *h, uint64_t at, uint64_t len) {
        if (err == cudaSuccess)
          err = cudaMemcpyAsync(d + at * v.es, h, len * v.es, cudaMemcpyHostToDevice, s);
      });
      return err;
    }
    if ((err = rings()))
      return err;
    v.pieces(o, n, [&](char *h, uint64_t at, uint64_t len) {
      const uint64_t bytes = len * v.es;
      for (uint64_t c = 0; c < bytes && err == cudaSuccess; c += slot_) {
        const size_t nb = size_t(std::min<uint64_t>(slot_, bytes - c));
        const int k = up_next_;
        up_next_ = (up_next_ + 1) % kSlots;
        if ((err = cudaEventSynchronize(up_ev_[k])))
          return;
        CopyPool::get().copy(up_[k], h + c, nb);
        if ((err = cudaMemcpyAsync(d + at * v.es + c, up_[k], nb, cudaMemcpyHostToDevice, s)))
          return;
        err = cudaEventRecord(up_ev_[k], s);
      }
    });
    return err;
  }

  // dev -> [o, o + n) of the view once `after` (recorded on the producing
  // stream) has completed.  Pinned views: async DMA on s_out; pageable: a job
  // for the worker.  drain() waits for every queued download.
  cudaError_t download(const HostView &v, uint64_t o, uint64_t n, const void *dev,
                       cudaEvent_t after) {
    if (v.pinned) {
      cudaError_t err = cudaStreamWaitEvent(s_out_, after, 0);
      v.pieces(o, n, [&](char *h, uint64_t at, uint64_t len) {
        if (err == cudaSuccess)
          err = cudaMemcpyAsync(h, static_cast<const char *>(dev) + at * v.es, len * v.es,
                                cudaMemcpyDeviceToHost, s_out_);
      });
      return err;
    }
    if (cudaError_t e = rings())
      return e;
    {
      std::lock_guard<std::mutex> lk(mu_);
      jobs_.push_back({v, o, n, static_cast<const char *>(dev), after});
      ++pending_;
    }
    cv_.notify_all();
    return cudaSuccess;
  }

  // wait for every download (both kinds); returns the first worker error
  cudaError_t drain() {
    std::unique_lock<std::mutex> lk(mu_);
    idle_cv_.wait(lk, [&] { return pending_ == 0; });
    lk.unlock();
    cudaError_t e = cudaStreamSynchronize(s_out_);
    lk.lock();
    const cudaError_t w = werr_;
    werr_ = cudaSuccess;
    return w ? w : e;
  }

private:
  struct Job {
    HostView v;
    uint64_t o, n;
    const char *dev;
    cudaEvent_t after;
  };
  struct Out { // a finished-DMA slot still to be copied out
    int slot;
    char *h;
    size_t nb;
  };
  void run() {
    cudaSetDevice(device_);
    std::deque<Out> outq;
    int next = 0;
    auto flush_one = [&]() {
      Out o = outq.front();
      outq.pop_front();
      cudaError_t e = cudaEventSynchronize(dn_ev_[o.slot]);
      if (e == cudaSuccess)
        CopyPool::get().copy(o.h, dn_[o.slot], o.nb);
      else
        note(e);
    };
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !jobs_.empty(); });
        if (jobs_.empty()) // stop_
          return;
        j = jobs_.front();
        jobs_.pop_front();
      }
      note(cudaStreamWaitEvent(s_out_, j.after, 0));
      j.v.pieces(j.o, j.n, [&](char *h, uint64_t at, uint64_t len) {
        const uint64_t bytes = len * j.v.es;
        for (uint64_t c = 0; c < bytes; c += slot_) {
          const size_t nb = size_t(std::min<uint64_t>(slot_, bytes - c));
          if (int(outq.size()) == kSlots)
            flush_one();
          const int k = next;
          next = (next + 1) % kSlots;
          note(cudaMemcpyAsync(dn_[k], j.dev + at * j.v.es + c, nb, cudaMemcpyDeviceToHost,
                               s_out_));
          note(cudaEventRecord(dn_ev_[k], s_out_));
          outq.push_back({k, h + c, nb});
        }
      });
      bool last;
      {
        std::lock_guard<std::mutex> lk(mu_);
        last = jobs_.empty();
      }
      if (last) // nothing else queued: finish the copies out now
        while (!outq.empty())
          flush_one();
      { // (outq is empty whenever pending_ reaches 0: it was flushed above)
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0)
          idle_cv_.notify_all();
      }
    }
  }
  // the pinned rings and the download worker, on first pageable use
  cudaError_t rings() {
    if (ready_)
      return cudaSuccess;
    for (int i = 0; i < kSlots; ++i) {
      cudaError_t e;
      if ((e = cudaHostAlloc(reinterpret_cast<void **>(&up_[i]), slot_, cudaHostAllocDefault)) ||
          (e = cudaHostAlloc(reinterpret_cast<void **>(&dn_[i]), slot_, cudaHostAllocDefault)) ||
          (e = cudaEventCreateWithFlags(&up_ev_[i], cudaEventDisableTiming)) ||
          (e = cudaEventCreateWithFlags(&dn_ev_[i], cudaEventDisableTiming)))
        return e;
    }
    worker_ = std::thread([this] { run(); });
    ready_ = true;
    return cudaSuccess;
  }
  void note(cudaError_t e) {
    if (e != cudaSuccess) {
      std::lock_guard<std::mutex> lk(mu_);
      if (werr_ == cudaSuccess)
        werr_ = e;
    }
  }

  int device_;
  bool ready_ = false;
  size_t slot_ = size_t(1) << 20;
  cudaStream_t s_out_ = nullptr;
  char *up_[kSlots] = {}, *dn_[kSlots] = {};
  cudaEvent_t up_ev_[kSlots] = {}, dn_ev_[kSlots] = {};
  int up_next_ = 0;
  std::thread worker_;
  std::deque<Job> jobs_;
  std::mutex mu_;
  std::condition_variable cv_, idle_cv_;
  int pending_ = 0;
  bool stop_ = false;
  cudaError_t werr_ = cudaSuccess;
};

} // namespace mgrg
