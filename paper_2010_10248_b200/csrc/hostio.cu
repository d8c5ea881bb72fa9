// Staged host <-> device transfers for large arrays (model upload, field and
// trace download of the public run() path).
//
// Pageable cudaMemcpy stages through the driver's own small pinned buffers
// on one thread (measured on the B200 box: ~11 GB/s H2D, ~5 GB/s for the
// pitched field download).  Here chunks of up to kChunk bytes go through a
// ring of kBufs pinned buffers: a pool of host threads copies chunk c
// between the user's pageable array and a pinned buffer while the copy
// engine moves chunk c-1 (download) / c (upload) over PCIe.  Pitched device
// layouts are (un)packed by the DMA engine (cudaMemcpy3DAsync into the dense
// pinned chunk), so no extra device pass is needed.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "stb_internal.cuh"

namespace stb {
namespace {

// Persistent worker threads; run(f) calls f(0..n-1) concurrently.
class CopyPool {
 public:
  explicit CopyPool(int n) : n_(std::max(1, n)) {
    for (int i = 1; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return n_; }
  void run(const std::function<void(int)>& f) {
    if (n_ == 1) {
      f(0);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      job_ = &f;
      remaining_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [this] { return remaining_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int i) {
    unsigned seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        f = job_;
      }
      (*f)(i);
      std::lock_guard<std::mutex> lk(m_);
      if (--remaining_ == 0) done_.notify_one();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  unsigned gen_ = 0;
  int remaining_ = 0;
  bool stop_ = false;
};

void par_memcpy(CopyPool& pool, void* dst, const void* src, size_t bytes) {
  const int n = pool.size();
  if (bytes < ((size_t)1 << 20) || n == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t part = ((bytes + n - 1) / n + 63) & ~(size_t)63;
  pool.run([&](int i) {
    const size_t lo = std::min(bytes, (size_t)i * part);
    const size_t hi = std::min(bytes, lo + part);
    if (hi > lo) std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo,
                             hi - lo);
  });
}

class HostIO {
 public:
  static constexpr size_t kChunk = (size_t)32 << 20;
  static constexpr int kBufs = 3;

  // one instance per device (its events belong to that device; the pinned
  // buffers are portable).  Intentionally leaked: pinned memory and events
  // must not be released during static destruction (after the CUDA runtime
  // may have shut down).
  static HostIO& get() {
    static std::mutex m;
    static HostIO* io[64] = {};
    int dev = 0;
    STB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(m);
    HostIO*& p = io[dev & 63];
    if (!p) p = new HostIO();
    return *p;
  }

  std::mutex mu;

  void ensure() {
    if (buf_[0]) return;
    for (int b = 0; b < kBufs; ++b) {
      STB_CUDA(cudaHostAlloc(&buf_[b], kChunk, cudaHostAllocPortable));
      STB_CUDA(cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming));
    }
  }

  void upload(void* dev, const void* host, size_t bytes, cudaStream_t st) {
    ensure();
    const size_t n = (bytes + kChunk - 1) / kChunk;
    for (size_t c = 0; c < n; ++c) {
      const int b = (int)(c % kBufs);
      const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      STB_CUDA(cudaEventSynchronize(ev_[b]));    // DMA that last read buf b
      par_memcpy(pool_, buf_[b], static_cast<const char*>(host) + off, len);
      STB_CUDA(cudaMemcpyAsync(static_cast<char*>(dev) + off, buf_[b], len,
                               cudaMemcpyHostToDevice, st));
      STB_CUDA(cudaEventRecord(ev_[b], st));
    }
  }

  // dense (nx, ny, row) host <- device rows of `row` bytes at
  // dev + (x * plane + y * pitch) bytes
  void download3d(void* host, const void* dev, size_t row, size_t ny, size_t nx, size_t pitch,
                  size_t plane, cudaStream_t st) {
    ensure();
    const size_t pbytes = row * ny;
    const size_t per = std::max<size_t>(1, kChunk / std::max<size_t>(pbytes, 1));
    if (pbytes > kChunk || nx == 0) {       // very large planes: one direct copy
      copy3d(host, dev, row, ny, nx, pitch, plane, st, cudaMemcpyDeviceToHost);
      STB_CUDA(cudaStreamSynchronize(st));
      return;
    }
    const size_t n = (nx + per - 1) / per;
    auto drain = [&](size_t c) {
      const int b = (int)(c % kBufs);
      const size_t x0 = c * per, cnt = std::min(per, nx - x0);
      STB_CUDA(cudaEventSynchronize(ev_[b]));
      par_memcpy(pool_, static_cast<char*>(host) + x0 * pbytes, buf_[b], cnt * pbytes);
    };
    for (size_t c = 0; c < n; ++c) {
      const int b = (int)(c % kBufs);
      const size_t x0 = c * per, cnt = std::min(per, nx - x0);
      copy3d(buf_[b], static_cast<const char*>(dev) + x0 * plane, row, ny, cnt, pitch, plane, st,
             cudaMemcpyDeviceToHost);
      STB_CUDA(cudaEventRecord(ev_[b], st));
      if (c >= 1) drain(c - 1);
    }
    drain(n - 1);
  }

 private:
  HostIO() : pool_(std::max(1, std::min(16, (int)std::thread::hardware_concurrency()))) {}

  static void copy3d(void* dst_dense, const void* src, size_t row, size_t ny, size_t nx,
                     size_t pitch, size_t plane, cudaStream_t st, cudaMemcpyKind kind) {
    if (pitch == row && plane == row * ny) {
      STB_CUDA(cudaMemcpyAsync(dst_dense, src, row * ny * nx, kind, st));
      return;
    }
    if (plane == pitch * ny) {
      STB_CUDA(cudaMemcpy2DAsync(dst_dense, row, src, pitch, row, ny * nx, kind, st));
      return;
    }
    cudaMemcpy3DParms p{};
    p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), pitch, row, plane / pitch);
    p.dstPtr = make_cudaPitchedPtr(dst_dense, row, row, ny);
    p.extent = make_cudaExtent(row, ny, nx);
    p.kind = kind;
    STB_CUDA(cudaMemcpy3DAsync(&p, st));
  }

  CopyPool pool_;
  void* buf_[kBufs] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_[kBufs] = {nullptr, nullptr, nullptr};
};

constexpr size_t kStageMin = (size_t)8 << 20;   // smaller copies: plain cudaMemcpy

}  // namespace

void host_to_device(void* dev, const void* host, size_t bytes, cudaStream_t st) {
  if (bytes < kStageMin) {
    STB_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st));
    return;
  }
  HostIO& io = HostIO::get();
  std::lock_guard<std::mutex> lk(io.mu);
  io.upload(dev, host, bytes, st);
}

void device_to_host_3d(void* host, const void* dev, size_t row, size_t ny, size_t nx,
                       size_t pitch, size_t plane, cudaStream_t st) {
  if (row * ny * nx < kStageMin) {
    if (pitch == row && plane == row * ny) {
      STB_CUDA(cudaMemcpyAsync(host, dev, row * ny * nx, cudaMemcpyDeviceToHost, st));
    } else {
      cudaMemcpy3DParms p{};
      p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(dev), pitch, row, plane / pitch);
      p.dstPtr = make_cudaPitchedPtr(host, row, row, ny);
      p.extent = make_cudaExtent(row, ny, nx);
      p.kind = cudaMemcpyDeviceToHost;
      STB_CUDA(cudaMemcpy3DAsync(&p, st));
    }
    STB_CUDA(cudaStreamSynchronize(st));
    return;
  }
  HostIO& io = HostIO::get();
  std::lock_guard<std::mutex> lk(io.mu);
  io.download3d(host, dev, row, ny, nx, pitch, plane, st);
}

void device_to_host(void* host, const void* dev, size_t bytes, cudaStream_t st) {
  // contiguous: 1 MiB rows (staged), then the remainder
  const size_t R = (size_t)1 << 20, nfull = bytes / R, rem = bytes - nfull * R;
  if (nfull) device_to_host_3d(host, dev, R, 1, nfull, R, R, st);
  if (rem) {
    STB_CUDA(cudaMemcpyAsync(static_cast<char*>(host) + nfull * R,
                             static_cast<const char*>(dev) + nfull * R, rem,
                             cudaMemcpyDeviceToHost, st));
    STB_CUDA(cudaStreamSynchronize(st));
  }
}

}  // namespace stb
