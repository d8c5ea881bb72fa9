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
#include <cstdint>
#include <cstdlib>
#include <cstring>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include <functional>
#include <mutex>
#include <thread>
#include <utility>
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

// Copy with non-temporal (streaming) stores: the destination -- a pinned
// staging buffer the DMA engine reads next, or the caller's result array --
// is not read back by these threads, so its lines need neither a
// read-for-ownership nor a place in the cache.  glibc's memcpy only switches
// to streaming stores above a per-thread size these 2 MB parts do not reach.
// SSE2 is the x86-64 baseline, so this runs on whatever host the library
// travels to.
void stream_copy(char* dst, const char* src, size_t n) {
#if defined(__SSE2__)
  const size_t head = std::min(n, (size_t)((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15));
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  for (size_t b = n / 64; b > 0; --b, src += 64, dst += 64) {
    const __m128i r0 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src));
    const __m128i r1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 16));
    const __m128i r2 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 32));
    const __m128i r3 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst), r0);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 16), r1);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 32), r2);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 48), r3);
  }
  _mm_sfence();
  std::memcpy(dst, src, n % 64);
#else
  std::memcpy(dst, src, n);
#endif
}

void par_memcpy(CopyPool& pool, void* dst, const void* src, size_t bytes) {
  const int n = pool.size();
  static const bool streaming = [] {
    const char* e = std::getenv("STB_STREAM_COPY");
    return !e || std::atoi(e) != 0;
  }();
  auto copy = [](char* d, const char* s, size_t len) {
    if (streaming) stream_copy(d, s, len);
    else std::memcpy(d, s, len);
  };
  if (bytes < ((size_t)1 << 20) || n == 1) {
    copy(static_cast<char*>(dst), static_cast<const char*>(src), bytes);
    return;
  }
  const size_t part = ((bytes + n - 1) / n + 63) & ~(size_t)63;
  pool.run([&](int i) {
    const size_t lo = std::min(bytes, (size_t)i * part);
    const size_t hi = std::min(bytes, lo + part);
    if (hi > lo) copy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
  });
}

// Pitched (x, y, row) device rows -> dense, 16 bytes per thread: the DMA
// engine then moves one linear block per chunk (a strided device-to-host
// copy of 2.3 KB rows ran at ~40 GB/s on the B200 box, a linear one at 57).
__global__ void pack_rows_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                 size_t row16, size_t ny, size_t nx, size_t pitch16,
                                 size_t plane16) {
  const size_t n = row16 * ny * nx;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t c = i % row16, r = i / row16;
    const size_t y = r % ny, x = r / ny;
    dst[i] = src[x * plane16 + y * pitch16 + c];
  }
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
    // strided layouts whose rows are whole 16-byte words: pack on the device
    // (stream-ordered before the copy that reads the pack buffer)
    const bool pack = !(pitch == row && plane == row * ny) && row % 16 == 0 && pitch % 16 == 0 &&
                      plane % 16 == 0 && reinterpret_cast<uintptr_t>(dev) % 16 == 0;
    if (pack && !dpack_) STB_CUDA(cudaMalloc(&dpack_, kChunk));
    for (size_t c = 0; c < n; ++c) {
      const int b = (int)(c % kBufs);
      const size_t x0 = c * per, cnt = std::min(per, nx - x0);
      const char* src = static_cast<const char*>(dev) + x0 * plane;
      if (pack) {
        pack_rows_kernel<<<592, 256, 0, st>>>(reinterpret_cast<const uint4*>(src),
                                              static_cast<uint4*>(dpack_), row / 16, ny, cnt,
                                              pitch / 16, plane / 16);
        STB_CHECK_LAUNCH();
        STB_CUDA(cudaMemcpyAsync(buf_[b], dpack_, cnt * pbytes, cudaMemcpyDeviceToHost, st));
      } else {
        copy3d(buf_[b], src, row, ny, cnt, pitch, plane, st, cudaMemcpyDeviceToHost);
      }
      STB_CUDA(cudaEventRecord(ev_[b], st));
      if (c >= 1) drain(c - 1);
    }
    drain(n - 1);
  }

  // page-locked destination: chunks are packed on the device into two
  // alternating buffers and copied straight into the caller's array
  void download3d_pinned(void* host, const void* dev, size_t row, size_t ny, size_t nx,
                         size_t pitch, size_t plane, cudaStream_t st) {
    const size_t pbytes = row * ny;
    const bool dense = pitch == row && plane == row * ny;
    const bool can_pack = row % 16 == 0 && pitch % 16 == 0 && plane % 16 == 0 &&
                          reinterpret_cast<uintptr_t>(dev) % 16 == 0 && pbytes <= kChunk;
    if (dense || !can_pack || nx == 0) {
      copy3d(host, dev, row, ny, nx, pitch, plane, st, cudaMemcpyDeviceToHost);
      STB_CUDA(cudaStreamSynchronize(st));
      return;
    }
    for (int b = 0; b < 2; ++b)
      if (!dpack2_[b]) STB_CUDA(cudaMalloc(&dpack2_[b], kChunk));
    if (!pst_) {
      STB_CUDA(cudaStreamCreateWithFlags(&pst_, cudaStreamNonBlocking));
      for (auto& e : pev_) STB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      for (auto& e : cev_) STB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    // pack kernels on st, copies on pst_: pack(c + 1) overlaps copy(c)
    const size_t per = std::max<size_t>(1, kChunk / pbytes), n = (nx + per - 1) / per;
    for (size_t c = 0; c < n; ++c) {
      const int b = (int)(c & 1);
      const size_t x0 = c * per, cnt = std::min(per, nx - x0);
      if (c >= 2) STB_CUDA(cudaStreamWaitEvent(st, cev_[b], 0));     // copy(c - 2) left buffer b
      pack_rows_kernel<<<592, 256, 0, st>>>(
          reinterpret_cast<const uint4*>(static_cast<const char*>(dev) + x0 * plane),
          static_cast<uint4*>(dpack2_[b]), row / 16, ny, cnt, pitch / 16, plane / 16);
      STB_CHECK_LAUNCH();
      STB_CUDA(cudaEventRecord(pev_[b], st));
      STB_CUDA(cudaStreamWaitEvent(pst_, pev_[b], 0));
      STB_CUDA(cudaMemcpyAsync(static_cast<char*>(host) + x0 * pbytes, dpack2_[b], cnt * pbytes,
                               cudaMemcpyDeviceToHost, pst_));
      STB_CUDA(cudaEventRecord(cev_[b], pst_));
    }
    STB_CUDA(cudaStreamSynchronize(pst_));
    STB_CUDA(cudaStreamSynchronize(st));
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
  void* dpack_ = nullptr;     // device staging of one packed chunk
  void* dpack2_[2] = {nullptr, nullptr};
  cudaStream_t pst_ = nullptr;
  cudaEvent_t pev_[2] = {nullptr, nullptr}, cev_[2] = {nullptr, nullptr};
  void* buf_[kBufs] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_[kBufs] = {nullptr, nullptr, nullptr};
};

constexpr size_t kStageMin = (size_t)8 << 20;   // smaller copies: plain cudaMemcpy

// Page-locked host memory (stb_host_alloc or any cudaHostAlloc / registered
// range): the DMA engine reads and writes it directly, no staging copy.
bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Cache of freed page-locked blocks, by exact size (cudaHostAlloc costs
// ~0.1 ms per MB; run() results are requested again and again at the same
// sizes).  Keeps at most kPoolCap bytes.
class PinnedPool {
 public:
  static constexpr size_t kPoolCap = (size_t)6 << 30;
  static PinnedPool& get() {
    static PinnedPool* p = new PinnedPool();    // leaked: see HostIO::get
    return *p;
  }
  void* alloc(size_t bytes) {
    {
      std::lock_guard<std::mutex> lk(m_);
      for (size_t i = 0; i < free_.size(); ++i)
        if (free_[i].second == bytes) {
          void* p = free_[i].first;
          cached_ -= bytes;
          free_.erase(free_.begin() + i);
          live_.emplace_back(p, bytes);
          return p;
        }
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      trim(0);                                  // give the cache back and retry once
      if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
    }
    std::lock_guard<std::mutex> lk(m_);
    live_.emplace_back(p, bytes);
    return p;
  }
  bool release(void* p) {
    size_t bytes = 0;
    {
      std::lock_guard<std::mutex> lk(m_);
      size_t i = 0;
      for (; i < live_.size(); ++i)
        if (live_[i].first == p) break;
      if (i == live_.size()) return false;
      bytes = live_[i].second;
      live_.erase(live_.begin() + i);
      if (bytes <= kPoolCap) {
        free_.emplace_back(p, bytes);
        cached_ += bytes;
        p = nullptr;
      }
    }
    if (p) cudaFreeHost(p);
    trim(kPoolCap);
    return true;
  }

 private:
  void trim(size_t cap) {
    for (;;) {
      void* victim = nullptr;
      {
        std::lock_guard<std::mutex> lk(m_);
        if (cached_ <= cap || free_.empty()) return;
        victim = free_.front().first;
        cached_ -= free_.front().second;
        free_.erase(free_.begin());
      }
      cudaFreeHost(victim);
    }
  }
  std::mutex m_;
  std::vector<std::pair<void*, size_t>> free_, live_;
  size_t cached_ = 0;
};

}  // namespace

void* host_pinned_alloc(size_t bytes) { return PinnedPool::get().alloc(bytes); }
bool host_pinned_free(void* p) { return PinnedPool::get().release(p); }

void host_to_device(void* dev, const void* host, size_t bytes, cudaStream_t st) {
  if (bytes < kStageMin) {
    STB_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st));
    return;
  }
  if (is_pinned(host)) {                  // direct DMA; the caller's array is free on return
    STB_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st));
    STB_CUDA(cudaStreamSynchronize(st));
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
  if (is_pinned(host)) io.download3d_pinned(host, dev, row, ny, nx, pitch, plane, st);
  else io.download3d(host, dev, row, ny, nx, pitch, plane, st);
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
