// Internal declarations shared by the libstb200 translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/stb200.h"

namespace stb {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_error(const std::string& msg);

#define STB_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      if (e_ == cudaErrorMemoryAllocation)                                    \
        throw ::stb::Error(STB_ERR_NOMEM, std::string(#call) + ": " +         \
                                               cudaGetErrorString(e_));       \
      throw ::stb::Error(STB_ERR_CUDA,                                        \
                         std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                         \
  } while (0)

#define STB_CHECK_LAUNCH() STB_CUDA(cudaGetLastError())

#define STB_REQUIRE(cond, code, msg)            \
  do {                                          \
    if (!(cond)) throw ::stb::Error(code, msg); \
  } while (0)

// Device allocations come from the stream-ordered pool of the current device
// with an unlimited release threshold: a process that runs many shots (or
// re-creates handles) reuses freed field buffers instead of paying
// cudaMalloc/page-mapping cost per handle.
inline void retain_freed_memory() {
  static thread_local int done_for = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  if (done_for == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_for = dev;
}

// Kernel attributes (cudaFuncSetAttribute) are per device: true the first
// time this kernel's configuration is needed on the current device.
inline bool first_use_on_device(std::atomic<uint64_t>& mask) {
  int dev = 0;
  STB_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  return (mask.fetch_or(bit) & bit) == 0;
}

// Owning device buffer.
// Large host <-> device copies staged through pinned buffers (hostio.cu).
// host_to_device is stream-ordered (returns once the host array may be
// reused); the device_to_host variants return when the data is on the host.
void host_to_device(void* dev, const void* host, size_t bytes, cudaStream_t st);
// page-locked host blocks from a size-keyed cache (hostio.cu)
void* host_pinned_alloc(size_t bytes);
bool host_pinned_free(void* p);
void device_to_host(void* host, const void* dev, size_t bytes, cudaStream_t st);
// dense (nx, ny, row bytes) host array <- rows at dev + x*plane + y*pitch bytes
void device_to_host_3d(void* host, const void* dev, size_t row, size_t ny, size_t nx,
                       size_t pitch, size_t plane, cudaStream_t st);

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) {
      retain_freed_memory();
      STB_CUDA(cudaMallocAsync(&p, count * sizeof(T), 0));
      STB_CUDA(cudaStreamSynchronize(0));
    }
  }
  void release() {
    if (p) {
      cudaFreeAsync(p, 0);
      cudaStreamSynchronize(0);
    }
    p = nullptr;
    n = 0;
  }
  void zero(cudaStream_t s = 0) {
    if (p) STB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void upload(const T* h, size_t count, cudaStream_t s = 0) {
    if (count) host_to_device(p, h, count * sizeof(T), s);
  }
  // synchronous: the data is on the host when this returns
  void download(T* h, size_t count, cudaStream_t s = 0) const {
    if (count) device_to_host(h, p, count * sizeof(T), s);
  }
  T* get() const { return p; }
};

// Geometry helpers ---------------------------------------------------------

struct Dims {
  int64_t nx, ny, nz;
  int64_t pitch;   // elements between consecutive (x, y) rows (>= nz)
  int64_t plane;   // ny * pitch
  int64_t total() const { return nx * plane; }
  int64_t npoints() const { return nx * ny * nz; }
};

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// Row pitch: rows start 128-byte aligned (and the pitch is a multiple of 16
// bytes as TMA requires).
inline Dims make_dims(const int64_t shape[3], size_t elem) {
  Dims d;
  d.nx = shape[0];
  d.ny = shape[1];
  d.nz = shape[2];
  const int64_t per128 = 128 / (int64_t)elem;
  d.pitch = round_up(d.nz, per128);
  d.plane = d.ny * d.pitch;
  return d;
}

// Inspector internals ------------------------------------------------------

struct Support {
  int64_t shape[3];
  double spacing[3], origin[3];
  int64_t n_points = 0;          // number of sparse points (sources/receivers)
  int64_t K = 0;                 // affected grid points
  int64_t M = 0;                 // kept (point, owner) entries
  bool keep_zero = false;
  // stencils of the sparse points
  DevBuf<int64_t> idx;           // n*8*3
  DevBuf<double> w;              // n*8
  // kept entries, sorted by (linear point key, entry index)
  DevBuf<int64_t> ent_key;       // M linear keys x*ny*nz + y*nz + z
  DevBuf<int32_t> ent_entry;     // M original entry index (owner*8 + corner)
  DevBuf<int64_t> ent_point;     // M point id (0..K-1)
  DevBuf<int64_t> seg_start;     // K+1 first entry of each point
  DevBuf<int64_t> keys;          // K unique linear keys (lexicographic)
  DevBuf<int64_t> row_ptr;       // nx*ny+1
  DevBuf<int32_t> nnz;           // nx*ny
};

void support_build(Support& s, const double* coords_host, int64_t n,
                   const stb_geometry& g, bool keep_zero, cudaStream_t st);
void support_from_points(Support& s, const int64_t* points_host, int64_t n,
                         const stb_geometry& g, cudaStream_t st);
void stencils_compute(const double* coords_dev, int64_t n, const stb_geometry& g,
                      int64_t margin, int64_t* idx_dev, double* w_dev, cudaStream_t st);
// src_dcmp on the device (nt x K, f64)
void support_decompose_dev(const Support& s, const double* wav_dev, int64_t nt_w,
                           const double* scale_dev, int64_t nt, double* out_dev,
                           cudaStream_t st);

void support_points_host(const Support& s, int64_t* points, cudaStream_t st);
void support_compress_host(const Support& s, int32_t* nnz, int64_t* row_ptr, int64_t* flat_z,
                           int32_t* flat_id, cudaStream_t st);
void support_masks_host(const Support& s, uint8_t* sm, int32_t* sid, cudaStream_t st);
void support_entries_host(const Support& s, int64_t* points, int64_t* owner, double* w,
                          cudaStream_t st);

}  // namespace stb

// Propagator handle (opaque to the C ABI) -----------------------------------

struct stb_prop_s {
  virtual ~stb_prop_s() = default;
  virtual void set_sources(stb::Support& s, const double* wav, int64_t nt_w,
                           const double* scale, int64_t nt) = 0;
  virtual void set_receivers(const double* coords, int64_t nrec) = 0;
  // field the receivers record (default: the reference's -- u / txx / p)
  virtual void set_receiver_field(int field) {
    STB_REQUIRE(field == 0, STB_ERR_ARG, "this handle records field 0 only");
  }
  virtual void run(int64_t t0, int64_t nsteps, int k, double* rec_out, int64_t* bad_step) = 0;
  virtual void read_field(int field, int64_t t, void* out) = 0;
  virtual void level_ptr(int field, int64_t t, void** dev, int64_t* plane, int64_t* pitch) = 0;
  virtual void reset() = 0;
  virtual void stats(int64_t* launches, double* ms, int64_t* updates, int64_t* all_launches,
                     double* run_ms) = 0;
  virtual std::string describe(int k) = 0;
  // deepest time_height one fused pass supports (requests above it are
  // split into blocks of this depth; schedule.py:171-207 accepts any T)
  virtual int max_time_height() const { return 1; }
  // max of the velocity the handle was built from (NaN: not known)
  virtual double velocity_max() const { return NAN; }
  // local field shape (x slab) and element size, for host-side copies
  virtual void field_info(int64_t shape[3], int* elem_bytes) = 0;
  // asynchronous stepping (multi-GPU x slabs): enqueue on stream() without
  // host synchronisation; traces and guard flags stay on the device until
  // async_finish.  Default: unsupported.
  virtual void* stream() { return nullptr; }
  virtual void set_damping(const double* const*) { throw_unsupported(); }
  virtual void async_begin(int64_t, int64_t) { throw_unsupported(); }
  virtual void step_async(int64_t, int, int64_t, int64_t) { throw_unsupported(); }
  virtual void step_async_peers(int64_t, int64_t, int64_t, const stb_peer_halo*) {
    throw_unsupported();
  }
  // elastic: one half step (0 = v, 1 = tau + injection) over local planes
  virtual void half_step_async(int64_t, int, int64_t, int64_t) { throw_unsupported(); }
  virtual void gather_async(int64_t, int) { throw_unsupported(); }
  virtual void async_finish(double*, int64_t*) { throw_unsupported(); }

 protected:
  [[noreturn]] static void throw_unsupported() {
    throw stb::Error(STB_ERR_ARG, "this handle does not support that asynchronous "
                                  "stepping call");
  }
};

struct stb_support_s {
  stb::Support s;
};

stb_prop_s* make_acoustic(const stb_acoustic_desc& d);
stb_prop_s* make_elastic(const stb_elastic_desc& d);
stb_prop_s* make_tti(const stb_tti_desc& d);
