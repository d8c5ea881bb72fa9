// Isotropic acoustic propagator (AcousticModel / acoustic_update,
// physics.py:124-213) with fused sparse operators.
//
// Per point, in the reference's exact IEEE order (physics.py:199-213):
//   lap = u1*c0;  for a in (x,y,z) active: for r in 1..R:
//                 lap = lap + (u1[+r] + u1[-r]) * c[a][r]
//   lap = lap*inv;  o = ((u1*2) - u0) + lap;  o = o*fac
// with fac = min(fx[x], fy[y], fz[z]) == f(1/(1+dt*max_a profile_a)) bit for
// bit (1-D tables), so the sponge costs no HBM stream.
//
// Device paths, all bitwise equal in EXACT mode:
//   fused      fp32, 3-D grids, R in {1, 2, 4, 6}; source injection fused
//              into the sweep, receivers gathered on a second stream.
//              K = 1: acoustic_fused<R,1> (the default; ~91 % of HBM at so=8).
//              K = 2: acoustic_wtb<R,2> (acoustic_wtb.cuh), the two-level
//              wavefront kernel with warp-specialised levels.  time_height = 0
//              measures K on the run's first blocks.
//   reference  thread-per-point kernel for fp64 and degenerate grids.
// Time level t lives in buffer t mod NB (NB = 6: distinct inputs/outputs
// for every K <= 4).
#include <climits>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <unordered_map>

#include <cub/cub.cuh>

#include "acoustic_fused.cuh"
#include "acoustic_kernels.cuh"
#include "acoustic_wtb.cuh"
#include "sparse_ops.cuh"

namespace stb {

namespace {

inline unsigned g1(int64_t n, int b = 256) { return (unsigned)((n + b - 1) / b); }

// order-preserving int64 key of a double (signed integer order == numeric
// order for non-NaN values), for atomicMax
__device__ __forceinline__ long long dkey(double x) {
  const long long b = __double_as_longlong(x);
  return b >= 0 ? b : b ^ 0x7fffffffffffffffLL;
}

template <typename T>
__global__ void inv_from_velocity_kernel(const double* __restrict__ v, const double* __restrict__ m,
                                         double dt2, Dims d, T* __restrict__ inv, int* bad_m,
                                         long long* vmax_key, int* v_nan) {
  const int64_t n = d.nx * d.ny * d.nz;
  long long mk = LLONG_MIN;
  int nan = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double mm;
    if (v) {
      const double vi = v[i];
      mm = rdiv(1.0, rmul(vi, vi));            // engine.py:243: 1/v**2
      nan |= vi != vi;
      mk = max(mk, dkey(vi));                  // max(v) for the sponge decay
    } else {
      mm = m[i];
    }
    if (mm <= 0.0) atomicExch(bad_m, 1);      // physics.py:149-150
    const int64_t z = i % d.nz, xy = i / d.nz;
    inv[xy * d.pitch + z] = from_f64<T>(rdiv(dt2, mm));   // physics.py:151
  }
  if (v) {
    for (int o = 16; o > 0; o >>= 1) {
      mk = max(mk, __shfl_xor_sync(0xffffffffu, mk, o));
      nan |= __shfl_xor_sync(0xffffffffu, nan, o);
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMax(vmax_key, mk);
      if (nan) atomicExch(v_nan, 1);
    }
  }
}

template <typename T>
__global__ void table_kernel(const double* __restrict__ src, int64_t n, T* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src ? from_f64<T>(src[i]) : T(1);
}

template <typename T>
__global__ void to_dtype_kernel(const double* __restrict__ src, int64_t n, T* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = from_f64<T>(src[i]);
}

__global__ void keys_to_offsets_kernel(const int64_t* __restrict__ keys, int64_t n, Dims d,
                                       int64_t* __restrict__ off) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t k = keys[i];
  const int64_t z = k % d.nz, xy = k / d.nz;
  off[i] = xy * d.pitch + z;
}

__global__ void shift_keys_kernel(const int64_t* __restrict__ keys, int64_t n, int64_t shift,
                                  int64_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = keys[i] - shift;
}

__global__ void idx_to_offsets_slab_kernel(const int64_t* __restrict__ idx, int64_t n8, Dims d,
                                           int64_t x_begin, int64_t* __restrict__ off,
                                           int* bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n8) return;
  const int64_t x = idx[i * 3] - x_begin;
  if (x < 0 || x >= d.nx) {
    atomicExch(bad, 1);
    off[i] = 0;
    return;
  }
  off[i] = (x * d.ny + idx[i * 3 + 1]) * d.pitch + idx[i * 3 + 2];
}



__global__ void plane_count_kernel(const int64_t* __restrict__ row_ptr, int64_t nx, int64_t ny,
                                   int* __restrict__ plane) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x < nx) plane[x] = (int)(row_ptr[(x + 1) * ny] - row_ptr[x * ny]);
}



// Per-tile source entry lists: point k (lexicographic id) is listed for every
// (TY x TZ) output tile whose level-1 region (tile widened by hy/hz) holds it.
__global__ void tile_count_kernel(const int64_t* __restrict__ keys, int64_t K, Dims d, int TY,
                                  int TZ, int hy, int hz, int nty, int ntz,
                                  int* __restrict__ cnt) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int64_t key = keys[k];
  const int z = (int)(key % d.nz), y = (int)((key / d.nz) % d.ny);
  int c = 0;
  for (int iy = max(0, (y - hy) / TY - 1); iy <= min(nty - 1, (y + hy) / TY + 1); ++iy)
    for (int iz = max(0, (z - hz) / TZ - 1); iz <= min(ntz - 1, (z + hz) / TZ + 1); ++iz)
      if (y >= iy * TY - hy && y < iy * TY + TY + hy && z >= iz * TZ - hz && z < iz * TZ + TZ + hz)
        ++c;
  cnt[k] = c;
}

__global__ void tile_fill_kernel(const int64_t* __restrict__ keys, int64_t K, Dims d, int TY,
                                 int TZ, int hy, int hz, int nty, int ntz,
                                 const int* __restrict__ off, int* __restrict__ tkey,
                                 int4* __restrict__ ent) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int64_t key = keys[k];
  const int z = (int)(key % d.nz), y = (int)((key / d.nz) % d.ny);
  const int x = (int)(key / (d.nz * d.ny));
  int o = off[k];
  for (int iy = max(0, (y - hy) / TY - 1); iy <= min(nty - 1, (y + hy) / TY + 1); ++iy)
    for (int iz = max(0, (z - hz) / TZ - 1); iz <= min(ntz - 1, (z + hz) / TZ + 1); ++iz)
      if (y >= iy * TY - hy && y < iy * TY + TY + hy && z >= iz * TZ - hz && z < iz * TZ + TZ + hz) {
        tkey[o] = iy * ntz + iz;
        ent[o] = make_int4(x, y, z, (int)k);
        ++o;
      }
}

// Per-thread source lists for the fused kernel of depth K: entry e of the
// per-tile list (tile-major, x-ordered within a tile) goes to the consumer
// thread (row, g) of that K's extended tile that owns its (y, z) point;
// key = tile * nwork + row * g1 + g (INT_MAX: outside), value {x, id*4 + zz}.
__global__ void thr_key_kernel(const int4* __restrict__ list, const int* __restrict__ tile_ptr,
                               int ntiles, int64_t n, int ntz, int TY, int TZ, int hy1, int hz1,
                               int hy1_rows, int g1, int* __restrict__ key,
                               int2* __restrict__ val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lo = 0, hi = ntiles;                      // tile of entry i: last t with ptr[t] <= i
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (tile_ptr[mid] <= i) lo = mid; else hi = mid;
  }
  const int t = lo;
  const int4 e = list[i];
  const int y0 = (t / ntz) * TY, z0 = (t % ntz) * TZ;
  const int row = e.y - (y0 - hy1), dz = e.z - (z0 - hz1);
  if (row < 0 || row >= hy1_rows || dz < 0 || dz >= 4 * g1) {
    key[i] = INT_MAX;
    val[i] = make_int2(0, 0);
    return;
  }
  key[i] = t * (hy1_rows * g1) + row * g1 + dz / 4;
  val[i] = make_int2(e.x, e.w * 4 + (dz & 3));
}

__global__ void tile_ptr_kernel(const int* __restrict__ tkey, int64_t n, int ntiles,
                                int* __restrict__ ptr) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  int64_t lo = 0, hi = n;              // first index with tkey >= t
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (tkey[mid] < t) lo = mid + 1; else hi = mid;
  }
  ptr[t] = (int)lo;
}

// Per-thread source lists for the wavefront kernels (acoustic_wtb, 1 or 2 levels):
// entry e of the per-tile list is keyed once for the level-1 thread owning
// its (y, z) point in the tile widened by (hy1, hz1) and once for the
// level-2 thread owning it in the tile itself (rows per thread ry); value
// {x, id*8 + (row % ry)*4 + (dz % 4)}.  Slots per tile: n1 + n2.
__global__ void wtb_key_kernel(const int4* __restrict__ list, const int* __restrict__ tile_ptr,
                               int ntiles, int64_t n, int ntz, int TY, int TZ, int hy1, int hz1,
                               int ry, int g1, int n1, int n2, int* __restrict__ key,
                               int2* __restrict__ val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lo = 0, hi = ntiles;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (tile_ptr[mid] <= i) lo = mid; else hi = mid;
  }
  const int t = lo;
  const int4 e = list[i];
  const int y0 = (t / ntz) * TY, z0 = (t % ntz) * TZ;
  const int base = t * (n1 + n2);
  int row = e.y - (y0 - hy1), dz = e.z - (z0 - hz1);
  if (row >= 0 && row < TY + 2 * hy1 && dz >= 0 && dz < TZ + 2 * hz1) {
    key[2 * i] = base + (row / ry) * g1 + dz / 4;
    val[2 * i] = make_int2(e.x, e.w * 8 + (row % ry) * 4 + (dz & 3));
  } else {
    key[2 * i] = INT_MAX;
    val[2 * i] = make_int2(0, 0);
  }
  row = e.y - y0;
  dz = e.z - z0;
  if (n2 > 0 && row >= 0 && row < TY && dz >= 0 && dz < TZ) {
    key[2 * i + 1] = base + n1 + (row / ry) * (TZ / 4) + dz / 4;
    val[2 * i + 1] = make_int2(e.x, e.w * 8 + (row % ry) * 4 + (dz & 3));
  } else {
    key[2 * i + 1] = INT_MAX;
    val[2 * i + 1] = make_int2(0, 0);
  }
}

// k measured by time_height = 0, remembered per (device, grid, order,
// arithmetic, medium kind) for the process: a second handle on the same
// configuration (a repeated run(), every shot of a survey) skips the trial.
struct KChoice {
  int k;
  float ms1, ms2;
};
std::mutex g_kcache_mu;
std::map<std::string, KChoice> g_kcache;

constexpr int NB = 6;
#ifndef STB_WTB_RY
#define STB_WTB_RY 0
#endif
constexpr int kWtbRYOverride = STB_WTB_RY;   // build-time A/B of the rows per thread
#ifndef STB_WTB_TY
#define STB_WTB_TY 0
#endif
constexpr int kWtbTYOverride = STB_WTB_TY;   // build-time A/B of the tile height
#ifndef STB_FUSED_TY1
#define STB_FUSED_TY1 32
#endif
constexpr int kFusedTY1 = STB_FUSED_TY1;     // acoustic_fused<R,1> tile height (0: 16)

}  // namespace

template <typename T>
class AcousticProp final : public stb_prop_s {
 public:
  explicit AcousticProp(const stb_acoustic_desc& desc) {
    R_ = desc.space_order / 2;
    arithmetic_ = desc.arithmetic;
    geom_ = desc.geom;
    x_begin_ = desc.x_begin;
    int64_t local_shape[3] = {desc.nx_local > 0 ? desc.nx_local : desc.geom.shape[0],
                              desc.geom.shape[1], desc.geom.shape[2]};
    STB_REQUIRE(x_begin_ >= 0 && x_begin_ + local_shape[0] <= desc.geom.shape[0], STB_ERR_ARG,
                "x slab [x_begin, x_begin + nx_local) leaves the grid");
    d_ = make_dims(local_shape, sizeof(T));
    zero_lo_ = x_begin_ == 0;
    zero_hi_ = x_begin_ + d_.nx == desc.geom.shape[0];
    STB_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    STB_CUDA(cudaStreamCreateWithFlags(&gst_, cudaStreamNonBlocking));
    for (auto& e : gev_) STB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    STB_CUDA(cudaEventCreateWithFlags(&sev_, cudaEventDisableTiming));
    for (int a = 0; a < 3; ++a) active_[a] = desc.active[a] != 0;
    // coefficients, rounded once to T exactly as NumPy's weak-scalar rule
    // rounds the Python floats _center/_lap_terms (physics.py:158-164).
    cf_.c0 = (T)desc.center;
    for (int a = 0; a < 3; ++a)
      for (int r = 0; r < 8; ++r) cf_.c[a][r] = (T)desc.coef[a][r];
    for (int a = 0; a < 3; ++a) cf_.active[a] = active_[a] ? 1 : 0;
    for (auto& b : lvl_) {
      b.alloc(d_.total());
      b.zero(st_);
    }
    if (desc.velocity || desc.m) {
      const int64_t n = d_.npoints();
      DevBuf<double> tmp(n);
      tmp.upload(desc.velocity ? desc.velocity : desc.m, n, st_);
      inv_.alloc(d_.total());
      inv_.zero(st_);
      // flags[0]: m <= 0, flags[1]: NaN velocity; vkey: max(v) key
      DevBuf<int> flags(2);
      flags.zero(st_);
      DevBuf<long long> vkey(1);
      const long long lo = LLONG_MIN;
      STB_CUDA(cudaMemcpyAsync(vkey.p, &lo, sizeof(lo), cudaMemcpyHostToDevice, st_));
      inv_from_velocity_kernel<T><<<1184, 256, 0, st_>>>(desc.velocity ? tmp.p : nullptr,
                                                         desc.velocity ? nullptr : tmp.p,
                                                         desc.dt2, d_, inv_.p, flags.p, vkey.p,
                                                         flags.p + 1);
      STB_CHECK_LAUNCH();
      int hf[2] = {0, 0};
      long long hk = lo;
      flags.download(hf, 2, st_);
      vkey.download(&hk, 1, st_);
      STB_CUDA(cudaStreamSynchronize(st_));
      STB_REQUIRE(hf[0] == 0, STB_ERR_ARG, "m must be positive everywhere");
      if (desc.velocity) {
        const long long b = hk >= 0 ? hk : hk ^ 0x7fffffffffffffffLL;
        double vm;
        std::memcpy(&vm, &b, sizeof(vm));
        vmax_ = hf[1] ? NAN : vm;             // np.max propagates NaN
      }
    } else {
      inv_scalar_ = (T)desc.inv_scalar;
    }
    set_damping(desc.damp);
    choose_path();
  }

  void set_damping(const double* const* damp) override {
    has_fac_ = damp[0] || damp[1] || damp[2];
    const int64_t n3[3] = {d_.nx, d_.ny, d_.nz};
    for (int a = 0; a < 3; ++a) {
      if (!fac_[a].p) fac_[a].alloc(n3[a]);
      DevBuf<double> tmp(damp[a] ? n3[a] : 0);
      // the x table is global: take this slab's planes
      if (damp[a]) tmp.upload(damp[a] + (a == 0 ? x_begin_ : 0), n3[a], st_);
      table_kernel<T><<<g1(n3[a]), 256, 0, st_>>>(damp[a] ? tmp.p : nullptr, n3[a], fac_[a].p);
      STB_CHECK_LAUNCH();
      STB_CUDA(cudaStreamSynchronize(st_));
    }
  }

  ~AcousticProp() override {
    // drain in-flight work: buffers are freed on stream 0, which a
    // non-blocking stream does not order against
    if (st_) cudaStreamSynchronize(st_);
    if (gst_) cudaStreamSynchronize(gst_);
    for (auto& e : events_) cudaEventDestroy(e);
    for (auto& e : run_ev_)
      if (e) cudaEventDestroy(e);
    for (auto& e : gev_)
      if (e) cudaEventDestroy(e);
    if (sev_) cudaEventDestroy(sev_);
    for (auto& e : cev_) cudaEventDestroy(e);
    if (cst_) {
      cudaStreamSynchronize(cst_);
      cudaStreamDestroy(cst_);
    }
    if (gst_) cudaStreamDestroy(gst_);
    if (st_) cudaStreamDestroy(st_);
  }

  void set_sources(Support& s, const double* wav, int64_t nt_w, const double* scale,
                   int64_t nt) override {
    check_same_geometry(s);
    src_nt_ = nt;
    K_ = 0;
    if (s.K == 0) return;
    // points of this slab: ids [k_lo, k_hi) of the global lexicographic list
    const int64_t plane = geom_.shape[1] * geom_.shape[2];
    std::vector<int64_t> rp_lohi(2);
    STB_CUDA(cudaMemcpyAsync(&rp_lohi[0], s.row_ptr.p + x_begin_ * geom_.shape[1],
                             sizeof(int64_t), cudaMemcpyDeviceToHost, st_));
    STB_CUDA(cudaMemcpyAsync(&rp_lohi[1], s.row_ptr.p + (x_begin_ + d_.nx) * geom_.shape[1],
                             sizeof(int64_t), cudaMemcpyDeviceToHost, st_));
    STB_CUDA(cudaStreamSynchronize(st_));
    const int64_t k_lo = rp_lohi[0], k_hi = rp_lohi[1];
    K_ = k_hi - k_lo;
    if (K_ == 0) return;
    STB_REQUIRE(K_ < INT32_MAX, STB_ERR_ARG, "too many affected source points");
    DevBuf<double> dwav(nt_w * s.n_points), dscale(s.n_points), dc(nt * s.K);
    dwav.upload(wav, nt_w * s.n_points, st_);
    dscale.upload(scale, s.n_points, st_);
    support_decompose_dev(s, dwav.p, nt_w, dscale.p, nt, dc.p, st_);
    DevBuf<double> dloc(nt * K_);
    STB_CUDA(cudaMemcpy2DAsync(dloc.p, K_ * sizeof(double), dc.p + k_lo, s.K * sizeof(double),
                               K_ * sizeof(double), nt, cudaMemcpyDeviceToDevice, st_));
    series_.alloc(nt * K_);
    to_dtype_kernel<T><<<g1(nt * K_), 256, 0, st_>>>(dloc.p, nt * K_, series_.p);
    // local keys (x shifted to the slab)
    src_keys_.alloc(K_);
    shift_keys_kernel<<<g1(K_), 256, 0, st_>>>(s.keys.p + k_lo, K_, x_begin_ * plane,
                                               src_keys_.p);
    src_off_.alloc(K_);
    keys_to_offsets_kernel<<<g1(K_), 256, 0, st_>>>(src_keys_.p, K_, d_, src_off_.p);
    STB_CHECK_LAUNCH();
    // per-plane counts for the fused epilogue (from the global CSR)
    src_plane_.alloc(d_.nx);
    plane_count_kernel<<<g1(d_.nx), 256, 0, st_>>>(s.row_ptr.p + x_begin_ * geom_.shape[1],
                                                   d_.nx, d_.ny, src_plane_.p);
    STB_CHECK_LAUNCH();
    if (path_ == Path::Fused) build_tile_lists();
    STB_CUDA(cudaStreamSynchronize(st_));
  }

  // Per-tile lists for the fused kernels (halo of the deepest supported K).
  void build_tile_lists() {
    const int hy = (max_k_ - 1) * R_;
    int hz = 0;
    for (int j = 1; j < max_k_; ++j) hz = (hz + R_ + 3) / 4 * 4;
    src_n_ = tile_lists(fused_ty(R_), kTZ, hy, hz, src_list_, src_tile_ptr_);
    thr_.clear();
    wtb_thr_[0].reset();
    wtb_thr_[1].reset();
  }

  // Point k of the inspector support is listed for every TY x TZ tile whose
  // region widened by (hy, hz) holds it; lists tile-major, x-ordered within a
  // tile (stable sort of the lexicographic support).  Returns the entry count.
  int64_t tile_lists(int TY, int TZ, int hy, int hz, DevBuf<int4>& list, DevBuf<int>& tptr) {
    const int nty = (int)((d_.ny + TY - 1) / TY), ntz = (int)((d_.nz + TZ - 1) / TZ);
    const int ntiles = nty * ntz;
    DevBuf<int> cnt(K_), off(K_ + 1);
    tile_count_kernel<<<g1(K_), 256, 0, st_>>>(src_keys_.p, K_, d_, TY, TZ, hy, hz, nty, ntz,
                                               cnt.p);
    STB_CHECK_LAUNCH();
    size_t tb = 0;
    STB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, off.p, (int)K_, st_));
    DevBuf<uint8_t> tmp(tb);
    STB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, off.p, (int)K_, st_));
    int last_off = 0, last_cnt = 0;
    STB_CUDA(cudaMemcpyAsync(&last_off, off.p + K_ - 1, sizeof(int), cudaMemcpyDeviceToHost, st_));
    STB_CUDA(cudaMemcpyAsync(&last_cnt, cnt.p + K_ - 1, sizeof(int), cudaMemcpyDeviceToHost, st_));
    STB_CUDA(cudaStreamSynchronize(st_));
    const int64_t n = (int64_t)last_off + last_cnt;
    DevBuf<int> tkey(n), tkey2(n);
    DevBuf<int4> ent(n);
    list.alloc(n);
    tile_fill_kernel<<<g1(K_), 256, 0, st_>>>(src_keys_.p, K_, d_, TY, TZ, hy, hz, nty, ntz,
                                              off.p, tkey.p, ent.p);
    STB_CHECK_LAUNCH();
    int bits = 1;
    while ((1 << bits) <= ntiles) ++bits;
    tb = 0;
    STB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, tkey.p, tkey2.p, ent.p, list.p, (int)n,
                                             0, bits, st_));
    tmp.alloc(tb);
    STB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, tkey.p, tkey2.p, ent.p, list.p, (int)n,
                                             0, bits, st_));
    tptr.alloc(ntiles + 1);
    tile_ptr_kernel<<<g1(ntiles + 1), 256, 0, st_>>>(tkey2.p, n, ntiles, tptr.p);
    STB_CHECK_LAUNCH();
    STB_CUDA(cudaStreamSynchronize(st_));
    return n;
  }

  // Per-thread lists for the fused kernel <R, K> (built on first use).
  struct ThrLists {
    DevBuf<int> ptr;     // ntiles * nwork + 1
    DevBuf<int2> list;
  };
  template <int R, int K>
  const ThrLists* thr_lists() {
    if (!K_ || src_n_ == 0) return nullptr;
    auto it = thr_.find(K);
    if (it != thr_.end()) return it->second.get();
    using C = FusedCfg<R, K, fused_ty(R), kTZ, pf_for(R)>;
    const int nty = (int)((d_.ny + C::TY_ - 1) / C::TY_), ntz = (int)((d_.nz + kTZ - 1) / kTZ);
    const int ntiles = nty * ntz;
    static_assert(K == 1, "acoustic_fused runs one step per pass; K = 2 is acoustic_wtb");
    const int4* tl = src_list_.p;
    const int* tp = src_tile_ptr_.p;
    int64_t n = src_n_;
    auto L = std::make_unique<ThrLists>();
    if (n == 0) {
      L->ptr.alloc(ntiles * C::NWORK + 1);
      L->ptr.zero(st_);
      STB_CUDA(cudaStreamSynchronize(st_));
      return thr_.emplace(K, std::move(L)).first->second.get();
    }
    DevBuf<int> key(n), key2(n);
    DevBuf<int2> val(n);
    L->list.alloc(n);
    thr_key_kernel<<<g1(n), 256, 0, st_>>>(tl, tp, ntiles, n, ntz, C::TY_,
                                           kTZ, C::hy(1), C::hz(1), C::HY1, C::G1, key.p, val.p);
    STB_CHECK_LAUNCH();
    size_t tb = 0;
    STB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key2.p, val.p, L->list.p,
                                             (int)n, 0, 32, st_));
    DevBuf<uint8_t> tmp(tb);
    STB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key2.p, val.p, L->list.p,
                                             (int)n, 0, 32, st_));
    const int nk = ntiles * C::NWORK;
    L->ptr.alloc(nk + 1);
    tile_ptr_kernel<<<g1(nk + 1), 256, 0, st_>>>(key2.p, n, nk, L->ptr.p);
    STB_CHECK_LAUNCH();
    STB_CUDA(cudaStreamSynchronize(st_));
    return thr_.emplace(K, std::move(L)).first->second.get();
  }

  // Per-thread lists for the two-level wavefront kernel (built on first use).
  template <int R, int LV>
  const ThrLists* wtb_thr_lists() {
    auto& cache = wtb_thr_[LV - 1];
    if (!K_ || src_n_ == 0) return nullptr;
    if (cache) return cache.get();
    using C = WtbCfg<R, LV, wtb_ry(R), kWtbPF, wtb_ty(R, LV)>;
    const int nty = (int)((d_.ny + C::TY - 1) / C::TY), ntz = (int)((d_.nz + kTZ - 1) / kTZ);
    const int ntiles = nty * ntz;
    // tile lists of this kernel's tile shape (the K = 1/2 fused lists when equal)
    DevBuf<int4> own_list;
    DevBuf<int> own_ptr;
    const int4* tl = src_list_.p;
    const int* tp = src_tile_ptr_.p;
    int64_t ne = src_n_;
    if (C::TY != fused_ty(R) || C::H1 != (max_k_ - 1) * R || C::HZ1 != (max_k_ > 1 ? (R + 3) / 4 * 4 : 0)) {
      ne = tile_lists(C::TY, kTZ, C::H1, C::HZ1, own_list, own_ptr);
      tl = own_list.p;
      tp = own_ptr.p;
    }
    auto L = std::make_unique<ThrLists>();
    if (ne == 0) {
      L->ptr.alloc(ntiles * C::NTHR + 1);
      L->ptr.zero(st_);
      STB_CUDA(cudaStreamSynchronize(st_));
      cache = std::move(L);
      return cache.get();
    }
    const int64_t n = 2 * ne;
    DevBuf<int> key(n), key2(n);
    DevBuf<int2> val(n);
    L->list.alloc(n);
    wtb_key_kernel<<<g1(ne), 256, 0, st_>>>(tl, tp, ntiles, ne, ntz, C::TY, kTZ, C::H1, C::HZ1,
                                            wtb_ry(R), C::G1, C::NW1T, C::NW2T, key.p, val.p);
    STB_CHECK_LAUNCH();
    size_t tb = 0;
    STB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key2.p, val.p, L->list.p,
                                             (int)n, 0, 32, st_));
    DevBuf<uint8_t> tmp(tb);
    STB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key2.p, val.p, L->list.p,
                                             (int)n, 0, 32, st_));
    const int nk = ntiles * C::NTHR;
    L->ptr.alloc(nk + 1);
    tile_ptr_kernel<<<g1(nk + 1), 256, 0, st_>>>(key2.p, n, nk, L->ptr.p);
    STB_CHECK_LAUNCH();
    STB_CUDA(cudaStreamSynchronize(st_));
    cache = std::move(L);
    return cache.get();
  }

  void set_receivers(const double* coords, int64_t nrec) override {
    nrec_ = nrec;
    if (nrec == 0) return;
    // stencils on the GLOBAL geometry (bitwise the reference's weights), then
    // corner planes shifted into this slab
    DevBuf<double> dc(nrec * 3);
    dc.upload(coords, nrec * 3, st_);
    DevBuf<int64_t> idx(nrec * 24);
    rec_w_.alloc(nrec * 8);
    stencils_compute(dc.p, nrec, geom_, -1, idx.p, rec_w_.p, st_);
    rec_off_.alloc(nrec * 8);
    DevBuf<int> bad(1);
    bad.zero(st_);
    idx_to_offsets_slab_kernel<<<g1(nrec * 8), 256, 0, st_>>>(idx.p, nrec * 8, d_, x_begin_,
                                                              rec_off_.p, bad.p);
    STB_CHECK_LAUNCH();
    int hb = 0;
    bad.download(&hb, 1, st_);
    STB_CUDA(cudaStreamSynchronize(st_));
    STB_REQUIRE(hb == 0, STB_ERR_ARG, "receiver corners leave this x slab");
  }

  void run(int64_t t0, int64_t nsteps, int k, double* rec_out, int64_t* bad_step) override {
    if (bad_step) *bad_step = -1;
    launches_ = all_launches_ = 0;
    updates_ = 0;
    run_ms_ = 0.0;
    if (nsteps <= 0) return;
    STB_REQUIRE(k >= 0, STB_ERR_PLAN, "time_height must be >= 1");
    STB_REQUIRE(K_ == 0 || t0 + nsteps <= src_nt_, STB_ERR_ARG,
                "run extends past the decomposed source series");
    // time_height = 0 and k not measured yet: time the first blocks of this
    // very run (K = 1, 1, 2, 2 -- real steps, the second of each kind timed
    // after its first-use costs) and continue with the faster; short runs
    // use the separate idempotent trial (autotune_k)
    const bool pinned_k = std::getenv("STB_DEFAULT_K") ||
                          (std::getenv("STB_AUTOTUNE") && std::atoi(std::getenv("STB_AUTOTUNE")) == 0);
    if (k == 0 && !tuned_k_ && path_ == Path::Fused && max_k_ >= 2 && !pinned_k) {
      std::lock_guard<std::mutex> lk(g_kcache_mu);
      auto it = g_kcache.find(kcache_key());
      if (it != g_kcache.end()) {
        tuned_k_ = it->second.k;
        tune_ms_[0] = it->second.ms1;
        tune_ms_[1] = it->second.ms2;
      }
    }
    bool trial = k == 0 && !tuned_k_ && path_ == Path::Fused && max_k_ >= 2 && nsteps >= 6 &&
                 !std::getenv("STB_DEFAULT_K") &&
                 !(std::getenv("STB_AUTOTUNE") && std::atoi(std::getenv("STB_AUTOTUNE")) == 0);
    if (k == 0 && !trial) autotune_k(t0);
    int kk = resolve_k(k);
    if (nrec_ && (int64_t)rec_dev_.n < nsteps * nrec_) rec_dev_.alloc(nsteps * nrec_);
    std::vector<int64_t> guard_steps;
    for (int64_t t = t0; t < t0 + nsteps; ++t)
      if (t > 0 && t % 32 == 0) guard_steps.push_back(t);
    if ((int64_t)guards_.n < (int64_t)guard_steps.size() + 1) guards_.alloc(guard_steps.size() + 1);
    guards_.zero(st_);
    ensure_events(nsteps + 1);
    STB_CUDA(cudaEventRecord(run_ev_[0], st_));
    // traces of completed step chunks are copied out (copy stream) while
    // later steps compute; chunk c = steps [c*kTraceChunk, ...) of this run
    const bool stream_traces =
        nrec_ && rec_out && (size_t)nsteps * nrec_ * sizeof(double) >= ((size_t)64 << 20);
    std::vector<int64_t> chunk_end;           // exclusive step index (relative)
    size_t gi = 0;
    int64_t t = t0;
    int64_t blk = 0;
    while (t < t0 + nsteps) {
      const int want = trial ? (blk < 2 ? 1 : 2) : kk;
      const int kb = (int)std::min<int64_t>(path_ == Path::Fused ? want : 1, t0 + nsteps - t);
      // guard steps inside this block
      int gmask = 0;
      int* gflag = nullptr;
      for (int j = 0; j < kb; ++j)
        if (gi < guard_steps.size() && guard_steps[gi] == t + j) {
          gmask |= 1 << j;
          gflag = guards_.p + gi;
          ++gi;
        }
      // receivers gather level s on a second stream (overlapping the next
      // steps); the block that rewrites ring slot s first waits for it
      if (nrec_)
        for (int j = 0; j < kb; ++j) STB_CUDA(cudaStreamWaitEvent(st_, gev_[slot(t + j)], 0));
      STB_CUDA(cudaEventRecord(events_[2 * launches_], st_));
      if (path_ == Path::Fused) {
        launch_fused_range(t, kb, gflag, gmask, 0, (int)d_.nx);
      } else {
        launch_reference_step<T>(R_, st_, lvl_[slot(t - 1)].p, lvl_[slot(t - 2)].p,
                                 lvl_[slot(t)].p, inv_.p, inv_scalar_, fac_[0].p, fac_[1].p,
                                 fac_[2].p, has_fac_, cf_, d_);
        if (gflag) {
          nonfinite_kernel<T><<<1184, 256, 0, st_>>>(lvl_[slot(t)].p, d_, gflag);
          STB_CHECK_LAUNCH();
          ++all_launches_;
        }
      }
      STB_CUDA(cudaEventRecord(events_[2 * launches_ + 1], st_));
      ++launches_;
      ++all_launches_;
      if (path_ != Path::Fused && K_) {
        inject_kernel<T><<<g1(K_), 256, 0, st_>>>(lvl_[slot(t)].p, src_off_.p,
                                                  series_.p + t * K_, K_);
        STB_CHECK_LAUNCH();
        ++all_launches_;
      }
      if (nrec_) {
        STB_CUDA(cudaEventRecord(sev_, st_));
        STB_CUDA(cudaStreamWaitEvent(gst_, sev_, 0));
        for (int j = 0; j < kb; ++j) {
          // levels t..t+kb-1 are all resident for kb <= 2 (the fused kernel
          // writes the last two levels), so receivers gather from HBM
          double* row = rec_dev_.p + (t + j - t0) * nrec_;
          gather_kernel<T><<<g1(nrec_), 256, 0, gst_>>>(lvl_[slot(t + j)].p, rec_off_.p,
                                                        rec_w_.p, nrec_, row);
          STB_CHECK_LAUNCH();
          STB_CUDA(cudaEventRecord(gev_[slot(t + j)], gst_));
          ++all_launches_;
        }
        const int64_t done = t + kb - t0;
        if (stream_traces && (done / kTraceChunk > (done - kb) / kTraceChunk || t + kb == t0 + nsteps)) {
          const size_t c = chunk_end.size();
          while (cev_.size() <= c) {
            cudaEvent_t e;
            STB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            cev_.push_back(e);
          }
          STB_CUDA(cudaEventRecord(cev_[c], gst_));
          chunk_end.push_back(done);
        }
      }
      t += kb;
      if (trial && ++blk == 4) {
        STB_CUDA(cudaEventSynchronize(events_[7]));
        float m1 = 0.f, m2 = 0.f;
        STB_CUDA(cudaEventElapsedTime(&m1, events_[2], events_[3]));   // block 1: K = 1
        STB_CUDA(cudaEventElapsedTime(&m2, events_[6], events_[7]));   // block 3: K = 2
        tune_ms_[0] = m1;
        tune_ms_[1] = m2 / 2;
        tuned_k_ = tune_ms_[1] < 0.95f * tune_ms_[0] ? 2 : 1;
        remember_k();
        kk = resolve_k(0);
        trial = false;
      }
    }
    if (nrec_) {                              // join the gather stream
      STB_CUDA(cudaEventRecord(sev_, gst_));
      STB_CUDA(cudaStreamWaitEvent(st_, sev_, 0));
    }
    STB_CUDA(cudaEventRecord(run_ev_[1], st_));
    updates_ = nsteps * d_.npoints();
    last_k_ = kk;
    if (stream_traces) {
      if (!cst_) STB_CUDA(cudaStreamCreateWithFlags(&cst_, cudaStreamNonBlocking));
      int64_t r0 = 0;
      for (size_t c = 0; c < chunk_end.size(); ++c) {
        STB_CUDA(cudaStreamWaitEvent(cst_, cev_[c], 0));
        device_to_host(rec_out + r0 * nrec_, rec_dev_.p + r0 * nrec_,
                       (size_t)(chunk_end[c] - r0) * nrec_ * sizeof(double), cst_);
        r0 = chunk_end[c];
      }
    } else if (nrec_ && rec_out) {
      rec_dev_.download(rec_out, nsteps * nrec_, st_);
    }
    std::vector<int> gh(guard_steps.size() + 1, 0);
    if (!guard_steps.empty()) guards_.download(gh.data(), guard_steps.size(), st_);
    STB_CUDA(cudaStreamSynchronize(st_));
    float rm = 0.f;
    STB_CUDA(cudaEventElapsedTime(&rm, run_ev_[0], run_ev_[1]));
    run_ms_ = rm;
    for (size_t i = 0; i < guard_steps.size(); ++i) {
      if (gh[i]) {
        if (bad_step) *bad_step = guard_steps[i];
        std::ostringstream os;
        os << "non-finite values in field group 'u' at step " << guard_steps[i];
        throw Error(STB_ERR_UNSTABLE, os.str());
      }
    }
  }

  // ---------------------------------------------------------------- async
  void* stream() override { return st_; }

  void async_begin(int64_t t0, int64_t nsteps) override {
    STB_REQUIRE(path_ == Path::Fused, STB_ERR_ARG, "asynchronous stepping needs the fused path");
    STB_REQUIRE(nsteps >= 0, STB_ERR_ARG, "nsteps must be >= 0");
    STB_REQUIRE(K_ == 0 || t0 + nsteps <= src_nt_, STB_ERR_ARG,
                "run extends past the decomposed source series");
    as_t0_ = t0;
    as_n_ = nsteps;
    as_guard_.clear();
    for (int64_t t = t0; t < t0 + nsteps; ++t)
      if (t > 0 && t % 32 == 0) as_guard_.push_back(t);
    if ((int64_t)guards_.n < (int64_t)as_guard_.size() + 1) guards_.alloc(as_guard_.size() + 1);
    guards_.zero(st_);
    if (nrec_ && (int64_t)rec_dev_.n < nsteps * nrec_) rec_dev_.alloc(nsteps * nrec_);
    launches_ = all_launches_ = 0;
    updates_ = 0;
    // up to three ranged launches per step (boundary, boundary, interior)
    ensure_events(3 * nsteps + 1);
    STB_CUDA(cudaEventRecord(run_ev_[0], st_));
    as_open_ = true;
  }

  // steps [t, t + kb) over local planes [x_lo, x_hi) (stencil + fused injection)
  // K = 1 step over local planes [x_lo, x_hi) whose boundary planes are
  // also written into the neighbour slabs' ghost planes (peer memory)
  void step_async_peers(int64_t t, int64_t x_lo, int64_t x_hi, const stb_peer_halo* peers) override {
    STB_REQUIRE(path_ == Path::Fused, STB_ERR_ARG, "peer halo stores need the fused path");
    peers_ = *peers;
    peers_on_ = true;
    try {
      step_async(t, 1, x_lo, x_hi);
    } catch (...) {
      peers_on_ = false;
      throw;
    }
    peers_on_ = false;
  }

  void step_async(int64_t t, int kb, int64_t x_lo, int64_t x_hi) override {
    STB_REQUIRE(as_open_, STB_ERR_ARG, "async_begin first");
    STB_REQUIRE(t >= as_t0_ && kb >= 1 && t + kb <= as_t0_ + as_n_, STB_ERR_ARG,
                "steps outside the async window");
    STB_REQUIRE(kb <= max_k_, STB_ERR_PLAN, "time_height exceeds the fused kernel's depth");
    STB_REQUIRE(0 <= x_lo && x_lo <= x_hi && x_hi <= d_.nx, STB_ERR_ARG, "plane range");
    if (x_hi == x_lo) return;
    int gmask = 0;
    int* gflag = nullptr;
    for (size_t g = 0; g < as_guard_.size(); ++g)
      for (int j = 0; j < kb; ++j)
        if (as_guard_[g] == t + j) {
          gmask |= 1 << j;
          gflag = guards_.p + g;
        }
    STB_REQUIRE(2 * launches_ + 1 < (int64_t)events_.size(), STB_ERR_ARG,
                "more than three launches per step in the async window");
    STB_CUDA(cudaEventRecord(events_[2 * launches_], st_));
    launch_fused_range(t, kb, gflag, gmask, (int)x_lo, (int)x_hi);
    STB_CUDA(cudaEventRecord(events_[2 * launches_ + 1], st_));
    ++launches_;
    ++all_launches_;
    updates_ += (int64_t)kb * (x_hi - x_lo) * d_.ny * d_.nz;
  }

  void gather_async(int64_t t, int kb) override {
    STB_REQUIRE(as_open_, STB_ERR_ARG, "async_begin first");
    if (!nrec_) return;
    for (int j = 0; j < kb; ++j) {
      double* row = rec_dev_.p + (t + j - as_t0_) * nrec_;
      gather_kernel<T><<<g1(nrec_), 256, 0, st_>>>(lvl_[slot(t + j)].p, rec_off_.p, rec_w_.p,
                                                   nrec_, row);
      STB_CHECK_LAUNCH();
      ++all_launches_;
    }
  }

  void async_finish(double* rec_out, int64_t* bad_step) override {
    STB_REQUIRE(as_open_, STB_ERR_ARG, "async_begin first");
    as_open_ = false;
    if (bad_step) *bad_step = -1;
    STB_CUDA(cudaEventRecord(run_ev_[1], st_));
    if (nrec_ && rec_out && as_n_) rec_dev_.download(rec_out, as_n_ * nrec_, st_);
    std::vector<int> gh(as_guard_.size() + 1, 0);
    if (!as_guard_.empty()) guards_.download(gh.data(), as_guard_.size(), st_);
    STB_CUDA(cudaStreamSynchronize(st_));
    float rm = 0.f;
    STB_CUDA(cudaEventElapsedTime(&rm, run_ev_[0], run_ev_[1]));
    run_ms_ = rm;
    for (size_t i = 0; i < as_guard_.size(); ++i)
      if (gh[i]) {
        if (bad_step) *bad_step = as_guard_[i];
        std::ostringstream os;
        os << "non-finite values in field group 'u' at step " << as_guard_[i];
        throw Error(STB_ERR_UNSTABLE, os.str());
      }
  }

  void read_field(int field, int64_t t, void* out) override {
    STB_REQUIRE(field == 0, STB_ERR_ARG, "acoustic handles have one field (u)");
    const T* src = lvl_[slot(t)].p;
    device_to_host_3d(out, src, d_.nz * sizeof(T), d_.ny, d_.nx, d_.pitch * sizeof(T),
                      d_.plane * sizeof(T), st_);
  }

  void level_ptr(int field, int64_t t, void** dev, int64_t* plane, int64_t* pitch) override {
    STB_REQUIRE(field == 0, STB_ERR_ARG, "acoustic handles have one field (u)");
    *dev = lvl_[slot(t)].p;
    if (plane) *plane = d_.plane;
    if (pitch) *pitch = d_.pitch;
  }

  void reset() override {
    for (auto& b : lvl_) b.zero(st_);
    STB_CUDA(cudaStreamSynchronize(st_));
  }

  void stats(int64_t* launches, double* ms, int64_t* updates, int64_t* all_launches,
             double* run_ms) override {
    double total = 0;
    for (int64_t i = 0; i < launches_; ++i) {
      float e = 0;
      STB_CUDA(cudaEventElapsedTime(&e, events_[2 * i], events_[2 * i + 1]));
      total += e;
    }
    if (launches) *launches = launches_;
    if (ms) *ms = total;
    if (updates) *updates = updates_;
    if (all_launches) *all_launches = all_launches_;
    if (run_ms) *run_ms = run_ms_;
  }

  void field_info(int64_t shape[3], int* elem_bytes) override {
    shape[0] = d_.nx;
    shape[1] = d_.ny;
    shape[2] = d_.nz;
    *elem_bytes = (int)sizeof(T);
  }

  std::string describe(int k) override {
    std::ostringstream os;
    const int kk = resolve_k(k);
    const int L = (int)d_.nx;
    if (path_ == Path::Fused && kk == 2) {
      os << "acoustic_wtb<f32,R=" << R_ << ",LV=2,TY=" << wtb_ty(R_) << ",TZ=" << kTZ
         << ",RY=" << wtb_ry(R_)
         << ",PF=" << kWtbPF << "," << (fast_ ? "fma" : "exact") << "> k=2 cx=" << wtb_cx(L)
         << " bytes_per_point=20";
    } else if (path_ == Path::Fused) {
      os << "acoustic_fused<f32,R=" << R_ << ",TY=" << fused_ty(R_) << ",TZ=" << kTZ
         << ",PF=" << pf_for(R_) << "," << (fast_ ? "fma" : "exact") << "> k=" << kk
         << " cx=" << fused_cx(L) << " bytes_per_point=16";
    } else {
      os << "acoustic_reference_step<" << (sizeof(T) == 4 ? "f32" : "f64") << ",R=" << R_
         << "> k=1 bytes_per_point=" << 4 * sizeof(T);
    }
    if (path_ == Path::Fused && k == 0 && tuned_k_ && tune_ms_[0] > 0.f)
      os << " autotuned(ms/step k1=" << tune_ms_[0] << " k2=" << tune_ms_[1] << ")";
    return os.str();
  }

  int max_time_height() const override { return path_ == Path::Fused ? max_k_ : 1; }
  double velocity_max() const override { return vmax_; }

 private:
  enum class Path { Reference, Fused };
  static constexpr int kTY = 16, kTZ = 64;
  // fused-kernel tile height.  K = 1: 32 rows in one CTA of 16 consumer
  // warps -- less y halo per staged plane and room for a deeper prefetch
  // (measured +1 % at so=4/8 and +10 % at so=12 over two 16-row CTAs per
  // SM).
  // R >= 7: 16-row tiles (one CTA of 8 consumer warps): the 2R+1-plane
  // register queue needs more registers than 16 warps of a 32-row tile get
  static constexpr int fused_ty(int R) { return R >= 7 ? 24 : (kFusedTY1 > 0 ? kFusedTY1 : kTY); }
  static constexpr int kWtbPF = 3;                // two-level kernel: TMA prefetch depth
  // rows per thread: 2 (measured at R = 2: RY = 1 gives 21 warps instead of
  // 11 but doubles the per-plane bookkeeping per point, 274 vs 328 GPts/s)
  static constexpr int wtb_ry(int) { return kWtbRYOverride ? kWtbRYOverride : 2; }
  // tile height.  Two levels: 24 at R = 2 (15 warps fit the register file,
  // level-1 redundancy 1.31 instead of 1.41), 16 at R = 4 (160 registers x 12
  // warps).  One level: 32 (8 consumer warps of 2 rows x 4 z points).
  static constexpr int wtb_ty(int R, int LV = 2) {
    return LV == 1 ? (R == 6 ? 28 : 32) : kWtbTYOverride ? kWtbTYOverride : (R <= 2 ? 24 : 16);
  }
  // TMA prefetch depth.  One-CTA 32-row tiles: 4 (R <= 4), 3 (R = 6, whose
  // planes are 40 % larger; measured 4 > 3, 5 at so=8).  Two-CTA 16-row
  // tiles: 3, and 2 at R = 6.
  static constexpr int pf_for(int R) {
    if (fused_ty(R) != kTY) return R >= 6 ? 3 : 4;
    return 2;
  }

  int slot(int64_t t) const { return (int)(((t % NB) + NB) % NB); }

  // time_height = 0: fused steps per launch chosen by measurement on this
  // handle's own grid.  A fused block is idempotent -- it recomputes levels
  // t.. from t-1, t-2 (injection included) into ring slots the real block
  // overwrites anyway -- so K = 1 and K = 2 launches are timed on the live
  // state before the first real step, without perturbing it.
  void autotune_k(int64_t t) {
    if (tuned_k_ || path_ != Path::Fused || max_k_ < 2) return;
    tuned_k_ = default_k_;
    if (std::getenv("STB_DEFAULT_K") || (K_ && t + 2 > src_nt_)) return;
    if (const char* e = std::getenv("STB_AUTOTUNE"))
      if (std::atoi(e) == 0) return;
    cudaEvent_t ev[3];
    for (auto& e : ev) STB_CUDA(cudaEventCreate(&e));
    launch_fused(t, 1, nullptr, 0);             // first launches: module load, maps
    launch_fused(t, 2, nullptr, 0);
    constexpr int kReps = 3;
    STB_CUDA(cudaEventRecord(ev[0], st_));
    for (int i = 0; i < kReps; ++i) launch_fused(t, 1, nullptr, 0);
    STB_CUDA(cudaEventRecord(ev[1], st_));
    for (int i = 0; i < kReps; ++i) launch_fused(t, 2, nullptr, 0);
    STB_CUDA(cudaEventRecord(ev[2], st_));
    STB_CUDA(cudaEventSynchronize(ev[2]));
    float m1 = 0.f, m2 = 0.f;
    STB_CUDA(cudaEventElapsedTime(&m1, ev[0], ev[1]));
    STB_CUDA(cudaEventElapsedTime(&m2, ev[1], ev[2]));
    for (auto& e : ev) cudaEventDestroy(e);
    tune_ms_[0] = m1 / kReps;                   // per step
    tune_ms_[1] = m2 / kReps / 2;
    tuned_k_ = tune_ms_[1] < 0.95f * tune_ms_[0] ? 2 : 1;
    remember_k();
  }

  std::string kcache_key() const {
    int dev = 0;
    cudaGetDevice(&dev);
    std::ostringstream os;
    os << dev << ':' << d_.nx << 'x' << d_.ny << 'x' << d_.nz << ":R" << R_ << ":f" << fast_
       << ":i" << (inv_.p != nullptr) << ":s" << (K_ > 0);
    return os.str();
  }
  void remember_k() {
    std::lock_guard<std::mutex> lk(g_kcache_mu);
    g_kcache[kcache_key()] = KChoice{tuned_k_, tune_ms_[0], tune_ms_[1]};
  }

  // x-chunk length for a launch over L planes: minimise waves x iterations,
  // ceil(c*tiles / slots) * (ceil(L/c) + 2KR), over the chunk count c
  // (592-plane grid: 4 chunks, as before; an 8-rank slab interior of 64
  // planes: 3 chunks instead of 1, i.e. 3.75 instead of 1.25 waves).
  int chunk_len(int L, int K, int ctas_per_sm, int ty = kTY) {
    if (L <= 0) return 1;
    if (std::getenv("STB_NCHUNK")) return cx_len_;
    if (!sm_count_) STB_CUDA(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, 0));
    const int64_t tiles = ((d_.ny + ty - 1) / ty) * ((d_.nz + kTZ - 1) / kTZ);
    const int64_t slots = (int64_t)sm_count_ * ctas_per_sm;
    int best_c = 1;
    int64_t best = INT64_MAX;
    for (int c = 1; c <= std::max(1, L / 8); ++c) {
      const int64_t waves = (c * tiles + slots - 1) / slots;
      const int64_t cost = waves * ((L + c - 1) / c + 2 * K * R_);
      if (cost < best) {
        best = cost;
        best_c = c;
      }
    }
    return (L + best_c - 1) / best_c;
  }

  // x-chunk lengths the launches use (describe() reports the same)
  template <int R>
  int fused_cx_r(int L) {
    using C = FusedCfg<R, 1, fused_ty(R), kTZ, pf_for(R)>;
    return chunk_len(L, 1, C::MINB, fused_ty(R));
  }
  template <int R>
  int wtb_cx_r(int L) {
    using C = WtbCfg<R, 2, wtb_ry(R), kWtbPF, wtb_ty(R, 2)>;
    int cx = chunk_len(L, 2, 1, C::TY);
    if (cx + 4 * R > C::MAXN) cx = C::MAXN - 4 * R;   // per-CTA damping table
    return cx;
  }
  int fused_cx(int L) {
    switch (R_) {
      case 1: return fused_cx_r<1>(L);
      case 2: return fused_cx_r<2>(L);
      case 4: return fused_cx_r<4>(L);
      case 3: return fused_cx_r<3>(L);
      case 5: return fused_cx_r<5>(L);
      case 6: return fused_cx_r<6>(L);
      case 7: return fused_cx_r<7>(L);
      case 8: return fused_cx_r<8>(L);
      default: return L;
    }
  }
  int wtb_cx(int L) {
    switch (R_) {
      case 1: return wtb_cx_r<1>(L);
      case 2: return wtb_cx_r<2>(L);
      case 4: return wtb_cx_r<4>(L);
      default: return L;
    }
  }

  int resolve_k(int k) const {
    if (path_ != Path::Fused) return 1;
    int kk = k < 1 ? (tuned_k_ ? tuned_k_ : default_k_) : k;
    if (kk > max_k_) kk = max_k_;
    return kk;
  }

  // fp32 grids with three active axes use the TMA kernels; fp64 and
  // degenerate (1-D/2-D) grids run the reference-order kernel.
  void choose_path() {
    path_ = Path::Reference;
    if constexpr (sizeof(T) == 4) {
      if (!(active_[0] && active_[1] && active_[2])) return;
      if (R_ < 1 || R_ > 8) return;
      const char* e = std::getenv("STB_PATH");
      if (e && std::strcmp(e, "reference") == 0) return;
      tcf_.c0 = cf_.c0;
      tcf_.nz = -0.0f;
      for (int r = 0; r < 8; ++r) {
        tcf_.cx[r] = cf_.c[0][r];
        tcf_.cy[r] = cf_.c[1][r];
        tcf_.cz[r] = cf_.c[2][r];
      }
      int64_t nch = (d_.nx + 149) / 150;
      if (const char* c = std::getenv("STB_NCHUNK")) nch = std::atoi(c);
      if (nch < 1) nch = 1;
      cx_len_ = (int)((d_.nx + nch - 1) / nch);
      fast_ = arithmetic_ == 1;
      max_k_ = (R_ == 4 || R_ == 2 || R_ == 1) ? 2 : 1;
      default_k_ = 1;
      if (const char* kd = std::getenv("STB_DEFAULT_K")) default_k_ = std::atoi(kd);
      if (default_k_ < 1) default_k_ = 1;
      if (default_k_ > max_k_) default_k_ = max_k_;
      path_ = Path::Fused;
    }
  }

  template <int R>
  void fused_maps(FusedMaps& m, int s_l0, int s_lm1) {
    using Cf = FusedCfg<R, 1, fused_ty(R), kTZ, pf_for(R)>;
    m.l0 = make_map3d_f32(reinterpret_cast<const float*>(lvl_[s_l0].p), d_, Cf::WZ0, Cf::HY0, 1);
    m.lm1 = make_map3d_f32(reinterpret_cast<const float*>(lvl_[s_lm1].p), d_, Cf::WZ1, Cf::HY1, 1);
    if (inv_.p)
      m.inv[0] = make_map3d_f32(reinterpret_cast<const float*>(inv_.p), d_, kTZ + 2 * Cf::hz(1),
                                Cf::TY_ + 2 * Cf::hy(1), 1);
  }

  // One step per pass: acoustic_fused<R, 1> (acoustic_fused.cuh).
  template <int R>
  void launch_fused_rk(int64_t t, int* gflag, int gmask, int x_lo, int x_hi) {
    constexpr int TY = fused_ty(R), PF = pf_for(R);
    const int cx = fused_cx_r<R>(x_hi - x_lo);
    // tensor maps are cached per input slots
    const int s_l0 = slot(t - 1), s_lm1 = slot(t - 2);
    const int key = (NB + s_l0) * NB + s_lm1;
    auto it = fmaps_.find(key);
    if (it == fmaps_.end()) {
      FusedMaps m{};
      fused_maps<R>(m, s_l0, s_lm1);
      it = fmaps_.emplace(key, m).first;
    }
    FusedArgs a = common_args(t, x_lo, x_hi, cx, gflag, gmask);
    a.out_km1 = nullptr;
    a.out_k = reinterpret_cast<float*>(lvl_[slot(t)].p);
    if (peers_on_) {
      a.peer_lo = static_cast<float*>(peers_.lo);
      a.peer_hi = static_cast<float*>(peers_.hi);
      a.peer_lo_end = (int)peers_.lo_end;
      a.peer_hi_begin = (int)peers_.hi_begin;
      a.peer_lo_shift = (int)peers_.lo_shift;
      a.peer_hi_shift = (int)peers_.hi_shift;
    }
    if (K_) {
      const ThrLists* tl = thr_lists<R, 1>();
      a.thr_ptr = tl ? tl->ptr.p : nullptr;
      a.thr_list = tl ? tl->list.p : nullptr;
    }
    const int nch = (x_hi - x_lo + cx - 1) / cx;
    if (fast_)
      FusedLauncher<R, 1, TY, kTZ, PF, true>::launch(st_, it->second, a, nch);
    else
      FusedLauncher<R, 1, TY, kTZ, PF, false>::launch(st_, it->second, a, nch);
  }

  // Two steps per pass: the two-level wavefront kernel (acoustic_wtb.cuh).
  template <int R>
  void launch_wtb_rk(int64_t t, int* gflag, int gmask, int x_lo, int x_hi) {
    using C = WtbCfg<R, 2, wtb_ry(R), kWtbPF, wtb_ty(R, 2)>;
    const int cx = wtb_cx_r<R>(x_hi - x_lo);
    const int s_l0 = slot(t - 1), s_lm1 = slot(t - 2);
    const int key = (2 * NB + s_l0) * NB + s_lm1;
    auto it = wmaps_.find(key);
    if (it == wmaps_.end()) {
      WtbMaps m{};
      const float* l0 = reinterpret_cast<const float*>(lvl_[s_l0].p);
      m.l0 = make_map3d_f32(l0, d_, C::WZ0, C::HY0, 1);
      m.lm1 = make_map3d_f32(reinterpret_cast<const float*>(lvl_[s_lm1].p), d_, C::WZ1, C::HY1,
                             1);
      m.c1 = make_map3d_f32(l0, d_, C::WZ1, C::TY, 1);
      if (inv_.p) {
        const float* iv = reinterpret_cast<const float*>(inv_.p);
        m.inv1 = make_map3d_f32(iv, d_, C::WZ1, C::HY1, 1);
        m.inv2 = make_map3d_f32(iv, d_, C::WZ1, C::TY, 1);
      }
      it = wmaps_.emplace(key, m).first;
    }
    FusedArgs a = common_args(t, x_lo, x_hi, cx, gflag, gmask);
    a.out_km1 = reinterpret_cast<float*>(lvl_[slot(t)].p);
    a.out_k = reinterpret_cast<float*>(lvl_[slot(t + 1)].p);
    if (K_) {
      const ThrLists* tl = wtb_thr_lists<R, 2>();
      a.thr_ptr = tl ? tl->ptr.p : nullptr;
      a.thr_list = tl ? tl->list.p : nullptr;
    }
    const int nch = (x_hi - x_lo + cx - 1) / cx;
    if (fast_)
      WtbLauncher<R, 2, wtb_ry(R), kWtbPF, wtb_ty(R, 2), true>::launch(st_, it->second, a, nch);
    else
      WtbLauncher<R, 2, wtb_ry(R), kWtbPF, wtb_ty(R, 2), false>::launch(st_, it->second, a, nch);
  }

  FusedArgs common_args(int64_t t, int x_lo, int x_hi, int cx, int* gflag, int gmask) {
    FusedArgs a{};
    a.fx = reinterpret_cast<const float*>(fac_[0].p);
    a.fy = reinterpret_cast<const float*>(fac_[1].p);
    a.fz = reinterpret_cast<const float*>(fac_[2].p);
    a.inv_scalar = (float)inv_scalar_;
    a.use_inv = inv_.p ? 1 : 0;
    a.cf = tcf_;
    a.d = d_;
    a.cx_len = cx;
    a.x_lo = x_lo;
    a.x_hi = x_hi;
    a.ntz = (int)((d_.nz + kTZ - 1) / kTZ);
    a.zero_lo = zero_lo_ ? 1 : 0;
    a.zero_hi = zero_hi_ ? 1 : 0;
    a.t0 = (int)t;
    if (K_) {
      a.series = reinterpret_cast<const float*>(series_.p);
      a.n_src = (int)K_;
    }
    a.nonfinite = gflag;
    a.guard_mask = gmask;
    return a;
  }

  // kb (1 or 2) fused steps from t over local planes [x_lo, x_hi)
  void launch_fused_range(int64_t t, int kb, int* gflag, int gmask, int x_lo, int x_hi) {
    if constexpr (sizeof(T) == 4) {
      STB_REQUIRE(kb >= 1 && kb <= max_k_, STB_ERR_PLAN,
                  "time_height exceeds the fused kernel's depth");
      switch (R_) {
        case 1: return kb == 2 ? launch_wtb_rk<1>(t, gflag, gmask, x_lo, x_hi)
                               : launch_fused_rk<1>(t, gflag, gmask, x_lo, x_hi);
        case 2: return kb == 2 ? launch_wtb_rk<2>(t, gflag, gmask, x_lo, x_hi)
                               : launch_fused_rk<2>(t, gflag, gmask, x_lo, x_hi);
        case 4: return kb == 2 ? launch_wtb_rk<4>(t, gflag, gmask, x_lo, x_hi)
                               : launch_fused_rk<4>(t, gflag, gmask, x_lo, x_hi);
        case 3: return launch_fused_rk<3>(t, gflag, gmask, x_lo, x_hi);
        case 5: return launch_fused_rk<5>(t, gflag, gmask, x_lo, x_hi);
        case 6: return launch_fused_rk<6>(t, gflag, gmask, x_lo, x_hi);
        case 7: return launch_fused_rk<7>(t, gflag, gmask, x_lo, x_hi);
        case 8: return launch_fused_rk<8>(t, gflag, gmask, x_lo, x_hi);
        default: throw Error(STB_ERR_ARG, "no fused kernel for this space order");
      }
    }
  }

  void launch_fused(int64_t t, int kb, int* gflag, int gmask) {
    launch_fused_range(t, kb, gflag, gmask, 0, (int)d_.nx);
  }

  void check_same_geometry(const Support& s) {
    for (int a = 0; a < 3; ++a)
      STB_REQUIRE(s.shape[a] == geom_.shape[a], STB_ERR_ARG,
                  "support was built for a different grid shape (supports are global)");
  }

  void ensure_events(int64_t n) {
    for (auto& e : run_ev_)
      if (!e) STB_CUDA(cudaEventCreate(&e));
    while ((int64_t)events_.size() < 2 * n) {
      cudaEvent_t e;
      STB_CUDA(cudaEventCreate(&e));
      events_.push_back(e);
    }
  }

  int R_ = 1;
  double vmax_ = NAN;            // max(velocity), reduced while forming inv
  Dims d_{};
  // async stepping state
  bool as_open_ = false;
  bool peers_on_ = false;         // the next K = 1 launch stores into peer ghosts
  stb_peer_halo peers_{};
  int64_t as_t0_ = 0, as_n_ = 0;
  std::vector<int64_t> as_guard_;
  stb_geometry geom_{};          // GLOBAL grid geometry
  int64_t x_begin_ = 0;          // global plane of local plane 0 (x slabs)
  bool zero_lo_ = true, zero_hi_ = true;
  bool active_[3]{};
  cudaStream_t st_ = nullptr;
  AcCoefs<T> cf_{};
  DevBuf<T> lvl_[NB];
  DevBuf<T> inv_;
  T inv_scalar_ = T(0);
  DevBuf<T> fac_[3];
  bool has_fac_ = false;
  // path selection
  Path path_ = Path::Reference;
  bool fast_ = false;
  int arithmetic_ = 0;
  int max_k_ = 1, default_k_ = 1, last_k_ = 1;
  int tuned_k_ = 0;                 // 0: not measured yet (time_height = 0)
  cudaStream_t gst_ = nullptr;      // receiver gathers (overlap the next steps)
  cudaEvent_t gev_[NB] = {};        // last gather of ring slot s
  cudaEvent_t sev_ = nullptr;
  static constexpr int64_t kTraceChunk = 64;     // steps per streamed trace chunk
  cudaStream_t cst_ = nullptr;                   // trace copies
  std::vector<cudaEvent_t> cev_;
  float tune_ms_[2] = {0.f, 0.f};   // measured ms per step at K = 1, 2
  int cx_len_ = 0;                  // STB_NCHUNK override of the x-chunk length
  int sm_count_ = 0;
  TiledCoefs tcf_{};
  std::unordered_map<int, FusedMaps> fmaps_;
  std::unordered_map<int, WtbMaps> wmaps_;
  // sources
  int64_t K_ = 0, src_nt_ = 0;
  DevBuf<T> series_;
  DevBuf<int64_t> src_off_;
  DevBuf<int> src_plane_;
  DevBuf<int64_t> src_keys_;
  DevBuf<int4> src_list_;
  DevBuf<int> src_tile_ptr_;
  int64_t src_n_ = 0;
  std::map<int, std::unique_ptr<ThrLists>> thr_;
  std::unique_ptr<ThrLists> wtb_thr_[2];   // acoustic_wtb lists per level count
  // receivers
  int64_t nrec_ = 0;
  DevBuf<int64_t> rec_off_;
  DevBuf<double> rec_w_;
  DevBuf<double> rec_dev_;
  DevBuf<int> guards_;
  // timing
  std::vector<cudaEvent_t> events_;
  cudaEvent_t run_ev_[2] = {nullptr, nullptr};
  int64_t launches_ = 0, all_launches_ = 0, updates_ = 0;
  double run_ms_ = 0.0;
};

}  // namespace stb

stb_prop_s* make_acoustic(const stb_acoustic_desc& d) {
  if (d.precision == 32) return new stb::AcousticProp<float>(d);
  return new stb::AcousticProp<double>(d);
}
