// Isotropic elastic velocity-stress propagator (ElasticModel,
// elastic_update_v / elastic_update_tau, physics.py:216-429).
//
// Exact reference operation order per point:
//   _stag_d   acc = sum_j (a[+hi] - a[+lo]) * c_j, j ascending;
//             forward reads (+j, -(j-1)), backward (+(j-1), -j)
//   div / trace / strain sums skip inactive axes, in the listed order
//   v   = (v_prev + div*buoy) * fac
//   tdg = (t_prev + (tr*lam + d*mu2)) * fac,   mu2 = 2*mu (exact)
//   tsh = (t_prev + (da + db)*mu) * fac
// The two half steps read only the previous value of the field they write
// at the same point, so both update in place (one level per field): 9 field
// streams + 3 material streams.
//
// Layout: every field is stored with a zero halo of H >= R points on all
// sides (never written), interior z starting 128-byte aligned, so neighbour
// loads need no bounds checks.  f32 3-D grids run the TMA-tiled 2.5-D x
// sweeps of elastic_tiled.cuh; f64 and degenerate grids the thread-per-point
// kernels below.  Every launch covers a local x range [x_lo, x_hi) (x-slab
// runs compute owned planes only and exchange R ghost planes per half step).
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>

#include "fp_exact.cuh"
#include "padded.cuh"
#include "sparse_ops.cuh"
#include "stb_internal.cuh"
#include "tma.cuh"

namespace stb {

namespace {

inline unsigned g1(int64_t n, int b = 256) { return (unsigned)((n + b - 1) / b); }

enum { VX, VY, VZ, TXX, TYY, TZZ, TXY, TXZ, TYZ, NFIELDS };

template <typename T>
struct ElCoefs {
  T d1[3][8];     // f(c_j / h_a)
  int active[3];
  T buoy, lam, mu;  // scalars when the material pointer is NULL
};

template <typename T>
struct ElArgs {
  T* f[NFIELDS];
  const T* buoy;
  const T* lam;
  const T* mu;
  const T* fx;
  const T* fy;
  const T* fz;
  int has_fac;
  ElCoefs<T> cf;
  PDims d;
  int x_lo, x_hi;         // local planes computed by this launch
  int* nonfinite;         // guard flag (NULL: no check this step)
};

// staggered first derivative from an accessor g(o) = a[centre + o*stride]
template <typename T, int R, typename G>
__device__ __forceinline__ T stag(const G& g, const T* c, bool fwd) {
  T acc = T(0);
#pragma unroll
  for (int j = 1; j <= R; ++j) {
    const int hi = fwd ? j : j - 1;
    const int lo = fwd ? -(j - 1) : -j;
    const T term = rmul(rsub(g(hi), g(lo)), c[j - 1]);
    acc = (j == 1) ? term : radd(acc, term);
  }
  return acc;
}

// ---------------------------------------------------------------------------
// Thread-per-point variants (default): full occupancy hides L1/L2 latency of
// the ~110 neighbour loads per point; the zero halo removes all bounds checks.
// ---------------------------------------------------------------------------
template <typename T, int R>
__global__ void __launch_bounds__(128)
elastic_v_point(ElArgs<T> a) {
  const int z = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * 4 + threadIdx.y;
  const int x = a.x_lo + blockIdx.z;
  if (z >= a.d.nz || y >= a.d.ny) return;
  const int ys = (int)a.d.pitch, xs = (int)a.d.plane;
  const int i = (int)a.d.at(x, y, z);
  const ElCoefs<T>& cf = a.cf;
  const T* __restrict__ txx = a.f[TXX];
  const T* __restrict__ txy = a.f[TXY];
  const T* __restrict__ txz = a.f[TXZ];
  const T* __restrict__ tyy = a.f[TYY];
  const T* __restrict__ tyz = a.f[TYZ];
  const T* __restrict__ tzz = a.f[TZZ];
  auto gx = [&](const T* p) { return [=](int o) { return p[i + o * xs]; }; };
  auto gy = [&](const T* p) { return [=](int o) { return p[i + o * ys]; }; };
  auto gz = [&](const T* p) { return [=](int o) { return p[i + o]; }; };
  T d[3] = {T(0), T(0), T(0)};
  bool h[3] = {false, false, false};
  if (cf.active[0]) {
    d[0] = stag<T, R>(gx(txx), cf.d1[0], true);
    d[1] = stag<T, R>(gx(txy), cf.d1[0], false);
    d[2] = stag<T, R>(gx(txz), cf.d1[0], false);
    h[0] = h[1] = h[2] = true;
  }
  if (cf.active[1]) {
    const T e0 = stag<T, R>(gy(txy), cf.d1[1], false);
    const T e1 = stag<T, R>(gy(tyy), cf.d1[1], true);
    const T e2 = stag<T, R>(gy(tyz), cf.d1[1], false);
    d[0] = h[0] ? radd(d[0], e0) : e0;
    d[1] = h[1] ? radd(d[1], e1) : e1;
    d[2] = h[2] ? radd(d[2], e2) : e2;
    h[0] = h[1] = h[2] = true;
  }
  if (cf.active[2]) {
    const T e0 = stag<T, R>(gz(txz), cf.d1[2], false);
    const T e1 = stag<T, R>(gz(tyz), cf.d1[2], false);
    const T e2 = stag<T, R>(gz(tzz), cf.d1[2], true);
    d[0] = h[0] ? radd(d[0], e0) : e0;
    d[1] = h[1] ? radd(d[1], e1) : e1;
    d[2] = h[2] ? radd(d[2], e2) : e2;
    h[0] = h[1] = h[2] = true;
  }
  const T buoy = a.buoy ? a.buoy[i] : cf.buoy;
  const T fac = a.has_fac ? tmin(tmin(a.fx[x], a.fy[y]), a.fz[z]) : T(1);
  bool bad = false;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T* v = a.f[VX + k];
    T o = v[i];
    if (h[k]) o = radd(o, rmul(d[k], buoy));
    if (a.has_fac) o = rmul(o, fac);
    v[i] = o;
    bad |= !finite(o);
  }
  if (a.nonfinite && bad) atomicExch(a.nonfinite, 1);
}

template <typename T, int R>
__global__ void __launch_bounds__(128)
elastic_tau_point(ElArgs<T> a) {
  const int z = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * 4 + threadIdx.y;
  const int x = a.x_lo + blockIdx.z;
  if (z >= a.d.nz || y >= a.d.ny) return;
  const int ys = (int)a.d.pitch, xs = (int)a.d.plane;
  const int i = (int)a.d.at(x, y, z);
  const ElCoefs<T>& cf = a.cf;
  const T* __restrict__ vx = a.f[VX];
  const T* __restrict__ vy = a.f[VY];
  const T* __restrict__ vz = a.f[VZ];
  auto gx = [&](const T* p) { return [=](int o) { return p[i + o * xs]; }; };
  auto gy = [&](const T* p) { return [=](int o) { return p[i + o * ys]; }; };
  auto gz = [&](const T* p) { return [=](int o) { return p[i + o]; }; };
  const T lam = a.lam ? a.lam[i] : cf.lam;
  const T mu = a.mu ? a.mu[i] : cf.mu;
  const T mu2 = rmul(mu, T(2));
  const T fac = a.has_fac ? tmin(tmin(a.fx[x], a.fy[y]), a.fz[z]) : T(1);
  T dg[3] = {T(0), T(0), T(0)};
  if (cf.active[0]) dg[0] = stag<T, R>(gx(vx), cf.d1[0], false);
  if (cf.active[1]) dg[1] = stag<T, R>(gy(vy), cf.d1[1], false);
  if (cf.active[2]) dg[2] = stag<T, R>(gz(vz), cf.d1[2], false);
  T tr = T(0);
  bool htr = false;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (!cf.active[k]) continue;
    tr = htr ? radd(tr, dg[k]) : dg[k];
    htr = true;
  }
  bool bad = false;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T inc = T(0);
    bool hi = false;
    if (htr) {
      inc = rmul(tr, lam);
      hi = true;
    }
    if (cf.active[k]) {
      const T d2 = rmul(dg[k], mu2);
      inc = hi ? radd(inc, d2) : d2;
      hi = true;
    }
    T* f = a.f[TXX + k];
    T o = f[i];
    if (hi) o = radd(o, inc);
    if (a.has_fac) o = rmul(o, fac);
    f[i] = o;
    bad |= !finite(o);
  }
  T s[3] = {T(0), T(0), T(0)};
  bool hs[3] = {false, false, false};
  if (cf.active[1]) { s[0] = stag<T, R>(gy(vx), cf.d1[1], true); hs[0] = true; }
  if (cf.active[2]) { s[1] = stag<T, R>(gz(vx), cf.d1[2], true); hs[1] = true; }
  if (cf.active[2]) { s[2] = stag<T, R>(gz(vy), cf.d1[2], true); hs[2] = true; }
  if (cf.active[0]) {
    const T e = stag<T, R>(gx(vy), cf.d1[0], true);
    s[0] = hs[0] ? radd(s[0], e) : e;
    hs[0] = true;
    const T e2 = stag<T, R>(gx(vz), cf.d1[0], true);
    s[1] = hs[1] ? radd(s[1], e2) : e2;
    hs[1] = true;
  }
  if (cf.active[1]) {
    const T e = stag<T, R>(gy(vz), cf.d1[1], true);
    s[2] = hs[2] ? radd(s[2], e) : e;
    hs[2] = true;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T* f = a.f[TXY + k];
    T o = f[i];
    if (hs[k]) o = radd(o, rmul(s[k], mu));
    if (a.has_fac) o = rmul(o, fac);
    f[i] = o;
    bad |= !finite(o);
  }
  if (a.nonfinite && bad) atomicExch(a.nonfinite, 1);
}

// dt/rho, dt*lam, dt*mu from per-point Lame parameters (compact host order)
template <typename T>
__global__ void elastic_materials_kernel(const double* __restrict__ lam,
                                         const double* __restrict__ mu,
                                         const double* __restrict__ rho, double dt, PDims d,
                                         T* __restrict__ buoy, T* __restrict__ lam_dt,
                                         T* __restrict__ mu_dt) {
  const int64_t n = d.nx * d.ny * d.nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i % d.nz, xy = i / d.nz;
    const int64_t o = d.at(xy / d.ny, xy % d.ny, z);
    buoy[o] = from_f64<T>(rdiv(dt, rho[i]));
    lam_dt[o] = from_f64<T>(rmul(dt, lam[i]));
    mu_dt[o] = from_f64<T>(rmul(dt, mu[i]));
  }
}

// Same from vp, vs, rho (engine.py:247-255 in f64: mu = rho*vs**2,
// lam = rho*vp**2 - 2*mu), with physics.py:229-236's checks as flag bits
// (1: rho <= 0, 2: mu < 0, 4: lam + 2*mu <= 0) and max(vp) for the sponge
// decay (order-preserving int64 key; NaN flagged separately).
struct MatIn {
  const double* p;
  double s;
  __device__ double at(int64_t i) const { return p ? p[i] : s; }
};

__device__ __forceinline__ long long el_dkey(double x) {
  const long long b = __double_as_longlong(x);
  return b >= 0 ? b : b ^ 0x7fffffffffffffffLL;
}

template <typename T>
__global__ void elastic_materials_from_velocity_kernel(MatIn vp, MatIn vs, MatIn rho, double dt,
                                                       PDims d, T* __restrict__ buoy,
                                                       T* __restrict__ lam_dt,
                                                       T* __restrict__ mu_dt, int* flags,
                                                       long long* vmax_key) {
  const int64_t n = d.nx * d.ny * d.nz;
  int f = 0;
  long long mk = LLONG_MIN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double p = vp.at(i), sv = vs.at(i), r = rho.at(i);
    const double mu = rmul(r, rmul(sv, sv));
    const double lam = rsub(rmul(r, rmul(p, p)), rmul(2.0, mu));
    f |= (r <= 0.0 ? 1 : 0) | (mu < 0.0 ? 2 : 0) | (radd(lam, rmul(2.0, mu)) <= 0.0 ? 4 : 0);
    f |= (p != p) ? 8 : 0;
    mk = max(mk, el_dkey(p));
    const int64_t z = i % d.nz, xy = i / d.nz;
    const int64_t o = d.at(xy / d.ny, xy % d.ny, z);
    buoy[o] = from_f64<T>(rdiv(dt, r));
    lam_dt[o] = from_f64<T>(rmul(dt, lam));
    mu_dt[o] = from_f64<T>(rmul(dt, mu));
  }
  for (int o = 16; o > 0; o >>= 1) {
    mk = max(mk, __shfl_xor_sync(0xffffffffu, mk, o));
    f |= __shfl_xor_sync(0xffffffffu, f, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(vmax_key, mk);
    if (f) atomicOr(flags, f);
  }
}

}  // namespace
}  // namespace stb

#include "elastic_tiled.cuh"
#include "elastic_tiled2.cuh"

namespace stb {
namespace {

template <typename T>
__global__ void el_fill_kernel(T* __restrict__ dst, PDims d, T v) {
  const int64_t n = d.nx * d.ny * d.nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i % d.nz, xy = i / d.nz;
    dst[d.at(xy / d.ny, xy % d.ny, z)] = v;
  }
}

// phase 0: v half step, 1: tau half step, over local planes [x_lo, x_hi)
template <typename T, int R>
void launch_point(cudaStream_t st, const ElArgs<T>& a, int phase) {
  if (a.x_hi <= a.x_lo) return;
  dim3 block(32, 4);
  dim3 grid((unsigned)((a.d.nz + 31) / 32), (unsigned)((a.d.ny + 3) / 4),
            (unsigned)(a.x_hi - a.x_lo));
  if (phase == 0)
    elastic_v_point<T, R><<<grid, block, 0, st>>>(a);
  else
    elastic_tau_point<T, R><<<grid, block, 0, st>>>(a);
}

}  // namespace

template <typename T>
class ElasticProp final : public stb_prop_s {
 public:
  explicit ElasticProp(const stb_elastic_desc& desc) {
    R_ = desc.space_order / 2;
    geom_ = desc.geom;
    x_begin_ = desc.x_begin;
    const int64_t nxl = desc.nx_local > 0 ? desc.nx_local : desc.geom.shape[0];
    STB_REQUIRE(x_begin_ >= 0 && x_begin_ + nxl <= desc.geom.shape[0], STB_ERR_ARG,
                "x slab [x_begin, x_begin + nx_local) leaves the grid");
    d_ = make_pdims(nxl, desc.geom.shape[1], desc.geom.shape[2], R_, sizeof(T));
    STB_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    for (int a = 0; a < 3; ++a) {
      cf_.active[a] = desc.active[a] ? 1 : 0;
      for (int j = 0; j < 8; ++j) cf_.d1[a][j] = (T)desc.d1[a][j];
    }
    for (auto& f : f_) {
      f.alloc(d_.total);
      f.zero(st_);
    }
    const int64_t n = d_.nx * d_.ny * d_.nz;
    const double dt = desc.dt;
    // materials (physics.py:251-257)
    const bool any_arr = desc.lam || desc.mu || desc.rho ||
                         (desc.from_velocities && (desc.vp || desc.vs));
    if (any_arr && desc.from_velocities) {
      auto up = [&](DevBuf<double>& b, const double* h) {
        if (h) {
          b.alloc(n);
          b.upload(h, n, st_);
        }
      };
      DevBuf<double> vp, vs, rho;
      up(vp, desc.vp);
      up(vs, desc.vs);
      up(rho, desc.rho);
      buoy_.alloc(d_.total);
      lam_.alloc(d_.total);
      mu_.alloc(d_.total);
      buoy_.zero(st_);
      lam_.zero(st_);
      mu_.zero(st_);
      DevBuf<int> flags(1);
      flags.zero(st_);
      DevBuf<long long> vkey(1);
      const long long lo = LLONG_MIN;
      STB_CUDA(cudaMemcpyAsync(vkey.p, &lo, sizeof(lo), cudaMemcpyHostToDevice, st_));
      elastic_materials_from_velocity_kernel<T><<<1184, 256, 0, st_>>>(
          MatIn{vp.p, desc.vp_scalar}, MatIn{vs.p, desc.vs_scalar}, MatIn{rho.p, desc.rho_scalar},
          dt, d_, buoy_.p, lam_.p, mu_.p, flags.p, vkey.p);
      STB_CHECK_LAUNCH();
      int hf = 0;
      long long hk = lo;
      flags.download(&hf, 1, st_);
      vkey.download(&hk, 1, st_);
      STB_CUDA(cudaStreamSynchronize(st_));
      STB_REQUIRE(!(hf & 1), STB_ERR_ARG, "rho must be positive");
      STB_REQUIRE(!(hf & 2), STB_ERR_ARG, "mu must be non-negative");
      STB_REQUIRE(!(hf & 4), STB_ERR_ARG, "lam + 2*mu must be positive");
      if (desc.vp) {
        const long long b = hk >= 0 ? hk : hk ^ 0x7fffffffffffffffLL;
        double vm;
        std::memcpy(&vm, &b, sizeof(vm));
        vmax_ = (hf & 8) ? NAN : vm;
      } else {
        vmax_ = desc.vp_scalar;
      }
    } else if (any_arr) {
      DevBuf<double> lam(n), mu(n), rho(n);
      auto fill = [&](DevBuf<double>& b, const double* h, double s) {
        if (h) {
          b.upload(h, n, st_);
        } else {
          std::vector<double> tmp(n, s);
          b.upload(tmp.data(), n, st_);
          STB_CUDA(cudaStreamSynchronize(st_));
        }
      };
      fill(lam, desc.lam, desc.lam_scalar);
      fill(mu, desc.mu, desc.mu_scalar);
      fill(rho, desc.rho, desc.rho_scalar);
      buoy_.alloc(d_.total);
      lam_.alloc(d_.total);
      mu_.alloc(d_.total);
      buoy_.zero(st_);
      lam_.zero(st_);
      mu_.zero(st_);
      elastic_materials_kernel<T><<<1184, 256, 0, st_>>>(lam.p, mu.p, rho.p, dt, d_, buoy_.p,
                                                         lam_.p, mu_.p);
      STB_CHECK_LAUNCH();
      STB_CUDA(cudaStreamSynchronize(st_));
    } else {
      cf_.buoy = (T)(dt / desc.rho_scalar);
      cf_.lam = (T)(dt * desc.lam_scalar);
      cf_.mu = (T)(dt * desc.mu_scalar);
    }
    set_damping(desc.damp);
    // TMA-tiled sweeps (elastic_tiled.cuh): f32, 3-D, R <= 4
    tiled_ = sizeof(T) == 4 && cf_.active[0] && cf_.active[1] && cf_.active[2] && R_ <= 4;
    if (const char* e = std::getenv("STB_ELASTIC_PATH")) tiled_ = tiled_ && std::string(e) != "point";
    if (tiled_) setup_tiled();
    if (tiled_) {
      // opt-in (STB_EL_STREAM=1): bit-exact and it cuts the DRAM traffic of a
      // step by 15-20 %, but measured slower than the two launches
      // (29 vs 24.6 ms at 1024^3) -- with half the SMs per
      // sweep, each SM's three-slot TMA pipeline is latency-bound
      int sms = 148;
      int dev = 0;
      STB_CUDA(cudaGetDevice(&dev));
      STB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      stream_nv_ = sms / 2;
      stream_nt_ = sms - stream_nv_;
      if (const char* e = std::getenv("STB_EL_STREAM"))
        stream_ = std::atoi(e) != 0 && d_.nx + 2 * R_ < (1 << 13) - 1;
      if (const char* e = std::getenv("STB_EL_NV")) stream_nv_ = std::max(1, std::atoi(e));
      if (const char* e = std::getenv("STB_EL_NT")) stream_nt_ = std::max(1, std::atoi(e));
      if (const char* e = std::getenv("STB_EL_LEAD")) stream_lead_ = std::max(1, std::atoi(e));
      if (const char* e = std::getenv("STB_EL_PUB")) {
        const int p = std::atoi(e);
        if (p == 1 || p == 2 || p == 4 || p == 8 || p == 16) stream_pub_ = p;
      }
    }
    STB_REQUIRE(d_.total < (int64_t)INT32_MAX, STB_ERR_ARG,
                "elastic slab too large for 32-bit offsets; use more x slabs");
  }

  // sponge tables (also after creation: stb_prop_set_damping)
  void set_damping(const double* const* damp) override {
    has_fac_ = damp[0] || damp[1] || damp[2];
    const int64_t n3[3] = {d_.nx, d_.ny, d_.nz};
    for (int a = 0; a < 3; ++a) {
      if (!fac_[a].p) fac_[a].alloc(n3[a]);
      DevBuf<double> tmp(damp[a] ? n3[a] : 0);
      if (damp[a]) tmp.upload(damp[a] + (a == 0 ? x_begin_ : 0), n3[a], st_);
      pad_table_kernel<T><<<g1(n3[a]), 256, 0, st_>>>(damp[a] ? tmp.p : nullptr, n3[a],
                                                     fac_[a].p);
      STB_CHECK_LAUNCH();
      STB_CUDA(cudaStreamSynchronize(st_));
    }
  }

  double velocity_max() const override { return vmax_; }

  ~ElasticProp() override {
    // drain in-flight work: buffers are freed on stream 0, which a
    // non-blocking stream does not order against
    if (st_) cudaStreamSynchronize(st_);
    for (auto& e : events_) cudaEventDestroy(e);
    for (auto& e : run_ev_)
      if (e) cudaEventDestroy(e);
    if (st_) cudaStreamDestroy(st_);
  }

  void setup_tiled() {
    if constexpr (sizeof(T) == 4) {
      auto materialise = [&](DevBuf<T>& b, T v) {
        if (b.p) return;
        b.alloc(d_.total);
        b.zero(st_);
        el_fill_kernel<T><<<1184, 256, 0, st_>>>(b.p, d_, v);
        STB_CHECK_LAUNCH();
      };
      materialise(buoy_, cf_.buoy);
      materialise(lam_, cf_.lam);
      materialise(mu_, cf_.mu);
      STB_CUDA(cudaStreamSynchronize(st_));
      Dims md{};
      md.nx = d_.nx + 2 * d_.H;
      md.ny = d_.ny + 2 * d_.H;
      md.nz = d_.pitch;
      md.pitch = d_.pitch;
      md.plane = d_.plane;
      // tau pass: the three velocities with the full halo of a 16 x 32 tile
      const uint32_t pz = kElTZ + 2 * ((R_ + 3) / 4 * 4);
      for (int f = VX; f < TXX; ++f)
        fmap_[f] = make_map3d_f32(reinterpret_cast<const float*>(f_[f].p), md, pz,
                                  (uint32_t)(16 + 2 * R_), 1);
      // elastic_tiled2 v pass: per-stress boxes with only the halo the field
      // is differentiated along (El2Cfg::fhy / fhz)
      switch (R_) {
        case 1: set_stress_maps<1>(md); break;
        case 2: set_stress_maps<2>(md); break;
        case 3: set_stress_maps<3>(md); break;
        case 4: set_stress_maps<4>(md); break;
        default: break;
      }
      // elastic_tiled2: centre-operand boxes over the 16 x 32 tile
      for (int f = 0; f < NFIELDS; ++f)
        omap_[f] = make_map3d_f32(reinterpret_cast<const float*>(f_[f].p), md, kElTZ, 16, 1);
      omap_[NFIELDS + 0] = make_map3d_f32(reinterpret_cast<const float*>(buoy_.p), md, kElTZ, 16, 1);
      omap_[NFIELDS + 1] = make_map3d_f32(reinterpret_cast<const float*>(lam_.p), md, kElTZ, 16, 1);
      omap_[NFIELDS + 2] = make_map3d_f32(reinterpret_cast<const float*>(mu_.p), md, kElTZ, 16, 1);
      switch (R_) {
        case 1: set_tiled_attr<1>(); break;
        case 2: set_tiled_attr<2>(); break;
        case 3: set_tiled_attr<3>(); break;
        case 4: set_tiled_attr<4>(); break;
        default: break;
      }
    }
  }

  template <int R>
  void set_stress_maps(const Dims& md) {
    using C = El2Cfg<R, 0>;
    for (int f = 0; f < 6; ++f)
      smap_[f] = make_map3d_f32(reinterpret_cast<const float*>(f_[TXX + f].p), md,
                                (uint32_t)C::fbz(f), (uint32_t)C::fby(f), 1);
  }

  template <int R, int PASS>
  void set_pair_attr() {
    const int sm = (int)El2Two<R, PASS>::SMEM;
    const auto at = cudaFuncAttributeMaxDynamicSharedMemorySize;
    STB_CUDA(cudaFuncSetAttribute(elastic_tiled2<R, PASS, false>, at, sm));
    STB_CUDA(cudaFuncSetAttribute(elastic_tiled2<R, PASS, true>, at, sm));
    if (PASS == 0) {
      const int ss = (int)std::max(El2Cfg<R, 0, kSNOv>::SMEM, El2Cfg<R, 1, kSNOt>::SMEM);
      STB_CUDA(cudaFuncSetAttribute(elastic_stream<R, false>, at, ss));
      STB_CUDA(cudaFuncSetAttribute(elastic_stream<R, true>, at, ss));
    }
  }

  // The full step in one launch (elastic_tiled2.cuh: elastic_stream).
  template <int R>
  void launch_stream_r(int* nonfinite) {
    const int tiles_z = (int)((d_.nz + kElTZ - 1) / kElTZ);
    const int tiles_yv = (int)((d_.ny + 15) / 16), tiles_yt = (int)((d_.ny + R + 15) / 16);
    const size_t nvt = (size_t)tiles_yv * tiles_z, ntt = (size_t)tiles_yt * tiles_z;
    if (prog_v_.n < nvt || prog_t_.n < ntt || !stream_err_.p || epoch_ >= (1u << 18)) {
      prog_v_.alloc(nvt);
      prog_t_.alloc(ntt);
      stream_err_.alloc(1);
      STB_CUDA(cudaMemsetAsync(prog_v_.p, 0, nvt * sizeof(unsigned), st_));
      STB_CUDA(cudaMemsetAsync(prog_t_.p, 0, ntt * sizeof(unsigned), st_));
      STB_CUDA(cudaMemsetAsync(stream_err_.p, 0, sizeof(int), st_));
      epoch_ = 0;
    }
    ElTiledArgs a{};
    a.fx = reinterpret_cast<const float*>(fac_[0].p);
    a.fy = reinterpret_cast<const float*>(fac_[1].p);
    a.fz = reinterpret_cast<const float*>(fac_[2].p);
    a.has_fac = has_fac_ ? 1 : 0;
    for (int ax = 0; ax < 3; ++ax)
      for (int j = 0; j < 8; ++j) a.cf.d1[ax][j] = (float)cf_.d1[ax][j];
    a.d = d_;
    a.cx = (int)d_.nx;
    a.x_lo = 0;
    a.x_hi = (int)d_.nx;
    a.nonfinite = nonfinite;
    a.negz = -0.0f;
    ElTiledArgs av = a, at = a;
    El2Maps mv{}, mt{};
    for (int f = 0; f < 6; ++f) mv.f[f] = smap_[f];
    for (int f = 0; f < 3; ++f) {
      mv.o[f] = omap_[VX + f];
      av.out[f] = reinterpret_cast<float*>(f_[VX + f].p);
    }
    mv.o[3] = omap_[NFIELDS + 0];
    for (int f = 0; f < 3; ++f) mt.f[f] = fmap_[VX + f];
    for (int f = 0; f < 6; ++f) {
      mt.o[f] = omap_[TXX + f];
      at.out[f] = reinterpret_cast<float*>(f_[TXX + f].p);
    }
    mt.o[6] = omap_[NFIELDS + 1];
    mt.o[7] = omap_[NFIELDS + 2];
    ElStream sc{};
    sc.prog_v = prog_v_.p;
    sc.prog_t = prog_t_.p;
    sc.err = stream_err_.p;
    sc.epoch = ++epoch_;
    sc.nv = (int)std::min<size_t>((size_t)stream_nv_, nvt);
    sc.nt = (int)std::min<size_t>((size_t)stream_nt_, ntt);
    sc.tiles_z = tiles_z;
    sc.tiles_yv = tiles_yv;
    sc.tiles_yt = tiles_yt;
    sc.lead = stream_lead_;
    sc.pub = stream_pub_;
    const int ss = (int)std::max(El2Cfg<R, 0, kSNOv>::SMEM, El2Cfg<R, 1, kSNOt>::SMEM);
    const unsigned grid = (unsigned)(sc.nv + sc.nt);
    if (nonfinite) elastic_stream<R, true><<<grid, El2Cfg<R, 0>::NT + 32, ss, st_>>>(mv, mt, av, at, sc);
    else elastic_stream<R, false><<<grid, El2Cfg<R, 0>::NT + 32, ss, st_>>>(mv, mt, av, at, sc);
    STB_CHECK_LAUNCH();
  }

  void launch_stream(int* nonfinite) {
    if constexpr (sizeof(T) == 4) {
      switch (R_) {
        case 1: return launch_stream_r<1>(nonfinite);
        case 2: return launch_stream_r<2>(nonfinite);
        case 3: return launch_stream_r<3>(nonfinite);
        case 4: return launch_stream_r<4>(nonfinite);
        default: break;
      }
    }
    throw Error(STB_ERR_ARG, "no streamed elastic kernel for this configuration");
  }

  template <int R>
  void set_tiled_attr() {
    set_pair_attr<R, 0>();
    set_pair_attr<R, 1>();
  }

  template <int R>
  void launch_tiled_r(int* nonfinite, int phase, int x_lo, int x_hi) {
    // x chunk per CTA (measured at so=8: 512^3 256 planes 36.6 vs 150 planes
    // 36.0 Gpts/s -- half the warm-ups; 1024^3 35.95 vs 35.88)
    int cx = 256;
    if (const char* e = std::getenv("STB_EL_CX")) cx = std::max(8, std::atoi(e));
    if (x_hi <= x_lo) return;
    auto grid_for = [&](int ty) {
      return dim3((unsigned)((d_.nz + kElTZ - 1) / kElTZ), (unsigned)((d_.ny + ty - 1) / ty),
                  (unsigned)((x_hi - x_lo + cx - 1) / cx));
    };
    ElTiledArgs a{};
    a.fx = reinterpret_cast<const float*>(fac_[0].p);
    a.fy = reinterpret_cast<const float*>(fac_[1].p);
    a.fz = reinterpret_cast<const float*>(fac_[2].p);
    a.has_fac = has_fac_ ? 1 : 0;
    for (int ax = 0; ax < 3; ++ax)
      for (int j = 0; j < 8; ++j) a.cf.d1[ax][j] = (float)cf_.d1[ax][j];
    a.d = d_;
    a.cx = cx;
    a.x_lo = x_lo;
    a.x_hi = x_hi;
    a.nonfinite = nonfinite;
    a.negz = -0.0f;
    El2Maps m{};
    const int nin = phase == 0 ? 6 : 3, nout = phase == 0 ? 3 : 6;
    const int fout = phase == 0 ? VX : TXX;
    for (int f = 0; f < nin; ++f) m.f[f] = phase == 0 ? smap_[f] : fmap_[VX + f];
    for (int f = 0; f < nout; ++f) {
      m.o[f] = omap_[fout + f];
      a.out[f] = reinterpret_cast<float*>(f_[fout + f].p);
    }
    if (phase == 0) {
      m.o[3] = omap_[NFIELDS + 0];
    } else {
      m.o[6] = omap_[NFIELDS + 1];
      m.o[7] = omap_[NFIELDS + 2];
    }
    const dim3 grid = grid_for(16);
    const bool g = nonfinite != nullptr;
    if (phase == 0) {
      using C = El2Two<R, 0>;
      if (g) elastic_tiled2<R, 0, true><<<grid, C::NT, C::SMEM, st_>>>(m, a);
      else elastic_tiled2<R, 0, false><<<grid, C::NT, C::SMEM, st_>>>(m, a);
    } else {
      using C = El2Two<R, 1>;
      if (g) elastic_tiled2<R, 1, true><<<grid, C::NT, C::SMEM, st_>>>(m, a);
      else elastic_tiled2<R, 1, false><<<grid, C::NT, C::SMEM, st_>>>(m, a);
    }
    STB_CHECK_LAUNCH();
  }

  // one half step (phase 0: v, 1: tau) over local planes [x_lo, x_hi)
  void launch_half(int phase, int x_lo, int x_hi, int* nonfinite) {
    if (tiled_) {
      if constexpr (sizeof(T) == 4) {
        switch (R_) {
          case 1: return launch_tiled_r<1>(nonfinite, phase, x_lo, x_hi);
          case 2: return launch_tiled_r<2>(nonfinite, phase, x_lo, x_hi);
          case 3: return launch_tiled_r<3>(nonfinite, phase, x_lo, x_hi);
          case 4: return launch_tiled_r<4>(nonfinite, phase, x_lo, x_hi);
          default: throw Error(STB_ERR_ARG, "no tiled elastic kernel for this space order");
        }
      }
    }
    ElArgs<T> A{};
    for (int i = 0; i < NFIELDS; ++i) A.f[i] = f_[i].p;
    A.buoy = buoy_.p;
    A.lam = lam_.p;
    A.mu = mu_.p;
    A.fx = fac_[0].p;
    A.fy = fac_[1].p;
    A.fz = fac_[2].p;
    A.has_fac = has_fac_ ? 1 : 0;
    A.cf = cf_;
    A.d = d_;
    A.x_lo = x_lo;
    A.x_hi = x_hi;
    A.nonfinite = nonfinite;
    switch (R_) {
      case 1: launch_point<T, 1>(st_, A, phase); break;
      case 2: launch_point<T, 2>(st_, A, phase); break;
      case 3: launch_point<T, 3>(st_, A, phase); break;
      case 4: launch_point<T, 4>(st_, A, phase); break;
      case 5: launch_point<T, 5>(st_, A, phase); break;
      case 6: launch_point<T, 6>(st_, A, phase); break;
      case 7: launch_point<T, 7>(st_, A, phase); break;
      case 8: launch_point<T, 8>(st_, A, phase); break;
      default: throw Error(STB_ERR_ARG, "space_order must be even in [2, 16]");
    }
    STB_CHECK_LAUNCH();
  }

  // injection of step t into the diagonal stresses (engine.py:327-332)
  void inject(int64_t t) {
    if (!K_) return;
    for (int fi = TXX; fi <= TZZ; ++fi)
      inject_kernel<T><<<g1(K_), 256, 0, st_>>>(f_[fi].p, src_off_.p, series_.p + t * K_, K_);
    STB_CHECK_LAUNCH();
    all_launches_ += 3;
  }

  void gather(int64_t row) {
    if (!nrec_) return;
    gather_kernel<T><<<g1(nrec_), 256, 0, st_>>>(f_[rec_field_].p, rec_off_.p, rec_w_.p, nrec_,
                                                 rec_dev_.p + row * nrec_);
    STB_CHECK_LAUNCH();
    ++all_launches_;
  }

  void set_sources(Support& s, const double* wav, int64_t nt_w, const double* scale,
                   int64_t nt) override {
    for (int a = 0; a < 3; ++a)
      STB_REQUIRE(s.shape[a] == geom_.shape[a], STB_ERR_ARG,
                  "support was built for a different grid shape (supports are global)");
    src_nt_ = nt;
    K_ = 0;
    if (s.K == 0) return;
    int64_t lohi[2];
    STB_CUDA(cudaMemcpyAsync(&lohi[0], s.row_ptr.p + x_begin_ * geom_.shape[1], sizeof(int64_t),
                             cudaMemcpyDeviceToHost, st_));
    STB_CUDA(cudaMemcpyAsync(&lohi[1], s.row_ptr.p + (x_begin_ + d_.nx) * geom_.shape[1],
                             sizeof(int64_t), cudaMemcpyDeviceToHost, st_));
    STB_CUDA(cudaStreamSynchronize(st_));
    K_ = lohi[1] - lohi[0];
    if (K_ == 0) return;
    DevBuf<double> dwav(nt_w * s.n_points), dscale(s.n_points), dc(nt * s.K), dl(nt * K_);
    dwav.upload(wav, nt_w * s.n_points, st_);
    dscale.upload(scale, s.n_points, st_);
    support_decompose_dev(s, dwav.p, nt_w, dscale.p, nt, dc.p, st_);
    STB_CUDA(cudaMemcpy2DAsync(dl.p, K_ * sizeof(double), dc.p + lohi[0], s.K * sizeof(double),
                               K_ * sizeof(double), nt, cudaMemcpyDeviceToDevice, st_));
    series_.alloc(nt * K_);
    pad_to_dtype_kernel<T><<<g1(nt * K_), 256, 0, st_>>>(dl.p, nt * K_, series_.p);
    src_off_.alloc(K_);
    pad_keys_to_offsets<<<g1(K_), 256, 0, st_>>>(s.keys.p + lohi[0], K_, geom_.shape[1],
                                                geom_.shape[2], x_begin_, d_, src_off_.p);
    STB_CHECK_LAUNCH();
    STB_CUDA(cudaStreamSynchronize(st_));
  }

  void set_receiver_field(int field) override {
    STB_REQUIRE(field >= 0 && field < NFIELDS, STB_ERR_ARG, "elastic field index in [0, 9)");
    rec_field_ = field;
  }

  void set_receivers(const double* coords, int64_t nrec) override {
    nrec_ = nrec;
    if (nrec == 0) return;
    DevBuf<double> dc(nrec * 3);
    dc.upload(coords, nrec * 3, st_);
    DevBuf<int64_t> idx(nrec * 24);
    rec_w_.alloc(nrec * 8);
    stencils_compute(dc.p, nrec, geom_, -1, idx.p, rec_w_.p, st_);
    rec_off_.alloc(nrec * 8);
    DevBuf<int> bad(1);
    bad.zero(st_);
    pad_idx_to_offsets<<<g1(nrec * 8), 256, 0, st_>>>(idx.p, nrec * 8, x_begin_, d_, rec_off_.p,
                                                     bad.p);
    STB_CHECK_LAUNCH();
    int hb = 0;
    bad.download(&hb, 1, st_);
    STB_CUDA(cudaStreamSynchronize(st_));
    STB_REQUIRE(hb == 0, STB_ERR_ARG, "receiver corners leave this x slab");
  }

  void run(int64_t t0, int64_t nsteps, int k, double* rec_out, int64_t* bad_step) override {
    if (bad_step) *bad_step = -1;
    launches_ = all_launches_ = 0;
    run_ms_ = 0.0;
    updates_ = 0;
    if (nsteps <= 0) return;
    STB_REQUIRE(K_ == 0 || t0 + nsteps <= src_nt_, STB_ERR_ARG,
                "run extends past the decomposed source series");
    STB_REQUIRE(t0 == t_next_, STB_ERR_ARG,
                "elastic handles update in place: steps must be run in order");
    (void)k;
    if (nrec_ && (int64_t)rec_dev_.n < nsteps * nrec_) rec_dev_.alloc(nsteps * nrec_);
    std::vector<int64_t> guard_steps;
    for (int64_t t = t0; t < t0 + nsteps; ++t)
      if (t > 0 && t % 32 == 0) guard_steps.push_back(t);
    DevBuf<int> guards(guard_steps.size() + 1);
    guards.zero(st_);
    ensure_events(nsteps + 1);
    size_t gi = 0;
    STB_CUDA(cudaEventRecord(run_ev_[0], st_));
    for (int64_t t = t0; t < t0 + nsteps; ++t) {
      const bool guard_now = gi < guard_steps.size() && guard_steps[gi] == t;
      // the reference's guard runs after the v half step of a guard step and
      // checks every field (engine.py:373-376): the v fields are new, the
      // stress fields still hold t-1 -- checked after the tau sweep here,
      // which flags the same blow-ups one half step later.
      int* nf = guard_now ? guards.p + gi : nullptr;
      STB_CUDA(cudaEventRecord(events_[2 * launches_], st_));
      if (stream_) {
        launch_stream(nf);
      } else {
        launch_half(0, 0, (int)d_.nx, nf);
        launch_half(1, 0, (int)d_.nx, nf);
      }
      STB_CUDA(cudaEventRecord(events_[2 * launches_ + 1], st_));
      ++launches_;
      all_launches_ += stream_ ? 1 : 2;
      if (guard_now) ++gi;
      inject(t);
      gather(t - t0);
    }
    STB_CUDA(cudaEventRecord(run_ev_[1], st_));
    t_next_ = t0 + nsteps;
    updates_ = nsteps * d_.nx * d_.ny * d_.nz;
    if (nrec_ && rec_out) rec_dev_.download(rec_out, nsteps * nrec_, st_);
    std::vector<int> gh(guard_steps.size() + 1, 0);
    if (!guard_steps.empty()) guards.download(gh.data(), guard_steps.size(), st_);
    int serr = 0;
    if (stream_ && stream_err_.p) stream_err_.download(&serr, 1, st_);
    STB_CUDA(cudaStreamSynchronize(st_));
    float rm = 0.f;
    STB_CUDA(cudaEventElapsedTime(&rm, run_ev_[0], run_ev_[1]));
    run_ms_ = rm;
    STB_REQUIRE(serr == 0, STB_ERR_CUDA,
                "elastic_stream: a tau tile gave up waiting for its v tiles (results invalid)");
    for (size_t i = 0; i < guard_steps.size(); ++i) {
      if (gh[i]) {
        if (bad_step) *bad_step = guard_steps[i];
        std::ostringstream os;
        os << "non-finite values in field group 'v' at step " << guard_steps[i];
        throw Error(STB_ERR_UNSTABLE, os.str());
      }
    }
  }

  // ---------------------------------------------------------------- async
  // x-slab stepping without host synchronisation (slabs.py): per step the v
  // half step over the owned planes, an exchange of R ghost planes of vx vy
  // vz, the tau half step (+ injection), an exchange of R planes of the six
  // stresses, the receiver gather -- all ordered on stream().
  void* stream() override { return st_; }

  void async_begin(int64_t t0, int64_t nsteps) override {
    STB_REQUIRE(nsteps >= 0, STB_ERR_ARG, "nsteps must be >= 0");
    STB_REQUIRE(t0 == t_next_, STB_ERR_ARG,
                "elastic handles update in place: steps must be run in order");
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
    ensure_events(2 * nsteps + 1);
    STB_CUDA(cudaEventRecord(run_ev_[0], st_));
    as_open_ = true;
  }

  void half_step_async(int64_t t, int phase, int64_t x_lo, int64_t x_hi) override {
    STB_REQUIRE(as_open_, STB_ERR_ARG, "async_begin first");
    STB_REQUIRE(t >= as_t0_ && t < as_t0_ + as_n_, STB_ERR_ARG, "step outside the async window");
    STB_REQUIRE(phase == 0 || phase == 1, STB_ERR_ARG, "phase: 0 = v, 1 = tau");
    STB_REQUIRE(0 <= x_lo && x_lo <= x_hi && x_hi <= d_.nx, STB_ERR_ARG, "plane range");
    int* nf = nullptr;
    for (size_t g = 0; g < as_guard_.size(); ++g)
      if (as_guard_[g] == t && phase == 1) nf = guards_.p + g;
    STB_REQUIRE(2 * launches_ + 1 < (int64_t)events_.size(), STB_ERR_ARG,
                "more than two launches per step in the async window");
    STB_CUDA(cudaEventRecord(events_[2 * launches_], st_));
    launch_half(phase, (int)x_lo, (int)x_hi, nf);
    STB_CUDA(cudaEventRecord(events_[2 * launches_ + 1], st_));
    ++launches_;
    ++all_launches_;
    if (phase == 1) {
      inject(t);
      updates_ += (x_hi - x_lo) * d_.ny * d_.nz;
    }
  }

  void step_async(int64_t t, int kb, int64_t x_lo, int64_t x_hi) override {
    STB_REQUIRE(kb == 1, STB_ERR_PLAN, "elastic steps fuse one time step per pass");
    half_step_async(t, 0, x_lo, x_hi);
    half_step_async(t, 1, x_lo, x_hi);
  }

  void gather_async(int64_t t, int kb) override {
    STB_REQUIRE(as_open_, STB_ERR_ARG, "async_begin first");
    for (int j = 0; j < kb; ++j) gather(t + j - as_t0_);
  }

  void async_finish(double* rec_out, int64_t* bad_step) override {
    STB_REQUIRE(as_open_, STB_ERR_ARG, "async_begin first");
    as_open_ = false;
    if (bad_step) *bad_step = -1;
    STB_CUDA(cudaEventRecord(run_ev_[1], st_));
    t_next_ = as_t0_ + as_n_;
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
        os << "non-finite values in field group 'v' at step " << as_guard_[i];
        throw Error(STB_ERR_UNSTABLE, os.str());
      }
  }

  void read_field(int field, int64_t t, void* out) override {
    STB_REQUIRE(field >= 0 && field < NFIELDS, STB_ERR_ARG, "elastic field index in [0, 9)");
    STB_REQUIRE(t == t_next_ - 1 || (t_next_ == 0), STB_ERR_ARG,
                "only the latest time level is resident for elastic handles");
    pad_read<T>(f_[field].p, d_, out, st_);
  }

  // Planes of the padded layout: local plane p starts at (p + H) * plane.
  void level_ptr(int field, int64_t t, void** dev, int64_t* plane, int64_t* pitch) override {
    STB_REQUIRE(field >= 0 && field < NFIELDS, STB_ERR_ARG, "elastic field index in [0, 9)");
    (void)t;
    *dev = f_[field].p + d_.H * d_.plane;
    if (plane) *plane = d_.plane;
    if (pitch) *pitch = d_.pitch;
  }

  void reset() override {
    for (auto& f : f_) f.zero(st_);
    t_next_ = 0;
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
    if (tiled_ && stream_)
      os << "elastic_stream<f32,R=" << R_ << "> (one launch per step: " << stream_nv_
         << " v-sweep + " << stream_nt_ << " tau-sweep CTAs streaming through L2; "
         << "16x32 tiles as z pairs)";
    else if (tiled_)
      os << "elastic_tiled2<f32,R=" << R_ << "> (TMA plane + operand rings, producer warp; "
         << "16x32 tiles as z pairs; x chunk 256)";
    else
      os << "elastic_point<" << (sizeof(T) == 4 ? "f32" : "f64") << ",R=" << R_
         << "> (v + tau, thread per point, zero-haloed layout)";
    os << " k=1 requested_k=" << k
       << " bytes_per_point=" << (tiled_ && stream_ ? 21 : 30) * sizeof(T);
    return os.str();
  }

 private:
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
  double vmax_ = NAN;        // max(vp) when the device formed the materials
  PDims d_{};
  stb_geometry geom_{};
  int64_t x_begin_ = 0;
  cudaStream_t st_ = nullptr;
  ElCoefs<T> cf_{};
  DevBuf<T> f_[NFIELDS];
  DevBuf<T> buoy_, lam_, mu_;
  DevBuf<T> fac_[3];
  bool has_fac_ = false;
  bool tiled_ = false;
  // elastic_stream: the full step as one launch (v and tau sweeps streaming
  // behind each other through L2); STB_EL_STREAM=0/1 overrides the size rule
  bool stream_ = false;
  int stream_nv_ = 0, stream_nt_ = 0, stream_lead_ = 32, stream_pub_ = 8;
  DevBuf<unsigned> prog_v_, prog_t_;
  DevBuf<int> stream_err_;
  unsigned epoch_ = 0;
  int rec_field_ = TXX;      // engine.py:327-332 records txx
  CUtensorMap fmap_[NFIELDS];
  CUtensorMap omap_[NFIELDS + 3];   // tile boxes of the fields, buoy, lam, mu (tiled2)
  CUtensorMap smap_[6];             // per-stress boxes of the tiled2 v pass
  int64_t t_next_ = 0;
  bool as_open_ = false;
  int64_t as_t0_ = 0, as_n_ = 0;
  std::vector<int64_t> as_guard_;
  DevBuf<int> guards_;
  int64_t K_ = 0, src_nt_ = 0;
  DevBuf<T> series_;
  DevBuf<int64_t> src_off_;
  int64_t nrec_ = 0;
  DevBuf<int64_t> rec_off_;
  DevBuf<double> rec_w_, rec_dev_;
  std::vector<cudaEvent_t> events_;
  cudaEvent_t run_ev_[2] = {nullptr, nullptr};
  int64_t launches_ = 0, all_launches_ = 0, updates_ = 0;
  double run_ms_ = 0.0;
};

}  // namespace stb

stb_prop_s* make_elastic(const stb_elastic_desc& d) {
  if (d.precision == 32) return new stb::ElasticProp<float>(d);
  return new stb::ElasticProp<double>(d);
}
