// Step-level operators on the reference's halo-padded time-level layout.
//
// stencil_tb lets a caller step a model itself: allocate_field /
// TimeBufferedField (grid.py:173-225) hold each time level as a C-order
// (nx+2h, ny+2h, nz+2h) array with a zero halo, and acoustic_update /
// elastic_update_v / elastic_update_tau (physics.py:181-429), scatter_box /
// fused_inject_row (precompute.py:209-252), gather_box (precompute.py:287-308)
// and inject_direct / record_receivers (sparse.py:176-207) each update one box
// of one level.  These kernels do the same on device memory in that layout
// (the Python mirror keeps the levels in torch CUDA tensors), thread per
// point, in the reference's exact IEEE operation order -- bitwise the NumPy
// results.  They are the drop-in for callers that drive the loop nest
// themselves; run() uses the fused sweep kernels instead.
#include <cstdint>

#include "fp_exact.cuh"
#include "sparse_ops.cuh"
#include "stb_internal.cuh"

namespace stb {
namespace {

struct Lay {
  int64_t px, py, pz;   // padded extents
  int64_t h;            // halo
  int64_t sx, sy;       // strides (elements)
  __device__ int64_t at(int64_t x, int64_t y, int64_t z) const {
    return (x + h) * sx + (y + h) * sy + (z + h);
  }
};

struct BoxD {
  int64_t lo[3], n[3];
};

Lay make_lay(const stb_layout& L) {
  Lay l;
  l.px = L.padded[0];
  l.py = L.padded[1];
  l.pz = L.padded[2];
  l.h = L.halo;
  l.sy = l.pz;
  l.sx = l.py * l.pz;
  return l;
}

BoxD check_box(const stb_layout& L, const stb_box& b) {
  BoxD d;
  for (int a = 0; a < 3; ++a) {
    const int64_t n = L.padded[a] - 2 * (int64_t)L.halo;
    STB_REQUIRE(b.lo[a] >= 0 && b.hi[a] <= n && b.lo[a] <= b.hi[a], STB_ERR_ARG,
                "box leaves the interior of the padded layout");
    d.lo[a] = b.lo[a];
    d.n[a] = b.hi[a] - b.lo[a];
  }
  return d;
}

void check_layout(const stb_layout* L) {
  STB_REQUIRE(L != nullptr, STB_ERR_ARG, "NULL layout");
  STB_REQUIRE(L->precision == 32 || L->precision == 64, STB_ERR_ARG, "precision must be 32/64");
  STB_REQUIRE(L->halo >= 0, STB_ERR_ARG, "halo must be >= 0");
  for (int a = 0; a < 3; ++a)
    STB_REQUIRE(L->padded[a] >= 2 * (int64_t)L->halo + 1, STB_ERR_ARG, "padded extent too small");
}

inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

dim3 box_grid(const BoxD& b) {
  return dim3(nblk(b.n[2], 128), (unsigned)b.n[1], (unsigned)b.n[0]);
}

bool box_empty(const BoxD& b) { return b.n[0] <= 0 || b.n[1] <= 0 || b.n[2] <= 0; }

template <typename T>
struct MatArg {
  const T* p;   // padded array, or NULL for the scalar
  T s;
  __device__ T at(int64_t i) const { return p ? p[i] : s; }
};

// ---------------------------------------------------------------------------
// acoustic_update (physics.py:181-213): lap = u1*c0; lap += (u1[+r]+u1[-r])*w
// per active axis / radius; lap *= inv; out = u1*2 - u0 + lap; out *= fac.
// ---------------------------------------------------------------------------
template <typename T>
struct AcBoxCoefs {
  T c0;
  T w[3][8];
  int active[3];
};

template <typename T, int R>
__global__ void __launch_bounds__(128)
box_acoustic_kernel(T* __restrict__ dst, const T* __restrict__ u1, const T* __restrict__ u0,
                    MatArg<T> inv, const T* __restrict__ fac, AcBoxCoefs<T> cf, Lay l, BoxD b) {
  const int64_t z = b.lo[2] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (z >= b.lo[2] + b.n[2]) return;
  const int64_t y = b.lo[1] + blockIdx.y, x = b.lo[0] + blockIdx.z;
  const int64_t i = l.at(x, y, z);
  const int64_t st[3] = {l.sx, l.sy, 1};
  const T uc = u1[i];
  T lap = rmul(uc, cf.c0);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (!cf.active[a]) continue;
#pragma unroll
    for (int r = 1; r <= R; ++r)
      lap = radd(lap, rmul(radd(u1[i + r * st[a]], u1[i - r * st[a]]), cf.w[a][r - 1]));
  }
  lap = rmul(lap, inv.at(i));
  T o = rmul(uc, T(2));
  o = rsub(o, u0[i]);
  o = radd(o, lap);
  if (fac) o = rmul(o, fac[i]);
  dst[i] = o;
}

// ---------------------------------------------------------------------------
// elastic_update_v / elastic_update_tau (physics.py:287-429).
// _stag_d: acc = sum_j (a[+hi] - a[+lo]) * c_j sequentially; forward reads
// (+j, -(j-1)), backward (+(j-1), -j).
// ---------------------------------------------------------------------------
template <typename T>
struct ElBoxCoefs {
  T d1[3][8];
  int active[3];
};

template <typename T, int R>
__device__ __forceinline__ T stag_d(const T* __restrict__ a, int64_t i, int64_t s, const T* c,
                                    bool fwd) {
  T acc = T(0);
#pragma unroll
  for (int j = 1; j <= R; ++j) {
    const int hi = fwd ? j : j - 1, lo = fwd ? -(j - 1) : -j;
    const T term = rmul(rsub(a[i + hi * s], a[i + lo * s]), c[j - 1]);
    acc = j == 1 ? term : radd(acc, term);
  }
  return acc;
}

// sum of the present parts in order (_acc_sum)
template <typename T>
__device__ __forceinline__ void acc_add(T& acc, bool& has, T v) {
  acc = has ? radd(acc, v) : v;
  has = true;
}

template <typename T>
struct ElVArgs {
  T* v[3];
  const T* vp[3];
  const T* tau[6];   // txx tyy tzz txy txz tyz at t-1
  MatArg<T> buoy;
  const T* fac;
};

template <typename T, int R>
__global__ void __launch_bounds__(128)
box_elastic_v_kernel(ElVArgs<T> a, ElBoxCoefs<T> cf, Lay l, BoxD b) {
  const int64_t z = b.lo[2] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (z >= b.lo[2] + b.n[2]) return;
  const int64_t y = b.lo[1] + blockIdx.y, x = b.lo[0] + blockIdx.z;
  const int64_t i = l.at(x, y, z);
  const int64_t st[3] = {l.sx, l.sy, 1};
  enum { XX, YY, ZZ, XY, XZ, YZ };
  // div_x = d_x(txx, fwd) + d_y(txy, bwd) + d_z(txz, bwd); div_y, div_z alike
  const int comp[3][3] = {{XX, XY, XZ}, {XY, YY, YZ}, {XZ, YZ, ZZ}};
  const T buoy = a.buoy.at(i);
  const T fac = a.fac ? a.fac[i] : T(1);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T div = T(0);
    bool has = false;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
      if (cf.active[ax]) acc_add(div, has, stag_d<T, R>(a.tau[comp[k][ax]], i, st[ax], cf.d1[ax],
                                                         ax == k));
    T o = a.vp[k][i];
    if (has) o = radd(o, rmul(div, buoy));
    if (a.fac) o = rmul(o, fac);
    a.v[k][i] = o;
  }
}

template <typename T>
struct ElTauArgs {
  T* tau[6];
  const T* tp[6];
  const T* v[3];     // vx vy vz at t
  MatArg<T> lam, mu, mu2;
  const T* fac;
};

template <typename T, int R>
__global__ void __launch_bounds__(128)
box_elastic_tau_kernel(ElTauArgs<T> a, ElBoxCoefs<T> cf, Lay l, BoxD b) {
  const int64_t z = b.lo[2] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (z >= b.lo[2] + b.n[2]) return;
  const int64_t y = b.lo[1] + blockIdx.y, x = b.lo[0] + blockIdx.z;
  const int64_t i = l.at(x, y, z);
  const int64_t st[3] = {l.sx, l.sy, 1};
  const T fac = a.fac ? a.fac[i] : T(1);
  T dg[3];
  T tr = T(0);
  bool htr = false;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    dg[k] = cf.active[k] ? stag_d<T, R>(a.v[k], i, st[k], cf.d1[k], false) : T(0);
    if (cf.active[k]) acc_add(tr, htr, dg[k]);
  }
  const T lam = a.lam.at(i), mu = a.mu.at(i), mu2 = a.mu2.at(i);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T inc = T(0);
    bool hi = false;
    if (htr) {
      inc = rmul(tr, lam);
      hi = true;
    }
    if (cf.active[k]) acc_add(inc, hi, rmul(dg[k], mu2));
    T o = a.tp[k][i];
    if (hi) o = radd(o, inc);
    if (a.fac) o = rmul(o, fac);
    a.tau[k][i] = o;
  }
  // txy: d_y(vx) + d_x(vy); txz: d_z(vx) + d_x(vz); tyz: d_z(vy) + d_y(vz)
  const int pa[3][2] = {{1, 0}, {2, 0}, {2, 1}};    // axes of the two parts
  const int pf[3][2] = {{0, 1}, {0, 2}, {1, 2}};    // velocity components
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T s = T(0);
    bool hs = false;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int ax = pa[k][q];
      if (cf.active[ax]) acc_add(s, hs, stag_d<T, R>(a.v[pf[k][q]], i, st[ax], cf.d1[ax], true));
    }
    T o = a.tp[3 + k][i];
    if (hs) o = radd(o, rmul(s, mu));
    if (a.fac) o = rmul(o, fac);
    a.tau[3 + k][i] = o;
  }
}

// ---------------------------------------------------------------------------
// Sparse operators.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool in_box(const int64_t* p, const BoxD& b) {
  return p[0] >= b.lo[0] && p[0] < b.lo[0] + b.n[0] && p[1] >= b.lo[1] &&
         p[1] < b.lo[1] + b.n[1] && p[2] >= b.lo[2] && p[2] < b.lo[2] + b.n[2];
}

// scatter_box: dst[p_k] += T(values[k]) for the support points in the box
// (each point once: the support is a set)
template <typename T>
__global__ void box_scatter_kernel(T* __restrict__ dst, const int64_t* __restrict__ pts,
                                   const double* __restrict__ vals, int64_t K, Lay l, BoxD b) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int64_t* p = pts + 3 * k;
  if (!in_box(p, b)) return;
  const int64_t i = l.at(p[0], p[1], p[2]);
  dst[i] = radd(dst[i], from_f64<T>(vals[k]));
}

// gather_box: contrib[m] = w[m] * f64(level[p_m]) for entries in the box
template <typename T>
__global__ void box_gather_kernel(const T* __restrict__ src, const int64_t* __restrict__ pts,
                                  const double* __restrict__ w, int64_t M, Lay l, BoxD b,
                                  double* __restrict__ contrib, uint8_t* __restrict__ mask) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int64_t* p = pts + 3 * m;
  const bool in = in_box(p, b);
  mask[m] = in ? 1 : 0;
  contrib[m] = in ? rmul(w[m], (double)src[l.at(p[0], p[1], p[2])]) : 0.0;
}

// record_receivers: 8 corners per receiver, NumPy's pairwise 8-sum
template <typename T>
__global__ void record_kernel(const T* __restrict__ src, const int64_t* __restrict__ idx,
                              const double* __restrict__ w, int64_t n, Lay l,
                              double* __restrict__ out) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  T v[8];
  double ww[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int64_t* p = idx + 24 * r + 3 * c;
    v[c] = src[l.at(p[0], p[1], p[2])];
    ww[c] = w[8 * r + c];
  }
  out[r] = pairwise8<T>(ww, v);
}

// ---------------------------------------------------------------------------
template <typename T, template <typename, int> class Launch, typename... A>
void dispatch_r(int R, A&&... args) {
  switch (R) {
    case 1: return Launch<T, 1>::go(args...);
    case 2: return Launch<T, 2>::go(args...);
    case 3: return Launch<T, 3>::go(args...);
    case 4: return Launch<T, 4>::go(args...);
    case 5: return Launch<T, 5>::go(args...);
    case 6: return Launch<T, 6>::go(args...);
    case 7: return Launch<T, 7>::go(args...);
    case 8: return Launch<T, 8>::go(args...);
    default: throw Error(STB_ERR_ARG, "radius must be in [1, 8]");
  }
}

template <typename T, int R>
struct AcL {
  static void go(cudaStream_t st, T* d, const T* u1, const T* u0, MatArg<T> inv, const T* fac,
                 AcBoxCoefs<T> cf, Lay l, BoxD b) {
    box_acoustic_kernel<T, R><<<box_grid(b), 128, 0, st>>>(d, u1, u0, inv, fac, cf, l, b);
  }
};
template <typename T, int R>
struct ElVL {
  static void go(cudaStream_t st, ElVArgs<T> a, ElBoxCoefs<T> cf, Lay l, BoxD b) {
    box_elastic_v_kernel<T, R><<<box_grid(b), 128, 0, st>>>(a, cf, l, b);
  }
};
template <typename T, int R>
struct ElTL {
  static void go(cudaStream_t st, ElTauArgs<T> a, ElBoxCoefs<T> cf, Lay l, BoxD b) {
    box_elastic_tau_kernel<T, R><<<box_grid(b), 128, 0, st>>>(a, cf, l, b);
  }
};

template <typename T>
MatArg<T> mat(const void* p, double s) {
  MatArg<T> m;
  m.p = static_cast<const T*>(p);
  m.s = (T)s;
  return m;
}

void check_radius(const stb_layout* L, int radius) {
  STB_REQUIRE(radius >= 1 && radius <= 8, STB_ERR_ARG, "radius must be in [1, 8]");
  STB_REQUIRE(L->halo >= radius, STB_ERR_ARG, "field halo is narrower than the stencil radius");
}

template <typename T>
void acoustic_t(const stb_layout* L, void* dst, const void* u1, const void* u0, int radius,
                const int32_t* active, double center, const double* weights, const void* inv,
                double inv_scalar, const void* dampfac, const BoxD& b, cudaStream_t st) {
  AcBoxCoefs<T> cf{};
  cf.c0 = (T)center;
  for (int a = 0; a < 3; ++a) {
    cf.active[a] = active[a] ? 1 : 0;
    for (int r = 0; r < radius; ++r) cf.w[a][r] = (T)weights[a * 8 + r];
  }
  dispatch_r<T, AcL>(radius, st, static_cast<T*>(dst), static_cast<const T*>(u1),
                     static_cast<const T*>(u0), mat<T>(inv, inv_scalar),
                     static_cast<const T*>(dampfac), cf, make_lay(*L), b);
  STB_CHECK_LAUNCH();
}

template <typename T>
ElBoxCoefs<T> el_coefs(int radius, const int32_t* active, const double* d1) {
  ElBoxCoefs<T> cf{};
  for (int a = 0; a < 3; ++a) {
    cf.active[a] = active[a] ? 1 : 0;
    for (int r = 0; r < radius; ++r) cf.d1[a][r] = (T)d1[a * 8 + r];
  }
  return cf;
}

}  // namespace
}  // namespace stb

#define STB_API extern "C" __attribute__((visibility("default")))
#define STB_GUARD_BEGIN try {
#define STB_GUARD_END                 \
  return STB_OK;                      \
  }                                   \
  catch (const stb::Error& e) {       \
    stb::set_error(e.what());         \
    return e.code;                    \
  }                                   \
  catch (const std::exception& e) {   \
    stb::set_error(e.what());         \
    return STB_ERR_CUDA;              \
  }

using stb::BoxD;

STB_API int stb_box_acoustic_update(const stb_layout* L, void* dst, const void* u1,
                                    const void* u0, int32_t radius, const int32_t* active,
                                    double center, const double* weights, const void* inv,
                                    double inv_scalar, const void* dampfac, const stb_box* box,
                                    void* stream) {
  STB_GUARD_BEGIN
  stb::check_layout(L);
  stb::check_radius(L, radius);
  STB_REQUIRE(dst && u1 && u0 && active && weights && box, STB_ERR_ARG, "NULL argument");
  const BoxD b = stb::check_box(*L, *box);
  if (stb::box_empty(b)) return STB_OK;
  auto st = static_cast<cudaStream_t>(stream);
  if (L->precision == 32)
    stb::acoustic_t<float>(L, dst, u1, u0, radius, active, center, weights, inv, inv_scalar,
                           dampfac, b, st);
  else
    stb::acoustic_t<double>(L, dst, u1, u0, radius, active, center, weights, inv, inv_scalar,
                            dampfac, b, st);
  STB_GUARD_END
}

STB_API int stb_box_elastic_v(const stb_layout* L, void* const* v_out, const void* const* v_prev,
                              const void* const* tau_prev, int32_t radius, const int32_t* active,
                              const double* d1, const void* buoy, double buoy_scalar,
                              const void* dampfac, const stb_box* box, void* stream) {
  STB_GUARD_BEGIN
  stb::check_layout(L);
  stb::check_radius(L, radius);
  STB_REQUIRE(v_out && v_prev && tau_prev && active && d1 && box, STB_ERR_ARG, "NULL argument");
  const BoxD b = stb::check_box(*L, *box);
  if (stb::box_empty(b)) return STB_OK;
  auto st = static_cast<cudaStream_t>(stream);
  auto go = [&](auto tag) {
    using T = decltype(tag);
    stb::ElVArgs<T> a{};
    for (int k = 0; k < 3; ++k) {
      a.v[k] = static_cast<T*>(v_out[k]);
      a.vp[k] = static_cast<const T*>(v_prev[k]);
    }
    for (int k = 0; k < 6; ++k) a.tau[k] = static_cast<const T*>(tau_prev[k]);
    a.buoy = stb::mat<T>(buoy, buoy_scalar);
    a.fac = static_cast<const T*>(dampfac);
    stb::dispatch_r<T, stb::ElVL>(radius, st, a, stb::el_coefs<T>(radius, active, d1),
                                  stb::make_lay(*L), b);
    STB_CHECK_LAUNCH();
  };
  if (L->precision == 32) go(float{}); else go(double{});
  STB_GUARD_END
}

STB_API int stb_box_elastic_tau(const stb_layout* L, void* const* tau_out,
                                const void* const* tau_prev, const void* const* v_cur,
                                int32_t radius, const int32_t* active, const double* d1,
                                const void* lam, double lam_scalar, const void* mu,
                                double mu_scalar, const void* mu2, double mu2_scalar,
                                const void* dampfac, const stb_box* box, void* stream) {
  STB_GUARD_BEGIN
  stb::check_layout(L);
  stb::check_radius(L, radius);
  STB_REQUIRE(tau_out && tau_prev && v_cur && active && d1 && box, STB_ERR_ARG, "NULL argument");
  const BoxD b = stb::check_box(*L, *box);
  if (stb::box_empty(b)) return STB_OK;
  auto st = static_cast<cudaStream_t>(stream);
  auto go = [&](auto tag) {
    using T = decltype(tag);
    stb::ElTauArgs<T> a{};
    for (int k = 0; k < 6; ++k) {
      a.tau[k] = static_cast<T*>(tau_out[k]);
      a.tp[k] = static_cast<const T*>(tau_prev[k]);
    }
    for (int k = 0; k < 3; ++k) a.v[k] = static_cast<const T*>(v_cur[k]);
    a.lam = stb::mat<T>(lam, lam_scalar);
    a.mu = stb::mat<T>(mu, mu_scalar);
    a.mu2 = stb::mat<T>(mu2, mu2_scalar);
    a.fac = static_cast<const T*>(dampfac);
    stb::dispatch_r<T, stb::ElTL>(radius, st, a, stb::el_coefs<T>(radius, active, d1),
                                  stb::make_lay(*L), b);
    STB_CHECK_LAUNCH();
  };
  if (L->precision == 32) go(float{}); else go(double{});
  STB_GUARD_END
}

STB_API int stb_box_scatter(const stb_layout* L, void* dst, const int64_t* points,
                            const double* values, int64_t K, const stb_box* box, void* stream) {
  STB_GUARD_BEGIN
  stb::check_layout(L);
  STB_REQUIRE(dst && box && K >= 0, STB_ERR_ARG, "bad argument");
  const BoxD b = stb::check_box(*L, *box);
  if (K == 0 || stb::box_empty(b)) return STB_OK;
  STB_REQUIRE(points && values, STB_ERR_ARG, "NULL argument");
  auto st = static_cast<cudaStream_t>(stream);
  const unsigned g = stb::nblk(K, 256);
  if (L->precision == 32)
    stb::box_scatter_kernel<float><<<g, 256, 0, st>>>(static_cast<float*>(dst), points, values,
                                                      K, stb::make_lay(*L), b);
  else
    stb::box_scatter_kernel<double><<<g, 256, 0, st>>>(static_cast<double*>(dst), points,
                                                       values, K, stb::make_lay(*L), b);
  STB_CHECK_LAUNCH();
  STB_GUARD_END
}

STB_API int stb_box_gather(const stb_layout* L, const void* src, const int64_t* points,
                           const double* weights, int64_t M, const stb_box* box, double* contrib,
                           uint8_t* in_box, void* stream) {
  STB_GUARD_BEGIN
  stb::check_layout(L);
  STB_REQUIRE(src && box && M >= 0, STB_ERR_ARG, "bad argument");
  const BoxD b = stb::check_box(*L, *box);
  if (M == 0) return STB_OK;
  STB_REQUIRE(points && weights && contrib && in_box, STB_ERR_ARG, "NULL argument");
  auto st = static_cast<cudaStream_t>(stream);
  const unsigned g = stb::nblk(M, 256);
  if (L->precision == 32)
    stb::box_gather_kernel<float><<<g, 256, 0, st>>>(static_cast<const float*>(src), points,
                                                     weights, M, stb::make_lay(*L), b, contrib,
                                                     in_box);
  else
    stb::box_gather_kernel<double><<<g, 256, 0, st>>>(static_cast<const double*>(src), points,
                                                      weights, M, stb::make_lay(*L), b, contrib,
                                                      in_box);
  STB_CHECK_LAUNCH();
  STB_GUARD_END
}

STB_API int stb_record_receivers(const stb_layout* L, const void* src, const int64_t* idx,
                                 const double* w, int64_t n, double* out, void* stream) {
  STB_GUARD_BEGIN
  stb::check_layout(L);
  STB_REQUIRE(src && n >= 0, STB_ERR_ARG, "bad argument");
  if (n == 0) return STB_OK;
  STB_REQUIRE(idx && w && out, STB_ERR_ARG, "NULL argument");
  auto st = static_cast<cudaStream_t>(stream);
  const unsigned g = stb::nblk(n, 256);
  if (L->precision == 32)
    stb::record_kernel<float><<<g, 256, 0, st>>>(static_cast<const float*>(src), idx, w, n,
                                                 stb::make_lay(*L), out);
  else
    stb::record_kernel<double><<<g, 256, 0, st>>>(static_cast<const double*>(src), idx, w, n,
                                                  stb::make_lay(*L), out);
  STB_CHECK_LAUNCH();
  STB_GUARD_END
}
