// Pseudo-acoustic TTI propagator (coupled p, q; eq. 2).
//
// The reference has no TTI; the discrete operator and its IEEE
// operation order are defined by this repo's oracle (oracle/stencil_oracle.py,
// class TTI), which these kernels reproduce bit for bit:
//
//   pass 1  g_a(u) = sum_k (u[+k] - u[-k]) * c_ak            (k = 1..r)
//           w      = sum_{a active} g_a(p) * n_a              (axis order)
//           F_a    = g_a(p) - w * n_a
//           G_a    = (sum_a g_a(q) * n_a) * n_a
//   pass 2  Lxy = sum_a D_a F_a ;  Lzz = sum_a D_a G_a
//           p'  = (((p*2) - p_prev) + ((Lxy*e2) + (Lzz*d2)) * inv) * fac
//           q'  = (((q*2) - q_prev) + ((Lxy*d2) + Lzz) * inv) * fac
//
// n = (sin t cos f, sin t sin f, cos t) is the symmetry axis, e2 = 1 + 2 eps,
// d2 = sqrt(1 + 2 delta), inv = dt^2/m with m = 1/vp^2 (all formed in f64 on
// the host/device and rounded once), r = space_order/4 (first derivatives of
// order so/2, so D_a D_a spans the acoustic footprint R = so/2).
//
// Layout: zero-haloed padded fields (padded.cuh, halo r): p and q keep two
// time levels each (level t in buffer t mod 2; pass 2 writes level t over
// level t-2, which each point reads only at itself before writing), plus six
// gradient streams F_a, G_a (halo zero, never written).  Thread per point,
// neighbours through L1: HBM-bound at ~104 B/point (f32):
//   pass 1: p, q, n_x, n_y, n_z in; F, G out          (5 + 6) x 4 B
//   pass 2: F, G, p, q, p_prev, q_prev, inv, e2, d2 in; p', q' out
//                                                    (13 + 2) x 4 B
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <sstream>

#include "fp_exact.cuh"
#include "padded.cuh"
#include "sparse_ops.cuh"
#include "stb_internal.cuh"
#include "tma.cuh"

namespace stb {

namespace {

inline unsigned g1t(int64_t n, int b = 256) { return (unsigned)((n + b - 1) / b); }

template <typename T>
struct TtiCoefs {
  T c[3][4];          // f(a_k / h_a), k = 1..r
  int active[3];
  T inv, e2, d2;      // scalars when the material pointer is NULL
  T n[3];
};

}  // namespace
}  // namespace stb

#include "tti_fused.cuh"
#include "tti_fused2.cuh"

namespace stb {
namespace {

template <typename T>
struct TtiArgs {
  const T* p1;        // level t-1
  const T* q1;
  T* p0;              // level t-2 in, level t out
  T* q0;
  T* F[3];
  T* G[3];
  const T* inv;
  const T* e2;
  const T* d2;
  const T* n[3];
  const T* fx;
  const T* fy;
  const T* fz;
  int has_fac;
  TtiCoefs<T> cf;
  PDims d;
  int x_lo;           // first local plane of this launch (grid.z = plane count)
  int* nonfinite;
};

// centred first derivative g = sum_k (u[i+k*s] - u[i-k*s]) * c_k
template <typename T, int r>
__device__ __forceinline__ T d1c(const T* __restrict__ u, int i, int s, const T* c) {
  T acc = rmul(rsub(u[i + s], u[i - s]), c[0]);
#pragma unroll
  for (int k = 2; k <= r; ++k) acc = radd(acc, rmul(rsub(u[i + k * s], u[i - k * s]), c[k - 1]));
  return acc;
}

template <typename T, int r>
__global__ void __launch_bounds__(128) tti_pass1(TtiArgs<T> a) {
  const int z = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * 4 + threadIdx.y;
  const int x = a.x_lo + blockIdx.z;
  if (z >= a.d.nz || y >= a.d.ny) return;
  const int st[3] = {(int)a.d.plane, (int)a.d.pitch, 1};
  const int i = (int)a.d.at(x, y, z);
  const TtiCoefs<T>& cf = a.cf;
  T gp[3], gq[3], n[3];
  T wp = T(0), wq = T(0);
  bool first = true;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    if (!cf.active[ax]) continue;
    gp[ax] = d1c<T, r>(a.p1, i, st[ax], cf.c[ax]);
    gq[ax] = d1c<T, r>(a.q1, i, st[ax], cf.c[ax]);
    n[ax] = a.n[ax] ? a.n[ax][i] : cf.n[ax];
    const T tp = rmul(gp[ax], n[ax]);
    const T tq = rmul(gq[ax], n[ax]);
    wp = first ? tp : radd(wp, tp);
    wq = first ? tq : radd(wq, tq);
    first = false;
  }
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    if (!cf.active[ax]) continue;
    a.F[ax][i] = rsub(gp[ax], rmul(wp, n[ax]));
    a.G[ax][i] = rmul(wq, n[ax]);
  }
}

template <typename T, int r>
__global__ void __launch_bounds__(128) tti_pass2(TtiArgs<T> a) {
  const int z = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * 4 + threadIdx.y;
  const int x = a.x_lo + blockIdx.z;
  if (z >= a.d.nz || y >= a.d.ny) return;
  const int st[3] = {(int)a.d.plane, (int)a.d.pitch, 1};
  const int i = (int)a.d.at(x, y, z);
  const TtiCoefs<T>& cf = a.cf;
  T lxy = T(0), lzz = T(0);
  bool any = false;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    if (!cf.active[ax]) continue;
    const T fa = d1c<T, r>(a.F[ax], i, st[ax], cf.c[ax]);
    const T ga = d1c<T, r>(a.G[ax], i, st[ax], cf.c[ax]);
    lxy = any ? radd(lxy, fa) : fa;
    lzz = any ? radd(lzz, ga) : ga;
    any = true;
  }
  const T inv = a.inv ? a.inv[i] : cf.inv;
  const T e2 = a.e2 ? a.e2[i] : cf.e2;
  const T d2 = a.d2 ? a.d2[i] : cf.d2;
  const T fac = a.has_fac ? tmin(tmin(a.fx[x], a.fy[y]), a.fz[z]) : T(1);
  T op = rsub(rmul(a.p1[i], T(2)), a.p0[i]);
  T oq = rsub(rmul(a.q1[i], T(2)), a.q0[i]);
  if (any) {
    op = radd(op, rmul(radd(rmul(lxy, e2), rmul(lzz, d2)), inv));
    oq = radd(oq, rmul(radd(rmul(lxy, d2), lzz), inv));
  }
  if (a.has_fac) {
    op = rmul(op, fac);
    oq = rmul(oq, fac);
  }
  a.p0[i] = op;
  a.q0[i] = oq;
  if (a.nonfinite && (!finite(op) || !finite(oq))) atomicExch(a.nonfinite, 1);
}

// inv = dt2 / (1/v^2) (engine.py:243, physics.py:151 -- same as acoustic),
// written into the padded layout; m <= 0 flagged.
template <typename T>
__global__ void tti_inv_kernel(const double* __restrict__ v, double dt2, PDims d,
                               T* __restrict__ inv, int* bad_m) {
  const int64_t n = d.nx * d.ny * d.nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double vi = v[i];
    const double mm = rdiv(1.0, rmul(vi, vi));
    if (mm <= 0.0) atomicExch(bad_m, 1);
    const int64_t z = i % d.nz, xy = i / d.nz;
    inv[d.at(xy / d.ny, xy % d.ny, z)] = from_f64<T>(rdiv(dt2, mm));
  }
}

template <typename T>
__global__ void tti_material_kernel(const double* __restrict__ src, PDims d, T* __restrict__ dst,
                                    int mode) {
  // mode 0: copy; 1: e2 = 1 + 2 eps; 2: d2 = sqrt(1 + 2 delta) -- the host's
  // f64 NumPy expressions (physics.py tti_medium), each op correctly rounded
  const int64_t n = d.nx * d.ny * d.nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i % d.nz, xy = i / d.nz;
    double v = src[i];
    if (mode) {
      v = __dadd_rn(1.0, __dmul_rn(2.0, v));
      if (mode == 2) v = __dsqrt_rn(v);
    }
    dst[d.at(xy / d.ny, xy % d.ny, z)] = from_f64<T>(v);
  }
}

// f32 axis components already rounded on the host (fp32 runs only)
template <typename T>
__global__ void tti_material32_kernel(const float* __restrict__ src, PDims d, T* __restrict__ dst) {
  const int64_t n = d.nx * d.ny * d.nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i % d.nz, xy = i / d.nz;
    dst[d.at(xy / d.ny, xy % d.ny, z)] = (T)src[i];
  }
}

template <typename T>
__global__ void tti_fill_kernel(T* __restrict__ dst, PDims d, T v) {
  const int64_t n = d.nx * d.ny * d.nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i % d.nz, xy = i / d.nz;
    dst[d.at(xy / d.ny, xy % d.ny, z)] = v;
  }
}

// pass 1 (gradient streams) over [x_lo - r, x_hi + r) within the slab, pass 2
// (divergences + update) over [x_lo, x_hi)
template <typename T, int r>
void launch_tti(cudaStream_t st, TtiArgs<T> a, int x_lo, int x_hi) {
  if (x_hi <= x_lo) return;
  dim3 block(32, 4);
  const int lo1 = std::max(x_lo - r, 0), hi1 = std::min<int>(x_hi + r, (int)a.d.nx);
  a.x_lo = lo1;
  dim3 grid1((unsigned)((a.d.nz + 31) / 32), (unsigned)((a.d.ny + 3) / 4), (unsigned)(hi1 - lo1));
  tti_pass1<T, r><<<grid1, block, 0, st>>>(a);
  a.x_lo = x_lo;
  dim3 grid2((unsigned)((a.d.nz + 31) / 32), (unsigned)((a.d.ny + 3) / 4),
             (unsigned)(x_hi - x_lo));
  tti_pass2<T, r><<<grid2, block, 0, st>>>(a);
}

}  // namespace

template <typename T>
class TtiProp final : public stb_prop_s {
 public:
  explicit TtiProp(const stb_tti_desc& desc) {
    STB_REQUIRE(desc.space_order % 4 == 0, STB_ERR_CONFIG,
                "space_order: TTI needs a multiple of 4 (first derivatives of order so/2)");
    r_ = desc.space_order / 4;
    geom_ = desc.geom;
    x_begin_ = desc.x_begin;
    const int64_t nxl = desc.nx_local > 0 ? desc.nx_local : desc.geom.shape[0];
    STB_REQUIRE(x_begin_ >= 0 && x_begin_ + nxl <= desc.geom.shape[0], STB_ERR_ARG,
                "x slab [x_begin, x_begin + nx_local) leaves the grid");
    d_ = make_pdims(nxl, desc.geom.shape[1], desc.geom.shape[2], r_, sizeof(T));
    STB_REQUIRE(d_.total < (int64_t)INT32_MAX, STB_ERR_ARG,
                "TTI slab too large for 32-bit offsets; use more x slabs");
    STB_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    for (int ax = 0; ax < 3; ++ax) {
      cf_.active[ax] = desc.active[ax] ? 1 : 0;
      for (int k = 0; k < 4; ++k) cf_.c[ax][k] = (T)desc.d1[ax][k];
    }
    for (int f = 0; f < 2; ++f)
      for (int l = 0; l < 2; ++l) {
        lv_[f][l].alloc(d_.total);
        lv_[f][l].zero(st_);
      }
    // fused single-pass path (f32, 3-D): the gradient streams F, G stay on chip
    fused_ = sizeof(T) == 4 && cf_.active[0] && cf_.active[1] && cf_.active[2];
    fast_ = desc.arithmetic == 1;
    STB_REQUIRE(!fast_ || fused_, STB_ERR_CONFIG,
                "schedule.arithmetic: 'fma' needs the fused f32 3-D TTI kernel");
    if (const char* e = std::getenv("STB_TTI_PATH")) {
      fused_ = fused_ && std::string(e) != "twopass";
      pair_ = std::string(e) != "fused1";
    }
    pair_ = pair_ && fused_ && r_ <= 2;
    for (int ax = 0; ax < 3 && !fused_; ++ax) {
      if (!cf_.active[ax]) continue;
      F_[ax].alloc(d_.total);
      G_[ax].alloc(d_.total);
      F_[ax].zero(st_);
      G_[ax].zero(st_);
    }
    const int64_t n = d_.nx * d_.ny * d_.nz;
    auto material = [&](const double* h, double scalar, DevBuf<T>& dst, T& cf, int mode = 0) {
      if (!h) {
        cf = (T)scalar;
        return;
      }
      DevBuf<double> tmp(n);
      tmp.upload(h, n, st_);
      dst.alloc(d_.total);
      dst.zero(st_);
      tti_material_kernel<T><<<1184, 256, 0, st_>>>(tmp.p, d_, dst.p, mode);
      STB_CHECK_LAUNCH();
      STB_CUDA(cudaStreamSynchronize(st_));
    };
    auto material32 = [&](const float* h, DevBuf<T>& dst) {
      DevBuf<float> tmp(n);
      tmp.upload(h, n, st_);
      dst.alloc(d_.total);
      dst.zero(st_);
      tti_material32_kernel<T><<<1184, 256, 0, st_>>>(tmp.p, d_, dst.p);
      STB_CHECK_LAUNCH();
      STB_CUDA(cudaStreamSynchronize(st_));
    };
    if (desc.velocity) {
      DevBuf<double> v(n);
      v.upload(desc.velocity, n, st_);
      inv_.alloc(d_.total);
      inv_.zero(st_);
      DevBuf<int> bad(1);
      bad.zero(st_);
      tti_inv_kernel<T><<<1184, 256, 0, st_>>>(v.p, desc.dt2, d_, inv_.p, bad.p);
      STB_CHECK_LAUNCH();
      int hb = 0;
      bad.download(&hb, 1, st_);
      STB_CUDA(cudaStreamSynchronize(st_));
      STB_REQUIRE(hb == 0, STB_ERR_ARG, "m must be positive");
    } else {
      cf_.inv = (T)desc.inv_scalar;
    }
    // raw_eps_delta: the e2/d2 pointers carry epsilon/delta, formed here
    material(desc.e2, desc.e2_scalar, e2_, cf_.e2, desc.raw_eps_delta ? 1 : 0);
    material(desc.d2, desc.d2_scalar, d2_, cf_.d2, desc.raw_eps_delta ? 2 : 0);
    for (int ax = 0; ax < 3; ++ax) {
      if (desc.axis32[ax]) {
        STB_REQUIRE(sizeof(T) == 4, STB_ERR_ARG, "f32 axis components need precision 32");
        material32(desc.axis32[ax], n_[ax]);
      } else {
        material(desc.axis[ax], desc.axis_scalar[ax], n_[ax], cf_.n[ax]);
      }
    }
    cx_ = 150;
    if (const char* e = std::getenv("STB_TTI_CX")) cx_ = std::max(1, std::atoi(e));
    if (fused_) {
      // scalar materials are materialised, so the fused loop has no pointer
      // tests
      auto materialise = [&](DevBuf<T>& b, T v) {
        if (b.p) return;
        b.alloc(d_.total);
        b.zero(st_);
        tti_fill_kernel<T><<<1184, 256, 0, st_>>>(b.p, d_, v);
        STB_CHECK_LAUNCH();
      };
      materialise(inv_, cf_.inv);
      materialise(e2_, cf_.e2);
      materialise(d2_, cf_.d2);
      for (int ax = 0; ax < 3; ++ax) materialise(n_[ax], cf_.n[ax]);
      STB_CUDA(cudaStreamSynchronize(st_));
      setup_fused();
    }
    set_damping(desc.damp);
  }

  // sponge tables (also after creation: stb_prop_set_damping)
  void set_damping(const double* const* damp) override {
    has_fac_ = damp[0] || damp[1] || damp[2];
    const int64_t n3[3] = {d_.nx, d_.ny, d_.nz};
    for (int ax = 0; ax < 3; ++ax) {
      if (!fac_[ax].p) fac_[ax].alloc(n3[ax]);
      DevBuf<double> tmp(damp[ax] ? n3[ax] : 0);
      if (damp[ax]) tmp.upload(damp[ax] + (ax == 0 ? x_begin_ : 0), n3[ax], st_);
      pad_table_kernel<T><<<g1t(n3[ax]), 256, 0, st_>>>(damp[ax] ? tmp.p : nullptr, n3[ax],
                                                        fac_[ax].p);
      STB_CHECK_LAUNCH();
      STB_CUDA(cudaStreamSynchronize(st_));
    }
  }

  ~TtiProp() override {
    // drain in-flight work: buffers are freed on stream 0, which a
    // non-blocking stream does not order against
    if (st_) cudaStreamSynchronize(st_);
    for (auto& e : events_) cudaEventDestroy(e);
    for (auto& e : run_ev_)
      if (e) cudaEventDestroy(e);
    if (st_) cudaStreamDestroy(st_);
  }

  void set_sources(Support& s, const double* wav, int64_t nt_w, const double* scale,
                   int64_t nt) override {
    for (int ax = 0; ax < 3; ++ax)
      STB_REQUIRE(s.shape[ax] == geom_.shape[ax], STB_ERR_ARG,
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
    pad_to_dtype_kernel<T><<<g1t(nt * K_), 256, 0, st_>>>(dl.p, nt * K_, series_.p);
    src_off_.alloc(K_);
    pad_keys_to_offsets<<<g1t(K_), 256, 0, st_>>>(s.keys.p + lohi[0], K_, geom_.shape[1],
                                                  geom_.shape[2], x_begin_, d_, src_off_.p);
    STB_CHECK_LAUNCH();
    STB_CUDA(cudaStreamSynchronize(st_));
  }

  void set_receiver_field(int field) override {
    STB_REQUIRE(field == 0 || field == 1, STB_ERR_ARG, "TTI field index: 0 = p, 1 = q");
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
    pad_idx_to_offsets<<<g1t(nrec * 8), 256, 0, st_>>>(idx.p, nrec * 8, x_begin_, d_,
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
    run_ms_ = 0.0;
    updates_ = 0;
    if (nsteps <= 0) return;
    STB_REQUIRE(K_ == 0 || t0 + nsteps <= src_nt_, STB_ERR_ARG,
                "run extends past the decomposed source series");
    STB_REQUIRE(t0 == t_next_, STB_ERR_ARG,
                "TTI handles keep two time levels: steps must be run in order");
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
      STB_CUDA(cudaEventRecord(events_[2 * launches_], st_));
      launch_step(t, 0, (int)d_.nx, guard_now ? guards.p + gi : nullptr);
      STB_CUDA(cudaEventRecord(events_[2 * launches_ + 1], st_));
      ++launches_;
      if (guard_now) ++gi;
      inject(t);
      gather(t, t - t0);
    }
    STB_CUDA(cudaEventRecord(run_ev_[1], st_));
    t_next_ = t0 + nsteps;
    if (nrec_ && rec_out) rec_dev_.download(rec_out, nsteps * nrec_, st_);
    std::vector<int> gh(guard_steps.size() + 1, 0);
    if (!guard_steps.empty()) guards.download(gh.data(), guard_steps.size(), st_);
    STB_CUDA(cudaStreamSynchronize(st_));
    float rm = 0.f;
    STB_CUDA(cudaEventElapsedTime(&rm, run_ev_[0], run_ev_[1]));
    run_ms_ = rm;
    for (size_t i = 0; i < guard_steps.size(); ++i) {
      if (gh[i]) {
        if (bad_step) *bad_step = guard_steps[i];
        std::ostringstream os;
        os << "non-finite values in field group 'pq' at step " << guard_steps[i];
        throw Error(STB_ERR_UNSTABLE, os.str());
      }
    }
  }

  // step t (level t from t-1, t-2) over local planes [x_lo, x_hi)
  void launch_step(int64_t t, int x_lo, int x_hi, int* nonfinite) {
    TtiArgs<T> A{};
    for (int ax = 0; ax < 3; ++ax) {
      A.F[ax] = F_[ax].p;
      A.G[ax] = G_[ax].p;
      A.n[ax] = n_[ax].p;
    }
    A.inv = inv_.p;
    A.e2 = e2_.p;
    A.d2 = d2_.p;
    A.fx = fac_[0].p;
    A.fy = fac_[1].p;
    A.fz = fac_[2].p;
    A.has_fac = has_fac_ ? 1 : 0;
    A.cf = cf_;
    A.d = d_;
    const int cur = (int)(t & 1), prev = cur ^ 1;
    A.p1 = lv_[0][prev].p;
    A.q1 = lv_[1][prev].p;
    A.p0 = lv_[0][cur].p;
    A.q0 = lv_[1][cur].p;
    A.nonfinite = nonfinite;
    if (fused_) {
      launch_fused(A, prev, x_lo, x_hi);
      all_launches_ += 1;
    } else {
      switch (r_) {
        case 1: launch_tti<T, 1>(st_, A, x_lo, x_hi); break;
        case 2: launch_tti<T, 2>(st_, A, x_lo, x_hi); break;
        case 3: launch_tti<T, 3>(st_, A, x_lo, x_hi); break;
        case 4: launch_tti<T, 4>(st_, A, x_lo, x_hi); break;
        default: throw Error(STB_ERR_CONFIG, "space_order: TTI supports 4, 8, 12, 16");
      }
      all_launches_ += 2;
    }
    STB_CHECK_LAUNCH();
    updates_ += (int64_t)(x_hi - x_lo) * d_.ny * d_.nz;
  }

  void inject(int64_t t) {
    if (!K_) return;
    const int cur = (int)(t & 1);
    for (int f = 0; f < 2; ++f)
      inject_kernel<T><<<g1t(K_), 256, 0, st_>>>(lv_[f][cur].p, src_off_.p, series_.p + t * K_,
                                                 K_);
    STB_CHECK_LAUNCH();
    all_launches_ += 2;
  }

  void gather(int64_t t, int64_t row) {
    if (!nrec_) return;
    gather_kernel<T><<<g1t(nrec_), 256, 0, st_>>>(lv_[rec_field_][t & 1].p, rec_off_.p, rec_w_.p,
                                                  nrec_, rec_dev_.p + row * nrec_);
    STB_CHECK_LAUNCH();
    ++all_launches_;
  }

  // ---------------------------------------------------------------- async
  // x-slab stepping without host synchronisation (slabs.py): per step one
  // launch over the owned planes (+ injection), then the exchange of R ghost
  // planes of p and q at level t, then the gather -- ordered on stream().
  void* stream() override { return st_; }

  void async_begin(int64_t t0, int64_t nsteps) override {
    STB_REQUIRE(nsteps >= 0, STB_ERR_ARG, "nsteps must be >= 0");
    STB_REQUIRE(t0 == t_next_, STB_ERR_ARG,
                "TTI handles keep two time levels: steps must be run in order");
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
    ensure_events(nsteps + 1);
    STB_CUDA(cudaEventRecord(run_ev_[0], st_));
    as_open_ = true;
  }

  void step_async(int64_t t, int kb, int64_t x_lo, int64_t x_hi) override {
    STB_REQUIRE(as_open_, STB_ERR_ARG, "async_begin first");
    STB_REQUIRE(kb == 1, STB_ERR_PLAN, "TTI steps fuse one time step per pass");
    STB_REQUIRE(t >= as_t0_ && t < as_t0_ + as_n_, STB_ERR_ARG, "step outside the async window");
    STB_REQUIRE(0 <= x_lo && x_lo <= x_hi && x_hi <= d_.nx, STB_ERR_ARG, "plane range");
    int* nf = nullptr;
    for (size_t g = 0; g < as_guard_.size(); ++g)
      if (as_guard_[g] == t) nf = guards_.p + g;
    STB_REQUIRE(2 * launches_ + 1 < (int64_t)events_.size(), STB_ERR_ARG,
                "more than one launch per step in the async window");
    STB_CUDA(cudaEventRecord(events_[2 * launches_], st_));
    launch_step(t, (int)x_lo, (int)x_hi, nf);
    STB_CUDA(cudaEventRecord(events_[2 * launches_ + 1], st_));
    ++launches_;
    inject(t);
  }

  void gather_async(int64_t t, int kb) override {
    STB_REQUIRE(as_open_, STB_ERR_ARG, "async_begin first");
    for (int j = 0; j < kb; ++j) gather(t + j, t + j - as_t0_);
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
        os << "non-finite values in field group 'pq' at step " << as_guard_[i];
        throw Error(STB_ERR_UNSTABLE, os.str());
      }
  }

  void read_field(int field, int64_t t, void* out) override {
    STB_REQUIRE(field == 0 || field == 1, STB_ERR_ARG, "TTI field index: 0 = p, 1 = q");
    STB_REQUIRE(t_next_ == 0 || t == t_next_ - 1 || t == t_next_ - 2, STB_ERR_ARG,
                "only the last two time levels are resident");
    pad_read<T>(lv_[field][t & 1].p, d_, out, st_);
  }

  void level_ptr(int field, int64_t t, void** dev, int64_t* plane, int64_t* pitch) override {
    STB_REQUIRE(field == 0 || field == 1, STB_ERR_ARG, "TTI field index: 0 = p, 1 = q");
    *dev = lv_[field][t & 1].p + d_.H * d_.plane;
    if (plane) *plane = d_.plane;
    if (pitch) *pitch = d_.pitch;
  }

  void reset() override {
    for (auto& f : lv_)
      for (auto& l : f) l.zero(st_);
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
    int nmat = (inv_.p ? 1 : 0) + (e2_.p ? 1 : 0) + (d2_.p ? 1 : 0);
    for (auto& b : n_) nmat += b.p ? 1 : 0;
    int na = cf_.active[0] + cf_.active[1] + cf_.active[2];
    std::ostringstream os;
    if (fused_) {
      const int bpp = (int)sizeof(T) * (2 + 2 + 2 + nmat);
      if (pair_)
        os << "tti_fused2<f32,r=" << r_ << "," << (fast_ ? "fma" : "exact")
           << "> (TMA p/q plane ring + operand ring, 16x32 tile as z pairs, halo warps, FG ring, x chunk "
           << cx_ << ") k=1 requested_k=" << k << " bytes_per_point=" << bpp;
      else
        os << "tti_fused<f32,r=" << r_ << ",ring=" << m_for_r(r_) << "x" << (2 * r_ + 1)
           << "," << (fast_ ? "fma" : "exact")
           << "> (TMA p/q plane ring, 16x32 tile, x chunk " << cx_
           << ", F/G on chip) k=1 requested_k=" << k << " bytes_per_point=" << bpp;
    } else {
      const int bpp = (int)sizeof(T) * (2 + 2 * na + 2 * na + 4 + 2 + nmat);
      os << "tti_pass1+pass2<" << (sizeof(T) == 4 ? "f32" : "f64") << ",r=" << r_
         << "> (thread per point, zero-haloed layout) k=1 requested_k=" << k
         << " bytes_per_point=" << bpp;
    }
    return os.str();
  }

 private:
  // ring of M (2r+1) plane slots: M = 2 leaves 2r+1 planes of TMA lead;
  // so=16 (r = 4) only fits M = 1 in shared memory
  static constexpr int m_for_r(int r) { return r <= 3 ? 2 : 1; }

  template <int r>
  void launch_pair(const TtiFusedArgs& fa, int prev) {
    using C = Tti2Cfg<r>;
    dim3 grid((unsigned)((d_.nz + C::TZ - 1) / C::TZ), (unsigned)((d_.ny + C::TY - 1) / C::TY),
              (unsigned)((fa.x_hi - fa.x_lo + cx_ - 1) / cx_));
    const bool g = fa.nonfinite != nullptr;
    if (fast_ && g)
      tti_fused2<r, true, true><<<grid, C::NT, C::SMEM, st_>>>(maps2_[prev], fa);
    else if (fast_)
      tti_fused2<r, true, false><<<grid, C::NT, C::SMEM, st_>>>(maps2_[prev], fa);
    else if (g)
      tti_fused2<r, false, true><<<grid, C::NT, C::SMEM, st_>>>(maps2_[prev], fa);
    else
      tti_fused2<r, false, false><<<grid, C::NT, C::SMEM, st_>>>(maps2_[prev], fa);
  }

  template <int r>
  void set_fused_attr() {
    if constexpr (r <= 2) {
      const int sm = (int)Tti2Cfg<r>::SMEM;
      const auto a = cudaFuncAttributeMaxDynamicSharedMemorySize;
      STB_CUDA(cudaFuncSetAttribute(tti_fused2<r, false, false>, a, sm));
      STB_CUDA(cudaFuncSetAttribute(tti_fused2<r, false, true>, a, sm));
      STB_CUDA(cudaFuncSetAttribute(tti_fused2<r, true, false>, a, sm));
      STB_CUDA(cudaFuncSetAttribute(tti_fused2<r, true, true>, a, sm));
    }
    constexpr int M = m_for_r(r);
    STB_CUDA(cudaFuncSetAttribute(tti_fused<r, M, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)TtiFusedCfg<r, M>::smem_bytes()));
    STB_CUDA(cudaFuncSetAttribute(tti_fused<r, M, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)TtiFusedCfg<r, M>::smem_bytes()));
  }

  void setup_fused() {
    if constexpr (sizeof(T) == 4) {
      const int r = r_;
      // TMA view of the padded layout: dims (pitch, ny + 2H, nx + 2H)
      Dims md{};
      md.nx = d_.nx + 2 * d_.H;
      md.ny = d_.ny + 2 * d_.H;
      md.nz = d_.pitch;
      md.pitch = d_.pitch;
      md.plane = d_.plane;
      const uint32_t pz = kTtiTZ + 2 * ((2 * r + 3) / 4 * 4), py = kTtiTY + 4 * r;
      for (int l = 0; l < 2; ++l) {
        maps_[l].p = make_map3d_f32(reinterpret_cast<const float*>(lv_[0][l].p), md, pz, py, 1);
        maps_[l].q = make_map3d_f32(reinterpret_cast<const float*>(lv_[1][l].p), md, pz, py, 1);
      }
      if (pair_) {
        // tti_fused2: p/q boxes as above; n boxes over the pass-1 extent,
        // p/q (t-2) and inv/e2/d2 boxes over the tile
        const uint32_t ez = kTtiTZ + 2 * ((2 * ((r + 1) / 2) + 3) / 4 * 4), ey = kTtiTY + 2 * r;
        auto f32p = [](const T* b) { return reinterpret_cast<const float*>(b); };
        for (int l = 0; l < 2; ++l) {        // l = buffer of level t-1
          Tti2Maps& m = maps2_[l];
          m.p = maps_[l].p;
          m.q = maps_[l].q;
          for (int ax = 0; ax < 3; ++ax) m.n[ax] = make_map3d_f32(f32p(n_[ax].p), md, ez, ey, 1);
          m.o[0] = make_map3d_f32(f32p(lv_[0][l ^ 1].p), md, kTtiTZ, kTtiTY, 1);
          m.o[1] = make_map3d_f32(f32p(lv_[1][l ^ 1].p), md, kTtiTZ, kTtiTY, 1);
          m.o[2] = make_map3d_f32(f32p(inv_.p), md, kTtiTZ, kTtiTY, 1);
          m.o[3] = make_map3d_f32(f32p(e2_.p), md, kTtiTZ, kTtiTY, 1);
          m.o[4] = make_map3d_f32(f32p(d2_.p), md, kTtiTZ, kTtiTY, 1);
        }
      }
      switch (r) {
        case 1: set_fused_attr<1>(); break;
        case 2: set_fused_attr<2>(); break;
        case 3: set_fused_attr<3>(); break;
        case 4: set_fused_attr<4>(); break;
        default: break;
      }
    }
  }

  template <int r>
  void launch_fused_r(const TtiFusedArgs& fa, int prev) {
    if (fa.x_hi <= fa.x_lo) return;
    dim3 grid((unsigned)((d_.nz + kTtiTZ - 1) / kTtiTZ), (unsigned)((d_.ny + kTtiTY - 1) / kTtiTY),
              (unsigned)((fa.x_hi - fa.x_lo + cx_ - 1) / cx_));
    if constexpr (r <= 2) {
      if (pair_) {
        launch_pair<r>(fa, prev);
        return;
      }
    }
    constexpr int M = m_for_r(r);
    if (fast_)
      tti_fused<r, M, true><<<grid, kTtiThreads, TtiFusedCfg<r, M>::smem_bytes(), st_>>>(
          maps_[prev], fa);
    else
      tti_fused<r, M, false><<<grid, kTtiThreads, TtiFusedCfg<r, M>::smem_bytes(), st_>>>(
          maps_[prev], fa);
  }

  void launch_fused(const TtiArgs<T>& A, int prev, int x_lo, int x_hi) {
    if constexpr (sizeof(T) == 4) {
      TtiFusedArgs fa{};
      fa.p0 = A.p0;
      fa.q0 = A.q0;
      fa.inv = A.inv;
      fa.e2 = A.e2;
      fa.d2 = A.d2;
      for (int ax = 0; ax < 3; ++ax) fa.n[ax] = A.n[ax];
      fa.fx = A.fx;
      fa.fy = A.fy;
      fa.fz = A.fz;
      fa.has_fac = A.has_fac;
      fa.cf = A.cf;
      fa.d = A.d;
      fa.cx = cx_;
      fa.x_lo = x_lo;
      fa.x_hi = x_hi;
      fa.nonfinite = A.nonfinite;
      fa.negz = -0.0f;
      switch (r_) {
        case 1: launch_fused_r<1>(fa, prev); break;
        case 2: launch_fused_r<2>(fa, prev); break;
        case 3: launch_fused_r<3>(fa, prev); break;
        case 4: launch_fused_r<4>(fa, prev); break;
        default: throw Error(STB_ERR_CONFIG, "space_order: TTI supports 4, 8, 12, 16");
      }
    } else {
      (void)A;
      (void)prev;
      (void)x_lo;
      (void)x_hi;
    }
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

  int r_ = 1;
  bool fused_ = false;
  bool pair_ = true;          // tti_fused2 (r <= 2) unless STB_TTI_PATH=fused1
  bool fast_ = false;
  int rec_field_ = 0;        // p
  int cx_ = 150;
  bool as_open_ = false;
  int64_t as_t0_ = 0, as_n_ = 0;
  std::vector<int64_t> as_guard_;
  DevBuf<int> guards_;
  TtiMaps maps_[2];           // [level buffer] p/q tensor maps (fused path)
  Tti2Maps maps2_[2];         // [level buffer] tti_fused2's operand maps
  PDims d_{};
  stb_geometry geom_{};
  int64_t x_begin_ = 0;
  cudaStream_t st_ = nullptr;
  TtiCoefs<T> cf_{};
  DevBuf<T> lv_[2][2];      // [p|q][t mod 2]
  DevBuf<T> F_[3], G_[3];
  DevBuf<T> inv_, e2_, d2_, n_[3];
  DevBuf<T> fac_[3];
  bool has_fac_ = false;
  int64_t t_next_ = 0;
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

stb_prop_s* make_tti(const stb_tti_desc& d) {
  if (d.precision == 32) return new stb::TtiProp<float>(d);
  return new stb::TtiProp<double>(d);
}
