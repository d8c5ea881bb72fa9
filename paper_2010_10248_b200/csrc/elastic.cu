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
#include <memory>
#include <sstream>

#include "fp_exact.cuh"
#include "sparse_ops.cuh"
#include "stb_internal.cuh"

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
struct ElFields {
  T* f[NFIELDS];
  const T* buoy;
  const T* lam;
  const T* mu;
  const T* fx;
  const T* fy;
  const T* fz;
  int has_fac;
};

template <typename T, int R>
__device__ __forceinline__ T stag(const T* __restrict__ a, int64_t i, int64_t stride,
                                  int64_t pos, int64_t n, const T* c, bool fwd) {
  T acc = T(0);
#pragma unroll
  for (int j = 1; j <= R; ++j) {
    const int hi = fwd ? j : j - 1;
    const int lo = fwd ? -(j - 1) : -j;
    const T vh = (pos + hi < n && pos + hi >= 0) ? a[i + hi * stride] : T(0);
    const T vl = (pos + lo < n && pos + lo >= 0) ? a[i + lo * stride] : T(0);
    const T term = rmul(rsub(vh, vl), c[j - 1]);
    acc = (j == 1) ? term : radd(acc, term);
  }
  return acc;
}

struct Pt {
  int64_t i, pos[3], n[3], stride[3];
};

__device__ __forceinline__ Pt make_pt(const Dims& d, int64_t x, int64_t y, int64_t z) {
  Pt p;
  p.i = x * d.plane + y * d.pitch + z;
  p.pos[0] = x; p.pos[1] = y; p.pos[2] = z;
  p.n[0] = d.nx; p.n[1] = d.ny; p.n[2] = d.nz;
  p.stride[0] = d.plane; p.stride[1] = d.pitch; p.stride[2] = 1;
  return p;
}

// Sum of the active terms in order (physics.py:314-321); has = any active.
template <typename T, int R>
__device__ __forceinline__ T dsum3(const ElCoefs<T>& cf, const Pt& p, const T* a0, int ax0,
                                   bool f0, const T* a1, int ax1, bool f1, const T* a2, int ax2,
                                   bool f2, bool& has) {
  const T* arr[3] = {a0, a1, a2};
  const int ax[3] = {ax0, ax1, ax2};
  const bool fw[3] = {f0, f1, f2};
  T acc = T(0);
  has = false;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (!cf.active[ax[k]]) continue;
    const T d = stag<T, R>(arr[k], p.i, p.stride[ax[k]], p.pos[ax[k]], p.n[ax[k]],
                           cf.d1[ax[k]], fw[k]);
    acc = has ? radd(acc, d) : d;
    has = true;
  }
  return acc;
}

template <typename T>
__device__ __forceinline__ T fac_at(const ElFields<T>& F, int64_t x, int64_t y, int64_t z) {
  return tmin(tmin(F.fx[x], F.fy[y]), F.fz[z]);
}

template <typename T, int R>
__global__ void __launch_bounds__(128)
elastic_v_step(ElFields<T> F, ElCoefs<T> cf, Dims d) {
  const int64_t z = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t y = blockIdx.y, x = blockIdx.z;
  if (z >= d.nz) return;
  const Pt p = make_pt(d, x, y, z);
  const T buoy = F.buoy ? F.buoy[p.i] : cf.buoy;
  bool h0, h1, h2;
  // elastic_update_v (physics.py:348-362)
  const T dvx = dsum3<T, R>(cf, p, F.f[TXX], 0, true, F.f[TXY], 1, false, F.f[TXZ], 2, false, h0);
  const T dvy = dsum3<T, R>(cf, p, F.f[TXY], 0, false, F.f[TYY], 1, true, F.f[TYZ], 2, false, h1);
  const T dvz = dsum3<T, R>(cf, p, F.f[TXZ], 0, false, F.f[TYZ], 1, false, F.f[TZZ], 2, true, h2);
  const T fac = F.has_fac ? fac_at(F, x, y, z) : T(1);
  const T incs[3] = {dvx, dvy, dvz};
  const bool has[3] = {h0, h1, h2};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T o = F.f[VX + k][p.i];
    if (has[k]) o = radd(o, rmul(incs[k], buoy));
    if (F.has_fac) o = rmul(o, fac);
    F.f[VX + k][p.i] = o;
  }
}

template <typename T, int R>
__global__ void __launch_bounds__(128)
elastic_tau_step(ElFields<T> F, ElCoefs<T> cf, Dims d) {
  const int64_t z = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t y = blockIdx.y, x = blockIdx.z;
  if (z >= d.nz) return;
  const Pt p = make_pt(d, x, y, z);
  const T lam = F.lam ? F.lam[p.i] : cf.lam;
  const T mu = F.mu ? F.mu[p.i] : cf.mu;
  const T mu2 = rmul(mu, T(2));
  const T fac = F.has_fac ? fac_at(F, x, y, z) : T(1);
  // elastic_update_tau (physics.py:385-429)
  T dg[3];
  bool hd[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    hd[a] = cf.active[a] != 0;
    dg[a] = hd[a] ? stag<T, R>(F.f[VX + a], p.i, p.stride[a], p.pos[a], p.n[a], cf.d1[a], false)
                  : T(0);
  }
  T tr = T(0);
  bool htr = false;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (!hd[a]) continue;
    tr = htr ? radd(tr, dg[a]) : dg[a];
    htr = true;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    T inc = T(0);
    bool hi = false;
    if (htr) {
      inc = rmul(tr, lam);
      hi = true;
    }
    if (hd[a]) {
      const T d2 = rmul(dg[a], mu2);
      inc = hi ? radd(inc, d2) : d2;
      hi = true;
    }
    T o = F.f[TXX + a][p.i];
    if (hi) o = radd(o, inc);
    if (F.has_fac) o = rmul(o, fac);
    F.f[TXX + a][p.i] = o;
  }
  // shear: (txy: d_y vx, d_x vy), (txz: d_z vx, d_x vz), (tyz: d_z vy, d_y vz)
  const int sa1[3] = {1, 2, 2}, sf1[3] = {VX, VX, VY};
  const int sa2[3] = {0, 0, 1}, sf2[3] = {VY, VZ, VZ};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T s = T(0);
    bool hs = false;
    if (cf.active[sa1[k]]) {
      s = stag<T, R>(F.f[sf1[k]], p.i, p.stride[sa1[k]], p.pos[sa1[k]], p.n[sa1[k]],
                     cf.d1[sa1[k]], true);
      hs = true;
    }
    if (cf.active[sa2[k]]) {
      const T d2 = stag<T, R>(F.f[sf2[k]], p.i, p.stride[sa2[k]], p.pos[sa2[k]], p.n[sa2[k]],
                              cf.d1[sa2[k]], true);
      s = hs ? radd(s, d2) : d2;
      hs = true;
    }
    T o = F.f[TXY + k][p.i];
    if (hs) o = radd(o, rmul(s, mu));
    if (F.has_fac) o = rmul(o, fac);
    F.f[TXY + k][p.i] = o;
  }
}

// dt/rho, dt*lam, dt*mu from per-point (or scalar) Lame parameters.
template <typename T>
__global__ void elastic_materials_kernel(const double* __restrict__ lam,
                                         const double* __restrict__ mu,
                                         const double* __restrict__ rho, double dt, Dims d,
                                         T* __restrict__ buoy, T* __restrict__ lam_dt,
                                         T* __restrict__ mu_dt) {
  const int64_t n = d.nx * d.ny * d.nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i % d.nz, xy = i / d.nz;
    const int64_t o = xy * d.pitch + z;
    if (buoy) buoy[o] = from_f64<T>(rdiv(dt, rho[i]));
    if (lam_dt) lam_dt[o] = from_f64<T>(rmul(dt, lam[i]));
    if (mu_dt) mu_dt[o] = from_f64<T>(rmul(dt, mu[i]));
  }
}

template <typename T>
__global__ void table_kernel_el(const double* __restrict__ src, int64_t n, T* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src ? from_f64<T>(src[i]) : T(1);
}

template <typename T>
__global__ void to_dtype_kernel_el(const double* __restrict__ src, int64_t n, T* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = from_f64<T>(src[i]);
}

__global__ void keys_to_offsets_el(const int64_t* __restrict__ keys, int64_t n, Dims d,
                                   int64_t* __restrict__ off) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t k = keys[i];
  off[i] = (k / d.nz) * d.pitch + k % d.nz;
}

__global__ void idx_to_offsets_el(const int64_t* __restrict__ idx, int64_t n8, Dims d,
                                  int64_t* __restrict__ off) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n8) return;
  off[i] = (idx[i * 3] * d.ny + idx[i * 3 + 1]) * d.pitch + idx[i * 3 + 2];
}

template <typename T, int R>
void launch_el(cudaStream_t st, const ElFields<T>& F, const ElCoefs<T>& cf, const Dims& d) {
  dim3 block(128), grid((unsigned)((d.nz + 127) / 128), (unsigned)d.ny, (unsigned)d.nx);
  elastic_v_step<T, R><<<grid, block, 0, st>>>(F, cf, d);
  elastic_tau_step<T, R><<<grid, block, 0, st>>>(F, cf, d);
}

}  // namespace

template <typename T>
class ElasticProp final : public stb_prop_s {
 public:
  explicit ElasticProp(const stb_elastic_desc& desc) {
    R_ = desc.space_order / 2;
    d_ = make_dims(desc.geom.shape, sizeof(T));
    geom_ = desc.geom;
    STB_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    for (int a = 0; a < 3; ++a) {
      cf_.active[a] = desc.active[a] ? 1 : 0;
      for (int j = 0; j < 8; ++j) cf_.d1[a][j] = (T)desc.d1[a][j];
    }
    for (auto& f : f_) {
      f.alloc(d_.total());
      f.zero(st_);
    }
    const int64_t n = d_.npoints();
    const double dt = desc.dt;
    // materials (physics.py:251-257)
    const bool any_arr = desc.lam || desc.mu || desc.rho;
    if (any_arr) {
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
      buoy_.alloc(d_.total());
      lam_.alloc(d_.total());
      mu_.alloc(d_.total());
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
    has_fac_ = desc.damp[0] || desc.damp[1] || desc.damp[2];
    const int64_t n3[3] = {d_.nx, d_.ny, d_.nz};
    for (int a = 0; a < 3; ++a) {
      fac_[a].alloc(n3[a]);
      DevBuf<double> tmp(desc.damp[a] ? n3[a] : 0);
      if (desc.damp[a]) tmp.upload(desc.damp[a], n3[a], st_);
      table_kernel_el<T><<<g1(n3[a]), 256, 0, st_>>>(desc.damp[a] ? tmp.p : nullptr, n3[a],
                                                     fac_[a].p);
      STB_CHECK_LAUNCH();
      STB_CUDA(cudaStreamSynchronize(st_));
    }
  }

  ~ElasticProp() override {
    for (auto& e : events_) cudaEventDestroy(e);
    if (st_) cudaStreamDestroy(st_);
  }

  void set_sources(Support& s, const double* wav, int64_t nt_w, const double* scale,
                   int64_t nt) override {
    for (int a = 0; a < 3; ++a)
      STB_REQUIRE(s.shape[a] == geom_.shape[a], STB_ERR_ARG,
                  "support was built for a different grid shape");
    K_ = s.K;
    src_nt_ = nt;
    if (K_ == 0) return;
    DevBuf<double> dwav(nt_w * s.n_points), dscale(s.n_points), dc(nt * K_);
    dwav.upload(wav, nt_w * s.n_points, st_);
    dscale.upload(scale, s.n_points, st_);
    support_decompose_dev(s, dwav.p, nt_w, dscale.p, nt, dc.p, st_);
    series_.alloc(nt * K_);
    to_dtype_kernel_el<T><<<g1(nt * K_), 256, 0, st_>>>(dc.p, nt * K_, series_.p);
    src_off_.alloc(K_);
    keys_to_offsets_el<<<g1(K_), 256, 0, st_>>>(s.keys.p, K_, d_, src_off_.p);
    STB_CHECK_LAUNCH();
    STB_CUDA(cudaStreamSynchronize(st_));
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
    idx_to_offsets_el<<<g1(nrec * 8), 256, 0, st_>>>(idx.p, nrec * 8, d_, rec_off_.p);
    STB_CHECK_LAUNCH();
    STB_CUDA(cudaStreamSynchronize(st_));
  }

  void run(int64_t t0, int64_t nsteps, int k, double* rec_out, int64_t* bad_step) override {
    if (bad_step) *bad_step = -1;
    if (nsteps <= 0) return;
    STB_REQUIRE(K_ == 0 || t0 + nsteps <= src_nt_, STB_ERR_ARG,
                "run extends past the decomposed source series");
    STB_REQUIRE(t0 == t_next_, STB_ERR_ARG,
                "elastic handles update in place: steps must be run in order");
    (void)k;
    DevBuf<double> rec(nrec_ && rec_out ? nsteps * nrec_ : 0);
    std::vector<int64_t> guard_steps;
    for (int64_t t = t0; t < t0 + nsteps; ++t)
      if (t > 0 && t % 32 == 0) guard_steps.push_back(t);
    DevBuf<int> guards(guard_steps.size() + 1);
    guards.zero(st_);
    ensure_events(nsteps);
    ElFields<T> F;
    for (int i = 0; i < NFIELDS; ++i) F.f[i] = f_[i].p;
    F.buoy = buoy_.p;
    F.lam = lam_.p;
    F.mu = mu_.p;
    F.fx = fac_[0].p;
    F.fy = fac_[1].p;
    F.fz = fac_[2].p;
    F.has_fac = has_fac_ ? 1 : 0;
    launches_ = 0;
    size_t gi = 0;
    for (int64_t t = t0; t < t0 + nsteps; ++t) {
      STB_CUDA(cudaEventRecord(events_[2 * launches_], st_));
      switch (R_) {
        case 1: launch_el<T, 1>(st_, F, cf_, d_); break;
        case 2: launch_el<T, 2>(st_, F, cf_, d_); break;
        case 3: launch_el<T, 3>(st_, F, cf_, d_); break;
        case 4: launch_el<T, 4>(st_, F, cf_, d_); break;
        case 5: launch_el<T, 5>(st_, F, cf_, d_); break;
        case 6: launch_el<T, 6>(st_, F, cf_, d_); break;
        case 7: launch_el<T, 7>(st_, F, cf_, d_); break;
        case 8: launch_el<T, 8>(st_, F, cf_, d_); break;
        default: throw Error(STB_ERR_ARG, "space_order must be even in [2, 16]");
      }
      STB_CHECK_LAUNCH();
      STB_CUDA(cudaEventRecord(events_[2 * launches_ + 1], st_));
      ++launches_;
      if (gi < guard_steps.size() && guard_steps[gi] == t) {
        for (int fi = 0; fi < NFIELDS; ++fi)
          nonfinite_kernel<T><<<1184, 256, 0, st_>>>(f_[fi].p, d_, guards.p + gi);
        STB_CHECK_LAUNCH();
        ++gi;
      }
      if (K_) {
        for (int fi = TXX; fi <= TZZ; ++fi)
          inject_kernel<T><<<g1(K_), 256, 0, st_>>>(f_[fi].p, src_off_.p, series_.p + t * K_, K_);
        STB_CHECK_LAUNCH();
      }
      if (rec.n) {
        gather_kernel<T><<<g1(nrec_), 256, 0, st_>>>(f_[TXX].p, rec_off_.p, rec_w_.p, nrec_,
                                                     rec.p + (t - t0) * nrec_);
        STB_CHECK_LAUNCH();
      }
    }
    t_next_ = t0 + nsteps;
    updates_ = nsteps * d_.npoints() * NFIELDS;
    if (rec.n) rec.download(rec_out, nsteps * nrec_, st_);
    std::vector<int> gh(guard_steps.size() + 1, 0);
    if (!guard_steps.empty()) guards.download(gh.data(), guard_steps.size(), st_);
    STB_CUDA(cudaStreamSynchronize(st_));
    for (size_t i = 0; i < guard_steps.size(); ++i) {
      if (gh[i]) {
        if (bad_step) *bad_step = guard_steps[i];
        std::ostringstream os;
        os << "non-finite values in field group 'v' at step " << guard_steps[i];
        throw Error(STB_ERR_UNSTABLE, os.str());
      }
    }
  }

  void read_field(int field, int64_t t, void* out) override {
    STB_REQUIRE(field >= 0 && field < NFIELDS, STB_ERR_ARG, "elastic field index in [0, 9)");
    STB_REQUIRE(t == t_next_ - 1 || (t_next_ == 0), STB_ERR_ARG,
                "only the latest time level is resident for elastic handles");
    STB_CUDA(cudaMemcpy2DAsync(out, d_.nz * sizeof(T), f_[field].p, d_.pitch * sizeof(T),
                               d_.nz * sizeof(T), d_.nx * d_.ny, cudaMemcpyDeviceToHost, st_));
    STB_CUDA(cudaStreamSynchronize(st_));
  }

  void level_ptr(int field, int64_t t, void** dev, int64_t* plane, int64_t* pitch) override {
    STB_REQUIRE(field >= 0 && field < NFIELDS, STB_ERR_ARG, "elastic field index in [0, 9)");
    (void)t;
    *dev = f_[field].p;
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
    if (all_launches) *all_launches = launches_ * 2;
    if (run_ms) *run_ms = total;
  }

  std::string describe(int k) override {
    std::ostringstream os;
    os << "elastic_reference_step<" << (sizeof(T) == 4 ? "f32" : "f64") << ",R=" << R_
       << "> k=" << (k < 1 ? 1 : k);
    return os.str();
  }

 private:
  void ensure_events(int64_t n) {
    while ((int64_t)events_.size() < 2 * n) {
      cudaEvent_t e;
      STB_CUDA(cudaEventCreate(&e));
      events_.push_back(e);
    }
  }

  int R_ = 1;
  Dims d_{};
  stb_geometry geom_{};
  cudaStream_t st_ = nullptr;
  ElCoefs<T> cf_{};
  DevBuf<T> f_[NFIELDS];
  DevBuf<T> buoy_, lam_, mu_;
  DevBuf<T> fac_[3];
  bool has_fac_ = false;
  int64_t t_next_ = 0;
  int64_t K_ = 0, src_nt_ = 0;
  DevBuf<T> series_;
  DevBuf<int64_t> src_off_;
  int64_t nrec_ = 0;
  DevBuf<int64_t> rec_off_;
  DevBuf<double> rec_w_;
  std::vector<cudaEvent_t> events_;
  int64_t launches_ = 0, updates_ = 0;
};

}  // namespace stb

stb_prop_s* make_elastic(const stb_elastic_desc& d) {
  if (d.precision == 32) return new stb::ElasticProp<float>(d);
  return new stb::ElasticProp<double>(d);
}
