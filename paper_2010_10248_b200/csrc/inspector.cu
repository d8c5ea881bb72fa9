// GPU inspector: off-grid point -> on-grid support, ids and compression.
//
// Restates, on the device, the reference's precompute pipeline
//   interp_stencil           sparse.py:136-173   (stencils_kernel)
//   find_support/_source_entries precompute.py:103-125 (keep w > 0)
//   build_masks              precompute.py:150-165 (lexicographic ids)
//   compress                 precompute.py:168-180 (nnz / row_ptr / flat_z)
//   decompose_wavefields     precompute.py:183-206 (f64, source-major order)
//   precompute_receivers     precompute.py:267-284 (entries by (point, rid))
// Lexicographic (x, y, z) order of grid points equals ascending linear key
// x*ny*nz + y*nz + z, so one stable radix sort of (key, entry) pairs yields
// the sorted point list, the per-point entry segments in source-major order,
// and the per-(x, y) column CSR -- no dense mask is needed unless the caller
// asks for sm/sid.
#include <cub/cub.cuh>

#include <cfloat>
#include <cmath>
#include <sstream>

#include "fp_exact.cuh"
#include "stb_internal.cuh"

namespace stb {

namespace {

constexpr double kEps = 1e-9;  // sparse.py:20

struct GeomDev {
  int64_t n[3];
  double h[3], o[3];
};

GeomDev to_dev(const stb_geometry& g) {
  GeomDev d;
  for (int a = 0; a < 3; ++a) {
    d.n[a] = g.shape[a];
    d.h[a] = g.spacing[a];
    d.o[a] = g.origin[a];
  }
  return d;
}

// One thread per sparse point; bad_first records the smallest offending
// point (and axis) for a deterministic error message.
__global__ void stencils_kernel(const double* __restrict__ coords, int64_t n, GeomDev g,
                                int64_t margin, int64_t* __restrict__ idx,
                                double* __restrict__ w, unsigned long long* bad_first) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t base[3];
  double f[3];
  for (int a = 0; a < 3; ++a) {
    const double c = coords[i * 3 + a];
    const double frac = rdiv(rsub(c, g.o[a]), g.h[a]);   // grid.py:67-71
    const int64_t na = g.n[a];
    const double hi = __dadd_rn((double)(na - 1), kEps);
    bool bad = (frac < -kEps) || (frac > hi);            // sparse.py:146
    if (margin >= 0) {                                    // sparse.py:231-234
      const int64_t lo_m = na > 1 ? margin : 0;
      const int64_t hi_m = na - 1 - lo_m;
      bad = bad || (frac < __dsub_rn((double)lo_m, kEps)) ||
            (frac > __dadd_rn((double)hi_m, kEps));
    }
    if (bad) {
      atomicMin(bad_first, (unsigned long long)(i * 4 + a));
      return;
    }
    if (na == 1) {
      base[a] = 0;
      f[a] = 0.0;
      continue;
    }
    double fa = fmin(fmax(frac, 0.0), (double)(na - 1));
    int64_t i0 = (int64_t)floor(fa);
    if (i0 >= na - 1) i0 = na - 2;                        // upper face snap
    base[a] = i0;
    f[a] = rsub(fa, (double)i0);
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int bx = (c >> 2) & 1, by = (c >> 1) & 1, bz = c & 1;
    const int b[3] = {bx, by, bz};
    double wa[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      wa[a] = b[a] ? f[a] : rsub(1.0, f[a]);
      idx[(i * 8 + c) * 3 + a] = (g.n[a] == 1) ? 0 : base[a] + b[a];
    }
    w[i * 8 + c] = rmul(rmul(wa[0], wa[1]), wa[2]);      // ((wx*wy)*wz)
  }
}

__global__ void entry_keys_kernel(const int64_t* __restrict__ idx, const double* __restrict__ w,
                                  int64_t n8, int64_t ny, int64_t nz, int64_t drop_key,
                                  int keep_zero, int64_t* __restrict__ keys,
                                  int32_t* __restrict__ ent, unsigned long long* kept) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n8) return;
  const bool keep = keep_zero || (w[e] > 0.0);
  keys[e] = keep ? (idx[e * 3] * ny + idx[e * 3 + 1]) * nz + idx[e * 3 + 2] : drop_key;
  ent[e] = (int32_t)e;
  if (keep) atomicAdd(kept, 1ull);
}

__global__ void head_flags_kernel(const int64_t* __restrict__ keys, int64_t M,
                                  int32_t* __restrict__ head) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void unique_kernel(const int64_t* __restrict__ keys, const int32_t* __restrict__ incl,
                              const int32_t* __restrict__ head, int64_t M, int64_t nz,
                              int64_t* __restrict__ ukeys, int64_t* __restrict__ seg,
                              int64_t* __restrict__ ent_point, int32_t* __restrict__ nnz) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  const int64_t id = incl[i] - 1;
  ent_point[i] = id;
  if (head[i]) {
    ukeys[id] = keys[i];
    seg[id] = i;
    atomicAdd(&nnz[keys[i] / nz], 1);
  }
}

__global__ void set_last_kernel(int64_t* p, int64_t idx, int64_t v) { p[idx] = v; }

// src_dcmp[t, id]: thread per (t, id), id fastest (coalesced rows).
__global__ void decompose_kernel(const int64_t* __restrict__ seg, const int32_t* __restrict__ ent,
                                 const double* __restrict__ w, const double* __restrict__ scale,
                                 const double* __restrict__ wav, int64_t nsrc, int64_t K,
                                 int64_t nt_w, int64_t nt, double* __restrict__ out) {
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t t = blockIdx.y + (int64_t)gridDim.y * blockIdx.z;
  if (id >= K || t >= nt) return;
  double acc = 0.0;
  if (t < nt_w) {
    for (int64_t e = seg[id]; e < seg[id + 1]; ++e) {
      const int32_t en = ent[e];
      const int64_t s = en >> 3;
      acc = radd(acc, rmul(rmul(w[en], scale[s]), wav[t * nsrc + s]));
    }
  }
  out[t * K + id] = acc;
}

__global__ void scatter_masks_kernel(const int64_t* __restrict__ ukeys, int64_t K,
                                     uint8_t* __restrict__ sm, int32_t* __restrict__ sid) {
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= K) return;
  if (sm) sm[ukeys[id]] = 1;
  if (sid) sid[ukeys[id]] = (int32_t)id;
}

__global__ void split_keys_kernel(const int64_t* __restrict__ keys, int64_t n, int64_t ny,
                                  int64_t nz, int64_t* __restrict__ pts,
                                  int64_t* __restrict__ fz) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t k = keys[i];
  const int64_t z = k % nz, xy = k / nz;
  if (pts) {
    pts[i * 3] = xy / ny;
    pts[i * 3 + 1] = xy % ny;
    pts[i * 3 + 2] = z;
  }
  if (fz) fz[i] = z;
}

__global__ void entries_kernel(const int32_t* __restrict__ ent, const double* __restrict__ w,
                               int64_t M, int64_t* __restrict__ owner,
                               double* __restrict__ ew) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  owner[i] = ent[i] >> 3;
  ew[i] = w[ent[i]];
}

__global__ void iota32_kernel(int32_t* p, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = (int32_t)i;
}

struct CastI64 {
  __host__ __device__ int64_t operator()(int32_t v) const { return (int64_t)v; }
};

inline unsigned grid1(int64_t n, int b = 256) { return (unsigned)((n + b - 1) / b); }

int bit_length(uint64_t v) {
  int b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

}  // namespace

void stencils_compute(const double* coords_dev, int64_t n, const stb_geometry& g,
                      int64_t margin, int64_t* idx_dev, double* w_dev, cudaStream_t st) {
  if (n == 0) return;
  DevBuf<unsigned long long> bad(1);
  const unsigned long long init = ~0ull;
  STB_CUDA(cudaMemcpyAsync(bad.p, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  stencils_kernel<<<grid1(n), 256, 0, st>>>(coords_dev, n, to_dev(g), margin, idx_dev, w_dev,
                                            bad.p);
  STB_CHECK_LAUNCH();
  unsigned long long h = 0;
  STB_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  STB_CUDA(cudaStreamSynchronize(st));
  if (h != ~0ull) {
    const int64_t i = (int64_t)(h / 4);
    const int a = (int)(h % 4);
    double c[3];
    STB_CUDA(cudaMemcpy(c, coords_dev + i * 3, sizeof(c), cudaMemcpyDeviceToHost));
    std::ostringstream os;
    os.precision(17);
    os << "coordinate (" << c[0] << ", " << c[1] << ", " << c[2] << ") [point " << i
       << "] outside allowed region on axis " << a;
    if (margin > 0) os << " (margin " << margin << " points)";
    throw Error(STB_ERR_DOMAIN, os.str());
  }
}

// Sort (key, entry) pairs (dropped entries carry key N and sort last), then
// derive unique lexicographic points, per-point entry segments and the
// per-column CSR (build_masks + compress, precompute.py:150-180).
static void finish_from_keys(Support& s, DevBuf<int64_t>& keys_in, DevBuf<int32_t>& ent_in,
                             int64_t n_entries, int64_t kept, cudaStream_t st) {
  const int64_t nx = s.shape[0], ny = s.shape[1], nz = s.shape[2];
  const int64_t N = nx * ny * nz;
  DevBuf<int64_t> keys_out(n_entries);
  DevBuf<int32_t> ent_out(n_entries);
  const int end_bit = bit_length((uint64_t)N);
  size_t tmp_bytes = 0;
  STB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in.p, keys_out.p, ent_in.p,
                                           ent_out.p, (int)n_entries, 0, end_bit, st));
  DevBuf<uint8_t> tmp(tmp_bytes);
  STB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys_in.p, keys_out.p, ent_in.p,
                                           ent_out.p, (int)n_entries, 0, end_bit, st));
  s.M = kept;
  if (s.M == 0) {
    s.K = 0;
    s.row_ptr.zero(st);
    s.seg_start.alloc(1);
    s.seg_start.zero(st);
    STB_CUDA(cudaStreamSynchronize(st));
    return;
  }
  DevBuf<int32_t> head(s.M), incl(s.M);
  head_flags_kernel<<<grid1(s.M), 256, 0, st>>>(keys_out.p, s.M, head.p);
  STB_CHECK_LAUNCH();
  tmp_bytes = 0;
  STB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, head.p, incl.p, (int)s.M, st));
  tmp.alloc(tmp_bytes);
  STB_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tmp_bytes, head.p, incl.p, (int)s.M, st));
  int32_t K = 0;
  STB_CUDA(cudaMemcpyAsync(&K, incl.p + (s.M - 1), sizeof(K), cudaMemcpyDeviceToHost, st));
  STB_CUDA(cudaStreamSynchronize(st));
  s.K = K;
  s.keys.alloc(K);
  s.seg_start.alloc(K + 1);
  s.ent_point.alloc(s.M);
  unique_kernel<<<grid1(s.M), 256, 0, st>>>(keys_out.p, incl.p, head.p, s.M, nz, s.keys.p,
                                            s.seg_start.p, s.ent_point.p, s.nnz.p);
  STB_CHECK_LAUNCH();
  set_last_kernel<<<1, 1, 0, st>>>(s.seg_start.p, K, s.M);
  // row_ptr = exclusive scan of per-column counts, row_ptr[nx*ny] = K
  tmp_bytes = 0;
  cub::TransformInputIterator<int64_t, CastI64, const int32_t*> cast_it(s.nnz.p, CastI64());
  STB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cast_it, s.row_ptr.p,
                                         (int)(nx * ny), st));
  tmp.alloc(tmp_bytes);
  STB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, cast_it, s.row_ptr.p,
                                         (int)(nx * ny), st));
  set_last_kernel<<<1, 1, 0, st>>>(s.row_ptr.p, nx * ny, (int64_t)K);
  STB_CHECK_LAUNCH();
  s.ent_key = std::move(keys_out);
  s.ent_entry = std::move(ent_out);
  s.ent_key.n = s.M;
  s.ent_entry.n = s.M;
  STB_CUDA(cudaStreamSynchronize(st));
}

void support_build(Support& s, const double* coords_host, int64_t n, const stb_geometry& g,
                   bool keep_zero, cudaStream_t st) {
  for (int a = 0; a < 3; ++a) {
    s.shape[a] = g.shape[a];
    s.spacing[a] = g.spacing[a];
    s.origin[a] = g.origin[a];
    STB_REQUIRE(g.shape[a] >= 1, STB_ERR_ARG, "every shape extent must be >= 1");
  }
  s.n_points = n;
  s.keep_zero = keep_zero;
  const int64_t nx = g.shape[0], ny = g.shape[1], nz = g.shape[2];
  const int64_t N = nx * ny * nz;
  s.nnz.alloc(nx * ny);
  s.nnz.zero(st);
  s.row_ptr.alloc(nx * ny + 1);
  if (n == 0) {
    s.K = s.M = 0;
    s.row_ptr.zero(st);
    s.seg_start.alloc(1);
    s.seg_start.zero(st);
    STB_CUDA(cudaStreamSynchronize(st));
    return;
  }
  STB_REQUIRE(8 * n < (int64_t)INT32_MAX, STB_ERR_ARG, "too many sparse points");
  DevBuf<double> coords(n * 3);
  coords.upload(coords_host, n * 3, st);
  s.idx.alloc(n * 24);
  s.w.alloc(n * 8);
  stencils_compute(coords.p, n, g, -1, s.idx.p, s.w.p, st);

  const int64_t n8 = n * 8;
  DevBuf<int64_t> keys_in(n8);
  DevBuf<int32_t> ent_in(n8);
  DevBuf<unsigned long long> kept(1);
  kept.zero(st);
  entry_keys_kernel<<<grid1(n8), 256, 0, st>>>(s.idx.p, s.w.p, n8, ny, nz, N, keep_zero ? 1 : 0,
                                               keys_in.p, ent_in.p, kept.p);
  STB_CHECK_LAUNCH();
  unsigned long long M = 0;
  STB_CUDA(cudaMemcpyAsync(&M, kept.p, sizeof(M), cudaMemcpyDeviceToHost, st));
  STB_CUDA(cudaStreamSynchronize(st));
  finish_from_keys(s, keys_in, ent_in, n8, (int64_t)M, st);
}

void support_from_points(Support& s, const int64_t* points_host, int64_t n,
                         const stb_geometry& g, cudaStream_t st) {
  for (int a = 0; a < 3; ++a) {
    s.shape[a] = g.shape[a];
    s.spacing[a] = g.spacing[a];
    s.origin[a] = g.origin[a];
  }
  s.n_points = 0;
  s.keep_zero = true;
  const int64_t nx = g.shape[0], ny = g.shape[1], nz = g.shape[2];
  s.nnz.alloc(nx * ny);
  s.nnz.zero(st);
  s.row_ptr.alloc(nx * ny + 1);
  if (n == 0) {
    s.K = s.M = 0;
    s.row_ptr.zero(st);
    s.seg_start.alloc(1);
    s.seg_start.zero(st);
    STB_CUDA(cudaStreamSynchronize(st));
    return;
  }
  STB_REQUIRE(n < (int64_t)INT32_MAX, STB_ERR_ARG, "too many points");
  std::vector<int64_t> keys(n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t x = points_host[3 * i], y = points_host[3 * i + 1], z = points_host[3 * i + 2];
    STB_REQUIRE(x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz, STB_ERR_ARG,
                "support indices leave the grid interior");
    keys[i] = (x * ny + y) * nz + z;
  }
  DevBuf<int64_t> keys_in(n);
  DevBuf<int32_t> ent_in(n);
  keys_in.upload(keys.data(), n, st);
  iota32_kernel<<<grid1(n), 256, 0, st>>>(ent_in.p, n);
  STB_CHECK_LAUNCH();
  finish_from_keys(s, keys_in, ent_in, n, n, st);
}

void support_decompose_dev(const Support& s, const double* wav_dev, int64_t nt_w,
                           const double* scale_dev, int64_t nt, double* out_dev,
                           cudaStream_t st) {
  if (s.K == 0 || nt == 0) return;
  const int64_t yz = nt;
  dim3 grid(grid1(s.K), (unsigned)std::min<int64_t>(yz, 65535),
            (unsigned)((yz + 65534) / 65535));
  decompose_kernel<<<grid, 256, 0, st>>>(s.seg_start.p, s.ent_entry.p, s.w.p, scale_dev, wav_dev,
                                         s.n_points, s.K, nt_w, nt, out_dev);
  STB_CHECK_LAUNCH();
}

void support_points_host(const Support& s, int64_t* points, cudaStream_t st) {
  if (s.K == 0) return;
  DevBuf<int64_t> pts(s.K * 3);
  split_keys_kernel<<<grid1(s.K), 256, 0, st>>>(s.keys.p, s.K, s.shape[1], s.shape[2], pts.p,
                                                nullptr);
  STB_CHECK_LAUNCH();
  pts.download(points, s.K * 3, st);
  STB_CUDA(cudaStreamSynchronize(st));
}

void support_compress_host(const Support& s, int32_t* nnz, int64_t* row_ptr, int64_t* flat_z,
                           int32_t* flat_id, cudaStream_t st) {
  const int64_t cols = s.shape[0] * s.shape[1];
  if (nnz) s.nnz.download(nnz, cols, st);
  if (row_ptr) s.row_ptr.download(row_ptr, cols + 1, st);
  if (s.K) {
    if (flat_z) {
      DevBuf<int64_t> fz(s.K);
      split_keys_kernel<<<grid1(s.K), 256, 0, st>>>(s.keys.p, s.K, s.shape[1], s.shape[2],
                                                    nullptr, fz.p);
      STB_CHECK_LAUNCH();
      fz.download(flat_z, s.K, st);
      STB_CUDA(cudaStreamSynchronize(st));
    }
    if (flat_id) {
      DevBuf<int32_t> fi(s.K);
      iota32_kernel<<<grid1(s.K), 256, 0, st>>>(fi.p, s.K);
      STB_CHECK_LAUNCH();
      fi.download(flat_id, s.K, st);
      STB_CUDA(cudaStreamSynchronize(st));
    }
  }
  STB_CUDA(cudaStreamSynchronize(st));
}

void support_masks_host(const Support& s, uint8_t* sm, int32_t* sid, cudaStream_t st) {
  const int64_t N = s.shape[0] * s.shape[1] * s.shape[2];
  DevBuf<uint8_t> dsm(sm ? N : 0);
  DevBuf<int32_t> dsid(sid ? N : 0);
  if (sm) STB_CUDA(cudaMemsetAsync(dsm.p, 0, N, st));
  if (sid) STB_CUDA(cudaMemsetAsync(dsid.p, 0xff, N * sizeof(int32_t), st));
  if (s.K) {
    scatter_masks_kernel<<<grid1(s.K), 256, 0, st>>>(s.keys.p, s.K, dsm.p, dsid.p);
    STB_CHECK_LAUNCH();
  }
  if (sm) dsm.download(sm, N, st);
  if (sid) dsid.download(sid, N, st);
  STB_CUDA(cudaStreamSynchronize(st));
}

void support_entries_host(const Support& s, int64_t* points, int64_t* owner, double* w,
                          cudaStream_t st) {
  if (s.M == 0) return;
  DevBuf<int64_t> pts(s.M * 3), own(s.M);
  DevBuf<double> ew(s.M);
  split_keys_kernel<<<grid1(s.M), 256, 0, st>>>(s.ent_key.p, s.M, s.shape[1], s.shape[2], pts.p,
                                                nullptr);
  entries_kernel<<<grid1(s.M), 256, 0, st>>>(s.ent_entry.p, s.w.p, s.M, own.p, ew.p);
  STB_CHECK_LAUNCH();
  if (points) pts.download(points, s.M * 3, st);
  if (owner) own.download(owner, s.M, st);
  if (w) ew.download(w, s.M, st);
  STB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace stb
