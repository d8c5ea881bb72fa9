// Sparse operators shared by the propagators: fused injection of the
// decomposed series (precompute.py:209-252) and the per-step receiver
// gather (sparse.py:197-207).
#pragma once

#include "fp_exact.cuh"
#include "stb_internal.cuh"

namespace stb {

// u[p] += T(src_dcmp[t, id]) for the K affected points (one add per point,
// as scatter_box does; the series is pre-rounded to T on upload, matching
// `dcmp.src_dcmp[t, m].astype(field.dtype)`).
template <typename T>
__global__ void inject_kernel(T* __restrict__ u, const int64_t* __restrict__ off,
                              const T* __restrict__ series_t, int64_t K) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int64_t o = off[k];
  u[o] = radd(u[o], series_t[k]);
}

// data[t, r] = sum_c w_c * u[corner_c] with NumPy's 8-wide pairwise
// summation (record_receivers -> ndarray.sum(axis=1) over 8 f64 products).
template <typename T>
__device__ __forceinline__ double pairwise8(const double* w, const T* v) {
  double p[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) p[c] = rmul(w[c], (double)v[c]);
  return radd(radd(radd(p[0], p[1]), radd(p[2], p[3])),
              radd(radd(p[4], p[5]), radd(p[6], p[7])));
}

template <typename T>
__global__ void gather_kernel(const T* __restrict__ u, const int64_t* __restrict__ off,
                              const double* __restrict__ w, int64_t nrec,
                              double* __restrict__ out_row) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  T v[8];
  double ww[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    v[c] = u[off[r * 8 + c]];
    ww[c] = w[r * 8 + c];
  }
  out_row[r] = pairwise8<T>(ww, v);
}

// Non-finite detection (engine.py:354-360) over a pitched interior.
template <typename T>
__global__ void nonfinite_kernel(const T* __restrict__ u, Dims d, int* flag) {
  const int64_t n = d.nx * d.ny * d.nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i % d.nz, xy = i / d.nz;
    if (!finite(u[xy * d.pitch + z])) {
      atomicExch(flag, 1);
      return;
    }
  }
}

}  // namespace stb
