// Zero-haloed field layout shared by the elastic and TTI propagators, and
// the small helper kernels that map compact (host-order) data onto it.
#pragma once

#include "fp_exact.cuh"
#include "stb_internal.cuh"

namespace stb {
namespace {

// Zero-haloed layout.
struct PDims {
  int64_t nx, ny, nz;     // interior
  int64_t H;              // halo width (>= R)
  int64_t zoff;           // interior z offset within a row (128-byte aligned)
  int64_t pitch;          // row length (elements)
  int64_t plane;          // (ny + 2H) * pitch
  int64_t total;          // (nx + 2H) * plane
  __host__ __device__ int64_t at(int64_t x, int64_t y, int64_t z) const {
    return ((x + H) * (ny + 2 * H) + (y + H)) * pitch + zoff + z;
  }
};

PDims make_pdims(int64_t nx, int64_t ny, int64_t nz, int R, size_t elem) {
  PDims p;
  p.nx = nx; p.ny = ny; p.nz = nz;
  p.H = R;
  const int64_t per128 = 128 / (int64_t)elem;
  p.zoff = round_up(R, per128);
  p.pitch = round_up(p.zoff + nz + R, per128);
  p.plane = (ny + 2 * p.H) * p.pitch;
  p.total = (nx + 2 * p.H) * p.plane;
  return p;
}

template <typename T>
__global__ void pad_table_kernel(const double* __restrict__ src, int64_t n, T* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src ? from_f64<T>(src[i]) : T(1);
}

template <typename T>
__global__ void pad_to_dtype_kernel(const double* __restrict__ src, int64_t n, T* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = from_f64<T>(src[i]);
}

__global__ void pad_keys_to_offsets(const int64_t* __restrict__ keys, int64_t n, int64_t gny,
                                   int64_t gnz, int64_t x_begin, PDims d,
                                   int64_t* __restrict__ off) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t k = keys[i];
  const int64_t z = k % gnz, xy = k / gnz;
  off[i] = d.at(xy / gny - x_begin, xy % gny, z);
}

__global__ void pad_idx_to_offsets(const int64_t* __restrict__ idx, int64_t n8, int64_t x_begin,
                                  PDims d, int64_t* __restrict__ off, int* bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n8) return;
  const int64_t x = idx[i * 3] - x_begin;
  if (x < 0 || x >= d.nx) {
    atomicExch(bad, 1);
    off[i] = 0;
    return;
  }
  off[i] = d.at(x, idx[i * 3 + 1], idx[i * 3 + 2]);
}

template <typename T>
__global__ void pad_nonfinite_kernel(const T* __restrict__ u, PDims d, int* flag) {
  const int64_t n = d.nx * d.ny * d.nz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i % d.nz, xy = i / d.nz;
    if (!finite(u[d.at(xy / d.ny, xy % d.ny, z)])) {
      atomicExch(flag, 1);
      return;
    }
  }
}


// Padded interior -> host (nx, ny, nz) array (staged, hostio.cu).
template <typename T>
void pad_read(const T* f, const PDims& d, void* out, cudaStream_t st) {
  device_to_host_3d(out, f + d.at(0, 0, 0), d.nz * sizeof(T), d.ny, d.nx, d.pitch * sizeof(T),
                    d.plane * sizeof(T), st);
}

}  // namespace
}  // namespace stb
