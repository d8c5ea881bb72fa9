// Acoustic stencil kernels.
#pragma once

#include "fp_exact.cuh"
#include "stb_internal.cuh"

namespace stb {

template <typename T>
struct AcCoefs {
  T c0;          // f(sum_a w0/h_a^2)
  T c[3][8];     // f(w_r/h_a^2), r = 1..R stored at [a][r-1]
  int active[3];
};

// ---------------------------------------------------------------------------
// Reference-order step, one thread per point (general: any R in 1..8, any
// grid incl. degenerate axes).  Neighbours outside the interior read the
// reference's zero halo.  Used for degenerate grids and as the baseline the
// tiled kernels are checked against.
// ---------------------------------------------------------------------------
template <typename T, int R>
__global__ void __launch_bounds__(128)
acoustic_reference_step(const T* __restrict__ u1, const T* __restrict__ u0, T* __restrict__ out,
                        const T* __restrict__ inv, T inv_scalar, const T* __restrict__ fx,
                        const T* __restrict__ fy, const T* __restrict__ fz, int has_fac,
                        AcCoefs<T> cf, Dims d) {
  const int64_t z = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t y = blockIdx.y;
  const int64_t x = blockIdx.z;
  if (z >= d.nz) return;
  const int64_t i = x * d.plane + y * d.pitch + z;
  const T uc = u1[i];
  T lap = rmul(uc, cf.c0);
  const int64_t n[3] = {d.nx, d.ny, d.nz};
  const int64_t pos[3] = {x, y, z};
  const int64_t stride[3] = {d.plane, d.pitch, 1};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (!cf.active[a]) continue;
#pragma unroll
    for (int r = 1; r <= R; ++r) {
      const T p = (pos[a] + r < n[a]) ? u1[i + r * stride[a]] : T(0);
      const T m = (pos[a] - r >= 0) ? u1[i - r * stride[a]] : T(0);
      lap = radd(lap, rmul(radd(p, m), cf.c[a][r - 1]));
    }
  }
  lap = rmul(lap, inv ? inv[i] : inv_scalar);
  T o = rmul(uc, T(2));
  o = rsub(o, u0[i]);
  o = radd(o, lap);
  if (has_fac) o = rmul(o, tmin(tmin(fx[x], fy[y]), fz[z]));
  out[i] = o;
}

template <typename T>
void launch_reference_step(int R, cudaStream_t st, const T* u1, const T* u0, T* out,
                           const T* inv, T inv_scalar, const T* fx, const T* fy, const T* fz,
                           bool has_fac, const AcCoefs<T>& cf, const Dims& d) {
  dim3 block(128);
  dim3 grid((unsigned)((d.nz + 127) / 128), (unsigned)d.ny, (unsigned)d.nx);
#define STB_REF_CASE(RR)                                                                 \
  case RR:                                                                               \
    acoustic_reference_step<T, RR><<<grid, block, 0, st>>>(u1, u0, out, inv, inv_scalar, \
                                                           fx, fy, fz, has_fac ? 1 : 0,  \
                                                           cf, d);                       \
    break;
  switch (R) {
    STB_REF_CASE(1)
    STB_REF_CASE(2)
    STB_REF_CASE(3)
    STB_REF_CASE(4)
    STB_REF_CASE(5)
    STB_REF_CASE(6)
    STB_REF_CASE(7)
    STB_REF_CASE(8)
    default:
      throw Error(STB_ERR_ARG, "space_order must be even in [2, 16]");
  }
#undef STB_REF_CASE
  STB_CHECK_LAUNCH();
}

}  // namespace stb
