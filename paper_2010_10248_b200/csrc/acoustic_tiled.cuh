// TMA-staged 2.5-D acoustic stencil kernel (one time step per launch), fp32.
//
// Each CTA owns a TY x TZ (y, z) tile and sweeps a chunk of x planes (x is
// the slowest axis).  Per plane:
//   * TMA (cp.async.bulk.tensor.3d, OOB zero-fill == the reference's zero
//     halo) stages the u[t-1] plane with a (R, RP) halo in y/z into a ring of
//     R+1+PF shared-memory slots, and the u[t-2] / inv tiles of the output
//     plane into a PF+1-slot ring; one mbarrier per slot, PF planes in flight.
//   * each thread owns 4 consecutive z points and keeps their u[t-1] values
//     for planes x-R..x+R in a register queue (x-neighbours), reads y/z
//     neighbours of the centre plane from shared memory (LDS.128), and
//     evaluates the update in the reference's exact IEEE order
//     (physics.py:199-213, no FMA contraction), so the result is bitwise the
//     NumPy oracle's.
// The x loop is unrolled by the queue length 2R+1 so every queue index is a
// compile-time register.
#pragma once

#include "acoustic_kernels.cuh"
#include "fp_exact.cuh"
#include "tma.cuh"

namespace stb {

template <int R, int TY, int TZ, int PF>
struct TiledCfg {
  static constexpr int RP = (R + 3) / 4 * 4;   // z halo rounded up to a float4
  static constexpr int W = TZ + 2 * RP;        // shared row length (floats)
  static constexpr int H = TY + 2 * R;         // shared rows per plane
  static constexpr int EXT = W * H;            // floats per staged u[t-1] plane
  static constexpr int TILE = TY * TZ;         // floats per u[t-2] / inv tile
  static constexpr int NS1 = R + 1 + PF;       // u[t-1] ring slots
  static constexpr int NS2 = PF + 1;           // u[t-2]/inv ring slots
  static constexpr int Q = 2 * R + 1;          // register queue length
  static constexpr int NT = TY * TZ / 4;       // threads per CTA
  static constexpr size_t RING1_BYTES = (size_t)NS1 * EXT * 4;
  static constexpr size_t RING2_BYTES = (size_t)NS2 * 2 * TILE * 4;
  static constexpr size_t SMEM = RING1_BYTES + RING2_BYTES + NS1 * 8;
  static_assert(TZ % 4 == 0, "TZ must hold whole float4 groups");
  static_assert((EXT * 4) % 128 == 0 || true, "");
};

struct TiledCoefs {
  float c0;
  float cx[8], cy[8], cz[8];
  float nz;     // -0.0f, a runtime value on purpose (see xmul2 in f32x2.cuh)
};

template <int R, int TY, int TZ, int PF>
__global__ void __launch_bounds__(TiledCfg<R, TY, TZ, PF>::NT, 2)
acoustic_tiled_step(const __grid_constant__ CUtensorMap m_u1, const __grid_constant__ CUtensorMap m_u0,
                    const __grid_constant__ CUtensorMap m_inv, float* __restrict__ out,
                    const float* __restrict__ fx, const float* __restrict__ fy,
                    const float* __restrict__ fz, int has_fac, int use_inv, float inv_scalar,
                    TiledCoefs cf, Dims d, int cx_len, int ntz, int* __restrict__ nonfinite) {
  using C = TiledCfg<R, TY, TZ, PF>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* ring1 = reinterpret_cast<float*>(smem_raw);
  float* ring2 = reinterpret_cast<float*>(smem_raw + C::RING1_BYTES);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + C::RING1_BYTES + C::RING2_BYTES);

  const int tid = threadIdx.x;
  const int ty = tid / (TZ / 4);
  const int tz4 = tid % (TZ / 4);
  const int tile = blockIdx.x;
  const int y0 = (tile / ntz) * TY;
  const int z0 = (tile % ntz) * TZ;
  const int x0 = blockIdx.y * cx_len;
  const int x1 = min(x0 + cx_len, (int)d.nx);
  const int J = (x1 - x0) + 2 * R;
  const int y = y0 + ty;
  const int z = z0 + 4 * tz4;
  const bool writer = (y < d.ny) && (z < d.nz);

  if (tid == 0) {
    for (int s = 0; s < C::NS1; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
    prefetch_map(&m_u1);
    prefetch_map(&m_u0);
    if (use_inv) prefetch_map(&m_inv);
  }
  __syncthreads();

  auto issue = [&](int j) {
    const int s1 = j % C::NS1;
    const int s2 = j % C::NS2;
    const int p = x0 - R + j;
    const bool outp = j >= 2 * R;
    const uint32_t bytes =
        C::EXT * 4 + (outp ? (use_inv ? 2u : 1u) * (uint32_t)C::TILE * 4u : 0u);
    mbar_arrive_expect_tx(&bar[s1], bytes);
    tma_load_3d(ring1 + (size_t)s1 * C::EXT, &m_u1, z0 - C::RP, y0 - R, p, &bar[s1]);
    if (outp) {
      float* a = ring2 + (size_t)s2 * 2 * C::TILE;
      tma_load_3d(a, &m_u0, z0, y0, p - R, &bar[s1]);
      if (use_inv) tma_load_3d(a + C::TILE, &m_inv, z0, y0, p - R, &bar[s1]);
    }
  };
  if (tid == 0) {
    for (int j = 0; j <= PF && j < J; ++j) issue(j);
  }

  // per-thread sponge factors min(fy[y], fz[z+i]); fx[x] is applied per plane
  float fyz[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    fyz[i] = 1.0f;
    if (has_fac && y < d.ny && z + i < d.nz) fyz[i] = tmin(__ldg(fy + y), __ldg(fz + z + i));
  }

  float q[C::Q][4];
#pragma unroll
  for (int s = 0; s < C::Q; ++s)
#pragma unroll
    for (int i = 0; i < 4; ++i) q[s][i] = 0.f;

  const int row_c = (ty + R) * C::W + C::RP + 4 * tz4;   // centre offset in a staged plane
  int bad = 0;

  for (int jb = 0; jb < J; jb += C::Q) {
#pragma unroll
    for (int qq = 0; qq < C::Q; ++qq) {
      const int j = jb + qq;
      if (j < J) {
        const int s1 = j % C::NS1;
        mbar_wait(&bar[s1], (uint32_t)((j / C::NS1) & 1));
        {
          const float4 v = *reinterpret_cast<const float4*>(ring1 + (size_t)s1 * C::EXT + row_c);
          q[qq][0] = v.x; q[qq][1] = v.y; q[qq][2] = v.z; q[qq][3] = v.w;
        }
        if (j >= 2 * R) {
          const int x = x0 - 2 * R + j;
          const float* cen = ring1 + (size_t)((j - R) % C::NS1) * C::EXT + row_c;
          constexpr int dummy = 0;
          (void)dummy;
          const int cs = (qq - R + C::Q) % C::Q;
          float lap[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) lap[i] = rmul(q[cs][i], cf.c0);
          // x neighbours from the register queue (axis 0 first, r ascending)
#pragma unroll
          for (int r = 1; r <= R; ++r) {
            const int sp = (qq - R + r + C::Q) % C::Q;
            const int sm = (qq - R - r + 2 * C::Q) % C::Q;
#pragma unroll
            for (int i = 0; i < 4; ++i)
              lap[i] = radd(lap[i], rmul(radd(q[sp][i], q[sm][i]), cf.cx[r - 1]));
          }
          // y neighbours
#pragma unroll
          for (int r = 1; r <= R; ++r) {
            const float4 pp = *reinterpret_cast<const float4*>(cen + r * C::W);
            const float4 mm = *reinterpret_cast<const float4*>(cen - r * C::W);
            lap[0] = radd(lap[0], rmul(radd(pp.x, mm.x), cf.cy[r - 1]));
            lap[1] = radd(lap[1], rmul(radd(pp.y, mm.y), cf.cy[r - 1]));
            lap[2] = radd(lap[2], rmul(radd(pp.z, mm.z), cf.cy[r - 1]));
            lap[3] = radd(lap[3], rmul(radd(pp.w, mm.w), cf.cy[r - 1]));
          }
          // z neighbours: window [z - RP, z + 4 + RP)
          float win[4 + 2 * C::RP];
#pragma unroll
          for (int w4 = 0; w4 < (4 + 2 * C::RP) / 4; ++w4) {
            const float4 v = *reinterpret_cast<const float4*>(cen - C::RP + 4 * w4);
            win[4 * w4 + 0] = v.x; win[4 * w4 + 1] = v.y;
            win[4 * w4 + 2] = v.z; win[4 * w4 + 3] = v.w;
          }
#pragma unroll
          for (int r = 1; r <= R; ++r)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              lap[i] = radd(lap[i], rmul(radd(win[C::RP + i + r], win[C::RP + i - r]),
                                         cf.cz[r - 1]));
          const float* aux = ring2 + (size_t)(j % C::NS2) * 2 * C::TILE + ty * TZ + 4 * tz4;
          const float4 u0 = *reinterpret_cast<const float4*>(aux);
          float iv[4];
          if (use_inv) {
            const float4 t4 = *reinterpret_cast<const float4*>(aux + C::TILE);
            iv[0] = t4.x; iv[1] = t4.y; iv[2] = t4.z; iv[3] = t4.w;
          } else {
            iv[0] = iv[1] = iv[2] = iv[3] = inv_scalar;
          }
          const float u0a[4] = {u0.x, u0.y, u0.z, u0.w};
          const float fxx = has_fac ? __ldg(fx + x) : 1.0f;
          float o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float l = rmul(lap[i], iv[i]);
            float v = rmul(q[cs][i], 2.0f);
            v = rsub(v, u0a[i]);
            v = radd(v, l);
            if (has_fac) v = rmul(v, tmin(fxx, fyz[i]));
            o[i] = v;
          }
          if (nonfinite) {
#pragma unroll
            for (int i = 0; i < 4; ++i) bad |= (writer && z + i < d.nz && !isfinite(o[i]));
          }
          if (writer) {
            *reinterpret_cast<float4*>(out + (int64_t)x * d.plane + (int64_t)y * d.pitch + z) =
                make_float4(o[0], o[1], o[2], o[3]);
          }
        }
        __syncthreads();
        if (tid == 0 && j + 1 + PF < J) {
          fence_proxy_async();
          issue(j + 1 + PF);
        }
      }
    }
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (tid & 31) == 0) atomicExch(nonfinite, 1);
}

// Host-side launcher holding the tensor maps for one grid.
template <int R, int TY, int TZ, int PF>
struct TiledAcousticLauncher {
  using C = TiledCfg<R, TY, TZ, PF>;
  static void configure() {
    static std::atomic<uint64_t> done{0};
    if (first_use_on_device(done))
      STB_CUDA(cudaFuncSetAttribute(acoustic_tiled_step<R, TY, TZ, PF>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  }
  static void launch(cudaStream_t st, const CUtensorMap& m_u1, const CUtensorMap& m_u0,
                     const CUtensorMap& m_inv, float* out, const float* fx, const float* fy,
                     const float* fz, bool has_fac, bool use_inv, float inv_scalar,
                     const TiledCoefs& cf, const Dims& d, int cx_len, int* nonfinite) {
    configure();
    const int ntz = (int)((d.nz + TZ - 1) / TZ);
    const int nty = (int)((d.ny + TY - 1) / TY);
    const int nch = (int)((d.nx + cx_len - 1) / cx_len);
    dim3 grid((unsigned)(ntz * nty), (unsigned)nch);
    acoustic_tiled_step<R, TY, TZ, PF><<<grid, C::NT, C::SMEM, st>>>(
        m_u1, m_u0, m_inv, out, fx, fy, fz, has_fac ? 1 : 0, use_inv ? 1 : 0, inv_scalar, cf,
        d, cx_len, ntz, nonfinite);
    STB_CHECK_LAUNCH();
  }
};

}  // namespace stb
