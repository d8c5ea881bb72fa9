// TMA-tiled elastic half steps (f32, 3-D grids, R <= 4): the v and tau
// updates of elastic.cu with the same IEEE operation order (stag(), sums in
// axis order, physics.py:287-429), restructured as 2.5-D x sweeps.
//
// Per CTA: a 16 x 32 (y, z) tile and an x chunk; 512 threads, one point per
// thread.  Thread 0 streams planes of the NF input fields (v pass: the six
// stresses; tau pass: the three velocities) with TMA into a ring of
// NS = 2R+1 slots (tile + R halo rows, z halo rounded to 16-byte boxes;
// out-of-range boxes are zero-filled, the padded layout's halo is zero).
// The fields differentiated along x live in per-thread register queues
// (2R+1 planes); y/z neighbours come from the slot of the output plane, which
// lags the newest plane by R.  The loop is unrolled by 2(2R+1) so every slot
// and queue index is static; the centre operands (old values of the updated
// fields, materials, fx) are loaded two iterations ahead with volatile loads.
// After one consumer barrier per plane, thread 0 refills the slot of the
// plane that just left the window (a barrier-free variant in which the last
// warp out of a slot refills it was measured slower: 33 vs 36 Gpts/s, the
// warps drift apart and refills wait on the slowest one).
//
// Compulsory HBM bytes per point (f32): v pass 6 tau + 3 v + buoy in, 3 v out
// = 52; tau pass 3 v + 6 tau + lam + mu in, 6 tau out = 68 (120 per step).
#pragma once

#include "fp_exact.cuh"
#include "padded.cuh"
#include "tma.cuh"

namespace stb {
namespace {

constexpr int kElTZ = 32;

// TY x 32 tiles; NS ring slots (a divisor of the unroll 2(2R+1), >= R + 2)
template <int R, int NF, int TY, int NS_>
struct ElTiledCfg {
  static constexpr int ZH = (R + 3) / 4 * 4;                  // z halo (16-byte boxes)
  static constexpr int PY = TY + 2 * R, PZ = kElTZ + 2 * ZH;
  static constexpr int FSLOT = (PY * PZ + 31) / 32 * 32;       // floats per field plane
  static constexpr int SLOT = NF * FSLOT;
  static constexpr int Q = 2 * R + 1;
  static constexpr int NS = NS_;
  static constexpr int THREADS = TY * kElTZ;
  static_assert((2 * Q) % NS == 0 && NS >= R + 2, "ring must divide the unroll");
  static constexpr size_t smem_bytes() { return (size_t)NS * SLOT * 4 + NS * 8 + 128; }
};

struct ElTiledMaps {
  CUtensorMap f[6];       // input fields (v pass: txx tyy tzz txy txz tyz; tau: vx vy vz)
};

struct ElTiledArgs {
  float* out[6];          // fields updated in place (v pass: vx vy vz; tau: 6 stresses)
  const float* m0;        // v pass: buoy; tau pass: lam
  const float* m1;        // tau pass: mu
  const float* fx;
  const float* fy;
  const float* fz;
  int has_fac;
  ElCoefs<float> cf;
  PDims d;
  int cx;
  int x_lo, x_hi;         // local planes of this launch, in cx chunks
  int* nonfinite;
  float negz;             // -0.0f, opaque to ptxas (exact packed products, f32x2.cuh)
};

__device__ __forceinline__ float el_ld_nc(const float* p) {
  float v;
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float el_ld_cg(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

constexpr int el_pmod(int a, int m) { return ((a % m) + m) % m; }

// PASS 0: v half step, PASS 1: tau half step.
template <int R, int PASS, int TY, int NS_, int MINB>
__global__ void __launch_bounds__(TY * 32, MINB)
elastic_tiled(const __grid_constant__ ElTiledMaps maps, ElTiledArgs a) {
  constexpr int NF = PASS == 0 ? 6 : 3;
  constexpr int NO = PASS == 0 ? 3 : 6;       // updated fields
  constexpr int NM = PASS == 0 ? 1 : 2;       // materials
  using C = ElTiledCfg<R, NF, TY, NS_>;
  constexpr int kElThreads = C::THREADS;
  constexpr int Q = C::Q, NS = C::NS, U = 2 * Q;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* ring = reinterpret_cast<float*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * C::SLOT);

  const int tid = threadIdx.x;
  const int ty = tid >> 5, tz = tid & 31;
  const int z0 = blockIdx.x * kElTZ, y0 = blockIdx.y * TY, x0 = a.x_lo + blockIdx.z * a.cx;
  const int ny = (int)a.d.ny, nz = (int)a.d.nz;
  const int x1 = min(x0 + a.cx, a.x_hi);
  const int y = y0 + ty, z = z0 + tz;
  const bool core_in = y < ny && z < nz;
  const int N = (x1 - x0) + 2 * R;            // sequence n = plane x0 - R + n

  const int H = (int)a.d.H;
  const int tc0 = (int)a.d.zoff + z0 - C::ZH, tc1 = H + y0 - R;
  auto issue = [&](int seq, int slot) {
    mbar_arrive_expect_tx(&full[slot], (uint32_t)NF * C::PY * C::PZ * 4u);
    const int xg = H + x0 - R + seq;
#pragma unroll
    for (int f = 0; f < NF; ++f)
      tma_load_3d(ring + slot * C::SLOT + f * C::FSLOT, &maps.f[f], tc0, tc1, xg, &full[slot]);
  };
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
#pragma unroll
    for (int f = 0; f < NF; ++f) prefetch_map(&maps.f[f]);
    for (int s = 0; s < NS && s < N; ++s) issue(s, s);
  }
  __syncthreads();

  const ElCoefs<float>& cf = a.cf;
  float cxk[R], cyk[R], czk[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    cxk[k] = cf.d1[0][k];
    cyk[k] = cf.d1[1][k];
    czk[k] = cf.d1[2][k];
  }
  const int plane = (int)a.d.plane;
  const int gcore = core_in ? (int)a.d.at(0, y, z) : 0;
  const bool has_fac = a.has_fac != 0;
  const float fyz = has_fac && core_in ? tmin(__ldg(a.fy + y), __ldg(a.fz + z)) : 1.f;
  const int coff = (ty + R) * C::PZ + (tz + C::ZH);   // centre within a field plane

  // centre operands of output plane x: NO old values, NM materials, fx
  constexpr int NOP = NO + NM + 1;
  auto load_ops = [&](int x, bool ok, float* o) {
    if (ok) {
      const int gi = gcore + x * plane;
#pragma unroll
      for (int f = 0; f < NO; ++f) o[f] = el_ld_cg(a.out[f] + gi);
      o[NO] = el_ld_nc(a.m0 + gi);
      if constexpr (NM == 2) o[NO + 1] = el_ld_nc(a.m1 + gi);
      o[NO + NM] = has_fac ? el_ld_nc(a.fx + x) : 1.f;
    }
  };
  float od[2][NOP];
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int k = 0; k < NOP; ++k) od[b][k] = 0.f;
  // outputs start at n = 2R >= 2, so nothing to preload

  // x queues (position n mod Q): v pass txx, txy, txz; tau pass vx, vy, vz
  float q0[Q], q1[Q], q2[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) q0[j] = q1[j] = q2[j] = 0.f;

  bool bad = false;
  for (int n0 = 0; n0 < N; n0 += U) {
    const int par0 = (n0 / NS) & 1;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int n = n0 + u;
      if (n >= N) break;
      const int sn = u % NS;                          // slot of sequence n
      mbar_wait_sleep(&full[sn], par0 ^ ((u / NS) & 1));
      // operands of this iteration's output plane (loaded two iterations
      // ago); then issue those of iteration n + 2 into the same buffer
      float ocur[NOP];
#pragma unroll
      for (int k = 0; k < NOP; ++k) ocur[k] = od[u & 1][k];
      {
        const int xo = x0 - R + (n + 2) - R;
        load_ops(xo, xo >= x0 && xo < x1 && core_in, od[u & 1]);
      }
      const float* sl = ring + sn * C::SLOT + coff;   // newest plane, centre
      // v pass queue fields: txx (0), txy (3), txz (4); tau pass: vx, vy, vz
      if constexpr (PASS == 0) {
        q0[u % Q] = sl[0 * C::FSLOT];
        q1[u % Q] = sl[3 * C::FSLOT];
        q2[u % Q] = sl[4 * C::FSLOT];
      } else {
        q0[u % Q] = sl[0 * C::FSLOT];
        q1[u % Q] = sl[1 * C::FSLOT];
        q2[u % Q] = sl[2 * C::FSLOT];
      }
      if (n >= 2 * R && core_in) {
        const int x = x0 - R + n - R;                 // output plane, sequence n - R
        const float* cp = ring + el_pmod(u - R, NS) * C::SLOT + coff;
        // x accessors from the queues: plane x + o sits at position (u - R + o)
        auto gq0 = [&](int o) { return q0[el_pmod(u - R + o, Q)]; };
        auto gq1 = [&](int o) { return q1[el_pmod(u - R + o, Q)]; };
        auto gq2 = [&](int o) { return q2[el_pmod(u - R + o, Q)]; };
        auto gy = [&](int f) { return [=](int o) { return cp[f * C::FSLOT + o * C::PZ]; }; };
        auto gz = [&](int f) { return [=](int o) { return cp[f * C::FSLOT + o]; }; };
        if constexpr (PASS == 0) {
          // fields: 0 txx, 1 tyy, 2 tzz, 3 txy, 4 txz, 5 tyz
          float d0 = stag<float, R>(gq0, cxk, true);
          d0 = radd(d0, stag<float, R>(gy(3), cyk, false));
          d0 = radd(d0, stag<float, R>(gz(4), czk, false));
          float d1 = stag<float, R>(gq1, cxk, false);
          d1 = radd(d1, stag<float, R>(gy(1), cyk, true));
          d1 = radd(d1, stag<float, R>(gz(5), czk, false));
          float d2 = stag<float, R>(gq2, cxk, false);
          d2 = radd(d2, stag<float, R>(gy(5), cyk, false));
          d2 = radd(d2, stag<float, R>(gz(2), czk, true));
          const float buoy = ocur[3];
          const float fac = has_fac ? tmin(ocur[4], fyz) : 1.f;
          const float dd[3] = {d0, d1, d2};
          const int gi = gcore + x * plane;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            float o = radd(ocur[k], rmul(dd[k], buoy));
            if (has_fac) o = rmul(o, fac);
            a.out[k][gi] = o;
            bad |= !finite(o);
          }
        } else {
          // fields: 0 vx, 1 vy, 2 vz; outputs txx tyy tzz txy txz tyz
          const float lam = ocur[6], mu = ocur[7];
          const float mu2 = rmul(mu, 2.f);
          const float fac = has_fac ? tmin(ocur[8], fyz) : 1.f;
          const float dg0 = stag<float, R>(gq0, cxk, false);
          const float dg1 = stag<float, R>(gy(1), cyk, false);
          const float dg2 = stag<float, R>(gz(2), czk, false);
          const float tr = radd(radd(dg0, dg1), dg2);
          const float dg[3] = {dg0, dg1, dg2};
          const int gi = gcore + x * plane;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            float o = radd(ocur[k], radd(rmul(tr, lam), rmul(dg[k], mu2)));
            if (has_fac) o = rmul(o, fac);
            a.out[k][gi] = o;
            bad |= !finite(o);
          }
          // txy = stag_y(vx, fwd) + stag_x(vy, fwd); txz = stag_z(vx) + stag_x(vz);
          // tyz = stag_z(vy) + stag_y(vz)   (elastic_tau_point order)
          const float s0 = radd(stag<float, R>(gy(0), cyk, true), stag<float, R>(gq1, cxk, true));
          const float s1 = radd(stag<float, R>(gz(0), czk, true), stag<float, R>(gq2, cxk, true));
          const float s2 = radd(stag<float, R>(gz(1), czk, true), stag<float, R>(gy(2), cyk, true));
          const float ss[3] = {s0, s1, s2};
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            float o = radd(ocur[3 + k], rmul(ss[k], mu));
            if (has_fac) o = rmul(o, fac);
            a.out[3 + k][gi] = o;
            bad |= !finite(o);
          }
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kElThreads) : "memory");
      // sequence n - R left the window: refill its slot with n - R + NS
      if (tid == 0 && n >= R && n - R + NS < N) {
        fence_proxy_async();
        issue(n - R + NS, el_pmod(u - R, NS));
      }
    }
  }
  if (a.nonfinite && bad) atomicExch(a.nonfinite, 1);
}

}  // namespace
}  // namespace stb
