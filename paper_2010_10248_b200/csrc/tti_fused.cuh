// Fused single-pass TTI step (f32, 3-D grids): one HBM sweep per time step.
//
// Same arithmetic, same IEEE order as tti_pass1 + tti_pass2 (tti.cu, and the
// oracle's TTI class), but the gradient streams F_a, G_a never leave the SM:
//
//   * a producer warp streams planes of p and q (level t-1) with TMA into a
//     ring of NS = M(2r+1) shared-memory slots; each slot holds the
//     (TY+4r) x (TZ+4r) tile plus the halo the two chained first
//     derivatives need (out-of-range boxes are zero-filled; the padded
//     layout's halo is zero too);
//   * 16 consumer warps sweep x.  At iteration i they run pass 1 at plane
//     xa = x0 - r + i for the TY x TZ core (one point per thread) and for
//     the y/z halo of the core (the points D_y F_y / D_z F_z need):
//       - F_x, G_x of the core go to per-thread register queues (2r+1 deep),
//       - F_y, G_y, F_z, G_z go to a double-buffered shared plane;
//     after a consumer barrier each thread forms D_y F_y, D_z F_z, D_y G_y,
//     D_z G_z at (xa, y, z) and queues them r planes deep;
//   * output plane x = xa - r (once the queues are full): Lxy = (D_x F_x +
//     D_y F_y) + D_z F_z, Lzz likewise, then the p/q update in place over
//     level t-2 (read only at the point itself).
//
// HBM traffic per point: p, q (t-1) once through TMA (+ L2-served halos),
// p, q (t-2), inv, e2, d2, n_x, n_y, n_z, and the p, q writes: 12 x 4 B =
// 48 B/point (vs 104 B/point for the two-pass path).
#pragma once

#include "fp_exact.cuh"
#include "padded.cuh"
#include "tma.cuh"

namespace stb {
namespace {

constexpr int kTtiTY = 16;
constexpr int kTtiTZ = 32;
constexpr int kTtiConsumers = kTtiTY * kTtiTZ;      // 512 threads, 16 warps
constexpr int kTtiThreads = kTtiConsumers;          // no separate producer warp:
                                                    // 16 warps = 4 per SM sub-
                                                    // partition, 128-reg budget

template <int r, int M>
struct TtiFusedCfg {
  static constexpr int TY = kTtiTY, TZ = kTtiTZ;
  // p/q slot: 2r halo rows; z halo rounded up to 4 floats so each TMA box
  // row starts 16-byte aligned in global memory
  static constexpr int ZH = (2 * r + 3) / 4 * 4;
  static constexpr int PY = TY + 4 * r, PZ = TZ + 2 * ZH;
  static constexpr int EY = TY + 2 * r, EZ = TZ + 2 * r;    // pass-1 extent
  static constexpr int Q = 2 * r + 1;                        // x stencil width
  static constexpr int NS = M * Q;                           // ring slots (= unroll)
  static constexpr int SLOT = (PY * PZ + 31) / 32 * 32;      // floats, 128-B aligned
  static constexpr int EPL = EY * EZ;                        // floats
  static constexpr int NHY = 2 * r * TZ;                     // y-halo points
  static constexpr int NHZ = 2 * r * TY;                     // z-halo points
  static constexpr size_t smem_bytes() {
    return (size_t)2 * NS * SLOT * 4 + (size_t)2 * 4 * EPL * 4 + NS * 8 + 128;
  }
};

struct TtiMaps {
  CUtensorMap p, q;   // level t-1 of p and q over the padded layout
};

struct TtiFusedArgs {
  float* p0;          // level t-2 in, level t out
  float* q0;
  const float* inv;
  const float* e2;
  const float* d2;
  const float* n[3];
  const float* fx;
  const float* fy;
  const float* fz;
  int has_fac;
  TtiCoefs<float> cf;
  PDims d;
  int cx;             // x planes per CTA
  int x_lo, x_hi;     // local output planes of this launch (in cx chunks)
  int* nonfinite;
  float negz;         // -0.0f, opaque to ptxas (exact packed products, f32x2.cuh)
};

// Loads issued as volatile asm so the compiler cannot sink them next to
// their use (it does so for plain loads, defeating the software pipeline):
// .nc for the read-only materials, .cg for the level the kernel overwrites.
__device__ __forceinline__ float ld_nc(const float* p) {
  float v;
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_cg(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

// acc + d*c: EXACT keeps the oracle's separate rounding of the product and
// the sum; FAST (ScheduleSpec.arithmetic = "fma") contracts them
template <bool FAST>
__device__ __forceinline__ float mac(float acc, float d, float c) {
  if constexpr (FAST) return __fmaf_rn(d, c, acc);
  else return radd(acc, rmul(d, c));
}

// centred first derivative from a strided shared-memory accessor
template <int r, bool FAST>
__device__ __forceinline__ float d1s(const float* c0, int s, const float* c) {
  float acc = rmul(rsub(c0[s], c0[-s]), c[0]);
#pragma unroll
  for (int k = 2; k <= r; ++k) acc = mac<FAST>(acc, rsub(c0[k * s], c0[-k * s]), c[k - 1]);
  return acc;
}

// pass 1 at one point: gradients of p, q (x via ring slots, y/z in-plane),
// w_p, w_q, then F_a, G_a.  ps[d] points at the (y, z) position of p in the
// slot of plane xa + d - r (d = 0..2r); q sits QOFF floats further.
template <int r, int PZ, int QOFF, bool FAST>
__device__ __forceinline__ void tti_point_pass1(const float* const* ps, const float* cx,
                                                const float* cy, const float* cz,
                                                const float n[3], float F[3], float G[3]) {
  float gpx = rmul(rsub(ps[r + 1][0], ps[r - 1][0]), cx[0]);
  float gqx = rmul(rsub(ps[r + 1][QOFF], ps[r - 1][QOFF]), cx[0]);
#pragma unroll
  for (int k = 2; k <= r; ++k) {
    gpx = mac<FAST>(gpx, rsub(ps[r + k][0], ps[r - k][0]), cx[k - 1]);
    gqx = mac<FAST>(gqx, rsub(ps[r + k][QOFF], ps[r - k][QOFF]), cx[k - 1]);
  }
  const float gpy = d1s<r, FAST>(ps[r], PZ, cy);
  const float gqy = d1s<r, FAST>(ps[r] + QOFF, PZ, cy);
  const float gpz = d1s<r, FAST>(ps[r], 1, cz);
  const float gqz = d1s<r, FAST>(ps[r] + QOFF, 1, cz);
  const float wp = mac<FAST>(mac<FAST>(rmul(gpx, n[0]), gpy, n[1]), gpz, n[2]);
  const float wq = mac<FAST>(mac<FAST>(rmul(gqx, n[0]), gqy, n[1]), gqz, n[2]);
  if constexpr (FAST) {
    F[0] = __fmaf_rn(-wp, n[0], gpx);
    F[1] = __fmaf_rn(-wp, n[1], gpy);
    F[2] = __fmaf_rn(-wp, n[2], gpz);
  } else {
    F[0] = rsub(gpx, rmul(wp, n[0]));
    F[1] = rsub(gpy, rmul(wp, n[1]));
    F[2] = rsub(gpz, rmul(wp, n[2]));
  }
  G[0] = rmul(wq, n[0]);
  G[1] = rmul(wq, n[1]);
  G[2] = rmul(wq, n[2]);
}

constexpr int pmod(int a, int m) { return ((a % m) + m) % m; }

template <int r, int M, bool FAST>
__global__ void __launch_bounds__(kTtiThreads, 1)
tti_fused(const __grid_constant__ TtiMaps maps, TtiFusedArgs a) {
  using C = TtiFusedCfg<r, M>;
  constexpr int Q = C::Q, NS = C::NS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // align by offsetting the __shared__ array itself (a uintptr_t round trip
  // would lose the address space and turn every access into a generic LD)
  float* sp = reinterpret_cast<float*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  float* sq = sp + NS * C::SLOT;
  float* fg = sq + NS * C::SLOT;                    // [2][4][EY][EZ]
  uint64_t* full = reinterpret_cast<uint64_t*>(fg + 2 * 4 * C::EPL);

  const int tid = threadIdx.x;
  const int z0 = blockIdx.x * C::TZ, y0 = blockIdx.y * C::TY;
  const int x0 = a.x_lo + blockIdx.z * a.cx;
  const int nx = (int)a.d.nx, ny = (int)a.d.ny, nz = (int)a.d.nz;
  const int x1 = min(x0 + a.cx, a.x_hi);
  const int n_iter = (x1 - x0) + 2 * r;             // pass-1 planes x0-r .. x1-1+r
  const int n_seq = n_iter + 2 * r;                 // p/q planes x0-2r .. x1-1+2r

  // TMA issue (thread 0): plane sequence s -> ring slot s mod NS.  The first
  // NS planes are issued up front; sequence j + NS is issued into slot
  // j mod NS right after the consumer barrier of iteration j: sequence j is
  // last read by iteration j, before that barrier.
  const int H = (int)a.d.H;
  const int tc0 = (int)a.d.zoff + z0 - C::ZH, tc1 = H + y0 - 2 * r;
  auto issue = [&](int seq, int slot) {
    mbar_arrive_expect_tx(&full[slot], 2u * C::PY * C::PZ * 4u);
    const int xg = H + x0 - 2 * r + seq;
    tma_load_3d(sp + slot * C::SLOT, &maps.p, tc0, tc1, xg, &full[slot]);
    tma_load_3d(sq + slot * C::SLOT, &maps.q, tc0, tc1, xg, &full[slot]);
  };
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    prefetch_map(&maps.p);
    prefetch_map(&maps.q);
    for (int s = 0; s < NS && s < n_seq; ++s) issue(s, s);
  }
  __syncthreads();

  // -------------------------------------------------------------- consumers
  const int ty = tid >> 5, tz = tid & 31;
  const int y = y0 + ty, z = z0 + tz;
  const bool core_in = (y < ny) && (z < nz);
  constexpr int QOFF = NS * C::SLOT;                // q ring follows the p ring

  // halo role: tid < NHY -> y-halo row point; NHY <= tid < NHY + NHZ -> z-halo
  int hy = -1, hz = -1;
  bool h_yrole = false;
  if (tid < C::NHY) {
    const int row = tid / C::TZ;                    // 0 .. 2r-1
    hy = row < r ? row : C::TY + row;               // ext rows [0,r) u [TY+r, TY+2r)
    hz = r + (tid % C::TZ);
    h_yrole = true;
  } else if (tid < C::NHY + C::NHZ) {
    const int j = tid - C::NHY;
    const int row = j / (2 * r), col = j % (2 * r);
    hy = r + row;
    hz = col < r ? col : C::TZ + col;
  }
  const bool has_halo = hy >= 0;
  const int hgy = y0 - r + hy, hgz = z0 - r + hz;   // global coords of the halo point
  const bool h_in = has_halo && hgy >= 0 && hgy < ny && hgz >= 0 && hgz < nz;

  float c0[r], c1[r], c2[r];
#pragma unroll
  for (int k = 0; k < r; ++k) {
    c0[k] = a.cf.c[0][k];
    c1[k] = a.cf.c[1][k];
    c2[k] = a.cf.c[2][k];
  }
  // every material is a per-point array on this path (the host materialises
  // scalars), so the loop has no pointer tests
  const int plane = (int)a.d.plane;
  const int gcore = core_in ? (int)a.d.at(0, y, z) : 0;
  const int ghalo = h_in ? (int)a.d.at(0, hgy, hgz) : 0;
  const float* __restrict__ n0 = a.n[0];
  const float* __restrict__ n1 = a.n[1];
  const float* __restrict__ n2 = a.n[2];
  const bool has_fac = a.has_fac != 0;
  const float fyz = has_fac && core_in ? tmin(__ldg(a.fy + y), __ldg(a.fz + z)) : 1.f;

  // software pipeline: the global operands of iteration i+1 are issued at
  // the top of iteration i (n at the pass-1 points, p/q(t-2), materials
  // and fx at the output point), hiding HBM latency behind one plane.
  auto load_n = [&](int xg, int base, bool ok, float* n) {
    if (ok) {
      const int gi = base + xg * plane;
      n[0] = ld_nc(n0 + gi);
      n[1] = ld_nc(n1 + gi);
      n[2] = ld_nc(n2 + gi);
    } else {
      n[0] = n[1] = n[2] = 0.f;
    }
  };
  auto load_out = [&](int x, bool ok, float* o) {
    if (ok) {
      const int gi = gcore + x * plane;
      o[0] = ld_cg(a.p0 + gi);
      o[1] = ld_cg(a.q0 + gi);
      o[2] = ld_nc(a.inv + gi);
      o[3] = ld_nc(a.e2 + gi);
      o[4] = ld_nc(a.d2 + gi);
      o[5] = has_fac ? ld_nc(a.fx + x) : 1.f;
    }
  };
  // prefetch distance PD iterations (register ping-pong; the buffer index
  // u % PD is static because NS is a multiple of PD)
  constexpr int PD = (NS % 2 == 0) ? 2 : 1;
  float nc[PD][3], nh[PD][3], od[PD][6];
#pragma unroll
  for (int j = 0; j < PD; ++j) {
    const int xa = x0 - r + j;
    load_n(xa, gcore, xa >= 0 && xa < nx && core_in, nc[j]);
    load_n(xa, ghalo, xa >= 0 && xa < nx && h_in, nh[j]);
#pragma unroll
    for (int k = 0; k < 6; ++k) od[j][k] = 0.f;   // outputs start at i = 2r >= PD
  }

  // circular register queues (period Q): position i mod Q holds the value
  // computed at iteration i; the loop is unrolled by NS (a multiple of Q),
  // so every position and ring slot below is a compile-time constant.
  float qF[Q], qG[Q], qDyF[Q], qDzF[Q], qDyG[Q], qDzG[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) qF[j] = qG[j] = qDyF[j] = qDzF[j] = qDyG[j] = qDzG[j] = 0.f;

  const int core_off = (ty + 2 * r) * C::PZ + (tz + C::ZH);
  const int halo_off = (hy + r) * C::PZ + (hz - r + C::ZH);
  const int ecore = (ty + r) * C::EZ + (tz + r);
  const int ehalo = hy * C::EZ + hz;
  for (int s = 0; s < 2 * r; ++s) mbar_wait_sleep(&full[s % NS], (s / NS) & 1);

  bool bad = false;
  for (int i0 = 0; i0 < n_iter; i0 += NS) {
    const int par0 = (i0 / NS) & 1;
#pragma unroll
    for (int u = 0; u < NS; ++u) {
      const int i = i0 + u;
      if (i >= n_iter) break;
      mbar_wait_sleep(&full[(u + 2 * r) % NS], par0 ^ (u + 2 * r >= NS ? 1 : 0));
      const int xa = x0 - r + i;
      const bool xa_in = xa >= 0 && xa < nx;
      float* fgb = fg + ((NS % 2 == 0) ? (u & 1) : (i & 1)) * 4 * C::EPL;
      // operands of this iteration (loaded PD iterations ago); issue those
      // of iteration i + PD into the same buffer
      const int b = u % PD;
      const float ncur[3] = {nc[b][0], nc[b][1], nc[b][2]};
      const float nhcur[3] = {nh[b][0], nh[b][1], nh[b][2]};
      const float ocur[6] = {od[b][0], od[b][1], od[b][2], od[b][3], od[b][4], od[b][5]};
      {
        const bool nx_ok = xa + PD >= 0 && xa + PD < nx;
        load_n(xa + PD, gcore, nx_ok && core_in, nc[b]);
        if (has_halo) load_n(xa + PD, ghalo, nx_ok && h_in, nh[b]);
        const int xo = xa + PD - r;                  // output plane of iteration i + PD
        load_out(xo, xo >= x0 && xo < x1 && core_in, od[b]);
      }

      // centre values of the output plane (sequence i), read before the
      // barrier so that slot i can be refilled right after it
      const float p1 = sp[(u % NS) * C::SLOT + core_off];
      const float q1 = sp[(u % NS) * C::SLOT + core_off + QOFF];
      // pass 1, core point
      {
        const float* ps[2 * r + 1];
#pragma unroll
        for (int dd = 0; dd <= 2 * r; ++dd) ps[dd] = sp + ((u + dd) % NS) * C::SLOT + core_off;
        float F[3] = {0.f, 0.f, 0.f}, G[3] = {0.f, 0.f, 0.f};
        if (xa_in && core_in) tti_point_pass1<r, C::PZ, QOFF, FAST>(ps, c0, c1, c2, ncur, F, G);
        qF[u % Q] = F[0];
        qG[u % Q] = G[0];
        fgb[0 * C::EPL + ecore] = F[1];
        fgb[1 * C::EPL + ecore] = G[1];
        fgb[2 * C::EPL + ecore] = F[2];
        fgb[3 * C::EPL + ecore] = G[2];
      }
      // pass 1, halo point (F_y/G_y for y-halo rows, F_z/G_z for z-halo cols)
      if (has_halo) {
        const float* ps[2 * r + 1];
#pragma unroll
        for (int dd = 0; dd <= 2 * r; ++dd) ps[dd] = sp + ((u + dd) % NS) * C::SLOT + halo_off;
        float F[3] = {0.f, 0.f, 0.f}, G[3] = {0.f, 0.f, 0.f};
        if (xa_in && h_in) tti_point_pass1<r, C::PZ, QOFF, FAST>(ps, c0, c1, c2, nhcur, F, G);
        const int comp = h_yrole ? 0 : 2;
        fgb[comp * C::EPL + ehalo] = h_yrole ? F[1] : F[2];
        fgb[(comp + 1) * C::EPL + ehalo] = h_yrole ? G[1] : G[2];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kTtiConsumers) : "memory");
      // every warp is done with sequence i: refill its slot with i + NS
      if (tid == 0 && i + NS < n_seq) {
        fence_proxy_async();
        issue(i + NS, u % NS);
      }

      // y / z divergence terms at plane xa
      qDyF[u % Q] = d1s<r, FAST>(fgb + 0 * C::EPL + ecore, C::EZ, c1);
      qDyG[u % Q] = d1s<r, FAST>(fgb + 1 * C::EPL + ecore, C::EZ, c1);
      qDzF[u % Q] = d1s<r, FAST>(fgb + 2 * C::EPL + ecore, 1, c2);
      qDzG[u % Q] = d1s<r, FAST>(fgb + 3 * C::EPL + ecore, 1, c2);

      // output plane x = xa - r: F_x of plane x + k sits at position
      // (u - r + k) mod Q; the y/z terms of plane x at (u - r) mod Q
      if (i >= 2 * r && core_in) {
        const int x = xa - r;
        float dxF = rmul(rsub(qF[pmod(u - r + 1, Q)], qF[pmod(u - r - 1, Q)]), c0[0]);
        float dxG = rmul(rsub(qG[pmod(u - r + 1, Q)], qG[pmod(u - r - 1, Q)]), c0[0]);
#pragma unroll
        for (int k = 2; k <= r; ++k) {
          dxF = mac<FAST>(dxF, rsub(qF[pmod(u - r + k, Q)], qF[pmod(u - r - k, Q)]), c0[k - 1]);
          dxG = mac<FAST>(dxG, rsub(qG[pmod(u - r + k, Q)], qG[pmod(u - r - k, Q)]), c0[k - 1]);
        }
        const int pr = pmod(u - r, Q);
        const float lxy = radd(radd(dxF, qDyF[pr]), qDzF[pr]);
        const float lzz = radd(radd(dxG, qDyG[pr]), qDzG[pr]);
        float op = rsub(rmul(p1, 2.f), ocur[0]);
        float oq = rsub(rmul(q1, 2.f), ocur[1]);
        if constexpr (FAST) {
          op = __fmaf_rn(__fmaf_rn(lzz, ocur[4], rmul(lxy, ocur[3])), ocur[2], op);
          oq = __fmaf_rn(__fmaf_rn(lxy, ocur[4], lzz), ocur[2], oq);
        } else {
          op = radd(op, rmul(radd(rmul(lxy, ocur[3]), rmul(lzz, ocur[4])), ocur[2]));
          oq = radd(oq, rmul(radd(rmul(lxy, ocur[4]), lzz), ocur[2]));
        }
        if (has_fac) {
          // min(min(fx, fy), fz) == min(fx, min(fy, fz)): min is exact
          const float fac = tmin(ocur[5], fyz);
          op = rmul(op, fac);
          oq = rmul(oq, fac);
        }
        const int gi = gcore + x * plane;
        a.p0[gi] = op;
        a.q0[gi] = oq;
        bad |= !finite(op) || !finite(oq);
      }
    }
  }
  if (a.nonfinite && bad) atomicExch(a.nonfinite, 1);
}

}  // namespace
}  // namespace stb
