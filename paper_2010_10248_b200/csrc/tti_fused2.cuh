// Fused single-pass TTI step, second kernel (f32, 3-D grids, r <= 2): two z
// points per thread in packed fp32, warp-specialised, no CTA barrier.
//
// Same arithmetic and IEEE order as tti_fused (and tti_pass1 + tti_pass2,
// and the oracle's TTI class): every packed lane is one correctly rounded
// scalar operation -- sums as FADD2, products as FFMA2 with an opaque -0
// addend (f32x2.cuh) -- so the results are bitwise those of the scalar
// kernels.
//
// What tti_fused's profile showed: 310 thread instructions
// per point, issue-bound, and a CTA barrier per plane behind which the 6
// halo warps (pass 1 of the tile's y/z halo) held the core warps.  Here:
//
//   producer warp  TMA of the p and q planes (tile + 2r rows, 16-byte aligned
//                  z halo, zero fill) into an NS-slot ring; full/empty
//                  mbarriers per slot.
//   core warps     (8) one z pair of the 16 x 32 tile per thread.  Pass 1 at
//                  plane xa: gradients by LDS.64 (x from the ring slots, y
//                  rows, z window of aligned pairs), w, F, G in packed math;
//                  F_x, G_x to register queues (2r+1 deep), F_y, G_y, F_z,
//                  G_z to a shared FG ring of NFG planes.  Pass 2 at plane
//                  xa - r: D_y F_y, D_z F_z, ... from the FG ring, D_x from
//                  the queues, the p/q update, 64-bit stores.
//   halo warps     pass 1 only, at the tile's y-halo rows (F_y, G_y) and
//                  z-halo pairs (F_z, G_z), into the same FG ring.
//
// FG slots carry full (all consumer threads wrote) and empty (core warps
// read) mbarriers, so the halo warps run ahead of the core warps by up to
// NFG - r planes instead of meeting them at a barrier every plane.
//
// Every operand arrives by TMA: besides the p/q planes, the producer stages
// per iteration n_x, n_y, n_z over the pass-1 extent and p, q (t-2), inv,
// e2, d2 over the tile at the output plane (plus fx) into a small operand
// ring, so no warp waits on a global load and no registers hold prefetched
// operands.  HBM bytes per point: 48, as tti_fused (p, q at t-1; p, q at
// t-2, inv, e2, d2, n_x, n_y, n_z; p, q out).
#pragma once

#include "f32x2.cuh"
#include "tti_fused.cuh"

namespace stb {
namespace {

template <int r>
struct Tti2Cfg {
  static constexpr int TY = kTtiTY, TZ = kTtiTZ, P = TZ / 2;  // 16 pairs per row
  static constexpr int HZP = (r + 1) / 2;                     // z-halo pairs per side
  static constexpr int ZH = (2 * r + 3) / 4 * 4;              // p/q slot z halo
  static constexpr int PY = TY + 4 * r, PZ = TZ + 2 * ZH;     // p/q TMA box
  static constexpr int SLOT = (PY * PZ + 31) / 32 * 32;
  // loop unrolled by Q (static queue positions); the p/q ring has 2Q slots,
  // addressed through two half-ring bases that swap every round
  static constexpr int Q = 2 * r + 1, NS = 2 * Q, NFG = Q;
  static constexpr int EY = TY + 2 * r, EZ = TZ + 4 * HZP;    // pass-1 extent (FG, n boxes)
  static constexpr int FPL = (EY * EZ + 31) / 32 * 32;
  static constexpr int TPL = TY * TZ;                         // tile plane (o boxes)
  // n boxes: the pass-1 extent with the z halo rounded up to 4 floats (TMA
  // box rows must start 16-byte aligned in global memory)
  static constexpr int NZH = (2 * HZP + 3) / 4 * 4, NEZ = TZ + 2 * NZH;
  static constexpr int NPL = (EY * NEZ + 31) / 32 * 32;
  // operand slot: n_x, n_y, n_z (NPL each), p0, q0, inv, e2, d2 (TPL each), fx
  static constexpr int NO = 4;
  static constexpr int OBASE = 3 * NPL;
  static constexpr int OSLOT = OBASE + 5 * TPL + 32;
  static constexpr int NCW = TY * P / 32;                     // core warps
  static constexpr int NHY = 2 * r * P, NHZ = TY * 2 * HZP;   // halo pairs
  static constexpr int NHW = (NHY + NHZ + 31) / 32;
  static constexpr int NW = NCW + NHW;                        // consumer warps
  static constexpr int NT = 32 * (NW + 1);                    // + the producer warp
  static constexpr size_t RING = (size_t)2 * NS * SLOT * 4;
  static constexpr size_t FGB = (size_t)4 * NFG * FPL * 4;
  static constexpr size_t OPB = (size_t)NO * OSLOT * 4;
  static constexpr size_t BARS = (size_t)(2 * NFG + 2 * NO) * 8;
  static constexpr size_t SMEM = RING + FGB + OPB + BARS + 128;
  static_assert((TY * P) % 32 == 0, "core pairs fill whole warps");
  static_assert(4 * HZP <= ZH, "z windows of the halo pairs stay inside the staged box");
  static_assert(NFG > r, "FG ring holds the planes between pass 1 and pass 2");
  static_assert(NS >= 2 * r + NO, "a free operand slot implies a free p/q slot");
  static_assert(SMEM <= 232448, "shared memory budget");
};

struct Tti2Maps {
  CUtensorMap p, q;           // level t-1, box PZ x PY
  CUtensorMap n[3];           // axis components, box EZ x EY
  CUtensorMap o[5];           // p, q (t-2), inv, e2, d2, box TZ x TY
};

__device__ __forceinline__ f2 lds2(const float* p) { return *reinterpret_cast<const f2*>(p); }
__device__ __forceinline__ void sts2(float* p, f2 v) { *reinterpret_cast<f2*>(p) = v; }
__device__ __forceinline__ f2 ld2_nc(const float* p) {
  f2 v;
  asm volatile("ld.global.nc.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ f2 ld2_cg(const float* p) {
  f2 v;
  asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ f2 neg2(f2 v) { return v ^ 0x8000000080000000ull; }

template <bool FAST>
__device__ __forceinline__ f2 mac2(f2 acc, f2 d, f2 c, f2 nz) {
  if constexpr (FAST) return fma2(d, c, acc);
  else return add2(acc, xmul2(d, c, nz));
}

// centred first derivative of the pair at c0 along a strided axis
template <int r, bool FAST>
__device__ __forceinline__ f2 d1p(const float* c0, int s, const f2* c, f2 nz) {
  f2 acc = xmul2(sub2(lds2(c0 + s), lds2(c0 - s)), c[0], nz);
#pragma unroll
  for (int k = 2; k <= r; ++k) acc = mac2<FAST>(acc, sub2(lds2(c0 + k * s), lds2(c0 - k * s)), c[k - 1], nz);
  return acc;
}

// along z: the window of aligned pairs z - 2HZP .. z + 2HZP + 1; odd offsets
// are re-paired in registers
template <int r, int HZP, bool FAST>
__device__ __forceinline__ f2 d1z(const float* c0, const f2* c, f2 nz) {
  f2 pr[2 * HZP + 1];
  float w[4 * HZP + 2];
#pragma unroll
  for (int j = 0; j <= 2 * HZP; ++j) {
    pr[j] = lds2(c0 + 2 * (j - HZP));
    upk(pr[j], w[2 * j], w[2 * j + 1]);
  }
  auto pair = [&](int off) -> f2 {       // (z + off, z + 1 + off)
    const int m = 2 * HZP + off;
    if (m % 2 == 0) return pr[m / 2];
    return pk(w[m], w[m + 1]);
  };
  f2 acc = xmul2(sub2(pair(1), pair(-1)), c[0], nz);
#pragma unroll
  for (int k = 2; k <= r; ++k) acc = mac2<FAST>(acc, sub2(pair(k), pair(-k)), c[k - 1], nz);
  return acc;
}

template <int r, bool FAST, bool GUARD>
__global__ void __launch_bounds__(Tti2Cfg<r>::NT, 1)
tti_fused2(const __grid_constant__ Tti2Maps maps, const __grid_constant__ TtiFusedArgs a) {
  using C = Tti2Cfg<r>;
  constexpr int Q = C::Q, NS = C::NS, NFG = C::NFG, NO = C::NO, HZP = C::HZP;
  constexpr int QOFF = NS * C::SLOT;                // q ring follows the p ring
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* sp = reinterpret_cast<float*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  float* fg = sp + 2 * NS * C::SLOT;                // [NFG][4 fields][FPL]
  float* opr = fg + 4 * NFG * C::FPL;               // [NO][OSLOT]
  uint64_t* fgfull = reinterpret_cast<uint64_t*>(opr + NO * C::OSLOT);
  uint64_t* fgempty = fgfull + NFG;
  uint64_t* ofull = fgempty + NFG;
  uint64_t* oempty = ofull + NO;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int z0 = blockIdx.x * C::TZ, y0 = blockIdx.y * C::TY;
  const int x0 = a.x_lo + blockIdx.z * a.cx;
  const int nx = (int)a.d.nx, ny = (int)a.d.ny, nz = (int)a.d.nz;
  const int x1 = min(x0 + a.cx, a.x_hi);
  const int n_iter = (x1 - x0) + 2 * r;             // pass-1 planes x0-r .. x1-1+r
                                                    // (p/q planes x0-2r .. x1-1+2r)
  const bool has_fac = a.has_fac != 0;

  if (tid == 0) {
    for (int g = 0; g < NFG; ++g) {
      mbar_init(&fgfull[g], C::NW * 32);
      mbar_init(&fgempty[g], C::NCW);
    }
    for (int o = 0; o < NO; ++o) {
      mbar_init(&ofull[o], 1);
      mbar_init(&oempty[o], C::NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ------------------------------------------------------------ producer
  // One thread, one transaction barrier per iteration i (slot i % NO): the
  // p/q plane sequence i + 2r (iteration 0 also 0 .. 2r-1), n_x, n_y, n_z
  // over the pass-1 extent of plane xa, and (output iterations) p, q (t-2),
  // inv, e2, d2 over the tile at plane xa - r plus fx.  Consumers release
  // slot i after iteration i; by then they are done with p/q sequence i too,
  // and NS >= 2r + NO makes a free operand slot imply a free p/q slot.
  if (warp == C::NW) {
    if (lane == 0) {
      const int H = (int)a.d.H, zo = (int)a.d.zoff;
      prefetch_map(&maps.p);
      prefetch_map(&maps.q);
      for (int k = 0; k < 3; ++k) prefetch_map(&maps.n[k]);
      for (int k = 0; k < 5; ++k) prefetch_map(&maps.o[k]);
      const int tc0 = zo + z0 - C::ZH, tc1 = H + y0 - 2 * r;
      constexpr uint32_t pq_bytes = 2u * C::PY * C::PZ * 4u;
      for (int i = 0; i < n_iter; ++i) {
        const int slot = i % NO;
        if (i >= NO) mbar_wait_sleep(&oempty[slot], (uint32_t)(((i / NO) - 1) & 1));
        float* os = opr + slot * C::OSLOT;
        const int xa = x0 - r + i, x = xa - r;
        const bool out = i >= 2 * r;                // output plane x in [x0, x1)
        if (out) os[C::OBASE + 5 * C::TPL] = has_fac ? __ldg(a.fx + x) : 1.f;
        const int s0 = i == 0 ? 0 : i + 2 * r;      // p/q sequences of this slot
        const int s1 = i + 2 * r;
        mbar_arrive_expect_tx(&ofull[slot],
                              (uint32_t)(s1 - s0 + 1) * pq_bytes +
                              (uint32_t)(3 * C::EY * C::NEZ + (out ? 5 * C::TPL : 0)) * 4u);
        for (int sq = s0; sq <= s1; ++sq) {
          const int ps = sq % NS, xg = H + x0 - 2 * r + sq;
          tma_load_3d(sp + ps * C::SLOT, &maps.p, tc0, tc1, xg, &ofull[slot]);
          tma_load_3d(sp + QOFF + ps * C::SLOT, &maps.q, tc0, tc1, xg, &ofull[slot]);
        }
        for (int k = 0; k < 3; ++k)
          tma_load_3d(os + k * C::NPL, &maps.n[k], zo + z0 - C::NZH, H + y0 - r, H + xa,
                      &ofull[slot]);
        if (out)
          for (int k = 0; k < 5; ++k)
            tma_load_3d(os + C::OBASE + k * C::TPL, &maps.o[k], zo + z0, H + y0, H + x,
                        &ofull[slot]);
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const bool core = warp < C::NCW;
  const int t = core ? tid : tid - 32 * C::NCW;
  bool work = true;
  int fy = 0, fzc = 0, yy = 0, zz = 0, comp = 0;   // comp: 0 all four, 1 F_y/G_y, 2 F_z/G_z
  int ooff = 0;                                     // core: pair offset in a tile box
  if (core) {
    const int ty = t / C::P, tzp = t % C::P;
    yy = y0 + ty;
    zz = z0 + 2 * tzp;
    fy = ty + r;
    fzc = 2 * HZP + 2 * tzp;
    ooff = ty * C::TZ + 2 * tzp;
  } else if (t < C::NHY) {
    const int row = t / C::P, j = t % C::P;         // rows [0, r) and [TY + r, TY + 2r)
    fy = row < r ? row : C::TY + row;
    yy = y0 - r + fy;
    fzc = 2 * HZP + 2 * j;
    zz = z0 + 2 * j;
    comp = 1;
  } else if (t < C::NHY + C::NHZ) {
    const int h = t - C::NHY;
    const int row = h / (2 * HZP), j = h % (2 * HZP);
    fy = r + row;
    yy = y0 + row;
    fzc = j < HZP ? 2 * j : C::TZ + 2 * j;
    zz = z0 - 2 * HZP + fzc;
    comp = 2;
  } else {
    work = false;                                   // corner slot (never read)
  }
  const bool yin = work && yy >= 0 && yy < ny;
  const bool zin0 = zz >= 0 && zz < nz, zin1 = zz + 1 >= 0 && zz + 1 < nz;
  const bool in0 = yin && zin0, in1 = yin && zin1;
  const bool any_in = in0 || in1;
  const f2 dmask = (in0 ? 0x00000000ffffffffull : 0ull) | (in1 ? 0xffffffff00000000ull : 0ull);
  const int gidx = any_in ? (int)a.d.at(0, yy, zz) : 0;       // even: zoff, pitch multiples of 32
  const int soff = work ? (yy - y0 + 2 * r) * C::PZ + (zz - z0 + C::ZH) : 2 * r * C::PZ + C::ZH;
  const int foff = fy * C::EZ + fzc;
  const int noff = fy * C::NEZ + fzc + (C::NZH - 2 * HZP);   // n offset in an operand slot

  const f2 nzr = bcast(a.negz);
  const f2 two = bcast(2.f);
  f2 cx[r], cy[r], cz[r];
#pragma unroll
  for (int k = 0; k < r; ++k) {
    cx[k] = bcast(a.cf.c[0][k]);
    cy[k] = bcast(a.cf.c[1][k]);
    cz[k] = bcast(a.cf.c[2][k]);
  }
  const int plane = (int)a.d.plane;
  float fyz0 = 1.f, fyz1 = 1.f;
  if (has_fac && core && any_in) {
    const float fyv = __ldg(a.fy + yy);
    fyz0 = in0 ? tmin(fyv, __ldg(a.fz + zz)) : 1.f;
    fyz1 = in1 ? tmin(fyv, __ldg(a.fz + zz + 1)) : 1.f;
  }

  f2 qF[Q], qG[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) qF[j] = qG[j] = 0ull;

  int os = 0;                                       // operand slot i % NO and its phase
  uint32_t oph = 0;
  bool bad = false;
  for (int i0 = 0, k = 0; i0 < n_iter; i0 += Q, ++k) {
    // half rings of this round (sequences kQ .. kQ+Q-1) and the next
    const int hc = (k & 1) * Q, hn = Q - hc;
    const float* rc = sp + hc * C::SLOT + soff;
    const float* rn = sp + hn * C::SLOT + soff;
    const uint32_t pk_ = (uint32_t)(k & 1);
#pragma unroll
    for (int u = 0; u < Q; ++u) {
      const int i = i0 + u;
      if (i >= n_iter) break;
      const int xa = x0 - r + i;
      mbar_wait(&ofull[os], oph);                   // p/q window and operands of iteration i
      const float* ob = opr + os * C::OSLOT;

      // ---- pass 1 at plane xa
      // (computed everywhere; points outside the grid are masked to +0)
      f2 F[3], G[3];
      f2 p1 = 0ull, q1 = 0ull;
      {
        const float* ps[2 * r + 1];
#pragma unroll
        for (int dd = 0; dd <= 2 * r; ++dd)
          ps[dd] = (u + dd < Q ? rc : rn) + ((u + dd) % Q) * C::SLOT;
        const f2 m = (xa >= 0 && xa < nx) ? dmask : 0ull;
        const f2 n0 = lds2(ob + noff), n1 = lds2(ob + C::NPL + noff),
                 n2 = lds2(ob + 2 * C::NPL + noff);
        f2 gpx = xmul2(sub2(lds2(ps[r + 1]), lds2(ps[r - 1])), cx[0], nzr);
        f2 gqx = xmul2(sub2(lds2(ps[r + 1] + QOFF), lds2(ps[r - 1] + QOFF)), cx[0], nzr);
#pragma unroll
        for (int kk = 2; kk <= r; ++kk) {
          gpx = mac2<FAST>(gpx, sub2(lds2(ps[r + kk]), lds2(ps[r - kk])), cx[kk - 1], nzr);
          gqx = mac2<FAST>(gqx, sub2(lds2(ps[r + kk] + QOFF), lds2(ps[r - kk] + QOFF)),
                           cx[kk - 1], nzr);
        }
        const f2 gpy = d1p<r, FAST>(ps[r], C::PZ, cy, nzr);
        const f2 gqy = d1p<r, FAST>(ps[r] + QOFF, C::PZ, cy, nzr);
        const f2 gpz = d1z<r, HZP, FAST>(ps[r], cz, nzr);
        const f2 gqz = d1z<r, HZP, FAST>(ps[r] + QOFF, cz, nzr);
        const f2 wp = mac2<FAST>(mac2<FAST>(xmul2(gpx, n0, nzr), gpy, n1, nzr), gpz, n2, nzr);
        const f2 wq = mac2<FAST>(mac2<FAST>(xmul2(gqx, n0, nzr), gqy, n1, nzr), gqz, n2, nzr);
        const f2 g[3] = {gpx, gpy, gpz};
        const f2 n[3] = {n0, n1, n2};
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          if constexpr (FAST) F[ax] = fma2(neg2(wp), n[ax], g[ax]);
          else F[ax] = sub2(g[ax], xmul2(wp, n[ax], nzr));
          G[ax] = xmul2(wq, n[ax], nzr);
          F[ax] &= m;
          G[ax] &= m;
        }
        if (core) {                                 // p, q (t-1) at the output plane xa - r
          p1 = lds2(ps[0]);
          q1 = lds2(ps[0] + QOFF);
        }
      }

      // ---- F_y, G_y, F_z, G_z of plane xa to FG slot u
      if (i >= NFG) mbar_wait(&fgempty[u], pk_ ^ 1u);
      {
        float* fgs = fg + u * 4 * C::FPL + foff;
        if (comp != 2) {
          sts2(fgs + 0 * C::FPL, F[1]);
          sts2(fgs + 1 * C::FPL, G[1]);
        }
        if (comp != 1) {
          sts2(fgs + 2 * C::FPL, F[2]);
          sts2(fgs + 3 * C::FPL, G[2]);
        }
        mbar_arrive(&fgfull[u]);
        // planes x0-r .. x0-1 only feed the x queues: nobody reads their FG
        // slot, so release it here (keeps every slot's phases in step)
        if (core && i < r) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&fgempty[u]);
        }
      }
      if (core) {
        qF[u] = F[0];
        qG[u] = G[0];
      }

      // ---- pass 2 (core warps): output plane x = xa - r, FG of iteration i - r
      if (core && i >= 2 * r) {
        const float* oo = ob + C::OBASE + ooff;
        const f2 o0 = lds2(oo), o1 = lds2(oo + C::TPL), o2 = lds2(oo + 2 * C::TPL),
                 o3 = lds2(oo + 3 * C::TPL), o4 = lds2(oo + 4 * C::TPL);
        const float fxc = ob[C::OBASE + 5 * C::TPL];
        const int g2 = (u - r + Q) % Q;
        mbar_wait(&fgfull[g2], u < r ? pk_ ^ 1u : pk_);
        const float* fq = fg + g2 * 4 * C::FPL + foff;
        const f2 dyF = d1p<r, FAST>(fq + 0 * C::FPL, C::EZ, cy, nzr);
        const f2 dyG = d1p<r, FAST>(fq + 1 * C::FPL, C::EZ, cy, nzr);
        const f2 dzF = d1z<r, HZP, FAST>(fq + 2 * C::FPL, cz, nzr);
        const f2 dzG = d1z<r, HZP, FAST>(fq + 3 * C::FPL, cz, nzr);
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&fgempty[g2]);
          mbar_arrive(&oempty[os]);
        }
        // F_x of plane x + kk sits at queue position (u - r + kk) mod Q
        f2 dxF = xmul2(sub2(qF[pmod(u - r + 1, Q)], qF[pmod(u - r - 1, Q)]), cx[0], nzr);
        f2 dxG = xmul2(sub2(qG[pmod(u - r + 1, Q)], qG[pmod(u - r - 1, Q)]), cx[0], nzr);
#pragma unroll
        for (int kk = 2; kk <= r; ++kk) {
          dxF = mac2<FAST>(dxF, sub2(qF[pmod(u - r + kk, Q)], qF[pmod(u - r - kk, Q)]),
                           cx[kk - 1], nzr);
          dxG = mac2<FAST>(dxG, sub2(qG[pmod(u - r + kk, Q)], qG[pmod(u - r - kk, Q)]),
                           cx[kk - 1], nzr);
        }
        const f2 lxy = add2(add2(dxF, dyF), dzF);
        const f2 lzz = add2(add2(dxG, dyG), dzG);
        f2 op = sub2(xmul2(p1, two, nzr), o0);
        f2 oq = sub2(xmul2(q1, two, nzr), o1);
        if constexpr (FAST) {
          op = fma2(fma2(lzz, o4, xmul2(lxy, o3, nzr)), o2, op);
          oq = fma2(fma2(lxy, o4, lzz), o2, oq);
        } else {
          op = add2(op, xmul2(add2(xmul2(lxy, o3, nzr), xmul2(lzz, o4, nzr)), o2, nzr));
          oq = add2(oq, xmul2(add2(xmul2(lxy, o4, nzr), lzz), o2, nzr));
        }
        if (has_fac) {
          // min(min(fx, fy), fz) == min(fx, min(fy, fz)): min is exact
          const f2 fac = pk(tmin(fxc, fyz0), tmin(fxc, fyz1));
          op = xmul2(op, fac, nzr);
          oq = xmul2(oq, fac, nzr);
        }
        if (any_in) {
          const int gi = gidx + (xa - r) * plane;
          float p_lo, p_hi, q_lo, q_hi;
          upk(op, p_lo, p_hi);
          upk(oq, q_lo, q_hi);
          if (in1) {
            *reinterpret_cast<f2*>(a.p0 + gi) = op;
            *reinterpret_cast<f2*>(a.q0 + gi) = oq;
            if constexpr (GUARD)
              bad |= !finite(p_lo) || !finite(q_lo) || !finite(p_hi) || !finite(q_hi);
          } else {
            a.p0[gi] = p_lo;
            a.q0[gi] = q_lo;
            if constexpr (GUARD) bad |= !finite(p_lo) || !finite(q_lo);
          }
        }
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&oempty[os]);
      }
      if (++os == NO) {
        os = 0;
        oph ^= 1u;
      }
    }
  }
  if constexpr (GUARD) {
    if (bad) atomicExch(a.nonfinite, 1);
  }
}

}  // namespace
}  // namespace stb
