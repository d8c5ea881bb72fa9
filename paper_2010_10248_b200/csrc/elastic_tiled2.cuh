// Elastic half steps, second TMA kernel (f32, 3-D grids, R <= 4): z pairs in
// packed fp32, a producer warp, no CTA barrier.
//
// Same arithmetic and IEEE order as elastic_tiled (and the point kernels,
// physics.py:287-429): each packed lane is one correctly rounded scalar
// operation -- sums as FADD2, products as FFMA2 with an opaque -0 addend
// (f32x2.cuh) -- so results are bitwise those of the scalar kernels.
//
// What elastic_tiled's profile showed: 236 (v) / 272 (tau)
// thread instructions per point, 27-30 % of the stall samples on the
// per-plane CTA barrier behind which thread 0 refilled the ring, and
// 17-23 % long-scoreboard on the centre operands loaded from global memory.
// Here, per CTA (16 x 32 tile, an x chunk):
//
//   producer warp  one transaction barrier per iteration n: the NF input
//                  field planes of sequence n (tile + the halo the field is
//                  differentiated along: R rows, 16-byte aligned z columns,
//                  zero fill) into a plane ring of NS = R + NO slots, and for output iterations the centre operands
//                  (old values of the updated fields, materials) over the
//                  tile plus fx into an NO-slot operand ring.
//   8 warps        one z pair of the tile per thread: x derivatives from
//                  register queues (2R+1 planes, pairs), y/z neighbours by
//                  LDS.64 from the slot of the output plane (R behind the
//                  newest), the update, 64-bit stores in place.  A warp
//                  releases iteration n's operand slot after its output;
//                  with NS = R + NO that also frees the plane slot the
//                  producer fills next.
//
// Compulsory HBM bytes per point unchanged: v pass 52, tau pass 68.
//
// el2_tile is one tile of one half step; elastic_tiled2 launches it per
// (tile, x chunk), elastic_stream (opt-in) runs both half steps of a step in
// one launch with the tau sweep trailing the v sweep through L2.
#pragma once

#include "elastic_tiled.cuh"
#include "f32x2.cuh"

namespace stb {
namespace {

template <int R, int PASS, int NO_ = 3>
struct El2Cfg {
  static constexpr int TY = 16, TZ = kElTZ, P = TZ / 2;       // 16 pairs per row
  static constexpr int NF = PASS == 0 ? 6 : 3;                // staged (differentiated) fields
  static constexpr int NOUT = PASS == 0 ? 3 : 6;              // updated fields
  static constexpr int NM = PASS == 0 ? 1 : 2;                // materials
  static constexpr int ZH = (R + 3) / 4 * 4;                  // z halo (16-byte boxes)
  static constexpr int PY = TY + 2 * R, PZ = TZ + 2 * ZH;
  // Per staged field, only the halo it is differentiated along: in the v pass
  // txx feeds the x queue alone (no halo), tyy / txy are differenced along y
  // (halo rows), tzz / txz along z (halo columns), tyz along both; in the tau
  // pass every velocity along both.  (Full boxes for all six cost 2.25 x the
  // tile's sectors per field, "Elastic".)
  static constexpr int fhy(int f) { return PASS == 1 || f == 1 || f == 3 || f == 5 ? R : 0; }
  static constexpr int fhz(int f) { return PASS == 1 || f == 2 || f == 4 || f == 5 ? ZH : 0; }
  static constexpr int fby(int f) { return TY + 2 * fhy(f); }
  static constexpr int fbz(int f) { return TZ + 2 * fhz(f); }
  static constexpr int fsz(int f) { return (fby(f) * fbz(f) + 31) / 32 * 32; }
  static constexpr int foff(int f) {
    int s = 0;
    for (int i = 0; i < f; ++i) s += fsz(i);
    return s;
  }
  static constexpr int boxf(int f) {                          // staged floats of fields [0, f)
    int s = 0;
    for (int i = 0; i < f; ++i) s += fby(i) * fbz(i);
    return s;
  }
  static constexpr int SLOT = foff(NF);
  static constexpr int BOXF = boxf(NF);
  static constexpr int Q = 2 * R + 1;
  static constexpr int NO = NO_, NS = R + NO;
  static constexpr int TPL = TY * TZ;
  static constexpr int OSLOT = (NOUT + NM) * TPL + 32;        // + fx
  static constexpr int HW = (R + 1) / 2;                      // z window: pairs -HW .. +HW
  static constexpr int NCW = TY * P / 32;
  static constexpr int NT = 32 * (NCW + 1);
  static constexpr size_t SMEM =
      (size_t)NS * SLOT * 4 + (size_t)NO * OSLOT * 4 + (size_t)2 * NO * 8 + 64 + 128;
  static_assert(2 * HW <= ZH, "z window inside the staged box");
  static_assert(SMEM <= 232448, "shared memory budget");
};

struct El2Maps {
  CUtensorMap f[6];       // staged inputs (v pass: txx tyy tzz txy txz tyz; tau: vx vy vz)
  CUtensorMap o[8];       // centre operands: updated fields' old values, then materials
};

// Control block of the streamed full step (elastic_stream below).  Progress
// words are (epoch << 13) | planes; a word of another epoch reads as 0.
struct ElStream {
  unsigned* prog_v;       // per v tile: x planes stored and visible
  unsigned* prog_t;       // per tau tile: x planes issued (throttle hint only)
  int* err;               // set when a dependency wait gave up
  unsigned epoch;
  int nv, nt;             // CTAs per role
  int tiles_z, tiles_yv, tiles_yt;
  int lead;               // planes a v tile may run ahead of the tau tile under it
  int pub;                // planes per published group (power of 2)
};

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_all() {
  asm volatile("fence.proxy.async;" ::: "memory");
}
__device__ __forceinline__ int ld_acquire_cta_s32(const volatile int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];"
               : "=r"(v) : "r"(smem_u32(const_cast<const int*>(p))) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_s32(volatile int* p, int v) {
  asm volatile("st.release.cta.shared.s32 [%0], %1;"
               ::"r"(smem_u32(const_cast<int*>(p))), "r"(v) : "memory");
}
constexpr int kElTauSeen = 8, kElHave = 9;          // wprog slots after the per-warp words
constexpr unsigned kElPlaneBits = 13, kElPlaneMask = (1u << kElPlaneBits) - 1u;

__device__ __forceinline__ f2 el_lds2(const float* p) { return *reinterpret_cast<const f2*>(p); }

// staggered first derivative of pairs: acc = sum_j (g(hi) - g(lo)) * c_j
template <int R, typename G>
__device__ __forceinline__ f2 stag2(const G& g, const f2* c, bool fwd, f2 nz) {
  f2 acc = 0ull;
#pragma unroll
  for (int j = 1; j <= R; ++j) {
    const int hi = fwd ? j : j - 1;
    const int lo = fwd ? -(j - 1) : -j;
    const f2 term = xmul2(sub2(g(hi), g(lo)), c[j - 1], nz);
    acc = (j == 1) ? term : add2(acc, term);
  }
  return acc;
}

// z window of a field around the pair at c0: pairs at offsets -2HW .. +2HW
template <int HW>
struct ZWin {
  f2 pr[2 * HW + 1];
  float w[4 * HW + 2];
  __device__ __forceinline__ void load(const float* c0) {
#pragma unroll
    for (int j = 0; j <= 2 * HW; ++j) {
      pr[j] = el_lds2(c0 + 2 * (j - HW));
      upk(pr[j], w[2 * j], w[2 * j + 1]);
    }
  }
  __device__ __forceinline__ f2 operator()(int o) const {   // (z + o, z + 1 + o)
    const int m = 2 * HW + o;
    if (m % 2 == 0) return pr[m / 2];
    return pk(w[m], w[m + 1]);
  }
};

// One tile (16 x 32 in y, z; x planes [x0, x1)) of one half step.  The caller
// has initialised the barriers ONCE: g0 counts the iterations this CTA ran on
// earlier tiles, and ring slots and barrier phases continue from there (an
// mbarrier.inval + init between tiles misbehaved on B200 whenever slot 0 had
// completed an odd number of phases).  Every thread returns.  STREAM adds the
// cross-CTA protocol of elastic_stream (publish / dependency waits / throttle).
template <int R, int PASS, bool GUARD, bool STREAM, int NO_ = 3>
__device__ __forceinline__ void el2_tile(const El2Maps& maps, const ElTiledArgs& a,
                                         const ElStream& sc, float* ring, float* opr,
                                         uint64_t* ofull, uint64_t* oempty, volatile int* wprog,
                                         const int y0, const int z0, const int x0, const int x1,
                                         const int tile, const int g0) {
  using C = El2Cfg<R, PASS, NO_>;
  constexpr int Q = C::Q, NS = C::NS, NO = C::NO, NF = C::NF, NOUT = C::NOUT, NM = C::NM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ny = (int)a.d.ny, nz = (int)a.d.nz;
  const int N = (x1 - x0) + 2 * R;                  // sequence n = plane x0 - R + n
  const bool has_fac = a.has_fac != 0;

  // ------------------------------------------------------------ producer
  if (warp == C::NCW) {
    if (lane == 0) {
      const int H = (int)a.d.H, zo = (int)a.d.zoff;
#pragma unroll
      for (int f = 0; f < NF; ++f) prefetch_map(&maps.f[f]);
#pragma unroll
      for (int k = 0; k < NOUT + NM; ++k) prefetch_map(&maps.o[k]);
      int have = 0;                                 // tau role: planes stored on every dependency
      int budget = 8000;                            // v role: throttle polls left for this tile
      for (int n = 0; n < N; ++n) {
        const int g = g0 + n;
        const int slot = g % NO;
        if constexpr (STREAM && PASS == 1) {
          // plane x0 - R + n of vx, vy, vz must be stored by every dependency
          // (which also means their sweeps have read the stress planes this
          // iteration's output overwrites, R behind); the sync warp polls the
          // dependencies and posts what it has acquired
          const int need = min(x0 - R + n + 1, x1) - x0;
          if (need > have) {
            while ((have = ld_acquire_cta_s32(&wprog[kElHave])) < need) __nanosleep(32);
            fence_proxy_async_all();                // their generic stores before our TMA reads
          }
          if ((n & 3) == 0)
            st_relaxed_u32(sc.prog_t + tile, (sc.epoch << kElPlaneBits) | (unsigned)n);
        }
        if constexpr (STREAM && PASS == 0) {
          // hold back while the tau tile under this tile is more than `lead`
          // planes behind, so what this sweep reads and writes is still in L2
          // when the tau sweep comes for it (bounded: a hint, not a dependency)
          while (budget > 0 && n - sc.lead > wprog[kElTauSeen]) {
            --budget;
            __nanosleep(128);
          }
        }
        if (g >= NO) mbar_wait_sleep(&oempty[slot], (uint32_t)(((g / NO) - 1) & 1));
        float* os = opr + slot * C::OSLOT;
        const bool out = n >= 2 * R;
        const int x = x0 - 2 * R + n;               // output plane of iteration n
        if (out) os[(NOUT + NM) * C::TPL] = has_fac ? __ldg(a.fx + x) : 1.f;
        mbar_arrive_expect_tx(&ofull[slot], (uint32_t)(C::BOXF +
                                                       (out ? (NOUT + NM) * C::TPL : 0)) * 4u);
        float* ps = ring + (g % NS) * C::SLOT;
#pragma unroll
        for (int f = 0; f < NF; ++f)
          tma_load_3d(ps + C::foff(f), &maps.f[f], zo + z0 - C::fhz(f), H + y0 - C::fhy(f),
                      H + x0 - R + n, &ofull[slot]);
        if (out) {
#pragma unroll
          for (int k = 0; k < NOUT + NM; ++k)
            tma_load_3d(os + k * C::TPL, &maps.o[k], zo + z0, H + y0, H + x, &ofull[slot]);
        }
      }
      if constexpr (STREAM && PASS == 1)
        st_relaxed_u32(sc.prog_t + tile, (sc.epoch << kElPlaneBits) | kElPlaneMask);
    }
    return;
  }

  // ------------------------------------------------------------ sync warp
  // (elastic_stream only) one thread that does the global-memory side of the
  // protocol, so neither the consumers nor the TMA-issuing thread wait on it.
  if (warp == C::NCW + 1) {
    if constexpr (STREAM) {
      if (lane == 0) {
        const int total = x1 - x0;
        const unsigned ep = sc.epoch << kElPlaneBits;
        if constexpr (PASS == 0) {
          // publish the planes every consumer warp has stored (the warps post
          // them with release.cta; the gpu-scope fence here is cumulative),
          // and keep the tau tile's progress at hand for the throttle
          int pubd = 0;
          for (unsigned it = 0; pubd < total; ++it) {
            int m = 1 << 30;
#pragma unroll
            for (int w = 0; w < C::NCW; ++w) m = min(m, ld_acquire_cta_s32(&wprog[w]));
            if (m >= pubd + sc.pub || (m >= total && pubd < total)) {
              __threadfence();
              st_relaxed_u32(sc.prog_v + tile, ep | (unsigned)m);
              pubd = m;
            }
            if ((it & 3) == 0) {
              const unsigned w = ld_relaxed_u32(sc.prog_t + tile);
              wprog[kElTauSeen] = (w >> kElPlaneBits) == sc.epoch ? (int)(w & kElPlaneMask) : 0;
            }
            __nanosleep(64);
          }
        } else {
          // the v tiles whose planes this tile stages (and whose sweeps read
          // the stresses this tile overwrites): rows ty-1, ty x columns
          // tz-1 .. tz+1 of the v tiling
          int dep[6];
          const int ty = tile / sc.tiles_z, tz = tile % sc.tiles_z;
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            const int dy = ty - 1 + k / 3, dz = tz - 1 + k % 3;
            dep[k] = (dy >= 0 && dy < sc.tiles_yv && dz >= 0 && dz < sc.tiles_z)
                         ? dy * sc.tiles_z + dz : -1;
          }
          int have = 0;
          for (unsigned spins = 0; have < total; ++spins) {
            unsigned w[6];
#pragma unroll
            for (int k = 0; k < 6; ++k)             // six independent loads in flight
              w[k] = dep[k] >= 0 ? ld_relaxed_u32(sc.prog_v + dep[k]) : (ep | kElPlaneMask);
            int m = 1 << 30;
#pragma unroll
            for (int k = 0; k < 6; ++k)
              m = min(m, (w[k] >> kElPlaneBits) == sc.epoch ? (int)(w[k] & kElPlaneMask) : 0);
            if (spins > (1u << 23)) {               // ~ seconds without progress: give up, report
              *sc.err = 1;
              m = total;
            }
            if (m > have) {
              __threadfence();                      // acquire: relaxed loads, then the fence
              st_release_cta_s32(&wprog[kElHave], m);
              have = m;
              spins = 0;
            }
            __nanosleep(64);
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int ty = tid / C::P, tzp = tid % C::P;
  const int y = y0 + ty, z = z0 + 2 * tzp;
  const bool in0 = y >= 0 && y < ny && z < nz, in1 = y >= 0 && y < ny && z + 1 < nz;
  const int gcore = in0 ? (int)a.d.at(0, y, z) : 0;
  // centre of field f in a ring slot: rows are TZ or PZ floats long
  const int b32 = ty * C::TZ + 2 * tzp, b40 = ty * C::PZ + 2 * tzp;
  auto cen = [&](int f) {
    return (C::fbz(f) == C::TZ ? b32 : b40) + (C::fhy(f) * C::fbz(f) + C::fhz(f) + C::foff(f));
  };
  const int ooff = ty * C::TZ + 2 * tzp;
  const int plane = (int)a.d.plane;
  const f2 nzr = bcast(a.negz);
  f2 cxk[R], cyk[R], czk[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    cxk[k] = bcast(a.cf.d1[0][k]);
    cyk[k] = bcast(a.cf.d1[1][k]);
    czk[k] = bcast(a.cf.d1[2][k]);
  }
  float fyz0 = 1.f, fyz1 = 1.f;
  if (has_fac && in0) {
    const float fyv = __ldg(a.fy + y);
    fyz0 = tmin(fyv, __ldg(a.fz + z));
    fyz1 = in1 ? tmin(fyv, __ldg(a.fz + z + 1)) : 1.f;
  }

  // x queues (position n mod Q): v pass txx, txy, txz; tau pass vx, vy, vz
  f2 q0[Q], q1[Q], q2[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) q0[j] = q1[j] = q2[j] = 0ull;
  constexpr int QF0 = 0, QF1 = PASS == 0 ? 3 : 1, QF2 = PASS == 0 ? 4 : 2;

  int os = g0 % NO, sn = g0 % NS, so = (g0 + NS - R) % NS;   // g % NO, g % NS, (g - R) % NS
  uint32_t oph = (uint32_t)((g0 / NO) & 1);
  bool bad = false;
  for (int n0 = 0; n0 < N; n0 += Q) {
#pragma unroll
    for (int u = 0; u < Q; ++u) {
      const int n = n0 + u;
      if (n >= N) break;
      mbar_wait(&ofull[os], oph);
      const float* sl = ring + sn * C::SLOT;         // newest plane
      q0[u] = el_lds2(sl + cen(QF0));
      q1[u] = el_lds2(sl + cen(QF1));
      q2[u] = el_lds2(sl + cen(QF2));
      if (n >= 2 * R) {
        const float* cp = ring + so * C::SLOT;          // output plane (sequence n - R)
        const float* ob = opr + os * C::OSLOT;
        auto gq0 = [&](int o) { return q0[el_pmod(u - R + o, Q)]; };
        auto gq1 = [&](int o) { return q1[el_pmod(u - R + o, Q)]; };
        auto gq2 = [&](int o) { return q2[el_pmod(u - R + o, Q)]; };
        auto gy = [&](int f) {
          const float* c0 = cp + cen(f);
          return [=](int o) { return el_lds2(c0 + o * C::fbz(f)); };
        };
        f2 res[NOUT];
        f2 fac = 0ull;
        if (has_fac) {
          const float fxv = ob[(NOUT + NM) * C::TPL];
          fac = pk(tmin(fxv, fyz0), tmin(fxv, fyz1));
        }
        if constexpr (PASS == 0) {
          // fields: 0 txx, 1 tyy, 2 tzz, 3 txy, 4 txz, 5 tyz
          ZWin<C::HW> w4, w5, w2;
          w4.load(cp + cen(4));
          w5.load(cp + cen(5));
          w2.load(cp + cen(2));
          f2 d0 = stag2<R>(gq0, cxk, true, nzr);
          d0 = add2(d0, stag2<R>(gy(3), cyk, false, nzr));
          d0 = add2(d0, stag2<R>(w4, czk, false, nzr));
          f2 d1 = stag2<R>(gq1, cxk, false, nzr);
          d1 = add2(d1, stag2<R>(gy(1), cyk, true, nzr));
          d1 = add2(d1, stag2<R>(w5, czk, false, nzr));
          f2 d2 = stag2<R>(gq2, cxk, false, nzr);
          d2 = add2(d2, stag2<R>(gy(5), cyk, false, nzr));
          d2 = add2(d2, stag2<R>(w2, czk, true, nzr));
          const f2 buoy = el_lds2(ob + 3 * C::TPL + ooff);
          const f2 dd[3] = {d0, d1, d2};
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            f2 o = add2(el_lds2(ob + k * C::TPL + ooff), xmul2(dd[k], buoy, nzr));
            if (has_fac) o = xmul2(o, fac, nzr);
            res[k] = o;
          }
        } else {
          // fields: 0 vx, 1 vy, 2 vz; outputs txx tyy tzz txy txz tyz
          ZWin<C::HW> w0, w1, w2;
          w0.load(cp + cen(0));
          w1.load(cp + cen(1));
          w2.load(cp + cen(2));
          const f2 lam = el_lds2(ob + 6 * C::TPL + ooff), mu = el_lds2(ob + 7 * C::TPL + ooff);
          const f2 mu2 = xmul2(mu, bcast(2.f), nzr);
          const f2 dg0 = stag2<R>(gq0, cxk, false, nzr);
          const f2 dg1 = stag2<R>(gy(1), cyk, false, nzr);
          const f2 dg2 = stag2<R>(w2, czk, false, nzr);
          const f2 tr = add2(add2(dg0, dg1), dg2);
          const f2 dg[3] = {dg0, dg1, dg2};
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            f2 o = add2(el_lds2(ob + k * C::TPL + ooff),
                        add2(xmul2(tr, lam, nzr), xmul2(dg[k], mu2, nzr)));
            if (has_fac) o = xmul2(o, fac, nzr);
            res[k] = o;
          }
          // txy = stag_y(vx, fwd) + stag_x(vy, fwd); txz = stag_z(vx) + stag_x(vz);
          // tyz = stag_z(vy) + stag_y(vz)   (elastic_tau_point order)
          const f2 s0 = add2(stag2<R>(gy(0), cyk, true, nzr), stag2<R>(gq1, cxk, true, nzr));
          const f2 s1 = add2(stag2<R>(w0, czk, true, nzr), stag2<R>(gq2, cxk, true, nzr));
          const f2 s2 = add2(stag2<R>(w1, czk, true, nzr), stag2<R>(gy(2), cyk, true, nzr));
          const f2 ss[3] = {s0, s1, s2};
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            f2 o = add2(el_lds2(ob + (3 + k) * C::TPL + ooff), xmul2(ss[k], mu, nzr));
            if (has_fac) o = xmul2(o, fac, nzr);
            res[3 + k] = o;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&oempty[os]);
        if (in0) {
          const int gi = gcore + (x0 - 2 * R + n) * plane;
#pragma unroll
          for (int k = 0; k < NOUT; ++k) {
            float lo, hi;
            upk(res[k], lo, hi);
            if (in1) {
              *reinterpret_cast<f2*>(a.out[k] + gi) = res[k];
              if constexpr (GUARD) bad |= !finite(lo) || !finite(hi);
            } else {
              a.out[k][gi] = lo;
              if constexpr (GUARD) bad |= !finite(lo);
            }
          }
        }
        if constexpr (STREAM && PASS == 0) {
          // post the planes this warp has stored (the sync warp publishes them)
          __syncwarp();
          if (lane == 0) st_release_cta_s32(&wprog[warp], n - 2 * R + 1);
        }
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&oempty[os]);
      }
      if (++os == NO) {
        os = 0;
        oph ^= 1u;
      }
      if (++sn == NS) sn = 0;
      if (++so == NS) so = 0;
    }
  }
  if constexpr (GUARD) {
    if (bad) atomicExch(a.nonfinite, 1);
  }
}

// shared memory of one pass: plane ring, operand ring, barriers, warp progress
template <int R, int PASS, int NO_ = 3>
struct El2Smem {
  using C = El2Cfg<R, PASS, NO_>;
  float* ring;
  float* opr;
  uint64_t* ofull;
  uint64_t* oempty;
  volatile int* wprog;
  __device__ __forceinline__ explicit El2Smem(unsigned char* raw) {
    ring = reinterpret_cast<float*>(raw + ((128u - (smem_u32(raw) & 127u)) & 127u));
    opr = ring + C::NS * C::SLOT;
    ofull = reinterpret_cast<uint64_t*>(opr + C::NO * C::OSLOT);
    oempty = ofull + C::NO;
    wprog = reinterpret_cast<volatile int*>(oempty + C::NO);
  }
  // barriers: once per CTA; the per-tile progress words: before every tile
  __device__ __forceinline__ void init(bool first) {
    if (first && threadIdx.x == 0) {
      for (int o = 0; o < C::NO; ++o) {
        mbar_init(&ofull[o], 1);
        mbar_init(&oempty[o], C::NCW);
      }
      fence_mbar_init();
    }
    if (threadIdx.x < 16) wprog[threadIdx.x] = 0;
    __syncthreads();
  }
};

// operand slots of the two-launch path per pass.  Since the v pass stages
// per-field boxes its ring has room for five (1024^3: 3 / 4 / 5 / 6 slots 43.7 /
// 45.4 / 45.9 / 45.7 GPts/s); the tau pass is best at three (2: 40.6, 4: 44.1,
// 5: 43.1 with five v slots -- its DRAM reads GROW with depth: 54.6 / 63.9 /
// 66.0 GB at 3 / 4 / 5 slots).
template <int PASS> constexpr int el2_two_no() { return PASS == 0 ? 5 : 3; }
template <int R, int PASS> using El2Two = El2Cfg<R, PASS, el2_two_no<PASS>()>;

// One half step as its own launch: a CTA per (tile, x chunk).
template <int R, int PASS, bool GUARD>
__global__ void __launch_bounds__(El2Cfg<R, PASS>::NT, 1)
elastic_tiled2(const __grid_constant__ El2Maps maps, const __grid_constant__ ElTiledArgs a) {
  using C = El2Two<R, PASS>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  El2Smem<R, PASS, C::NO> sm(smem_raw);
  sm.init(true);
  const int x0 = a.x_lo + blockIdx.z * a.cx;
  const ElStream none{};
  el2_tile<R, PASS, GUARD, false, C::NO>(maps, a, none, sm.ring, sm.opr, sm.ofull, sm.oempty, sm.wprog,
                                  blockIdx.y * C::TY, blockIdx.x * C::TZ, x0,
                                  min(x0 + a.cx, a.x_hi), 0, 0);
}

// The full step (v sweep, then tau sweep) as ONE launch, the two sweeps
// streaming through L2 behind each other -- the reference's wavefront over
// the two half steps (schedule.py:81-90: tau follows v with an offset of R),
// with B200's L2 in the role of the CPU's last-level cache.
//
// CTAs [0, nv) run the v sweep, CTAs [nv, nv + nt) the tau sweep, each CTA
// taking tiles rank, rank + n_role, ... and streaming the whole x extent per
// tile.  The tau tiling is shifted by -R rows in y, so a tau tile only
// overwrites stress rows no later v tile reads, and it trails the v tiles it
// depends on by R planes in x plus the publish granularity: what the v sweep
// read (six stresses) and wrote (three velocities) a few microseconds earlier
// is what the tau sweep reads next, out of L2.  DRAM then sees ~84 B per point
// per step (each field read and written once, three materials) instead of the
// two launches' 120 B.
//
// v tiles never wait on anything but a bounded throttle, and they are the
// lower block indices, so the dependency waits of the tau role cannot
// deadlock whatever the residency of the grid.
// operand slots per sweep in the streamed launch: with half the SMs per sweep
// a deeper TMA pipeline per SM keeps the sweep fed (1024^3: 3 slots 33.0 ms,
// 5 slots 29.0 ms, 6 slots 29.1 ms; the two launches: 24.6 ms)
constexpr int kSNOv = 5, kSNOt = 5;

template <int R, bool GUARD>
__global__ void __launch_bounds__(El2Cfg<R, 0>::NT + 32, 1)
elastic_stream(const __grid_constant__ El2Maps mv, const __grid_constant__ El2Maps mt,
               const __grid_constant__ ElTiledArgs av, const __grid_constant__ ElTiledArgs at,
               const __grid_constant__ ElStream sc) {
  static_assert(El2Cfg<R, 0>::NT == El2Cfg<R, 1>::NT, "both roles share the thread layout");
  static_assert(2 * R <= El2Cfg<R, 0>::TY, "tau rows shifted by R stay clear of the next v row");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const bool tau = (int)blockIdx.x >= sc.nv;
  const int rank = tau ? (int)blockIdx.x - sc.nv : (int)blockIdx.x;
  const int N = (av.x_hi - av.x_lo) + 2 * R;         // iterations per tile
  int g0 = 0;
  if (!tau) {
    using C = El2Cfg<R, 0, kSNOv>;
    El2Smem<R, 0, kSNOv> sm(smem_raw);
    for (int t = rank; t < sc.tiles_yv * sc.tiles_z; t += sc.nv, g0 += N) {
      sm.init(g0 == 0);
      el2_tile<R, 0, GUARD, true, kSNOv>(mv, av, sc, sm.ring, sm.opr, sm.ofull, sm.oempty, sm.wprog,
                                  (t / sc.tiles_z) * C::TY, (t % sc.tiles_z) * C::TZ, av.x_lo,
                                  av.x_hi, t, g0);
      __syncthreads();
    }
  } else {
    using C = El2Cfg<R, 1, kSNOt>;
    El2Smem<R, 1, kSNOt> sm(smem_raw);
    for (int t = rank; t < sc.tiles_yt * sc.tiles_z; t += sc.nt, g0 += N) {
      sm.init(g0 == 0);
      el2_tile<R, 1, GUARD, true, kSNOt>(mt, at, sc, sm.ring, sm.opr, sm.ofull, sm.oempty, sm.wprog,
                                  (t / sc.tiles_z) * C::TY - R, (t % sc.tiles_z) * C::TZ, at.x_lo,
                                  at.x_hi, t, g0);
      __syncthreads();
    }
  }
}

}  // namespace
}  // namespace stb
