// Wavefront temporal blocking with warp-specialised levels (LV = 2), and
// the same machinery for a single level (LV = 1, measured slower than
// acoustic_fused<R, 1>; kept behind STB_WTB1).
//
// The paper's wavefront schedule (Alg. 6, schedule.py:171-310) with
// time-tile height 2, carried to one SM.  A CTA owns a TY x 64 (y, z) output
// tile and an x chunk and sweeps x once.  It produces u[t] and u[t+1] from
// one read of u[t-1], u[t-2] and inv: 20 B per point per two steps instead
// of 2 x 16 B.  Level 2 lags level 1 by R planes (the skew of
// schedule.py:139-168).  Level 1 is computed on the tile widened by H1 rows
// (R rounded up to RY) and round_up4(R) columns: overlapped tiling, so the
// halo is recomputed, never exchanged.  The inspector turned off-grid
// sources into per-thread entry lists, so injection happens inside the sweep
// right after each level's update.  That removes the dependency that blocks
// temporal blocking with off-grid sources (precompute.py:209-252).
//
// Unlike acoustic_fused<R, 2>, where the same threads compute both levels
// and level 2 idles the halo threads behind a CTA barrier per plane, the
// levels run on separate warp groups:
//
//   producer warp  TMA of the u[t-1] plane (level-1 region + R rows, OOB zero
//                  fill) into an NS1-slot ring.  Per iteration it also loads
//                  the u[t-2]/inv boxes of level 1 and the u[t-1]/inv boxes
//                  of level 2 into an NSB-slot ring, all on one transaction
//                  mbarrier.
//   level-1 warps  Register queue of their own u[t-1] columns (x
//                  neighbours), y/z neighbours from the staged plane.  Each
//                  plane goes first to a shared ring of NL level-1 planes
//                  (full/empty mbarriers per slot), then to HBM (owned
//                  points).
//   level-2 warps  Register queue of their level-1 columns read from that
//                  ring, y/z neighbours from the ring; result to HBM.
//                  (Letting only these warps release the producer's slots
//                  -- their progress implies level 1's -- measured -2 %.)
//
// Both groups run ONE role-parameterised code body.  Their rings share the
// row stride, so shared addressing stays static.  Separate 9-way-unrolled
// bodies (147 KB of SASS) stalled on instruction fetch.
//
// Each thread owns RY consecutive y rows x 4 consecutive z points.  The y
// neighbours of its rows are loaded once (RY + 2R rows per RY x 4 points),
// and the centre rows come from its queue.  With RY = 2 a level update
// costs 10 (level 1) / 9 (level 2) LDS.128 per 4 points, against 14 in the
// K = 1 kernel.
//
// Arithmetic: the reference's IEEE operation order (physics.py:199-213) on
// packed fp32 pairs: sums as FADD2, exact products as FFMA2 with an opaque
// -0 addend (see f32x2.cuh).  FAST contracts the Laplacian terms into FFMA2.
// Measured numbers and profile: DESIGN.md §6.
#pragma once

#include "acoustic_fused.cuh"

// consumer-side barrier waits: plain try_wait spin (STB_WTB_SLEEP=1: with the
// suspend-time hint)
#if defined(STB_WTB_SLEEP) && STB_WTB_SLEEP
#define STB_WTB_WAIT mbar_wait_sleep
#else
#define STB_WTB_WAIT mbar_wait
#endif

namespace stb {

template <int R, int LV, int RY, int PF, int TY_ = 16>
struct WtbCfg {
  static_assert(LV == 1 || LV == 2, "one or two levels per sweep");
  static constexpr int TY = TY_, TZ = 64;
  static constexpr int RP = kRoundUp4(R);
  // level-1 y halo: R rows, rounded up so a thread's rows are all inside
  // or all outside the tile
  static constexpr int H1 = LV == 2 ? (R + RY - 1) / RY * RY : 0;
  static constexpr int HZ1 = LV == 2 ? RP : 0;        // level-1 z halo (float4 aligned)
  static constexpr int HZ0 = kRoundUp4(HZ1 + R);      // staged u[t-1] z halo
  static constexpr int HY1 = TY + 2 * H1, WZ1 = TZ + 2 * HZ1;
  static constexpr int HY0 = HY1 + 2 * R, WZ0 = TZ + 2 * HZ0;
  static_assert(HY1 % RY == 0 && TY % RY == 0 && H1 % RY == 0,
                "rows per thread must tile the regions");
  static constexpr int G1 = WZ1 / 4, G2 = TZ / 4;
  static constexpr int NW1T = (HY1 / RY) * G1;        // level-1 work threads
  static constexpr int NW2T = LV == 2 ? (TY / RY) * G2 : 0;   // level-2 work threads
  static constexpr int NTHR = NW1T + NW2T;            // per-tile thread slots (source lists)
  static constexpr int NW1 = (NW1T + 31) / 32, NW2 = (NW2T + 31) / 32;
  static constexpr int NT = 32 * (1 + NW1 + NW2);
  // per-thread register cap for one CTA per SM: registers are allocated for
  // whole 4-warp groups (a 288-thread CTA is charged as 384 threads)
  static constexpr int NTA = (NT + 127) / 128 * 128;
  static constexpr int MAXREG = (65536 / NTA) / 8 * 8 > 255 ? 255 : (65536 / NTA) / 8 * 8;
  static constexpr int Q = 2 * R + 1;
  static constexpr int NSB = PF + 1;                  // iteration ring (aux boxes, barriers)
  static constexpr int NS1 = R + NSB;                 // staged u[t-1] planes
  static constexpr int NL = LV == 2 ? R + 2 : 0;      // level-1 plane ring
  static constexpr int E0 = HY0 * WZ0, E1 = HY1 * WZ1;
  static_assert(E0 % 32 == 0 && E1 % 32 == 0 && (TY * WZ1) % 32 == 0 && (HY1 * WZ0) % 4 == 0,
                "TMA destinations must stay 128-byte aligned");
  static constexpr int ET = TY * WZ1;                 // level-2 aux boxes: tile rows, WZ1 wide
  static constexpr int EL = HY1 * WZ0;                // level-1 ring plane (row stride WZ0)
  // u[t-2], inv (level 1); u[t-1], inv (level 2)
  static constexpr int AUX = 2 * E1 + (LV == 2 ? 2 * ET : 0);
  static constexpr int MAXN = 1024;                   // planes per CTA sweep (x chunk + 2 LV R)
  static constexpr size_t RING1 = (size_t)NS1 * E0 * 4;
  static constexpr size_t RING2 = (size_t)NSB * AUX * 4;
  static constexpr size_t LBUF = (size_t)NL * EL * 4;
  static constexpr size_t FXS = (size_t)MAXN * 4;
  static constexpr size_t BARS = (size_t)(2 * NSB + 2 * NL) * 8;
  static constexpr size_t SMEM = RING1 + RING2 + LBUF + FXS + BARS;
  static_assert(SMEM <= 232448, "shared memory budget");
};

struct WtbMaps {
  CUtensorMap l0;     // u[t-1], box WZ0 x HY0 (level-1 input plane)
  CUtensorMap lm1;    // u[t-2], box WZ1 x HY1
  CUtensorMap c1;     // u[t-1], box WZ1 x TY (level-2 "u0")
  CUtensorMap inv1;   // inv, box WZ1 x HY1
  CUtensorMap inv2;   // inv, box WZ1 x TY
};

// RY rows x 4 z points.  xq: register queue (centre slot cs); cen: the
// thread's row-0 centre in a shared plane of row stride W.
template <bool FAST, int R, int Q, int RY, int W>
__device__ __forceinline__ void wtb_update(const float (&xq)[Q][RY][4], const int cs,
                                           const float* cen, const float (&u0)[RY][4],
                                           const float (&iv)[RY][4], const float (&fac)[RY][4],
                                           const TiledCoefs& cf, float (&o)[RY][4]) {
  const f2 nz = bcast(cf.nz);
  // y rows d in [-R, RY + R): centre rows from the queue, the rest from smem
  float yr[RY + 2 * R][4];
#pragma unroll
  for (int d = -R; d < RY + R; ++d) {
    if (d >= 0 && d < RY) {
#pragma unroll
      for (int i = 0; i < 4; ++i) yr[d + R][i] = xq[cs][d][i];
    } else {
      const float4 v = *reinterpret_cast<const float4*>(cen + d * W);
      yr[d + R][0] = v.x; yr[d + R][1] = v.y; yr[d + R][2] = v.z; yr[d + R][3] = v.w;
    }
  }
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    const f2 c01 = pk(xq[cs][r][0], xq[cs][r][1]);
    const f2 c23 = pk(xq[cs][r][2], xq[cs][r][3]);
    f2 L01, L23;
    if constexpr (FAST) {
      L01 = mul2(c01, bcast(cf.c0));
      L23 = mul2(c23, bcast(cf.c0));
    } else {
      L01 = xmul2(c01, bcast(cf.c0), nz);
      L23 = xmul2(c23, bcast(cf.c0), nz);
    }
    // x neighbours (axis 0 first, r ascending -- the reference's term order)
#pragma unroll
    for (int k = 1; k <= R; ++k) {
      const int sp = (cs + k) % Q, sm = (cs - k + Q) % Q;
      L01 = term2<FAST>(L01, pk(xq[sp][r][0], xq[sp][r][1]), pk(xq[sm][r][0], xq[sm][r][1]),
                        cf.cx[k - 1], nz);
      L23 = term2<FAST>(L23, pk(xq[sp][r][2], xq[sp][r][3]), pk(xq[sm][r][2], xq[sm][r][3]),
                        cf.cx[k - 1], nz);
    }
    // y neighbours
#pragma unroll
    for (int k = 1; k <= R; ++k) {
      const float* pp = yr[r + k + R];
      const float* mm = yr[r - k + R];
      L01 = term2<FAST>(L01, pk(pp[0], pp[1]), pk(mm[0], mm[1]), cf.cy[k - 1], nz);
      L23 = term2<FAST>(L23, pk(pp[2], pp[3]), pk(mm[2], mm[3]), cf.cy[k - 1], nz);
    }
    // z neighbours: window [z - R, z + 4 + R), centre from the queue
    float win[4 + 2 * R];
    const float* cr = cen + r * W;
    {
      // left part [-R, 0): scalar / float2 heads up to 16-byte alignment
      int d = -R;
      if (d & 1) {
        win[d + R] = cr[d];
        d += 1;
      }
      if (((d % 4) + 4) % 4 == 2) {
        const float2 v = *reinterpret_cast<const float2*>(cr + d);
        win[d + R] = v.x; win[d + R + 1] = v.y;
        d += 2;
      }
#pragma unroll
      for (; d < 0; d += 4) {
        const float4 v = *reinterpret_cast<const float4*>(cr + d);
        win[d + R] = v.x; win[d + R + 1] = v.y; win[d + R + 2] = v.z; win[d + R + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) win[R + i] = xq[cs][r][i];
      // right part [4, 4 + R): float4 body, float2 / scalar tails
      d = 4;
#pragma unroll
      for (; d + 4 <= 4 + R; d += 4) {
        const float4 v = *reinterpret_cast<const float4*>(cr + d);
        win[d + R] = v.x; win[d + R + 1] = v.y; win[d + R + 2] = v.z; win[d + R + 3] = v.w;
      }
      if (d + 2 <= 4 + R) {
        const float2 v = *reinterpret_cast<const float2*>(cr + d);
        win[d + R] = v.x; win[d + R + 1] = v.y;
        d += 2;
      }
      if (d < 4 + R) win[d + R] = cr[d];
    }
#pragma unroll
    for (int k = 1; k <= R; ++k) {
      if ((R + k) % 2 == 0) {
        L01 = term2<FAST>(L01, pk(win[R + k], win[R + k + 1]), pk(win[R - k], win[R - k + 1]),
                          cf.cz[k - 1], nz);
        L23 = term2<FAST>(L23, pk(win[R + k + 2], win[R + k + 3]),
                          pk(win[R - k + 2], win[R - k + 3]), cf.cz[k - 1], nz);
      } else {
        L01 = term2s<FAST>(L01, win[R + k], win[R - k], win[R + k + 1], win[R - k + 1],
                           cf.cz[k - 1], nz);
        L23 = term2s<FAST>(L23, win[R + k + 2], win[R - k + 2], win[R + k + 3],
                           win[R - k + 3], cf.cz[k - 1], nz);
      }
    }
    // epilogue: o = ((c*2 - u0) + lap*inv) * fac   (c*2 == c+c exactly)
    f2 v01 = sub2(add2(c01, c01), pk(u0[r][0], u0[r][1]));
    f2 v23 = sub2(add2(c23, c23), pk(u0[r][2], u0[r][3]));
    if constexpr (FAST) {
      v01 = fma2(L01, pk(iv[r][0], iv[r][1]), v01);
      v23 = fma2(L23, pk(iv[r][2], iv[r][3]), v23);
    } else {
      v01 = add2(v01, xmul2(L01, pk(iv[r][0], iv[r][1]), nz));
      v23 = add2(v23, xmul2(L23, pk(iv[r][2], iv[r][3]), nz));
    }
    v01 = xmul2(v01, pk(fac[r][0], fac[r][1]), nz);
    v23 = xmul2(v23, pk(fac[r][2], fac[r][3]), nz);
    upk(v01, o[r][0], o[r][1]);
    upk(v23, o[r][2], o[r][3]);
  }
}

template <int RY>
__device__ __forceinline__ void ld_rows(float (&dst)[RY][4], const float* src, int stride) {
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    const float4 v = *reinterpret_cast<const float4*>(src + r * stride);
    dst[r][0] = v.x; dst[r][1] = v.y; dst[r][2] = v.z; dst[r][3] = v.w;
  }
}

// Per-thread state of one level group: geometry, damping, source window.
template <int RY>
struct WtbLane {
  int y, z;                 // first row / first z point
  bool zdom[RY][4];
  float fyz[RY][4];
  bool own[RY];             // row inside the output tile and the grid
  int wk;                   // source window: (x << 3) | (row << 2) | lane
  float wv;
  int cur, e_end;
  int bad;

  __device__ __forceinline__ void init(const FusedArgs& a, bool work, int y_, int z_,
                                       bool in_tile) {
    y = y_;
    z = z_;
    bad = 0;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const bool ydom = work && y + r >= 0 && y + r < a.d.ny;
      own[r] = in_tile && ydom && z < a.d.nz;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        zdom[r][i] = ydom && (z + i >= 0) && (z + i < a.d.nz);
        fyz[r][i] = zdom[r][i] ? tmin(__ldg(a.fy + y + r), __ldg(a.fz + z + i)) : 1.0f;
      }
    }
  }
  __device__ __forceinline__ void fetch(const FusedArgs& a, int level) {
    if (cur < e_end) {
      const int2 e = __ldg(a.thr_list + cur);
      wk = (e.x << 3) | (e.y & 7);
      wv = __ldg(a.series + (size_t)(a.t0 + level - 1) * a.n_src + (e.y >> 3));
    } else {
      wk = 0x7fffffff;
      wv = 0.f;
    }
    ++cur;
  }
  // entry list of this thread slot; entries before plane pfirst are skipped
  __device__ __forceinline__ void src_init(const FusedArgs& a, bool work, int slot, int pfirst,
                                           int level) {
    wk = 0x7fffffff;
    wv = 0.f;
    cur = e_end = 0;
    if (a.thr_list == nullptr || !work) return;
    cur = __ldg(a.thr_ptr + slot);
    e_end = __ldg(a.thr_ptr + slot + 1);
    while (cur < e_end && __ldg(&a.thr_list[cur].x) < pfirst) ++cur;
    fetch(a, level);
  }
  // NaN guard (on the stencil result, as the reference's check sees it), then
  // fused injection from the window
  template <bool GUARD>
  __device__ __forceinline__ void epilogue(const FusedArgs& a, float (&o)[RY][4], int level,
                                           int p, int x0, int x1, bool active) {
    if constexpr (GUARD) {
      if ((a.guard_mask & (1 << (level - 1))) && p >= x0 && p < x1 && p >= 0 && p < a.d.nx) {
#pragma unroll
        for (int r = 0; r < RY; ++r)
          if (own[r])
#pragma unroll
            for (int i = 0; i < 4; ++i) bad |= (zdom[r][i] && !isfinite(o[r][i]));
      }
    }
    while ((wk >> 3) == p) {
      if (active) {
#pragma unroll
        for (int r = 0; r < RY; ++r)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (r * 4 + i == (wk & 7)) o[r][i] = __fadd_rn(o[r][i], wv);
      }
      fetch(a, level);
    }
  }
  __device__ __forceinline__ void store(const FusedArgs& a, float* gb, const float (&o)[RY][4],
                                        int p) const {
    float* base = gb + (int64_t)p * a.d.plane;
#pragma unroll
    for (int r = 0; r < RY; ++r)
      if (own[r])
        *reinterpret_cast<float4*>(base + (int64_t)r * a.d.pitch) =
            make_float4(o[r][0], o[r][1], o[r][2], o[r][3]);
  }
};

template <int R, int LV, int RY, int PF, int TY_, bool FAST, bool GUARD>
__global__ void __maxnreg__((WtbCfg<R, LV, RY, PF, TY_>::MAXREG))
acoustic_wtb(const __grid_constant__ WtbMaps maps, const __grid_constant__ FusedArgs a) {
  using C = WtbCfg<R, LV, RY, PF, TY_>;
  constexpr int TY = C::TY, TZ = C::TZ, Q = C::Q, W = C::WZ0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* ring1 = reinterpret_cast<float*>(smem_raw);
  float* ring2 = reinterpret_cast<float*>(smem_raw + C::RING1);
  float* lbuf = reinterpret_cast<float*>(smem_raw + C::RING1 + C::RING2);
  float* fxs = reinterpret_cast<float*>(smem_raw + C::RING1 + C::RING2 + C::LBUF);
  uint64_t* full =
      reinterpret_cast<uint64_t*>(smem_raw + C::RING1 + C::RING2 + C::LBUF + C::FXS);
  uint64_t* done = full + C::NSB;
  uint64_t* lfull = done + C::NSB;
  uint64_t* lempty = lfull + C::NL;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int tile = blockIdx.x;
  const int y0 = (tile / a.ntz) * TY;
  const int z0 = (tile % a.ntz) * TZ;
  const int x0 = a.x_lo + blockIdx.y * a.cx_len;
  const int x1 = min(x0 + a.cx_len, a.x_hi);
  const int N = (x1 - x0) + 2 * LV * R;
  const int ibase = x0 - LV * R;
  const int pofs1 = x0 - (LV + 1) * R;          // level-1 plane of loop counter c: c + pofs1

  // damping x factors of the planes this CTA touches: fxs[j] = fx(pofs1 + j)
  for (int j = tid; j < N; j += blockDim.x)
    fxs[j] = __ldg(a.fx + min(max(pofs1 + j, 0), (int)a.d.nx - 1));
  if (tid == 0) {
    for (int s = 0; s < C::NSB; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], C::NW1 + C::NW2);
    }
    for (int s = 0; s < C::NL; ++s) {
      mbar_init(&lfull[s], C::NW1 * 32);
      mbar_init(&lempty[s], C::NW2);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const bool use_inv = a.use_inv != 0;

  // ------------------------------------------------------------ producer warp
  if (warp == C::NW1 + C::NW2) {
    if (lane == 0) {
      prefetch_map(&maps.l0);
      prefetch_map(&maps.lm1);
      if (LV == 2) prefetch_map(&maps.c1);
      for (int n = 0; n < N; ++n) {
        const int sb = n % C::NSB;
        if (n >= C::NSB) mbar_wait_sleep(&done[sb], (uint32_t)(((n / C::NSB) - 1) & 1));
        uint32_t bytes = (uint32_t)C::E0 * 4u;
        if (n >= 2 * R) bytes += (uint32_t)C::E1 * (use_inv ? 8u : 4u);
        if (LV == 2 && n >= 4 * R) bytes += (uint32_t)C::ET * (use_inv ? 8u : 4u);
        mbar_arrive_expect_tx(&full[sb], bytes);
        tma_load_3d(ring1 + (size_t)(n % C::NS1) * C::E0, &maps.l0, z0 - C::HZ0,
                    y0 - C::H1 - R, ibase + n, &full[sb]);
        float* ab = ring2 + (size_t)sb * C::AUX;
        if (n >= 2 * R) {
          tma_load_3d(ab, &maps.lm1, z0 - C::HZ1, y0 - C::H1, ibase + n - R, &full[sb]);
          if (use_inv)
            tma_load_3d(ab + C::E1, &maps.inv1, z0 - C::HZ1, y0 - C::H1, ibase + n - R,
                        &full[sb]);
        }
        if (LV == 2 && n >= 4 * R) {
          tma_load_3d(ab + 2 * C::E1, &maps.c1, z0 - C::HZ1, y0, ibase + n - 2 * R, &full[sb]);
          if (use_inv)
            tma_load_3d(ab + 2 * C::E1 + C::ET, &maps.inv2, z0 - C::HZ1, y0, ibase + n - 2 * R,
                        &full[sb]);
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------ level warps
  // Both levels run the same code (one copy in the instruction cache) on
  // role-specific bases: level 1 reads the staged u[t-1] ring, level 2 the
  // level-1 ring; both rings have row stride W, so all addressing inside
  // the update is static.  Loop counter c: level 1 = iteration n, level 2 =
  // level-1 plane m = n - 2R; both push plane c into queue slot c % Q and
  // compute plane c - R once c >= 2R.
  const bool r1 = warp < C::NW1;
  const int t = r1 ? tid : tid - C::NW1 * 32;
  const bool work = t < (r1 ? C::NW1T : C::NW2T);
  const int gw = r1 ? C::G1 : C::G2;
  const int row = work ? (t / gw) * RY : 0;
  const int g = work ? t % gw : 0;
  const int ylo = r1 ? y0 - C::H1 + row : y0 + row;
  const int zlo = r1 ? z0 - C::HZ1 + 4 * g : z0 + 4 * g;
  // level 1: rows of a thread are all in or all out of the tile (H1, TY multiples of RY)
  const bool in_tile =
      !r1 || (row >= C::H1 && row < C::H1 + TY && 4 * g >= C::HZ1 && 4 * g < C::HZ1 + TZ);
  WtbLane<RY> L;
  L.init(a, work, ylo, zlo, in_tile);
  const int level = r1 ? 1 : 2;
  L.src_init(a, work, tile * C::NTHR + (r1 ? t : C::NW1T + t), r1 ? x0 - (LV - 1) * R : x0, level);
  // CTA-uniform: does the level-1 region leave the grid?  Interior CTAs skip
  // the zero-halo masking.  (One level: nothing reads values outside the
  // grid, and they are never stored.)
  const bool edge = LV == 2 && ((y0 - C::H1 < 0) || (y0 + TY + C::H1 > a.d.ny) ||
                                (z0 - C::HZ1 < 0) || (z0 + TZ + C::HZ1 > a.d.nz));

  const int cnt = r1 ? N : N - 2 * R;
  const int noff = r1 ? 0 : 2 * R;
  const int pofs = r1 ? pofs1 : x0 - 2 * R;
  const int fxo = r1 ? 0 : R;
  const int NS = r1 ? C::NS1 : C::NL;
  const int ES = r1 ? C::E0 : C::EL;
  const float* pring = r1 ? ring1 : lbuf;
  const int offP =
      r1 ? (row + R) * W + 4 * g + (C::HZ0 - C::HZ1) : (row + C::H1) * W + 4 * g + C::HZ1;
  const int offA = r1 ? row * C::WZ1 + 4 * g : 2 * C::E1 + row * C::WZ1 + 4 * g + C::HZ1;
  const int invA = r1 ? C::E1 : C::ET;
  // this thread's (y, z) column in the output level; plane offsets added per store
  float* dst = ((r1 && LV == 2) ? a.out_km1 : a.out_k) + ((int64_t)ylo * a.d.pitch + zlo);
  const int offW = row * W + 4 * g;              // level 1: own point in the level-1 ring

  float q[Q][RY][4];
#pragma unroll
  for (int s = 0; s < Q; ++s)
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i) q[s][r][i] = 0.f;

  int ps = 0, pph = 0;        // c % NS (push slot) and, for level 2, the lfull phase
  int ys = NS - R;            // (c - R) % NS
  int ls = 0, lph = 0;        // level 1: (c - 2R) % NL and its phase

  // level 2 starts at iteration 2R; it still releases iterations 0..2R-1
  // (after their TMA completed, so the arrivals land in the right phase)
  if (LV == 2 && !r1) {
    for (int n = 0; n < 2 * R; ++n) {
      mbar_wait_sleep(&full[n % C::NSB], (uint32_t)((n / C::NSB) & 1));
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[n % C::NSB]);
    }
  }

  for (int nb = 0; nb < cnt; nb += Q) {
#pragma unroll
    for (int qq = 0; qq < Q; ++qq) {
      const int c = nb + qq;
      if (c < cnt) {
        const unsigned un = (unsigned)(c + noff);
        const int sb = (int)(un % C::NSB);
        STB_WTB_WAIT(&full[sb], (uint32_t)((un / C::NSB) & 1u));
        if (!r1) STB_WTB_WAIT(&lfull[ps], (uint32_t)pph);
        if (work) ld_rows<RY>(q[qq], pring + ps * ES + offP, W);
        if (c >= 2 * R) {
          const int p = c + pofs;
          const int cs = (qq - R + Q) % Q;
          float o[RY][4];
#pragma unroll
          for (int r = 0; r < RY; ++r)
#pragma unroll
            for (int i = 0; i < 4; ++i) o[r][i] = 0.f;
          if (work) {
            const float* aux = ring2 + (size_t)sb * C::AUX + offA;
            float u0[RY][4], iv[RY][4], fac[RY][4];
            ld_rows<RY>(u0, aux, C::WZ1);
            if (use_inv) {
              ld_rows<RY>(iv, aux + invA, C::WZ1);
            } else {
#pragma unroll
              for (int r = 0; r < RY; ++r)
#pragma unroll
                for (int i = 0; i < 4; ++i) iv[r][i] = a.inv_scalar;
            }
            const float fxx = fxs[c + fxo];
#pragma unroll
            for (int r = 0; r < RY; ++r)
#pragma unroll
              for (int i = 0; i < 4; ++i) fac[r][i] = tmin(fxx, L.fyz[r][i]);
            wtb_update<FAST, R, Q, RY, W>(q, cs, pring + ys * ES + offP, u0, iv, fac, a.cf, o);
            // zero halo: planes outside the grid (uniform), points outside
            // the y/z extent (edge CTAs only)
            const bool live = (p >= 0 && p < a.d.nx) || (p < 0 ? !a.zero_lo : !a.zero_hi);
            if (edge || !live) {
#pragma unroll
              for (int r = 0; r < RY; ++r)
#pragma unroll
                for (int i = 0; i < 4; ++i) o[r][i] = (live && L.zdom[r][i]) ? o[r][i] : 0.f;
            }
          }
          L.template epilogue<GUARD>(a, o, level, p, x0, x1, work);
          if (LV == 2 && r1) {
            // hand the plane to level 2 first (its warps wait on it), then
            // the fire-and-forget HBM store
            if (c - 2 * R >= C::NL) STB_WTB_WAIT(&lempty[ls], (uint32_t)(lph ^ 1));
            if (work) {
              float* lb = lbuf + ls * C::EL + offW;
#pragma unroll
              for (int r = 0; r < RY; ++r)
                *reinterpret_cast<float4*>(lb + r * W) =
                    make_float4(o[r][0], o[r][1], o[r][2], o[r][3]);
            }
            mbar_arrive(&lfull[ls]);
            if (++ls == C::NL) { ls = 0; lph ^= 1; }
          }
          if (p >= x0 && p < x1) L.store(a, dst, o, p);
        }
        if (!r1 && c >= R) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&lempty[ys]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[sb]);
        if (++ps == NS) { ps = 0; pph ^= 1; }
        if (++ys == NS) ys = 0;
      }
    }
  }
  if constexpr (GUARD) {
    if (__any_sync(0xffffffffu, L.bad) && lane == 0) atomicExch(a.nonfinite, 1);
  }
}

template <int R, int LV, int RY, int PF, int TY_, bool FAST>
struct WtbLauncher {
  using C = WtbCfg<R, LV, RY, PF, TY_>;
  template <bool GUARD>
  static void launch_g(cudaStream_t st, const WtbMaps& maps, const FusedArgs& a, int nchunks) {
    static std::atomic<uint64_t> configured{0};
    if (first_use_on_device(configured))
      STB_CUDA(cudaFuncSetAttribute(acoustic_wtb<R, LV, RY, PF, TY_, FAST, GUARD>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    const int nty = (int)((a.d.ny + C::TY - 1) / C::TY);
    dim3 grid((unsigned)(a.ntz * nty), (unsigned)nchunks);
    acoustic_wtb<R, LV, RY, PF, TY_, FAST, GUARD><<<grid, C::NT, C::SMEM, st>>>(maps, a);
    STB_CHECK_LAUNCH();
  }
  static void launch(cudaStream_t st, const WtbMaps& maps, const FusedArgs& a, int nchunks) {
    if (nchunks <= 0) return;
    if (a.guard_mask && a.nonfinite)
      launch_g<true>(st, maps, a, nchunks);
    else
      launch_g<false>(st, maps, a, nchunks);
  }
};

}  // namespace stb
