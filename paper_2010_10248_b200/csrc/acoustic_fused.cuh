// Temporally blocked acoustic kernel: K time steps fused per HBM pass.
//
// The paper's wavefront temporal blocking (Alg. 6, schedule.py
// 171-310) carried to a B200 SM: each CTA owns an output tile TY x TZ in
// (y, z) and an x chunk, and sweeps x once while computing all K time levels
// in a pipeline.  Level j (1..K) lags level j-1 by R planes (the skew of
// schedule.py:139-168) and is computed on the tile widened by (K-j)*R in y/z
// (overlapped tiling; halo values are recomputed, never exchanged).  Because
// the inspector turned off-grid sources into per-tile entry lists, injection
// is applied inside the sweep right after each level's update -- the
// dependency that forbids temporal blocking with off-grid sources is gone.
//
// Dataflow per iteration n (input plane i = x0 - K*R + n):
//   producer warp : waits until iteration n-NSB is done, then TMA-loads the
//                   u[t-1] plane i (tile + K*R halo, OOB zero-fill) into a
//                   ring of R+NSB slots and the u[t-2] / inv boxes into an
//                   NSB ring, all on one transaction mbarrier.
//   consumers     : q0 <- own 4 z-points of plane i (register queue = x nbrs)
//                   level 1 at plane i-R: y/z nbrs from the staged plane
//                   level j>1 at plane i-jR: queue centre -> smem buffer,
//                   named barrier, y/z nbrs from the buffer, x nbrs from the
//                   level j-1 queue, u[t+j-3] centre = oldest level j-2 entry;
//                   one "done" arrival per warp per iteration.
// Points outside the grid are forced to +0 at every level (the reference's
// zero halo), so overlapped halos are exact.  Only the last two levels are
// written to HBM (20 B/pt per K-step block in fp32; 16 B/pt for K = 1).
//
// Arithmetic runs on packed fp32 pairs (FADD2/FMUL2/FFMA2).  EXACT mode
// keeps the reference's IEEE operation order (physics.py:199-213): sums and
// differences packed, products as scalar FMULs (see f32x2.cuh) -> bitwise
// equal to stencil_tb.  FAST mode accumulates the Laplacian with FFMA2 (one
// rounding per term instead of two); tests bound it at 1e-5 relative L2.
#pragma once

#include "acoustic_kernels.cuh"
#include "f32x2.cuh"
#include "fp_exact.cuh"
#include "tma.cuh"

namespace stb {

constexpr int kRoundUp4(int v) { return (v + 3) / 4 * 4; }

// Stencil coefficients of the fp32 sweep kernels, rounded once to fp32 as
// NumPy's weak-scalar rule rounds the Python floats (physics.py:158-164).
struct TiledCoefs {
  float c0;
  float cx[8], cy[8], cz[8];
  float nz;     // -0.0f, a runtime value on purpose (see xmul2 in f32x2.cuh)
};

template <int R, int K, int TY, int TZ, int PF>
struct FusedCfg {
  static constexpr int hy(int j) { return (K - j) * R; }
  static constexpr int hz(int j) { return j >= K ? 0 : kRoundUp4(hz(j + 1) + R); }
  static constexpr int RP = kRoundUp4(R);
  static constexpr int TY_ = TY;
  static constexpr int HY0 = TY + 2 * hy(0), WZ0 = TZ + 2 * hz(0);   // staged u[t-1]
  static constexpr int HY1 = TY + 2 * hy(1), WZ1 = TZ + 2 * hz(1);   // thread grid
  static constexpr int G1 = WZ1 / 4;
  static constexpr int NWORK = HY1 * G1;
  static constexpr int NTC = (NWORK + 31) / 32 * 32;
  static constexpr int NT = NTC + 32;
  static constexpr int NCW = NTC / 32;
  static constexpr int Q = 2 * R + 1;
  static constexpr int NSB = PF + 1;                  // iteration ring (barriers, aux)
  static constexpr int NS1 = R + NSB;                 // staged u[t-1] planes
  static constexpr int E0 = HY0 * WZ0;
  static constexpr int E1 = HY1 * WZ1;
  // TMA destinations start 128-byte aligned: slots and boxes padded to 32 floats
  static constexpr int pad32(int v) { return (v + 31) / 32 * 32; }
  static constexpr int E0S = pad32(E0);
  static constexpr int ebox(int j) { return (TY + 2 * hy(j)) * (TZ + 2 * hz(j)); }
  static constexpr int aux_floats() {
    int s = pad32(E1);
    for (int j = 1; j <= K; ++j) s += pad32(ebox(j));
    return s;
  }
  static constexpr int AUX = aux_floats();
  static constexpr int aux_inv_off(int j) {
    int s = pad32(E1);
    for (int jj = 1; jj < j; ++jj) s += pad32(ebox(jj));
    return s;
  }
  static constexpr int NBUF = K > 1 ? (K - 1) : 0;
  static constexpr size_t RING1 = (size_t)NS1 * E0S * 4;
  static constexpr size_t RING2 = (size_t)NSB * AUX * 4;
  static constexpr size_t BUFS = (size_t)NBUF * 2 * E1 * 4;
  static constexpr size_t BARS = (size_t)(2 * NSB) * 8;
  static constexpr size_t SMEM = RING1 + RING2 + BUFS + BARS;
  // resident CTAs per SM the launch bounds ask for: two for the 9-warp
  // K = 1 tiles (and the K = 2 R <= 2 kernel), one otherwise
  static constexpr int MINB = K == 1 ? (NT <= 320 && R <= 6 ? 2 : 1) : (R <= 2 ? 2 : 1);
};

struct FusedMaps {
  CUtensorMap l0;        // u[t-1], box WZ0 x HY0 x 1
  CUtensorMap lm1;       // u[t-2], box WZ1 x HY1 x 1
  CUtensorMap inv[4];    // inv, box of level j+1
};

struct FusedArgs {
  float* out_km1;        // level K-1 (u[t+K-2]), unused for K == 1
  float* out_k;          // level K   (u[t+K-1])
  const float* fx;
  const float* fy;
  const float* fz;
  float inv_scalar;
  int use_inv;
  TiledCoefs cf;
  Dims d;
  int cx_len, ntz;
  int x_lo, x_hi;        // planes swept by this launch: [x_lo, x_hi) in cx_len chunks
  int zero_lo, zero_hi;  // planes < 0 / >= nx are the reference's zero halo
  int t0;                // time step of level 1
  const int* thr_ptr;    // per (tile, consumer thread): range in thr_list
  const int2* thr_list;  // {x, id*4 + z lane}, x ascending per thread
  const float* series;   // (nt, n_src), pre-rounded to fp32
  int n_src;
  int* nonfinite;
  int guard_mask;        // bit j-1: step t0+j-1 is a guard step
  // x-slab halo exchange fused into the K = 1 sweep: owned planes p <
  // peer_lo_end (p >= peer_hi_begin) are also stored, over NVLink peer
  // memory, into the lower (upper) neighbour slab's ghost planes at its
  // local plane p + peer_lo_shift (p + peer_hi_shift).  NULL: no peer.
  float* peer_lo;
  float* peer_hi;
  int peer_lo_end, peer_hi_begin;
  int peer_lo_shift, peer_hi_shift;
};

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// One Laplacian term for two packed points: lap + (p + m) * c.
template <bool FAST>
__device__ __forceinline__ f2 term2(f2 lap, f2 p, f2 m, float c, f2 nz) {
  const f2 s = add2(p, m);
  if constexpr (FAST)
    return fma2(s, bcast(c), lap);
  else
    return add2(lap, xmul2(s, bcast(c), nz));
}

// Same term when the two sums come from scalars (odd z offsets, where the
// packed operands would straddle register pairs).
template <bool FAST>
__device__ __forceinline__ f2 term2s(f2 lap, float p0, float m0, float p1, float m1, float c,
                                     f2 nz) {
  const f2 s = pk(__fadd_rn(p0, m0), __fadd_rn(p1, m1));
  if constexpr (FAST)
    return fma2(s, bcast(c), lap);
  else
    return add2(lap, xmul2(s, bcast(c), nz));
}

// Update of 4 consecutive z points.  xq: register queue of the input level
// (centre slot cs); cen: shared-memory pointer to the thread's centre in the
// input plane (row stride W); u0/iv/fac per point.  Result in o (unmasked).
template <bool FAST, int R, int Q, int RP, int W>
__device__ __forceinline__ void update4(const float (&xq)[Q][4], const int cs, const float* cen,
                                        const float (&u0)[4], const float (&iv)[4],
                                        const float (&fac)[4], const TiledCoefs& cf,
                                        float (&o)[4]) {
  const f2 c01 = pk(xq[cs][0], xq[cs][1]);
  const f2 c23 = pk(xq[cs][2], xq[cs][3]);
  const f2 nz = bcast(cf.nz);
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
  for (int r = 1; r <= R; ++r) {
    const int sp = (cs + r) % Q, sm = (cs - r + Q) % Q;
    L01 = term2<FAST>(L01, pk(xq[sp][0], xq[sp][1]), pk(xq[sm][0], xq[sm][1]), cf.cx[r - 1], nz);
    L23 = term2<FAST>(L23, pk(xq[sp][2], xq[sp][3]), pk(xq[sm][2], xq[sm][3]), cf.cx[r - 1], nz);
  }
  // y neighbours
#pragma unroll
  for (int r = 1; r <= R; ++r) {
    const float4 pp = *reinterpret_cast<const float4*>(cen + r * W);
    const float4 mm = *reinterpret_cast<const float4*>(cen - r * W);
    L01 = term2<FAST>(L01, pk(pp.x, pp.y), pk(mm.x, mm.y), cf.cy[r - 1], nz);
    L23 = term2<FAST>(L23, pk(pp.z, pp.w), pk(mm.z, mm.w), cf.cy[r - 1], nz);
  }
  // z neighbours: window [z - RP, z + 4 + RP); only [z - R, z + 4 + R) is
  // loaded (8-byte heads/tails where R is not a multiple of 4) and the
  // centre comes from the queue
  float win[4 + 2 * RP];
  {
    int d = -R;
    if (d & 1) {
      win[RP + d] = cen[d];
      d += 1;
    }
    if (((d % 4) + 4) % 4 == 2) {
      const float2 v = *reinterpret_cast<const float2*>(cen + d);
      win[RP + d] = v.x; win[RP + d + 1] = v.y;
      d += 2;
    }
#pragma unroll
    for (; d < 0; d += 4) {
      const float4 v = *reinterpret_cast<const float4*>(cen + d);
      win[RP + d] = v.x; win[RP + d + 1] = v.y; win[RP + d + 2] = v.z; win[RP + d + 3] = v.w;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) win[RP + i] = xq[cs][i];
    d = 4;
#pragma unroll
    for (; d + 4 <= 4 + R; d += 4) {
      const float4 v = *reinterpret_cast<const float4*>(cen + d);
      win[RP + d] = v.x; win[RP + d + 1] = v.y; win[RP + d + 2] = v.z; win[RP + d + 3] = v.w;
    }
    if (d + 2 <= 4 + R) {
      const float2 v = *reinterpret_cast<const float2*>(cen + d);
      win[RP + d] = v.x; win[RP + d + 1] = v.y;
      d += 2;
    }
    if (d < 4 + R) win[RP + d] = cen[d];
  }
#pragma unroll
  for (int r = 1; r <= R; ++r) {
    if ((RP + r) % 2 == 0) {
      L01 = term2<FAST>(L01, pk(win[RP + r], win[RP + r + 1]), pk(win[RP - r], win[RP - r + 1]),
                        cf.cz[r - 1], nz);
      L23 = term2<FAST>(L23, pk(win[RP + r + 2], win[RP + r + 3]),
                        pk(win[RP - r + 2], win[RP - r + 3]), cf.cz[r - 1], nz);
    } else {
      L01 = term2s<FAST>(L01, win[RP + r], win[RP - r], win[RP + r + 1], win[RP - r + 1],
                         cf.cz[r - 1], nz);
      L23 = term2s<FAST>(L23, win[RP + r + 2], win[RP - r + 2], win[RP + r + 3],
                         win[RP - r + 3], cf.cz[r - 1], nz);
    }
  }
  // epilogue: o = ((c*2 - u0) + lap*inv) * fac   (c*2 == c+c exactly)
  f2 v01 = sub2(add2(c01, c01), pk(u0[0], u0[1]));
  f2 v23 = sub2(add2(c23, c23), pk(u0[2], u0[3]));
  if constexpr (FAST) {
    v01 = fma2(L01, pk(iv[0], iv[1]), v01);
    v23 = fma2(L23, pk(iv[2], iv[3]), v23);
  } else {
    v01 = add2(v01, xmul2(L01, pk(iv[0], iv[1]), nz));
    v23 = add2(v23, xmul2(L23, pk(iv[2], iv[3]), nz));
  }
  v01 = xmul2(v01, pk(fac[0], fac[1]), nz);
  v23 = xmul2(v23, pk(fac[2], fac[3]), nz);
  upk(v01, o[0], o[1]);
  upk(v23, o[2], o[3]);
}

template <int R, int K, int TY, int TZ, int PF, bool FAST, bool GUARD>
__global__ void __launch_bounds__(FusedCfg<R, K, TY, TZ, PF>::NT, FusedCfg<R, K, TY, TZ, PF>::MINB)
acoustic_fused(const __grid_constant__ FusedMaps maps, const __grid_constant__ FusedArgs a) {
  using C = FusedCfg<R, K, TY, TZ, PF>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* ring1 = reinterpret_cast<float*>(smem_raw);
  float* ring2 = reinterpret_cast<float*>(smem_raw + C::RING1);
  float* bufs = reinterpret_cast<float*>(smem_raw + C::RING1 + C::RING2);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + C::RING1 + C::RING2 + C::BUFS);
  uint64_t* done = full + C::NSB;

  const int tid = threadIdx.x;
  const int tile = blockIdx.x;
  const int y0 = (tile / a.ntz) * TY;
  const int z0 = (tile % a.ntz) * TZ;
  const int x0 = a.x_lo + blockIdx.y * a.cx_len;
  const int x1 = min(x0 + a.cx_len, a.x_hi);
  const int N = (x1 - x0) + 2 * K * R;
  const int ibase = x0 - K * R;

  if (tid == 0) {
    for (int s = 0; s < C::NSB; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], C::NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ------------------------------------------------------------ producer warp
  if (tid >= C::NTC) {
    if (tid == C::NTC) {
      prefetch_map(&maps.l0);
      prefetch_map(&maps.lm1);
      const bool use_inv = a.use_inv != 0;
      for (int n = 0; n < N; ++n) {
        const int sb = n % C::NSB;
        if (n >= C::NSB) mbar_wait_sleep(&done[sb], (uint32_t)(((n / C::NSB) - 1) & 1));
        uint32_t bytes = (uint32_t)C::E0 * 4u;
        if (n >= 2 * R) {
          bytes += (uint32_t)C::E1 * 4u;
          if (use_inv) {
#pragma unroll
            for (int j = 1; j <= K; ++j)
              if (n >= 2 * j * R) bytes += (uint32_t)C::ebox(j) * 4u;
          }
        }
        mbar_arrive_expect_tx(&full[sb], bytes);
        tma_load_3d(ring1 + (size_t)(n % C::NS1) * C::E0S, &maps.l0, z0 - C::hz(0),
                    y0 - C::hy(0), ibase + n, &full[sb]);
        if (n >= 2 * R) {
          float* ab = ring2 + (size_t)sb * C::AUX;
          tma_load_3d(ab, &maps.lm1, z0 - C::hz(1), y0 - C::hy(1), ibase + n - R, &full[sb]);
          if (use_inv) {
#pragma unroll
            for (int j = 1; j <= K; ++j)
              if (n >= 2 * j * R)
                tma_load_3d(ab + C::aux_inv_off(j), &maps.inv[j - 1], z0 - C::hz(j),
                            y0 - C::hy(j), ibase + n - j * R, &full[sb]);
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const int lane = tid & 31;
  const bool work = tid < C::NWORK;
  const int row = work ? tid / C::G1 : 0;
  const int g = work ? tid % C::G1 : 0;
  const int y = y0 - C::hy(1) + row;
  const int z = z0 - C::hz(1) + 4 * g;
  bool inE[K + 1];
#pragma unroll
  for (int j = 1; j <= K; ++j) {
    const int dy = C::hy(1) - C::hy(j), dz = C::hz(1) - C::hz(j);
    inE[j] = work && row >= dy && row < C::HY1 - dy && 4 * g >= dz && 4 * g < C::WZ1 - dz;
  }
  const bool ydom = y >= 0 && y < a.d.ny;
  bool zdom[4];
  float fyz[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    zdom[i] = ydom && (z + i >= 0) && (z + i < a.d.nz);
    fyz[i] = zdom[i] ? tmin(__ldg(a.fy + y), __ldg(a.fz + z + i)) : 1.0f;
  }
  const bool tile_owner = inE[K] && ydom && z < a.d.nz;
  const bool use_inv = a.use_inv != 0;
  // CTA-uniform: does any level region of this CTA leave the grid?  Interior
  // CTAs skip all zero-halo masking.
  const bool edge = (y0 - C::hy(1) < 0) || (y0 + TY + C::hy(1) > a.d.ny) ||
                    (z0 - C::hz(1) < 0) || (z0 + TZ + C::hz(1) > a.d.nz) ||
                    (x0 - (K - 1) * R < 0) || (x1 + (K - 1) * R > a.d.nx);
  const int nxm1 = (int)a.d.nx - 1;
  const int64_t gbase = (int64_t)y * a.d.pitch + z;      // global offset within a plane

  float q[K][C::Q][4];
#pragma unroll
  for (int j = 0; j < K; ++j)
#pragma unroll
    for (int s = 0; s < C::Q; ++s)
#pragma unroll
      for (int i = 0; i < 4; ++i) q[j][s][i] = 0.f;

  const int off0 = (row + (C::hy(0) - C::hy(1))) * C::WZ0 + 4 * g + (C::hz(0) - C::hz(1));
  const int off1 = row * C::WZ1 + 4 * g;
  int bad = 0;

  // Fused injection: each consumer thread walks its own entry list (the
  // points of its 4 z lanes, x ascending) with a two-entry window per level
  // whose series values are loaded when the entry enters the window -- a
  // plane without an entry for this thread costs one register compare, and
  // consuming an entry never waits on memory (the next one, possibly on the
  // very next plane, is already in the window).
  // window depth: two entries; one at R = 6 and for K >= 2 (register budget)
  constexpr int W = (R >= 6 || K >= 2) ? 1 : 2;
  int e_end = 0;
  int cur[K];
  int wk[K][W];          // (x << 2) | z lane of the window entries per level
  float wv[K][W];        // their series values
  const bool has_src = a.thr_list != nullptr && work;
  auto fetch = [&](int j, int c, int& k, float& v) {
    if (c < e_end) {
      const int2 e = __ldg(a.thr_list + c);
      k = (e.x << 2) | (e.y & 3);
      v = __ldg(a.series + (size_t)(a.t0 + j - 1) * a.n_src + (e.y >> 2));
    } else {
      k = 0x7fffffff;
      v = 0.f;
    }
  };
#pragma unroll
  for (int j = 0; j < K; ++j) {
    cur[j] = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      wk[j][w] = 0x7fffffff;
      wv[j][w] = 0.f;
    }
  }
  if (has_src) {
    const int base = tile * C::NWORK + tid;
    const int c0 = __ldg(a.thr_ptr + base);
    e_end = __ldg(a.thr_ptr + base + 1);
#pragma unroll
    for (int j = 1; j <= K; ++j) {
      // level j first computes plane x0 - (K - j) R: skip earlier entries
      const int pfirst = x0 - (K - j) * R;
      int c = c0;
      while (c < e_end && __ldg(&a.thr_list[c].x) < pfirst) ++c;
#pragma unroll
      for (int w = 0; w < W; ++w) fetch(j, c + w, wk[j - 1][w], wv[j - 1][w]);
      cur[j - 1] = c + W;
    }
  }

  // guard (before injection, as the reference's NaN check sees the stencil
  // result) then fused injection from this thread's entry window
  auto sparse_epilogue = [&](float (&o)[4], int j, int p, bool active) {
    if constexpr (GUARD) {
      if (a.guard_mask & (1 << (j - 1))) {
        const bool pin = p >= 0 && p < a.d.nx;
        if (active && tile_owner && pin && p >= x0 && p < x1) {
#pragma unroll
          for (int i = 0; i < 4; ++i) bad |= (zdom[i] && !isfinite(o[i]));
        }
      }
    }
    while ((wk[j - 1][0] >> 2) == p) {   // rare: an entry of this thread on this plane
      if (active) {
        const int lane = wk[j - 1][0] & 3;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i == lane) o[i] = __fadd_rn(o[i], wv[j - 1][0]);
      }
#pragma unroll
      for (int w = 0; w + 1 < W; ++w) {
        wk[j - 1][w] = wk[j - 1][w + 1];
        wv[j - 1][w] = wv[j - 1][w + 1];
      }
      fetch(j, cur[j - 1], wk[j - 1][W - 1], wv[j - 1][W - 1]);
      ++cur[j - 1];
    }
  };

  auto level_mask = [&](float (&o)[4], int p) {
    const bool pin = p >= 0 && p < a.d.nx;
    const bool live = pin || (p < 0 ? !a.zero_lo : !a.zero_hi);
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = (live && zdom[i]) ? o[i] : 0.0f;
  };

  auto fac4 = [&](float (&fac)[4], int p) {
    const float fxx = __ldg(a.fx + min(max(p, 0), nxm1));
#pragma unroll
    for (int i = 0; i < 4; ++i) fac[i] = tmin(fxx, fyz[i]);
  };

  for (int nb = 0; nb < N; nb += C::Q) {
#pragma unroll
    for (int qq = 0; qq < C::Q; ++qq) {
      const int n = nb + qq;
      if (n < N) {
        const unsigned un = (unsigned)n;
        const int sb = (int)(un % C::NSB);
        mbar_wait_sleep(&full[sb], (uint32_t)((un / C::NSB) & 1u));
        if (work) {
          const float4 v =
              *reinterpret_cast<const float4*>(ring1 + (size_t)(un % C::NS1) * C::E0S + off0);
          q[0][qq][0] = v.x; q[0][qq][1] = v.y; q[0][qq][2] = v.z; q[0][qq][3] = v.w;
        }
        const int cs = (qq - R + C::Q) % C::Q;          // centre slot (plane of level j)
        const int os = (qq - 2 * R + 2 * C::Q) % C::Q;  // oldest slot
        if (n >= 2 * R) {
          const float* aux = ring2 + (size_t)sb * C::AUX;
          // ================= level 1 (plane i - R) from the staged plane
          {
            const int p = ibase + n - R;
            float o[4] = {0.f, 0.f, 0.f, 0.f};
            if (work) {
              const float* cen = ring1 + (size_t)((un - R) % C::NS1) * C::E0S + off0;
              const float4 u04 = *reinterpret_cast<const float4*>(aux + off1);
              const float u0[4] = {u04.x, u04.y, u04.z, u04.w};
              float iv[4];
              if (use_inv) {
                const float4 t4 =
                    *reinterpret_cast<const float4*>(aux + C::aux_inv_off(1) + off1);
                iv[0] = t4.x; iv[1] = t4.y; iv[2] = t4.z; iv[3] = t4.w;
              } else {
                iv[0] = iv[1] = iv[2] = iv[3] = a.inv_scalar;
              }
              float fac[4];
              fac4(fac, p);
              update4<FAST, R, C::Q, C::RP, C::WZ0>(q[0], cs, cen, u0, iv, fac, a.cf, o);
              if (edge) level_mask(o, p);
            }
            sparse_epilogue(o, 1, p, work);
            if constexpr (K >= 2) {
#pragma unroll
              for (int i = 0; i < 4; ++i) q[1][qq][i] = o[i];
            }
            if constexpr (K <= 2) {
              if (work && tile_owner && p >= x0 && p < x1) {
                float* dst = (K == 1) ? a.out_k : a.out_km1;
                const float4 v4 = make_float4(o[0], o[1], o[2], o[3]);
                *reinterpret_cast<float4*>(dst + (int64_t)p * a.d.plane + gbase) = v4;
                if constexpr (K == 1) {
                  // fused halo exchange: the boundary planes go straight into
                  // the neighbours' ghost zones (plane-uniform branches)
                  if (a.peer_lo && p < a.peer_lo_end)
                    *reinterpret_cast<float4*>(
                        a.peer_lo + (int64_t)(p + a.peer_lo_shift) * a.d.plane + gbase) = v4;
                  if (a.peer_hi && p >= a.peer_hi_begin)
                    *reinterpret_cast<float4*>(
                        a.peer_hi + (int64_t)(p + a.peer_hi_shift) * a.d.plane + gbase) = v4;
                }
              }
            }
          }
          // ================= levels 2..K (plane i - jR) from the smem buffers
#pragma unroll
          for (int j = 2; j <= K; ++j) {
            if (n >= 2 * j * R) {
              float* buf = bufs + ((size_t)(j - 2) * 2 + (n & 1)) * C::E1;
              if (inE[j - 1]) {
                *reinterpret_cast<float4*>(buf + off1) = make_float4(
                    q[j - 1][cs][0], q[j - 1][cs][1], q[j - 1][cs][2], q[j - 1][cs][3]);
              }
              named_bar_sync(1, C::NTC);
              const int p = ibase + n - j * R;
              float o[4] = {0.f, 0.f, 0.f, 0.f};
              if (inE[j]) {
                float iv[4];
                if (use_inv) {
                  const int dy = C::hy(1) - C::hy(j), dz = C::hz(1) - C::hz(j);
                  const float4 t4 = *reinterpret_cast<const float4*>(
                      aux + C::aux_inv_off(j) + (row - dy) * (TZ + 2 * C::hz(j)) + 4 * g - dz);
                  iv[0] = t4.x; iv[1] = t4.y; iv[2] = t4.z; iv[3] = t4.w;
                } else {
                  iv[0] = iv[1] = iv[2] = iv[3] = a.inv_scalar;
                }
                const float u0[4] = {q[j - 2][os][0], q[j - 2][os][1], q[j - 2][os][2],
                                     q[j - 2][os][3]};
                float fac[4];
                fac4(fac, p);
                update4<FAST, R, C::Q, C::RP, C::WZ1>(q[j - 1], cs, buf + off1, u0, iv, fac,
                                                      a.cf, o);
                if (edge) level_mask(o, p);
              }
              sparse_epilogue(o, j, p, inE[j]);
              if (j < K) {
#pragma unroll
                for (int i = 0; i < 4; ++i) q[j][qq][i] = o[i];
              }
              if (tile_owner && (j == K || (j == K - 1 && p >= x0 && p < x1))) {
                float* dst = (j == K) ? a.out_k : a.out_km1;
                *reinterpret_cast<float4*>(dst + (int64_t)p * a.d.plane + gbase) =
                    make_float4(o[0], o[1], o[2], o[3]);
              }
            }
          }
        }
        // iteration n done: its aux slot and the staged plane n-R (level-1
        // centre) may be refilled by the producer
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[sb]);
      }
    }
  }
  if constexpr (GUARD) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(a.nonfinite, 1);
  }
}

template <int R, int K, int TY, int TZ, int PF, bool FAST>
struct FusedLauncher {
  using C = FusedCfg<R, K, TY, TZ, PF>;
  template <bool GUARD>
  static void launch_g(cudaStream_t st, const FusedMaps& maps, const FusedArgs& a, int nchunks) {
    static std::atomic<uint64_t> configured{0};
    if (first_use_on_device(configured))
      STB_CUDA(cudaFuncSetAttribute(acoustic_fused<R, K, TY, TZ, PF, FAST, GUARD>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    const int nty = (int)((a.d.ny + TY - 1) / TY);
    dim3 grid((unsigned)(a.ntz * nty), (unsigned)nchunks);
    acoustic_fused<R, K, TY, TZ, PF, FAST, GUARD><<<grid, C::NT, C::SMEM, st>>>(maps, a);
    STB_CHECK_LAUNCH();
  }
  static void launch(cudaStream_t st, const FusedMaps& maps, const FusedArgs& a, int nchunks) {
    if (nchunks <= 0) return;
    if (a.guard_mask && a.nonfinite)
      launch_g<true>(st, maps, a, nchunks);
    else
      launch_g<false>(st, maps, a, nchunks);
  }
};

}  // namespace stb
