// Shared declarations of the TMA-tiled elastic half steps (elastic_tiled2.cuh):
// the launch arguments, the z-tile width and the ring-index helper.  (The
// first TMA kernel that lived here -- one point per thread, a CTA barrier per
// plane, 36.4 GPts/s -- was superseded by elastic_tiled2 and removed.)
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

constexpr int el_pmod(int a, int m) { return ((a % m) + m) % m; }

}  // namespace
}  // namespace stb
