// mr_stream2d.cuh -- column-strip streaming FIR engine for the 2D velocity
// v = -K*(z grad I) (integrator.py:93-94; kernel.py:36-45,71-73).
//
// One CTA owns a strip of OX output columns of one pair and walks down all rows:
//   per group of G new input rows
//     TMA  : I rows (+-1) and z rows of the strip + R-column halo -> smem
//            (the next group's boxes are in flight while this group is filtered)
//     prod : m_c = z * d_c I for the group, written with an odd pitch
//     H    : horizontal FIR of the new rows only (no y halo) -> ring of filtered rows
//   per block of G output rows
//     V    : vertical FIR over the ring (register blocking, lanes <-> columns)
//     epi  : v = -(...) straight to HBM (coalesced), velocity guard
//     shift: drop the G oldest ring rows
// Each input row is staged and multiplied once per strip (x halo RX/OX only);
// FIR work is exactly 2 * (2R+1) FFMA per output and component.  Replicate
// borders: rows above 0 / below H-1 are copies of the border rows' filtered
// rows; columns outside the image replicate inside the product stage.
#pragma once

#include "mr_kernels2d.cuh"

namespace mr {

template <typename T, int R>
struct StreamCfg {
  static constexpr int OX = 64;           // output columns per strip
  static constexpr int G = 32;            // rows per group / output block
  static constexpr int A = 16 / (int)sizeof(T);
  static constexpr int RX = OX + 2 * R;   // input columns
  static constexpr int PXI = round_up(RX + 2 + A - 1, A);  // I box width (aligned start)
  static constexpr int PXZ = round_up(RX + A - 1, A);      // z box width
  static constexpr int PP = (RX % 2) ? RX : RX + 1;        // product pitch (odd)
  static constexpr int RING = G + 2 * R;  // filtered rows kept
  static constexpr int RP = OX + 4;       // ring pitch: 16-B rows (float4 stores/copies),
                                          // 8-byte column pairs; 68 = 4 mod 32 keeps the
                                          // quarter-warp float4 stores conflict-free
  // smem layout (elements after the 128-B head)
  static constexpr int o_ist = 0;
  static constexpr int n_ist = round_up((G + 2) * PXI + A, 32);
  static constexpr int o_zst = o_ist + n_ist;
  static constexpr int n_zst = round_up(G * PXZ + A, 32);
  static constexpr int o_p = o_zst + n_zst;
  static constexpr int n_p = round_up(2 * G * PP, 32);
  static constexpr int o_ring = o_p + n_p;
  static constexpr int n_ring = round_up(2 * RING * RP, 32);
  static constexpr size_t head = 128;
  static constexpr size_t bytes = head + sizeof(T) * (size_t)(o_ring + n_ring);
};

template <typename T, int R>
__global__ void __launch_bounds__(kThreads)
    k_velocity2d_stream(VelArgs<T> a, Taps<T> tp, const __grid_constant__ CUtensorMap mapI,
                        const __grid_constant__ CUtensorMap mapZ) {
  using C = StreamCfg<T, R>;
  constexpr int OX = C::OX, G = C::G, RX = C::RX, PXI = C::PXI, PXZ = C::PXZ, PP = C::PP,
                RING = C::RING, RP = C::RP;
  static_assert(sizeof(T) == 4 && OX == 64 && G == 32, "fp32 FFMA2 layout");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  T* base = reinterpret_cast<T*>(smem_raw + C::head);
  T* ist0 = base + C::o_ist;
  T* zst0 = base + C::o_zst;
  T* P = base + C::o_p;        // [2][G][PP]
  T* ring = base + C::o_ring;  // [2][RING][RP], ring row 0 <-> image row ring_lo

  const int H = a.g.H, W = a.g.W;
  const int b = blockIdx.y;
  const int x0 = blockIdx.x * OX;
  const int xs = x0 - R;  // first input column
  const int offI = align_shift(xs - 1, C::A), offZ = align_shift(xs, C::A);
  const T* ist = ist0 + offI;  // staged I element (r, i) at ist[r*PXI + i], r=0 <-> row u0-1
  const T* zst = zst0 + offZ;  // staged z element (r, i) at zst[r*PXZ + i]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long N = a.g.N;
  T* v0 = a.v + (long long)b * 2 * N;
  T* v1 = v0 + N;

  // in-image input columns of the strip window
  const int i_lo = max(0, -xs), i_hi = min(RX, W - xs);
  // every in-image column has both x neighbours in the image
  const bool x_interior = (xs + i_lo >= 1) && (xs + i_hi - 1 <= W - 2);

  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  unsigned phase = 0;
  auto issue = [&](int u0) {  // TMA of the group starting at image row u0 (thread 0)
    mbar_expect_tx(bar, (unsigned)(sizeof(T) * (PXI * (G + 2) + PXZ * G)));
    tma_load_3d(ist0, &mapI, xs - 1 - offI, u0 - 1, b, bar);
    tma_load_3d(zst0, &mapZ, xs - offZ, u0, b, bar);
  };
  if (tid == 0) issue(0);

  unsigned flags = 0;
  int ring_lo = -R;   // image row of ring row 0
  int next_u = 0;     // next image row to produce (rows < 0 are replicas of row 0)
  for (int y0 = 0; y0 < H; y0 += G) {
    const int need_hi = y0 + G + R;  // rows [.., need_hi) must be in the ring
    while (next_u < need_hi) {
      const int u0 = next_u;
      const int cnt = min(G, need_hi - u0);
      if (u0 < H) {
        // ---- product of the in-image rows of this group ----
        const int cin = min(cnt, H - u0);
        mbar_wait(bar, phase);
        phase ^= 1u;
        for (int r = warp; r < cin; r += kNW) {
          const int u = u0 + r;
          const T* crow = ist + (r + 1) * PXI + 1;
          const T* zrow = zst + r * PXZ;
          T* p0 = P + r * PP;
          T* p1 = P + G * PP + r * PP;
          const bool yin = u > 0 && u < H - 1;  // warp-uniform
          if (yin && x_interior) {              // branch-free central differences
            for (int i = i_lo + lane; i < i_hi; i += 32) {
              // z * ((a - b) / 2) == (z / 2) * (a - b) exactly (halving is exact)
              const T* c = crow + i;
              const T hz = T(0.5) * zrow[i];
              p0[i] = hz * (c[PXI] - c[-PXI]);
              p1[i] = hz * (c[1] - c[-1]);
            }
          } else {
            for (int i = i_lo + lane; i < i_hi; i += 32) {
              const T* c = crow + i;
              const T f0 = c[0];
              const T g0 = grad1(c[-PXI], f0, c[PXI], u, H);
              const T g1 = grad1(c[-1], f0, c[1], xs + i, W);
              const T zz = zrow[i];
              p0[i] = zz * g0;
              p1[i] = zz * g1;
            }
          }
        }
        __syncthreads();
        // staging is free again: prefetch the next group's rows
        const int nu = u0 + cnt;
        if (tid == 0 && nu < H) {
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          issue(nu);
        }
        // replicate the border columns inside the product rows
        if (i_lo > 0 || i_hi < RX) {
          const int nl = i_lo, nr = RX - i_hi;
          for (int r = warp; r < cin; r += kNW)
            for (int t = lane; t < nl + nr; t += 32) {
              const int i = t < nl ? t : i_hi + (t - nl);
              const int ir = t < nl ? i_lo : i_hi - 1;
              P[r * PP + i] = P[r * PP + ir];
              P[G * PP + r * PP + i] = P[G * PP + r * PP + ir];
            }
          __syncthreads();
        }
        // ---- horizontal FIR of the new rows -> ring: rows (r, r+16) per thread (FFMA2) ----
        constexpr int NB = OX / kRB;
        for (int cb = warp; cb < NB; cb += kNW) {  // (c, column-block pair)
          const int r = lane & 15;
          // half-warps 16 columns apart: complementary bank sets with the odd pitch
          const int pb = cb % (NB / 2);
          const int ib = (pb & 1) + 4 * (pb >> 1) + 2 * (lane >> 4);
          const int c = cb / (NB / 2);
          if (r >= cin) continue;
          const T* s0 = P + c * G * PP + r * PP + ib * kRB;
          const T* s1 = s0 + 16 * PP;
          float2 acc[kRB];
#pragma unroll
          for (int o = 0; o < kRB; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
          for (int t = 0; t < kRB + 2 * R; ++t) {
            const float2 x = make_float2(s0[t], s1[t]);
#pragma unroll
            for (int o = 0; o < kRB; ++o) {
              const int tap = t - o;
              if (tap >= 0 && tap <= 2 * R) acc[o] = ffma2(x, (float)tp.w[tap], acc[o]);
            }
          }
          float4* d0 = reinterpret_cast<float4*>(ring + c * RING * RP + (u0 + r - ring_lo) * RP +
                                                 ib * kRB);
          d0[0] = make_float4(acc[0].x, acc[1].x, acc[2].x, acc[3].x);
          d0[1] = make_float4(acc[4].x, acc[5].x, acc[6].x, acc[7].x);
          if (r + 16 < cin) {
            float4* d1 = d0 + 16 * RP / 4;
            d1[0] = make_float4(acc[0].y, acc[1].y, acc[2].y, acc[3].y);
            d1[1] = make_float4(acc[4].y, acc[5].y, acc[6].y, acc[7].y);
          }
        }
        __syncthreads();
        if (u0 == 0) {  // rows above the image replicate row 0 (only in the first block)
          for (int j = warp; j < 2 * (0 - ring_lo); j += kNW) {
            const int c = j / (0 - ring_lo), rr = j % (0 - ring_lo);
            for (int i = lane; i < OX; i += 32)
              ring[c * RING * RP + rr * RP + i] = ring[c * RING * RP + (0 - ring_lo) * RP + i];
          }
          __syncthreads();
        }
        if (u0 + cnt > H) {  // rows below the image in this group replicate row H-1
          for (int j = warp; j < 2 * (u0 + cnt - H); j += kNW) {
            const int n = u0 + cnt - H;
            const int c = j / n, rr = H + j % n;
            for (int i = lane; i < OX; i += 32)
              ring[c * RING * RP + (rr - ring_lo) * RP + i] =
                  ring[c * RING * RP + (H - 1 - ring_lo) * RP + i];
          }
          __syncthreads();
        }
      } else {  // whole group below the image: replicas of row H-1
        for (int j = warp; j < 2 * cnt; j += kNW) {
          const int c = j / cnt, rr = u0 + j % cnt;
          for (int i = lane; i < OX; i += 32)
            ring[c * RING * RP + (rr - ring_lo) * RP + i] =
                ring[c * RING * RP + (H - 1 - ring_lo) * RP + i];
        }
        __syncthreads();
      }
      next_u = u0 + cnt;
    }

    // ---- vertical FIR over the ring for output rows [y0, y0+G): lanes <-> column pairs ----
    constexpr int NBV = G / kRB;
    for (int cb = warp; cb < 2 * NBV; cb += kNW) {
      const int jb = cb % NBV, c = cb / NBV;
      const int i = 2 * lane;  // OX == 64: one column pair per lane
      const float2* src = reinterpret_cast<const float2*>(
          ring + c * RING * RP + (y0 + jb * kRB - R - ring_lo) * RP + i);
      float2 acc[kRB];
#pragma unroll
      for (int o = 0; o < kRB; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < kRB + 2 * R; ++t) {
        const float2 x = src[t * (RP / 2)];
#pragma unroll
        for (int o = 0; o < kRB; ++o) {
          const int tap = t - o;
          if (tap >= 0 && tap <= 2 * R) acc[o] = ffma2(x, (float)tp.w[tap], acc[o]);
        }
      }
      const int gx = x0 + i;
      T* vo = (c == 0 ? v0 : v1) + gx;
      const bool pair_ok = gx + 1 < W && ((W & 1) == 0);  // 8-byte aligned float2 store
      const int gyb = y0 + jb * kRB;
      if (pair_ok && gyb + kRB <= H) {  // whole block in the image: plain float2 stores
        float2* vrow = reinterpret_cast<float2*>(vo + gyb * W);  // < N per component
        bool big = false;
#pragma unroll
        for (int o = 0; o < kRB; ++o) {
          const float2 val = make_float2(-acc[o].x, -acc[o].y);
          vrow[o * (W / 2)] = val;
          big |= !(fabsf(val.x) <= 1e6f && fabsf(val.y) <= 1e6f);
        }
        if (big) {  // exact guard bits only when a value failed the one-compare test
#pragma unroll
          for (int o = 0; o < kRB; ++o) {
            flags |= guard_bits(-acc[o].x, MR_GUARD_VELOCITY_NONFINITE);
            flags |= guard_bits(-acc[o].y, MR_GUARD_VELOCITY_NONFINITE);
          }
        }
        continue;
      }
#pragma unroll
      for (int o = 0; o < kRB; ++o) {
        const int gy = y0 + jb * kRB + o;
        if (gy < H) {
          const T a0 = -acc[o].x, a1 = -acc[o].y;
          if (pair_ok) {
            *reinterpret_cast<float2*>(vo + (long long)gy * W) = make_float2(a0, a1);
          } else {
            if (gx < W) vo[(long long)gy * W] = a0;
            if (gx + 1 < W) vo[(long long)gy * W + 1] = a1;
          }
          // one compare on the common path; exact guard bits only when it fails
          if (!(fabsf(a0) <= 1e6f && fabsf(a1) <= 1e6f)) {
            if (gx < W) flags |= guard_bits(a0, MR_GUARD_VELOCITY_NONFINITE);
            if (gx + 1 < W) flags |= guard_bits(a1, MR_GUARD_VELOCITY_NONFINITE);
          }
        }
      }
    }
    __syncthreads();
    // ---- shift: keep ring rows [y0+G-R, y0+G+R) at the front (drop G rows) ----
    // bands of G rows so that source and destination never overlap within a band
#pragma unroll
    for (int band = 0; band < 2 * R; band += G) {
      const int nrow = (2 * R - band) < G ? (2 * R - band) : G;  // compile-time per band
      // float4 copy: each warp moves two rows (16 float4 per row and component)
      for (int t = warp * 32 + lane; t < nrow * 2 * (OX / 4); t += kThreads) {
        const int q4 = t % (OX / 4), rest = t / (OX / 4);
        const int c = rest & 1, rr = band + (rest >> 1);
        float4* dst = reinterpret_cast<float4*>(ring + c * RING * RP + rr * RP) + q4;
        const float4* src = reinterpret_cast<const float4*>(ring + c * RING * RP + (rr + G) * RP) + q4;
        *dst = *src;
      }
      __syncthreads();
    }
    ring_lo = y0 + G - R;
  }
  if (a.guard) flush_flags(flags, a.guard + (long long)b * a.guard_stride);
}

}  // namespace mr

namespace mr {

// ---------------------------------------------------------------------------------
// Streaming adjoint of the velocity (objective.py:157-161, 165-169):
//   mbar = -K^T vbar (kernel.py:48-68: zero-padded correlation + cumulative-weight
//   edge taps at index 0 and n-1); zb += mbar . grad I; ib += G^T(mbar z).
// Strip of OX computed columns (owners OX-2, one column of halo each side for
// G^T); blocks of G computed rows (owners G-2).  vbar rows are TMA-staged
// (zero fill outside the image = the transpose's zero padding), copied to an
// odd pitch, filtered horizontally into the ring, then filtered vertically.
// The epilogue operands (I, z, ib|v0, zb) of the block arrive by TMA while the
// passes run.
// ---------------------------------------------------------------------------------
template <typename T, int R>
struct StreamAdjCfg {
  static constexpr int OX = 64;  // computed columns (owners OX-2)
  static constexpr int G = 32;   // computed rows per block (owners G-2)
  static constexpr int ADV = G - 2;
  static constexpr int A = 16 / (int)sizeof(T);
  static constexpr int RX = OX + 2 * R;
  static constexpr int PXZ = round_up(RX + A - 1, A);  // vbar box width
  static constexpr int PP = (RX % 2) ? RX : RX + 1;
  static constexpr int RING = G + 2 * R;
  static constexpr int RP = OX + 4;  // 16-B rows: float4 ring stores / copies, float2 column pairs
  static constexpr int OXP = OX + A;                   // epilogue box width
  static constexpr int EPL = round_up(G * OXP, 32);    // one epilogue operand (I or z)
  static constexpr int o_st = 0;  // vbar staging [2][G][PXZ]; after a block's last group: I, z
  static constexpr int n_st1 = round_up(G * PXZ + A, 32);
  static constexpr int o_p = o_st + 2 * n_st1;         // P [2][G][PP]; later res [2][G][RP]
  static constexpr int n_p = round_up(2 * G * (PP > RP ? PP : RP), 32);
  static constexpr int o_ring = o_p + n_p;
  static constexpr int n_ring = round_up(2 * RING * RP, 32);
  static constexpr size_t head = 128;
  static constexpr size_t bytes_reg = head + sizeof(T) * (size_t)(o_ring + n_ring);
  static constexpr size_t bytes_noreg = bytes_reg;
  static_assert(2 * G * RP <= n_p, "result must fit in the product buffer");
  static_assert(2 * EPL <= 2 * n_st1, "epilogue I/z must fit in the staging buffer");
};

constexpr int kAdjStreamThreads = 256;

template <typename T, int R, bool REG>
__global__ void __launch_bounds__(kAdjStreamThreads)
    k_velocity_adj2d_stream(VelAdjArgs<T> a, Taps<T> tp, const __grid_constant__ VelAdjMaps maps) {
  using C = StreamAdjCfg<T, R>;
  constexpr int NW = kAdjStreamThreads / 32;
  constexpr int OX = C::OX, G = C::G, ADV = C::ADV, RX = C::RX, PXZ = C::PXZ, PP = C::PP,
                RING = C::RING, RP = C::RP, OXP = C::OXP, EPL = C::EPL;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);  // [0]: vbar groups, [1]: epilogue
  T* base = reinterpret_cast<T*>(smem_raw + C::head);
  T* st0 = base + C::o_st;
  T* P = base + C::o_p;
  T* ring = base + C::o_ring;
  T* epi0 = base + C::o_st;  // epilogue I, z reuse the staging buffer

  const int H = a.g.H, W = a.g.W;
  const long long N = a.g.N;
  const int b = blockIdx.y;
  const int x_org = blockIdx.x * (OX - 2) - 1;  // computed column 0
  const int xs = x_org - R;                     // first input column
  const int offV = align_shift(xs, C::A), offE = align_shift(x_org, C::A);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_barrier_init();
  }
  __syncthreads();
  unsigned ph0 = 0, ph1 = 0;
  auto issue_v = [&](int u0) {
    mbar_expect_tx(bar, (unsigned)(sizeof(T) * 2 * PXZ * G));
    tma_load_3d(st0, &maps.vbar, xs - offV, u0, 2 * b, bar);
    tma_load_3d(st0 + C::n_st1, &maps.vbar, xs - offV, u0, 2 * b + 1, bar);
  };
  auto issue_e = [&](int yc0) {
    mbar_expect_tx(bar + 1, (unsigned)(sizeof(T) * OXP * G * 2));
    const int xa = x_org - offE;
    tma_load_3d(epi0, &maps.I, xa, yc0, b, bar + 1);
    tma_load_3d(epi0 + EPL, &maps.z, xa, yc0, b, bar + 1);
  };
  if (tid == 0) issue_v(0);

  unsigned bad = 0;
  int ring_lo = -1 - R;  // image row of ring row 0
  int next_u = -1 - R;   // next image row to produce (outside the image: zero rows)
  for (int yb = 0; yb < H; yb += ADV) {
    const int yc0 = yb - 1;  // computed row 0 of this block
    const int need_hi = yc0 + G + R;
    while (next_u < need_hi) {
      const int u0 = next_u;
      if (u0 < 0 || u0 >= H) {  // zero rows up to the image edge or to need_hi
        const int cnt = u0 < 0 ? min(-u0, need_hi - u0) : need_hi - u0;
        for (int j = warp; j < 2 * cnt; j += NW) {
          const int c = j / cnt, rr = u0 + j % cnt;
          for (int i = lane; i < OX; i += 32) ring[c * RING * RP + (rr - ring_lo) * RP + i] = T(0);
        }
        next_u = u0 + cnt;
        continue;
      }
      const int cnt = min(G, need_hi - u0);
      const int cin = min(cnt, H - u0);
      mbar_wait(bar, ph0);
      ph0 ^= 1u;
      // vbar rows -> odd-pitch P (zeros outside the image came from the TMA fill)
      // (consecutive lanes on both sides: conflict-free loads and stores)
      for (int rc = warp; rc < 2 * cin; rc += NW) {
        const int r = rc >> 1, c = rc & 1;
        const T* srow = st0 + c * C::n_st1 + r * PXZ + offV;
        T* prow = P + c * G * PP + r * PP;
#pragma unroll
        for (int i = lane; i < RX; i += 32) prow[i] = srow[i];
      }
      __syncthreads();
      const int nu = u0 + cnt;
      if (tid == 0 && nu < H && nu < need_hi) {  // next group of this block
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue_v(nu);
      }
      // horizontal transposed FIR of the new rows -> ring: rows (r, r+16) per thread (FFMA2)
      constexpr int NB = OX / kRB;
      static_assert(NB % 2 == 0 && 2 * (NB / 2) == NW, "one (component, column-block pair) per warp");
      {
        const int cb = warp;
        const int r = lane & 15;
        const int pb = cb % (NB / 2);
        const int ib = (pb & 1) + 4 * (pb >> 1) + 2 * (lane >> 4);
        const int c = cb / (NB / 2);
        if (r < cin) {
          const T* s0 = P + c * G * PP + r * PP + ib * kRB;
          const T* s1 = s0 + 16 * PP;
          float2 acc[kRB];
#pragma unroll
          for (int o = 0; o < kRB; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
          for (int t = 0; t < kRB + 2 * R; ++t) {
            const float2 x = make_float2(s0[t], s1[t]);
#pragma unroll
            for (int o = 0; o < kRB; ++o) {
              const int tap = t - o;
              if (tap >= 0 && tap <= 2 * R) acc[o] = ffma2(x, (float)tp.w[tap], acc[o]);
            }
          }
          const int gx0 = x_org + ib * kRB;
          if (gx0 <= 0 && gx0 + kRB > 0) {  // column 0: sum_{d=0..R} W[R-d] g[d]
            const int o = -gx0;
            float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int d = 0; d <= R; ++d)
              s2 = ffma2(make_float2(s0[o + R + d], s1[o + R + d]), (float)tp.e[R - d], s2);
#pragma unroll
            for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s2;
          }
          if (gx0 <= W - 1 && gx0 + kRB > W - 1) {  // column n-1
            const int o = W - 1 - gx0;
            float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int d = -R; d <= 0; ++d)
              s2 = ffma2(make_float2(s0[o + R + d], s1[o + R + d]), (float)tp.e[R + d], s2);
#pragma unroll
            for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s2;
          }
          float4* d0 = reinterpret_cast<float4*>(ring + c * RING * RP + (u0 + r - ring_lo) * RP +
                                                 ib * kRB);
          d0[0] = make_float4(acc[0].x, acc[1].x, acc[2].x, acc[3].x);
          d0[1] = make_float4(acc[4].x, acc[5].x, acc[6].x, acc[7].x);
          if (r + 16 < cin) {
            float4* d1 = d0 + 16 * RP / 4;
            d1[0] = make_float4(acc[0].y, acc[1].y, acc[2].y, acc[3].y);
            d1[1] = make_float4(acc[4].y, acc[5].y, acc[6].y, acc[7].y);
          }
        }
      }
      __syncthreads();
      next_u = u0 + cin;
    }
    __syncthreads();
    // staging is free: fetch the epilogue's I and z tiles while the vertical pass runs
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue_e(yc0);
    }

    // ---- owner operands of the epilogue into registers (in flight during the pass) ----
    constexpr int NJ = (G - 2 + NW - 1) / NW, NI = (OX - 2 + 31) / 32;
    T pre_a[NJ][NI], pre_b[NJ][NI], pre_c[NJ][NI];
    const T* __restrict__ zb_p = a.zb + b * N;
    const T* __restrict__ o2_p = REG ? a.v0 + b * 2 * N : a.ib + b * N;
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
      for (int ii = 0; ii < NI; ++ii) {
        const int j = 1 + warp + jj * NW, i = 1 + lane + ii * 32;
        const int gy = yc0 + j, gx = x_org + i;
        const bool ok = j < G - 1 && i < OX - 1 && gy < H && gx < W;
        const int q = ok ? gy * W + gx : 0;  // < N < 2^31 per pair
        pre_a[jj][ii] = ok ? zb_p[q] : T(0);
        pre_b[jj][ii] = ok ? o2_p[q] : T(0);
        pre_c[jj][ii] = (REG && ok) ? o2_p[N + q] : T(0);
      }

    // ---- vertical transposed FIR for computed rows [yc0, yc0+G) -> res (= P):
    //      lanes <-> column pairs (FFMA2), one (component, row block) per warp ----
    T* res = P;  // [2][G][RP], holds mbar = -K^T vbar
    constexpr int NBV = G / kRB;
    static_assert(2 * NBV == NW && OX == 64, "one (component, row block) per warp");
    {
      const int jb = warp % NBV, c = warp / NBV;
      const int i = 2 * lane;
      const float2* src = reinterpret_cast<const float2*>(
          ring + c * RING * RP + (yc0 + jb * kRB - R - ring_lo) * RP + i);
      float2 acc[kRB];
#pragma unroll
      for (int o = 0; o < kRB; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < kRB + 2 * R; ++t) {
        const float2 x = src[t * (RP / 2)];
#pragma unroll
        for (int o = 0; o < kRB; ++o) {
          const int tap = t - o;
          if (tap >= 0 && tap <= 2 * R) acc[o] = ffma2(x, (float)tp.w[tap], acc[o]);
        }
      }
      const int gy0 = yc0 + jb * kRB;
      if (gy0 <= 0 && gy0 + kRB > 0) {
        const int o = -gy0;
        float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int d = 0; d <= R; ++d) s2 = ffma2(src[(o + R + d) * (RP / 2)], (float)tp.e[R - d], s2);
#pragma unroll
        for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s2;
      }
      if (gy0 <= H - 1 && gy0 + kRB > H - 1) {
        const int o = H - 1 - gy0;
        float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int d = -R; d <= 0; ++d) s2 = ffma2(src[(o + R + d) * (RP / 2)], (float)tp.e[R + d], s2);
#pragma unroll
        for (int q = 0; q < kRB; ++q) if (q == o) acc[q] = s2;
      }
      float2* dst = reinterpret_cast<float2*>(res + c * G * RP + jb * kRB * RP + i);
#pragma unroll
      for (int o = 0; o < kRB; ++o) dst[o * (RP / 2)] = make_float2(-acc[o].x, -acc[o].y);
    }
    mbar_wait(bar + 1, ph1);
    ph1 ^= 1u;
    __syncthreads();

    // ---- epilogue on owners: rows j in [1, G-1), cols i in [1, OX-1) ----
    const T* tI = epi0 + offE;
    const T* tz = tI + EPL;
    T* __restrict__ zb_o = a.zb + b * N;
    T* __restrict__ ib_o = a.ib + b * N;
    // every owner >= 2 away from the image edges: central stencils, no edge terms
    const bool interior = !REG && yc0 + 1 >= 2 && yc0 + G - 2 <= H - 3 && x_org + 1 >= 2 &&
                          x_org + OX - 2 <= W - 3;
    if (interior) {
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
        for (int ii = 0; ii < NI; ++ii) {
          const int j = 1 + warp + jj * NW, i = 1 + lane + ii * 32;
          if (j >= G - 1 || i >= OX - 1) continue;
          const int q = (yc0 + j) * W + (x_org + i);
          const int e = j * OXP + i;
          const T g0 = (tI[e + OXP] - tI[e - OXP]) / T(2);
          const T g1 = (tI[e + 1] - tI[e - 1]) / T(2);
          const T m0 = res[j * RP + i];
          const T m1 = res[G * RP + j * RP + i];
          zb_o[q] = pre_a[jj][ii] + (m0 * g0 + m1 * g1);  // objective.py:159
          if (a.zero_a) {
            a.zero_a[b * N + q] = T(0);
            a.zero_b[b * N + q] = T(0);
          }
          // G^T(mbar z): 0.5 q[j-1] - 0.5 q[j+1] per axis (fields.py:148-158)
          const T gm = res[(j - 1) * RP + i] * tz[e - OXP];
          const T gp = res[(j + 1) * RP + i] * tz[e + OXP];
          const T hm = res[G * RP + j * RP + i - 1] * tz[e - 1];
          const T hp = res[G * RP + j * RP + i + 1] * tz[e + 1];
          const T t0 = T(0.5) * gm - T(0.5) * gp;
          const T t1 = T(0.5) * hm - T(0.5) * hp;
          ib_o[q] = pre_b[jj][ii] + (t0 + t1);
        }
    } else {
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
    for (int ii = 0; ii < NI; ++ii) {
      const int j = 1 + warp + jj * NW, i = 1 + lane + ii * 32;
      const int gy = yc0 + j, gx = x_org + i;
      if (j >= G - 1 || i >= OX - 1 || gy >= H || gx >= W) continue;
      {
        const int q = gy * W + gx;
        const int e = j * OXP + i;
        const T cI = tI[e];
        const T g0 = grad1(tI[e - OXP], cI, tI[e + OXP], gy, H);
        const T g1 = grad1(tI[e - 1], cI, tI[e + 1], gx, W);
        const T m0 = res[j * RP + i];
        const T m1 = res[G * RP + j * RP + i];
        T zb_new = pre_a[jj][ii] + (m0 * g0 + m1 * g1);  // objective.py:159
        if (REG) {
          const T km = -(pre_b[jj][ii] * g0 + pre_c[jj][ii] * g1);
          zb_new = zb_new + a.lam * (km + a.two_rho * tz[e]);
          a.zout[b * N + q] = zb_new;
          bad |= isfinite(zb_new) ? 0u : 1u;
        } else {
          zb_o[q] = zb_new;
          if (a.zero_a) {  // the consumed ibar/zbar of step k+1 = next step's scatter targets
            a.zero_a[b * N + q] = T(0);
            a.zero_b[b * N + q] = T(0);
          }
          auto q0 = [&](int jr) { return res[jr * RP + i] * tz[jr * OXP + i]; };
          auto q1 = [&](int ic) { return res[G * RP + j * RP + ic] * tz[j * OXP + ic]; };
          const T zc = tz[e];
          const T qc0 = m0 * zc, qc1 = m1 * zc;
          const T gm = (gy > 0) ? q0(j - 1) : T(0);
          const T gp = (gy < H - 1) ? q0(j + 1) : T(0);
          const T gf = (gy == 0) ? qc0 : ((gy == 1) ? gm : T(0));
          const T gl = (gy == H - 1) ? qc0 : ((gy == H - 2) ? gp : T(0));
          const T t0 = diff_adj1(gm, gp, gf, gl, gy, H);
          const T hm = (gx > 0) ? q1(i - 1) : T(0);
          const T hp = (gx < W - 1) ? q1(i + 1) : T(0);
          const T hf = (gx == 0) ? qc1 : ((gx == 1) ? hm : T(0));
          const T hl = (gx == W - 1) ? qc1 : ((gx == W - 2) ? hp : T(0));
          const T t1 = diff_adj1(hm, hp, hf, hl, gx, W);
          ib_o[q] = pre_b[jj][ii] + (t0 + t1);
        }
      }
    }
    }
    __syncthreads();
    // ---- shift the ring by ADV rows (float4 copies, bands that never overlap) ----
    const int keep_lo = yc0 + ADV - R;  // first row needed by the next block
    constexpr int drop = ADV;           // == keep_lo - ring_lo
    constexpr int keep = G + 2 * R - ADV;  // == next_u - keep_lo
#pragma unroll
    for (int band = 0; band < keep; band += drop) {
      const int nrow = (keep - band) < drop ? (keep - band) : drop;
      for (int t = tid; t < nrow * 2 * (OX / 4); t += kAdjStreamThreads) {
        const int q4 = t % (OX / 4), rest = t / (OX / 4);
        const int c = rest & 1, rr = band + (rest >> 1);
        float4* dst = reinterpret_cast<float4*>(ring + c * RING * RP + rr * RP) + q4;
        *dst = *(reinterpret_cast<const float4*>(ring + c * RING * RP + (rr + drop) * RP) + q4);
      }
      __syncthreads();
    }
    ring_lo = keep_lo;
    if (tid == 0 && next_u < H) {  // the next block's first group
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue_v(next_u);
    }
  }
  if (REG) {
    unsigned all = __reduce_or_sync(0xffffffffu, bad);
    if (all && lane == 0) atomicOr(reinterpret_cast<int*>(a.flags + b), 1);
  }
}

}  // namespace mr
