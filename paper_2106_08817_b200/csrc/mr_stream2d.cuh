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
  static constexpr int RP = OX + 1;       // ring pitch (odd)
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
        // ---- horizontal FIR of the new rows -> ring (lanes <-> rows) ----
        constexpr int NB = OX / kRB;
        for (int cb = warp; cb < 2 * NB; cb += kNW) {
          const int r = lane;
          if (r >= cin) continue;
          const int ib = cb % NB, c = cb / NB;
          const T* src = P + c * G * PP + r * PP + ib * kRB;
          T acc[kRB];
#pragma unroll
          for (int o = 0; o < kRB; ++o) acc[o] = T(0);
#pragma unroll
          for (int t = 0; t < kRB + 2 * R; ++t) {
            const T x = src[t];
#pragma unroll
            for (int o = 0; o < kRB; ++o) {
              const int tap = t - o;
              if (tap >= 0 && tap <= 2 * R) acc[o] = fma(tp.w[tap], x, acc[o]);
            }
          }
          T* dst = ring + c * RING * RP + (u0 + r - ring_lo) * RP + ib * kRB;
#pragma unroll
          for (int o = 0; o < kRB; ++o) dst[o] = acc[o];
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

    // ---- vertical FIR over the ring for output rows [y0, y0+G) (lanes <-> columns) ----
    constexpr int NBV = G / kRB;
    for (int cb = warp; cb < 2 * NBV; cb += kNW) {
      const int jb = cb % NBV, c = cb / NBV;
      for (int i = lane; i < OX; i += 32) {
        const T* src = ring + c * RING * RP + (y0 + jb * kRB - R - ring_lo) * RP + i;
        T acc[kRB];
#pragma unroll
        for (int o = 0; o < kRB; ++o) acc[o] = T(0);
#pragma unroll
        for (int t = 0; t < kRB + 2 * R; ++t) {
          const T x = src[t * RP];
#pragma unroll
          for (int o = 0; o < kRB; ++o) {
            const int tap = t - o;
            if (tap >= 0 && tap <= 2 * R) acc[o] = fma(tp.w[tap], x, acc[o]);
          }
        }
        const int gx = x0 + i;
        if (gx < W) {
          T* vo = (c == 0 ? v0 : v1) + gx;
#pragma unroll
          for (int o = 0; o < kRB; ++o) {
            const int gy = y0 + jb * kRB + o;
            if (gy < H) {
              const T val = -acc[o];
              vo[(long long)gy * W] = val;
              flags |= guard_bits(val, MR_GUARD_VELOCITY_NONFINITE);
            }
          }
        }
      }
    }
    __syncthreads();
    // ---- shift: keep ring rows [y0+G-R, next_u) at the front ----
    const int keep_lo = y0 + G - R;
    const int drop = keep_lo - ring_lo;  // == G
    const int keep = next_u - keep_lo;   // == 2R (<= RING - G)
    for (int band = 0; band < keep; band += drop) {
      const int nrow = min(drop, keep - band);
      for (int j = warp; j < 2 * nrow; j += kNW) {
        const int c = j / nrow, rr = band + j % nrow;
        for (int i = lane; i < OX; i += 32)
          ring[c * RING * RP + rr * RP + i] = ring[c * RING * RP + (rr + drop) * RP + i];
      }
      __syncthreads();
    }
    ring_lo = keep_lo;
  }
  if (a.guard) flush_flags(flags, a.guard + (long long)b * a.guard_stride);
}

}  // namespace mr
