// dgm_tc.cuh -- fused Maxwell stage kernel on the 5th-gen tensor cores (fp32 via 3xTF32).
//
// The whole semidiscrete RHS of one component c is a single GEMM row per
// element (oracle.py:67-93 regrouped):
//
//   rhs_c = sum_mu D_mu w_mu^(c) + LIFT f^(c)
//   w_mu^(c) = (sum over the curl's two terms of +-rx[mu][nu] u_g) / (eps|mu)
//   f^(c)    = upwind_bracket_c * face_jacobian / det_J / (eps|mu)
//
// because d/dx_nu u = sum_mu rx[mu][nu] D_mu u and rx is constant per element.
// So with A[e][k] = [w_0 | w_1 | w_2 | pad | f_face0 | .. | f_face3] and the
// constant B[n][k] = [D_0 | D_1 | D_2 | 0 | LIFT_face0 | .. ] (rows n = output
// node; every face block padded to NFPK = ceil8(Nfp) so a flux K-step never
// straddles two faces), one tcgen05.mma chain per component computes the full
// RHS of 128 elements (M = 128 TMEM lanes, one element per lane).  fp32
// accuracy comes from 3xTF32 (A_hi B_hi + A_lo B_hi + A_hi B_lo), exact splits.
//
// Roles (544 threads, one CTA per SM, persistent over 128-element tiles):
//   warps 0-15 producers.
//     A K-step: thread-per-row (row = TMEM lane); warp w serves lane quadrant
//     w%4, component group (w/8: E components from H fields, or H components
//     from E fields) and K half ((w/4)%2); tcgen05.st of hi and lo parts into
//     a 2-stage A ring in TMEM.
//     Surface flux: once per face (all NFPK node slots, 2 K-steps at N=3,4),
//     node-major mapping (NFPK lanes per element row, coalesced neighbour
//     gathers, all loads in flight before any use) into smem staging.
//     Epilogue: per component, one quadrant-complete warp group moves the
//     accumulator TMEM -> smem (double-buffered) while all producers apply the
//     LSRK update of the previous component with coalesced 16-B accesses; u
//     comes from the tile's smem rows, res was L2-prefetched at tile start.
//     After component c the smem slab of field c is released to the loader.
//   warp 16 (control, warp-uniform; one elected lane issues):
//     cp.async.bulk of each tile's geometry / connectivity rows (as soon as
//     the producers finish the K-loop) and field slabs (as soon as the
//     epilogue releases them), L2 prefetch of the residual, of the next tile
//     and of every out-of-tile face neighbour's rows, the B operand ring (two
//     K-steps ahead), and the 18 MMAs of each K-step as one burst.
// TMEM: [0, 6*NB) accumulators; two A stages of 6 x (8 hi + 8 lo) columns.
#pragma once

#include "dgm_stage.cuh"
#include "tc05.cuh"

namespace dgm {

#ifdef DGM_TC_TRACE
// Test-only phase timeline of CTA 0 (libdgm_trace.so): two tracing threads
// (producer tid 0, control warp) append (tag, clock64) to their own global
// slice with plain stores; no atomics on the timed path.
__device__ long long g_tc_trace[2][2 * 4096];
__device__ int g_tc_trace_n[2];
#define TC_TRACE_DECL int tc_tn = 0
#define TC_TRACE(who, tag)                                     \
  do {                                                         \
    if (blockIdx.x == 0 && tc_tn < 4096) {                     \
      g_tc_trace[who][2 * tc_tn] = (tag);                      \
      g_tc_trace[who][2 * tc_tn + 1] = clock64();              \
      ++tc_tn;                                                 \
      g_tc_trace_n[who] = tc_tn;                               \
    }                                                          \
  } while (0)
#else
#define TC_TRACE_DECL \
  do {                \
  } while (0)
#define TC_TRACE(who, tag) \
  do {                     \
  } while (0)
#endif

template <int N>
struct TcCfg {
  using C = Cfg<N, float>;
  static constexpr int NP = C::NP, NFP = C::NFP, NF4 = C::NF4, NPG = C::NPG;
  static constexpr int NPK = (NP + 3) / 4 * 4;     // K extent of one volume block
  static constexpr int NFPK = (NFP + 7) / 8 * 8;   // K extent of one face block
  static constexpr int NB = (NP + 15) / 16 * 16;   // MMA N (M=128, A in TMEM: N % 16 == 0)
  static constexpr int KV = (3 * NPK + 7) / 8 * 8; // volume part of K, padded to a K step
  static constexpr int KT = KV + 4 * NFPK;
  static constexpr int KS = KT / 8;                // K steps (one kind::tf32 MMA each)
  static constexpr int TE = 128;
  static constexpr int PWARPS = 16;
  static constexpr int PROD = 32 * PWARPS;         // producer threads
  static constexpr int THREADS = PROD + 32;
  static constexpr int ACC_COLS = 6 * NB;
  static constexpr int A_COL0 = (ACC_COLS + 31) / 32 * 32;
  static constexpr int A_STAGE_COLS = 6 * 16;      // 6 components x (8 hi + 8 lo)
  static constexpr int TMEM_COLS = 512;
  static_assert(A_COL0 + 2 * A_STAGE_COLS <= TMEM_COLS, "TMEM budget");
  static constexpr int SROW = TE + 4;              // flux staging row stride
  static constexpr int B_STEP_BYTES = 2 * 2 * NB * 16;   // hi/lo x 2 chunks x NB rows x 16 B
  static constexpr int NBS = 4;                    // B ring slots (two K-steps ahead of the MMAs)
  static constexpr uint32_t ROWS_BYTES = TE * NPG * 4;   // one field slab of one tile
  static constexpr int ITEMS = TE * NFPK / PROD;   // (row, face node) flux items per thread
  static_assert(ITEMS * PROD == TE * NFPK, "flux items must tile the producers");
  // shared-memory carve-up (bytes)
  static constexpr size_t OFF_U = 0;
  static constexpr size_t OFF_GEO = OFF_U + (size_t)6 * ROWS_BYTES;
  static constexpr size_t OFF_NBR = OFF_GEO + (size_t)TE * GEO_WORDS * 4;
  static constexpr size_t OFF_CODE = OFF_NBR + (size_t)TE * 4 * 4;
  static constexpr size_t OFF_B = OFF_CODE + (size_t)TE * 4 * 4;
  static constexpr size_t FLUX_BYTES = (size_t)6 * NFPK * SROW * 4;
  static constexpr size_t EPI_BYTES = (size_t)2 * ROWS_BYTES;
  static constexpr size_t OFF_STAGE = OFF_B + (size_t)NBS * B_STEP_BYTES;
  static constexpr size_t OFF_BAR = OFF_STAGE + (FLUX_BYTES > EPI_BYTES ? FLUX_BYTES : EPI_BYTES);
  static constexpr size_t OFF_FMASK = OFF_BAR + 256;  // 17 mbarriers + TMEM base address
  static constexpr size_t OFF_PTAB = OFF_FMASK + (4 * NFP + 15) / 16 * 16;
  static constexpr size_t SMEM_FIXED = OFF_PTAB;   // + ncodes * NFP
  static constexpr size_t B_FLOATS = (size_t)KS * 2 * 2 * NB * 4;  // packed operand in global
};

struct TcArgs {
  StageArgs<float> s;
  const float* bpack;  // [KS][hi,lo][2 chunks][NB][4]
  int num_tiles;
};

template <int N, int MODE>
__global__ void __launch_bounds__(TcCfg<N>::THREADS, 1) tc_stage_kernel(const TcArgs args) {
  using T = TcCfg<N>;
  using namespace tc;
  constexpr int TE = T::TE, NPG = T::NPG, NP = T::NP, NFP = T::NFP, NB = T::NB, NFPK = T::NFPK;
  constexpr int KS = T::KS, KV = T::KV, NPK = T::NPK, SROW = T::SROW, PROD = T::PROD, NBS = T::NBS;
  constexpr int ITEMS = T::ITEMS;
  const StageArgs<float>& a = args.s;

  extern __shared__ __align__(1024) unsigned char smem[];
  float* s_u = reinterpret_cast<float*>(smem + T::OFF_U);
  float* s_geo = reinterpret_cast<float*>(smem + T::OFF_GEO);
  int* s_nbr = reinterpret_cast<int*>(smem + T::OFF_NBR);
  int* s_code = reinterpret_cast<int*>(smem + T::OFF_CODE);
  unsigned char* s_b = smem + T::OFF_B;
  float* s_stage = reinterpret_cast<float*>(smem + T::OFF_STAGE);  // flux of one face | 2 epilogue rows buffers
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
  uint64_t* full = bar + 0;        // [2] producers -> MMA (A stage written)
  uint64_t* empty = bar + 2;       // [2] MMA commit -> A stage / B slot reusable
  uint64_t* load_full = bar + 4;   // tile rows landed
  uint64_t* acc_full = bar + 5;    // accumulators final
  uint64_t* tile_free = bar + 6;   // producers finished the K-loop (geometry / connectivity reusable)
  uint64_t* slab_free = bar + 7;   // [6] epilogue finished reading field slab c
  uint64_t* b_full = bar + 13;     // [NBS] B ring slot landed
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bar + 17);
  uint8_t* s_fmask = smem + T::OFF_FMASK;
  uint8_t* s_ptab = smem + T::OFF_PTAB;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t fstride = a.kf * NPG;

  if (warp == 0) tmem_alloc(s_tmem, T::TMEM_COLS);
  if (tid == PROD) {
    mbar_init(&full[0], T::PWARPS);
    mbar_init(&full[1], T::PWARPS);
    mbar_init(&empty[0], 1);
    mbar_init(&empty[1], 1);
    mbar_init(load_full, 1);
    mbar_init(acc_full, 1);
    mbar_init(tile_free, T::PWARPS);
    for (int c = 0; c < 6; ++c) mbar_init(&slab_free[c], 1);
    for (int i = 0; i < NBS; ++i) mbar_init(&b_full[i], 1);
    mbar_init_fence();
  }
  for (int c = tid; c < 4 * NFP; c += blockDim.x) s_fmask[c] = a.fmask[c];
  for (int c = tid; c < a.ncodes * NFP; c += blockDim.x) s_ptab[c] = a.ptab[c];
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = *s_tmem;
  TC_TRACE_DECL;

  if (warp == T::PWARPS) {
    // ================= control warp =================
    const uint32_t idesc = idesc_tf32(128, NB);
    const int my_tiles =
        (int)blockIdx.x < args.num_tiles ? (args.num_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const uint32_t total_steps = (uint32_t)my_tiles * KS;
    auto load_b = [&](uint32_t step) {  // B operand of global K-step `step` into its ring slot
      if (step >= total_steps) return;
      const uint32_t slot = step % NBS;
      mbar_expect_tx(&b_full[slot], T::B_STEP_BYTES);
      bulk_g2s(s_b + slot * T::B_STEP_BYTES, args.bpack + (size_t)(step % KS) * (T::B_STEP_BYTES / 4),
               T::B_STEP_BYTES, &b_full[slot]);
    };
    if (elect_one()) {
      load_b(0);
      load_b(1);
    }
    __syncwarp();
    uint32_t g = 0;  // global K-step counter
    int it = 0;
    for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x, ++it) {
      const int64_t e0 = a.e_begin + (int64_t)tile * TE;
      const int nv = (int)min((int64_t)TE, a.e_end - e0);
      const uint32_t rowbytes = (uint32_t)nv * NPG * 4;
      // ---- this tile's rows: geometry/connectivity once the K-loop of the previous tile is done,
      //      each field slab once the previous tile's epilogue released it ----
      if (it > 0) mbar_wait(tile_free, (it - 1) & 1);
      if (elect_one()) {
        const uint32_t geobytes = (uint32_t)nv * GEO_WORDS * 4, conbytes = (uint32_t)nv * 16;
        mbar_expect_tx(load_full, 6 * rowbytes + geobytes + 2 * conbytes);
        bulk_g2s(s_geo, a.geo + e0 * GEO_WORDS, geobytes, load_full);
        bulk_g2s(s_nbr, a.nbr + e0 * 4, conbytes, load_full);
        bulk_g2s(s_code, a.code + e0 * 4, conbytes, load_full);
      }
      __syncwarp();
      for (int f = 0; f < 6; ++f) {
        if (it > 0) mbar_wait(&slab_free[f], (it - 1) & 1);
        if (elect_one()) bulk_g2s(s_u + f * TE * NPG, a.u + (int64_t)f * fstride + e0 * NPG, rowbytes, load_full);
        __syncwarp();
      }
      if (it < 4) TC_TRACE(1, 1000 * it + 400);  // tile loads issued
      if (elect_one()) {
        if (MODE == MODE_LSRK && !a.a_zero)
          for (int f = 0; f < 6; ++f) prefetch_l2(a.res + (int64_t)f * fstride + e0 * NPG, rowbytes);
        const int nt = tile + gridDim.x;  // warm L2 with the next tile of this CTA
        if (nt < args.num_tiles) {
          const int64_t n0 = a.e_begin + (int64_t)nt * TE;
          const uint32_t nn = (uint32_t)min((int64_t)TE, a.e_end - n0);
          for (int f = 0; f < 6; ++f) prefetch_l2(a.u + (int64_t)f * fstride + n0 * NPG, nn * NPG * 4);
          prefetch_l2(a.geo + n0 * GEO_WORDS, nn * GEO_WORDS * 4);
          prefetch_l2(a.nbr + n0 * 4, nn * 16);
          prefetch_l2(a.code + n0 * 4, nn * 16);
        }
      }
      __syncwarp();
      // ---- K loop: B ring two steps ahead, one MMA burst per step ----
      for (int s = 0; s < KS; ++s, ++g) {
        const int slot = g & 1;
        if (g >= 2) mbar_wait(&empty[slot], ((g - 2) >> 1) & 1);  // MMA(g-2) done: its B slot is free
        if (elect_one()) load_b(g + 2);
        __syncwarp();
        mbar_wait(&b_full[g % NBS], (g / NBS) & 1);
        mbar_wait(&full[slot], (g >> 1) & 1);
        if (it < 4) TC_TRACE(1, 1000 * it + 500 + 2 * s);  // stage full
        fence_after_sync();
        if (elect_one()) {
          const uint32_t bh = smem_u32(s_b + (g % NBS) * T::B_STEP_BYTES);
          const uint64_t dbh = desc_kmajor(bh, NB * 16, 128);
          const uint64_t dbl = desc_kmajor(bh + 2 * NB * 16, NB * 16, 128);
          const uint32_t abase = tmem + T::A_COL0 + slot * T::A_STAGE_COLS;
          const uint32_t acc0 = s > 0 ? 1u : 0u;
          // pass-major order: consecutive MMAs hit different accumulators
#pragma unroll
          for (int c = 0; c < 6; ++c) mma_tf32_ts(tmem + c * NB, abase + c * 16, dbh, idesc, acc0);
#pragma unroll
          for (int c = 0; c < 6; ++c) mma_tf32_ts(tmem + c * NB, abase + c * 16 + 8, dbh, idesc, 1u);
#pragma unroll
          for (int c = 0; c < 6; ++c) mma_tf32_ts(tmem + c * NB, abase + c * 16, dbl, idesc, 1u);
          mma_commit(&empty[slot]);
          if (s == KS - 1) mma_commit(acc_full);
        }
        __syncwarp();
      }
    }
    if (elect_one()) bulk_wait<0>();
    __syncwarp();
  } else {
    // ================= producers =================
    const int quad = warp & 3;               // TMEM lane quadrant
    const int khalf = (warp >> 2) & 1;       // which 4 of a K step's 8 columns
    const int grp = (warp >> 3) & 1;         // 0: E components (from H fields), 1: H components (from E fields)
    const int egrp = warp >> 2;              // epilogue: TMEM -> smem mover for components egrp, egrp + 4
    const int row = quad * 32 + lane;        // element row = TMEM lane
    const uint32_t lane_addr = static_cast<uint32_t>(quad * 32) << 16;
    const float inv_m = grp == 0 ? a.inv_eps : a.inv_mu;
    constexpr int RV = NPG / 4;              // 16-byte chunks per row
    constexpr int PER = (TE * RV + PROD - 1) / PROD;
    uint32_t pstep = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x, ++it) {
      const int64_t e0 = a.e_begin + (int64_t)tile * TE;
      const int nv = (int)min((int64_t)TE, a.e_end - e0);
      if (tid == 0 && it < 4) TC_TRACE(0, 1000 * it + 1);  // tile start
      mbar_wait(load_full, it & 1);
      if (tid == 0 && it < 4) TC_TRACE(0, 1000 * it + 2);  // rows landed

      {  // warm L2 with the rows of every face neighbour outside the tile (read by the face K-steps)
        const int e = tid;  // one (row, face) entry per producer thread
        if (e < nv * 4) {
          const int code = s_code[e];
          const int64_t nb = s_nbr[e];
          if (code >= 0 && (nb < e0 || nb >= e0 + nv)) {
#pragma unroll
            for (int f = 0; f < 6; ++f) {
              const float* p = a.u + (int64_t)f * fstride + nb * NPG;
              prefetch_line_l2(p);
              prefetch_line_l2(p + NPG - 1);
            }
          }
        }
      }
      const bool row_ok = row < nv;
      float prx[9];  // geometric factors of the owned row, pre-scaled by 1/eps or 1/mu
#pragma unroll
      for (int q = 0; q < 9; ++q) prx[q] = row_ok ? s_geo[row * GEO_WORDS + q] * inv_m : 0.f;

      for (int s = 0; s < KS; ++s, ++pstep) {
        const int slot = pstep & 1;
        const int k0 = s * 8;
        if (tid == 0 && it < 4) TC_TRACE(0, 1000 * it + 100 + 4 * s);  // step begin
        // ---- surface flux of a whole face at its first K-step ----
        if (k0 >= KV && (k0 - KV) % NFPK == 0) {
          const int face = (k0 - KV) / NFPK;
          named_sync(1, PROD);  // every thread finished reading the previous face's staging
          float up[ITEMS][6];
#pragma unroll
          for (int i = 0; i < ITEMS; ++i) {  // u+ gathers first: all loads in flight together
            const int item = tid + i * PROD;
            const int r = item / NFPK, node = item % NFPK;
            const bool live = node < NFP && r < nv;
            const int im = s_fmask[face * NFP + (node < NFP ? node : 0)];
            const float* src = s_u + r * NPG + im;  // PEC walls mirror the own trace below
            int64_t fs = TE * NPG;
            const int code = live ? s_code[r * 4 + face] : -1;
            if (code >= 0) {
              const int nb = s_nbr[r * 4 + face];
              const int jn = s_ptab[code * NFP + node];
              const int64_t loc = (int64_t)nb - e0;
              if (loc >= 0 && loc < nv) {
                src = s_u + (int)loc * NPG + jn;
              } else {
                src = a.u + (int64_t)nb * NPG + jn;
                fs = fstride;
              }
            }
#pragma unroll
            for (int f = 0; f < 6; ++f) up[i][f] = src[f * fs];
          }
#pragma unroll
          for (int i = 0; i < ITEMS; ++i) {
            const int item = tid + i * PROD;
            const int r = item / NFPK, node = item % NFPK;
            const bool live = node < NFP && r < nv;
            const int im = s_fmask[face * NFP + (node < NFP ? node : 0)];
            float um[6];
#pragma unroll
            for (int f = 0; f < 6; ++f) um[f] = s_u[(f * TE + r) * NPG + im];
            const float* gk = s_geo + r * GEO_WORDS;
            const float nx = gk[10 + 3 * face], ny = gk[11 + 3 * face], nz = gk[12 + 3 * face];
            if (live && s_code[r * 4 + face] < 0) {  // PEC mirror (maxwell.py:117-132)
              const float nde = nx * um[0] + ny * um[1] + nz * um[2];
              const float ndh = nx * um[3] + ny * um[4] + nz * um[5];
              up[i][0] = -um[0] + 2.f * nde * nx;
              up[i][1] = -um[1] + 2.f * nde * ny;
              up[i][2] = -um[2] + 2.f * nde * nz;
              up[i][3] = um[3] - 2.f * ndh * nx;
              up[i][4] = um[4] - 2.f * ndh * ny;
              up[i][5] = um[5] - 2.f * ndh * nz;
            }
            float out[6];
            upwind(um, up[i], nx, ny, nz, a, out);
            const float sc = live ? gk[22 + face] * gk[9] : 0.f;
            const float se = sc * a.inv_eps, sh = sc * a.inv_mu;
#pragma unroll
            for (int c = 0; c < 3; ++c) s_stage[(c * NFPK + node) * SROW + r] = out[c] * se;
#pragma unroll
            for (int c = 3; c < 6; ++c) s_stage[(c * NFPK + node) * SROW + r] = out[c] * sh;
          }
          named_sync(1, PROD);
          if (tid == 0 && it < 4) TC_TRACE(0, 1000 * it + 103 + 4 * s);  // face flux staged
        }

        // ---- A K-step (this warp's 4 columns, 3 components) into TMEM, thread-per-row ----
        float v[3][4];
        {
          const int k = k0 + 4 * khalf;
          if (k < 3 * NPK) {
            const int mu = k / NPK, j0 = k - mu * NPK;
            const float p0 = prx[mu * 3 + 0], p1 = prx[mu * 3 + 1], p2 = prx[mu * 3 + 2];
            const int fb = grp == 0 ? 3 : 0;  // E comps read H fields and vice versa
            const float4 x = *reinterpret_cast<const float4*>(s_u + ((fb + 0) * TE + row) * NPG + j0);
            const float4 y = *reinterpret_cast<const float4*>(s_u + ((fb + 1) * TE + row) * NPG + j0);
            const float4 z = *reinterpret_cast<const float4*>(s_u + ((fb + 2) * TE + row) * NPG + j0);
            const float xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w}, zs[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (grp == 0) {  // (curl H)_x,y,z
                v[0][q] = p1 * zs[q] - p2 * ys[q];
                v[1][q] = p2 * xs[q] - p0 * zs[q];
                v[2][q] = p0 * ys[q] - p1 * xs[q];
              } else {         // -(curl E)_x,y,z
                v[0][q] = p2 * ys[q] - p1 * zs[q];
                v[1][q] = p0 * zs[q] - p2 * xs[q];
                v[2][q] = p1 * xs[q] - p0 * ys[q];
              }
            }
          } else if (k >= KV) {
            const int node = (k - KV) % NFPK;
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int c = 0; c < 3; ++c) v[c][q] = s_stage[((3 * grp + c) * NFPK + node + q) * SROW + row];
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int c = 0; c < 3; ++c) v[c][q] = 0.f;
          }
        }
        float hi[3][4], lo[3][4];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int q = 0; q < 4; ++q) split_tf32(row_ok ? v[c][q] : 0.f, hi[c][q], lo[c][q]);
        if (tid == 0 && it < 4) TC_TRACE(0, 1000 * it + 101 + 4 * s);  // A values ready
        mbar_wait(&empty[slot], ((pstep >> 1) & 1) ^ 1);
        if (tid == 0 && it < 4) TC_TRACE(0, 1000 * it + 102 + 4 * s);  // stage free
        fence_after_sync();
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const uint32_t col = T::A_COL0 + slot * T::A_STAGE_COLS + (3 * grp + c) * 16 + 4 * khalf;
          tmem_st4(tmem + lane_addr + col, hi[c]);
          tmem_st4(tmem + lane_addr + col + 8, lo[c]);
        }
        tmem_st_wait();
        fence_before_sync();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&full[slot]);
          if (s == KS - 1) mbar_arrive(tile_free);  // geometry / connectivity may be refilled
        }
      }

      // ================= epilogue: accumulators -> LSRK update =================
      if (tid == 0 && it < 4) TC_TRACE(0, 1000 * it + 3);  // all steps produced
      mbar_wait(acc_full, it & 1);
      if (tid == 0 && it < 4) TC_TRACE(0, 1000 * it + 4);  // accumulators final
      fence_after_sync();
      // TMEM -> smem rows buffer (thread-per-row), done by one quadrant-complete warp group
      auto move_acc = [&](int comp) {
        float* dst = s_stage + (size_t)(comp & 1) * TE * NPG + row * NPG;
#pragma unroll
        for (int c0 = 0; c0 < NB; c0 += 8) {
          float r8[8];
          tmem_ld8(tmem + lane_addr + comp * NB + c0, r8);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 8; q += 4) {
            const int i = c0 + q;
            if (i < NPG) {
              float4 o;
              o.x = (i + 0 < NP) ? r8[q + 0] : 0.f;
              o.y = (i + 1 < NP) ? r8[q + 1] : 0.f;
              o.z = (i + 2 < NP) ? r8[q + 2] : 0.f;
              o.w = (i + 3 < NP) ? r8[q + 3] : 0.f;
              *reinterpret_cast<float4*>(dst + i) = o;
            }
          }
        }
      };
      const int nvec = nv * RV;
      auto load_res = [&](int comp, float4* ro) {
#pragma unroll
        for (int p = 0; p < PER; ++p) {
          const int c = tid + p * PROD;
          ro[p] = (MODE == MODE_LSRK && !a.a_zero && c < nvec)
                      ? __ldcs(reinterpret_cast<const float4*>(a.res + ((int64_t)comp * a.kf + e0) * NPG) + c)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      float4 ro[PER], rn[PER];
      if (egrp == 0) move_acc(0);
      load_res(0, ro);
      named_sync(1, PROD);
#pragma unroll 1
      for (int comp = 0; comp < 6; ++comp) {
        if (comp + 1 < 6) {
          if (egrp == ((comp + 1) & 3)) move_acc(comp + 1);
          load_res(comp + 1, rn);
        }
        const float4* rs = reinterpret_cast<const float4*>(s_stage + (size_t)(comp & 1) * TE * NPG);
        const float4* us = reinterpret_cast<const float4*>(s_u + (size_t)comp * TE * NPG);
        const int64_t gbase = ((int64_t)comp * a.kf + e0) * NPG;
#pragma unroll
        for (int p = 0; p < PER; ++p) {
          const int c = tid + p * PROD;
          if (c < nvec) {
            const float4 rh = rs[c];
            if (MODE == MODE_RHS) {
              *reinterpret_cast<float4*>(a.out + gbase + (int64_t)c * 4) = rh;
            } else {
              float4 r;
              if (a.a_zero) {
                r = make_float4(a.dt * rh.x, a.dt * rh.y, a.dt * rh.z, a.dt * rh.w);
              } else {
                r = make_float4(a.a * ro[p].x + a.dt * rh.x, a.a * ro[p].y + a.dt * rh.y,
                                a.a * ro[p].z + a.dt * rh.z, a.a * ro[p].w + a.dt * rh.w);
              }
              const float4 uo = us[c];
              __stcs(reinterpret_cast<float4*>(a.res + gbase) + c, r);
              __stcs(reinterpret_cast<float4*>(a.u_out + gbase) + c,
                     make_float4(uo.x + a.b * r.x, uo.y + a.b * r.y, uo.z + a.b * r.z, uo.w + a.b * r.w));
            }
          }
        }
        named_sync(1, PROD);  // rows buffer `comp & 1` and field slab `comp` fully read
        if (tid == 0) mbar_arrive(&slab_free[comp]);
#pragma unroll
        for (int p = 0; p < PER; ++p) ro[p] = rn[p];
      }
      if (tid == 0 && it < 4) TC_TRACE(0, 1000 * it + 5);  // epilogue done
      fence_before_sync();
    }
  }
  __syncthreads();
  fence_after_sync();
  if (warp == 0) tmem_dealloc(tmem, T::TMEM_COLS);
}

}  // namespace dgm
