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
// So with A[row][k] = [w_0 | w_1 | w_2 | pad | f_face0 | .. | f_face3] and the
// constant B[n][k] = [D_0 | D_1 | D_2 | 0 | LIFT_face0 | .. ] (rows n = output
// node; every face block padded to NFPK = ceil8(Nfp) so a flux K-step never
// straddles two faces), tcgen05.mma chains compute the full RHS.  fp32
// accuracy comes from 3xTF32 (A_hi B_hi + A_lo B_hi + A_hi B_lo), exact splits.
//
// Tiling: a CTA owns TE = 64 consecutive elements.  The 6 x 64 GEMM rows are
// three M = 128 tiles; M-tile t holds component t (E_t) of the 64 elements in
// TMEM lanes 0-63 and component t+3 (H_t) in lanes 64-127, so every MMA is a
// full 128-lane instruction and a CTA needs only 3*NB accumulator columns plus
// a 2-stage A ring (<= 256 TMEM columns) and ~103 KB of shared memory at N=4:
// two CTAs share an SM and hide each other's gather / barrier latencies.
//
// Roles (320 threads):
//   warps 0-7 producers, thread-per-TMEM-lane: warp w serves lane quadrant
//     q = w%4 (lanes 32q..32q+31: element (q%2)*32 + lane, E components for
//     q < 2, H components for q >= 2) and K half w/4.
//     A K-step: 4 columns x 3 M-tiles, tcgen05.st of the tf32 hi and lo parts.
//     Surface flux: once per face (all NFPK node slots), node-major mapping
//     (coalesced neighbour gathers, all loads in flight before any use) into
//     smem staging that the face K-steps read.
//     Epilogue per M-tile: quadrant warps move the accumulator TMEM -> smem,
//     then all producers apply the LSRK update with coalesced 16-B accesses
//     (u from the tile's smem rows, res L2-prefetched at CTA start).
//   warp 8 (MMA, warp-uniform; one elected lane issues): the 9 MMAs of each
//     K-step as one burst, committed to the A stage's `empty` barrier.
//   warp 9 (loader): cp.async.bulk of the tile's rows (one mbarrier with a tx
//     count), L2 prefetch of the residual, and the B operand ring (BAHEAD
//     K-steps ahead, a slot refilled once the MMAs that read it completed) --
//     kept off the MMA warp because bulk-copy issue can stall on the TMA queue.
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
#elif defined(DGM_TC_TIMING)
// Test-only phase timing of every CTA (libdgm_timing.so): producer thread 0 stores 5 clock64 stamps.
__device__ long long g_tc_phase[1 << 16][5];
#define TC_TRACE_DECL \
  do {                \
  } while (0)
#define TC_TRACE(who, tag)                                                          \
  do {                                                                              \
    if ((who) == 0 && (tag) >= 1 && (tag) <= 5 && blockIdx.x < (1u << 16))          \
      g_tc_phase[blockIdx.x][(tag) - 1] = clock64();                                \
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
  // Lane mapping.  MAP 0 (N <= 4, 6): 64 elements per CTA, M-tile t = [E_t of the 64 elements |
  // H_t of the 64 elements].  MAP 1 (N = 7, 8, where a 64-element u tile no longer fits in smem),
  // M-tiles component-major: N=8, 32 elements per CTA, tile 0 = [E_x | E_y | E_z | H_x], tile 1 =
  // [H_y | H_z | pad | pad] (32 lanes per component); N=5, 7, 42 elements, tile 0 = [E_x | E_y | E_z],
  // tile 1 = [H_x | H_y | H_z] (42 lanes per component, 2 pad lanes).
  // MAP 2 (N = 9): TE = 21 elements per CTA, one M-tile holding all six components, lane = TE c + e
  // (126 of 128 lanes used).
#ifdef DGM_TC_N4_SMALL
  // Experiment knob (measured 2.73 ms vs 1.63 ms per C3 stage): N=4 on 16-element CTAs
  // with 4 producer warps (both K halves per thread) and 3 CTAs per SM.
  static constexpr bool SMALL = N == 4;
#else
  static constexpr bool SMALL = false;
#endif
  // N=5 on the 42-element three-component MAP 1 tiles at two CTAs per SM (TMEM 128 + 4 x 32 columns,
  // 107 KB smem, role-based registers) instead of one 64-element MAP 0 CTA: C2 N=5 168.5 -> 139.1 us
  // per stage, -12 % at 547k tets (profiles/r02/ab_n5_map1.txt); -DDGM_TC_N5_MAP0 restores MAP 0
#ifdef DGM_TC_N5_MAP0
  static constexpr bool N5M1 = false;
#else
  static constexpr bool N5M1 = N == 5 && !SMALL;
#endif
  static constexpr int MAP = SMALL ? 2 : (N5M1 ? 1 : (N <= 6 ? 0 : (N <= 8 ? 1 : 2)));
#ifdef DGM_TC_INLINE_FLUX
  // experiment: each producer computes its own face values inside the K-loop (no flux passes)
  static constexpr bool INLINE_FLUX = MAP == 0;
#else
  static constexpr bool INLINE_FLUX = false;
#endif
  // MAP 2 tile: 21 elements fill 126 of the 128 lanes (16 used 96: C2 N=9 917 -> 816 us per stage,
  // profiles/r02/ab_map2_te21.txt); DGM_TC_TE9 overrides it for experiments
#ifdef DGM_TC_TE9
  static constexpr int TE_MAP2 = SMALL ? 16 : DGM_TC_TE9;
#else
  static constexpr int TE_MAP2 = SMALL ? 16 : 21;
#endif
  // MAP 1 tile at N=7: 42 elements, three components per M-tile (252 of 256 lanes; 32 elements used
  // 192: C2 N=7 439 -> 384 us per stage, profiles/r02/ab_map1_te42.txt); N=8 has no shared memory for
  // more than 32.  DGM_TC_TE7 overrides it for experiments
#ifdef DGM_TC_TE7
  static constexpr int TE_MAP1 = (N == 7 || N5M1) ? DGM_TC_TE7 : 32;
#else
  static constexpr int TE_MAP1 = (N == 7 || N5M1) ? 42 : 32;
#endif
  // MAP 1 with TE != 32: three components per M-tile (tile t = components 3t..3t+2, lane = TE c' + e)
  static constexpr bool M1C3 = MAP == 1 && TE_MAP1 != 32;
  static constexpr int TE = MAP == 0 ? 64 : (MAP == 1 ? TE_MAP1 : TE_MAP2);  // elements per CTA
  static constexpr int MT = MAP == 0 ? 3 : (MAP == 1 ? 2 : 1);     // M-tiles
#if defined(DGM_TC_WIDE_MASK)
  // experiment knob: bit N set -> 16 producer warps with 2 K-columns per thread at order N
  static constexpr bool WIDE = ((DGM_TC_WIDE_MASK) >> N) & 1;
#elif defined(DGM_TC_W16)
  static constexpr bool WIDE = N <= 4;   // experiment: 16 producer warps, 2 K-columns per thread
#else
  static constexpr bool WIDE = false;
#endif
  // producer warps: 4 lane quadrants x NQ column groups
  static constexpr int PWARPS = SMALL ? 4 : (WIDE ? 16 : 8);
  static constexpr int NQ = PWARPS / 4;            // producer warps per lane quadrant
  static constexpr int CW = PWARPS == 16 ? 2 : 4;  // K columns per group (tcgen05.st width)
  static constexpr int KH = 8 / CW / NQ;           // column groups per producer thread and K-step
  static constexpr int FB = PWARPS == 16 ? 2 : 4;  // face nodes per flux work unit
  static constexpr int PROD = 32 * PWARPS;         // producer threads
#ifdef DGM_TC_MERGE
  // experiment: the loader's work in the MMA warp at 2 CTAs/SM (9 warps per CTA: 112 registers)
  static constexpr bool MERGE = !SMALL && N <= 4;  // the CTAS == 2 kernels
#else
  static constexpr bool MERGE = false;
#endif
  // Role-based registers at 2 CTAs/SM (setmaxnreg): a 12-warp CTA (warpgroup 2 = MMA, loader and two
  // idle warps) launches at 80 registers per thread; warpgroup 2 drops to REG_AUX and the producers
  // rise to REG_PROD = 104 (from the 96 of a 10-warp CTA), which holds the incremental K-step counters
  // and the packed fp32x2 build without spills: C3 1369 -> 1358 us per stage, N=3 60.7 -> 59.4
  // (profiles/r02/ab_rreg.txt); -DDGM_TC_NO_RREG restores the 10-warp CTA
#ifdef DGM_TC_NO_RREG
  static constexpr bool RREG = false;
#else
  static constexpr bool RREG = !SMALL && !MERGE && (N <= 4 || N5M1) && PWARPS == 8;
#endif
  static constexpr int REG_AUX = 32, REG_PROD = 104;
  // flux pass: u+ of in-tile and out-of-tile neighbours through one generic-address load path
  // (A/B, profiles/r02/ab_generic_up.txt: N=4 -0.35 %, N=5 -0.6 %, N=3 +0.7 %, N=6 +0.9 %)
#ifdef DGM_TC_GENERIC_UP
  static constexpr bool GENERIC_UP = true;
#else
  static constexpr bool GENERIC_UP = N == 4 || N == 5;
#endif
  // packed fp32x2 A-operand build and tf32 split (FMUL2 / FFMA2 / FADD2): measured per order against
  // the scalar form (profiles/r02/ab_f32x2.txt): N=2 -3.6 %, N=3, 5, 6 within 0.6 %, N=4 +5.7 %
  // (12 B of spills at the 96-register cap); with the role-based registers (104, no spills) N=3 -1.5 %,
  // N=4 -0.4 %, N=6 +0.6 % (profiles/r02/ab_rreg.txt): on where it wins, everywhere with DGM_TC_F32X2
#ifdef DGM_TC_F32X2
  static constexpr bool F32X2 = MAP == 0;
#else
  static constexpr bool F32X2 = N == 2 || RREG;
#endif
  static constexpr int THREADS = PROD + (MERGE ? 32 : (RREG ? 128 : 64));  // + MMA warp (+ loader warp)
  static constexpr int ACC_COLS = MT * NB;
  static constexpr int A_COL0 = (ACC_COLS + 31) / 32 * 32;
  static constexpr int A_STAGE_COLS = MT * 16;     // M-tiles x (8 hi + 8 lo)
  static constexpr int CTAS = SMALL ? 3 : ((N <= 4 || N5M1) ? 2 : 1);  // CTAs per SM (TMEM and smem split between them)
  static constexpr int TMEM_COLS = CTAS == 3 ? 128 : 512 / CTAS;  // power of two
  static constexpr int AST0 = (TMEM_COLS - A_COL0) / A_STAGE_COLS;
  static constexpr int AST = AST0 > 6 ? 6 : AST0;   // A ring stages in TMEM
  static_assert(AST >= 2, "TMEM budget");
  // flux staging row stride TE + pad: the pad minimises the shared-bank multiplicity of the flux
  // pass stores (lanes = (row, node block) units) plus the MAP 2 staging reads (two components
  // per warp); TE + 4 had 2-way (N=3,4) up to 7-way (N=9) store conflicts
  static constexpr int bank_mult(const int* addr, int n) {
    int cnt[32] = {}, m = 0;
    for (int i = 0; i < n; ++i) {
      const int b = addr[i] % 32;
      m = ++cnt[b] > m ? cnt[b] : m;
    }
    return m;
  }
  static constexpr int srow_cost(int pad) {  // x NBF: integer arithmetic
    const int S = TE + pad, NBF = NFPK / FB;
    int tot = 0, warps = 0;
    for (int w = 0; w < NBF; ++w) {
      int addr[32] = {}, n = 0;
      for (int u = w * 32; u < w * 32 + 32; ++u)
        if (u / NBF < TE) addr[n++] = (u % NBF) * FB * S + u / NBF;
      if (n) tot += bank_mult(addr, n), ++warps;
    }
    int rd = 1;
    if (MAP == 2) {
      int addr[32] = {};
      for (int l = 0; l < 32; ++l) addr[l] = (l / TE) * NFPK * S + (l % TE);
      rd = bank_mult(addr, 32);
    } else if (M1C3) {  // staging reads of the four quadrants (lane 32 q + l: component slot, row)
      int r4 = 0;
      for (int q = 0; q < 4; ++q) {
        int addr[32] = {}, n = 0;
        for (int l = 0; l < 32; ++l)
          if ((32 * q + l) / TE < 3) addr[n++] = ((32 * q + l) / TE) * NFPK * S + (32 * q + l) % TE;
        r4 += n ? bank_mult(addr, n) : 0;
      }
      rd = (r4 + 3) / 4;
    }
    return (tot * 64) / warps + rd * 64;
  }
  static constexpr int srow_pad() {
    int best = 0;
    for (int p = 1; p < 32; ++p)
      if (srow_cost(p) < srow_cost(best)) best = p;
    return best;
  }
#ifdef DGM_TC_SROW_OLD
  static constexpr int SROW = TE + 4;  // experiment: the previous fixed padding
#else
  static constexpr int SROW = TE + srow_pad();
#endif
  static constexpr int B_STEP_BYTES = 2 * 2 * NB * 16;   // hi/lo x 2 chunks x NB rows x 16 B
  static constexpr int NBS = (N <= 5 && !N5M1) ? 6 : 4;       // B ring slots (a slot is refilled when its MMAs complete)
  static constexpr uint32_t ROWS_BYTES = TE * NPG * 4;   // one field slab of the tile
  // shared-memory carve-up (bytes)
  static constexpr size_t OFF_U = 0;
  static constexpr size_t OFF_GEO = OFF_U + (size_t)6 * ROWS_BYTES;
  static constexpr size_t OFF_NBR = OFF_GEO + (size_t)TE * GEO_WORDS * 4;
  static constexpr size_t OFF_CODE = OFF_NBR + (size_t)TE * 4 * 4;
  static constexpr size_t OFF_B = (OFF_CODE + (size_t)TE * 4 * 4 + 127) / 128 * 128;
  // Flux staging layout.  Default: [component][face node][row] (row stride SROW), read as scalars.
  // FT (MAP 0, NFPK = 16, i.e. N = 3, 4): [component][row][4 node chunks of 16 B], the chunk index
  // XOR-swizzled by bits 1-2 of the row, so the flux pass writes and the A build reads one 16-byte
  // vector per (component, row, 4 nodes) and both are bank-conflict-free.  C3 1353 -> 1338 us per
  // stage; N=3 +0.3 % (profiles/r02/ab_flux_layout.txt), so N=4 only (DGM_TC_FT: N=3 too)
#ifdef DGM_TC_FT
  static constexpr bool FT = MAP == 0 && NFPK == 16 && FB == 4 && CW == 4;
#else
  static constexpr bool FT = MAP == 0 && NFPK == 16 && FB == 4 && CW == 4 && N == 4;
#endif
  __host__ __device__ static constexpr int ft_off(int c, int row, int nb) {  // float offset, FT layout
    return ((c * TE + row) * 4 + (nb ^ ((row >> 1) & 3))) * 4;
  }
  static constexpr size_t FLUX_BYTES = FT ? (size_t)6 * TE * 16 * 4 : (size_t)6 * NFPK * SROW * 4;
  static constexpr size_t EPI_BYTES = (size_t)2 * ROWS_BYTES;
  static constexpr size_t OFF_STAGE = OFF_B + (size_t)NBS * B_STEP_BYTES;
  static constexpr size_t OFF_BAR = OFF_STAGE + (FLUX_BYTES > EPI_BYTES ? FLUX_BYTES : EPI_BYTES);
  static constexpr size_t OFF_FMASK = OFF_BAR + 256;  // mbarriers + TMEM base address
  static constexpr size_t OFF_PTAB = OFF_FMASK + (4 * NFP + 15) / 16 * 16;
  static constexpr size_t SMEM_FIXED = OFF_PTAB;   // + ncodes * NFP
  static constexpr size_t B_FLOATS = (size_t)KS * 2 * 2 * NB * 4;  // packed operand in global

  // component held by TMEM lane (quadrant q, lane l) in M-tile t (>= 6: padding lanes)
  __host__ __device__ static constexpr int comp_of(int t, int q, int l) {
    return MAP == 0 ? t + 3 * (q >> 1)
                    : (MAP == 1 ? (M1C3 ? ((32 * q + l) / TE < 3 ? 3 * t + (32 * q + l) / TE : 6) : 4 * t + q)
                                : (32 * q + l) / TE);
  }
  // element row of lane (q, l)
  __host__ __device__ static constexpr int row_of(int q, int l) {
    return MAP == 0 ? (q & 1) * 32 + l : (MAP == 1 && !M1C3 ? l : (32 * q + l) % TE);
  }
  // MAP 2: quadrant q holds lanes of epilogue phase p's two components (lanes [2p TE, 2p TE + 2 TE))
  __host__ __device__ static constexpr bool map2_quad_in_phase(int q, int p) {
    return 32 * q < (2 * p + 2) * TE && 32 * q + 32 > 2 * p * TE;
  }
  // MAP 1: the M-tile from which quadrant q moves epilogue phase p's components, -1 if none (no
  // quadrant needs both tiles in one phase)
  __host__ __device__ static constexpr int map1_epi_tile(int p, int q) {
    for (int which = 0; which < 2; ++which) {
      const int c = 2 * p + which;
      if (M1C3) {
        const int lo = (c % 3) * TE;
        if (32 * q < lo + TE && 32 * q + 32 > lo) return c / 3;
      } else if (c % 4 == q) {
        return c / 4;
      }
    }
    return -1;
  }
  // epilogue phase p moves two components (which = 0, 1) through the rows buffer
  __host__ __device__ static constexpr int epi_comp(int p, int which) { return MAP == 0 ? p + 3 * which : 2 * p + which; }
};

// CW consecutive floats from shared memory as one vector load (16 or 8 bytes, aligned by layout).
template <int CW>
__device__ __forceinline__ void lds_vec(const float* p, float (&v)[CW]) {
  if constexpr (CW == 4) {
    const float4 x = *reinterpret_cast<const float4*>(p);
    v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
  } else {
    static_assert(CW == 2, "column groups of 2 or 4");
    const float2 x = *reinterpret_cast<const float2*>(p);
    v[0] = x.x, v[1] = x.y;
  }
}

struct TcArgs {
  StageArgs<float> s;
  const float* bpack;  // [KS][hi,lo][2 chunks][NB][4]
  int num_tiles;
  int wave;            // CTAs resident at once (CTAS x SMs): tile + wave runs next on this SM
};

template <int N, int MODE>
__global__ void __launch_bounds__(TcCfg<N>::THREADS, TcCfg<N>::CTAS) tc_stage_kernel(const TcArgs args) {
  using T = TcCfg<N>;
  using namespace tc;
  constexpr int TE = T::TE, NPG = T::NPG, NP = T::NP, NFP = T::NFP, NB = T::NB, NFPK = T::NFPK;
  constexpr int KS = T::KS, KV = T::KV, NPK = T::NPK, SROW = T::SROW, PROD = T::PROD, NBS = T::NBS;
  constexpr int MT = T::MT, AST = T::AST;
  const StageArgs<float>& a = args.s;

  extern __shared__ __align__(1024) unsigned char smem[];
  float* s_u = reinterpret_cast<float*>(smem + T::OFF_U);
  float* s_geo = reinterpret_cast<float*>(smem + T::OFF_GEO);
  int* s_nbr = reinterpret_cast<int*>(smem + T::OFF_NBR);
  int* s_code = reinterpret_cast<int*>(smem + T::OFF_CODE);
  unsigned char* s_b = smem + T::OFF_B;
  float* s_stage = reinterpret_cast<float*>(smem + T::OFF_STAGE);  // flux of one face | epilogue rows
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
  uint64_t* full = bar;            // [AST] producers -> MMA (A stage written)
  uint64_t* empty = full + AST;    // [AST] MMA commit -> A stage reusable
  uint64_t* b_full = empty + AST;  // [NBS] B ring slot landed
  uint64_t* b_empty = b_full + NBS;  // [NBS] MMA commit -> B slot reusable
  uint64_t* load_full = b_empty + NBS;  // tile rows landed
  uint64_t* acc_full = load_full + 1;   // accumulators final
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acc_full + 1);
  static_assert((2 * AST + 2 * NBS + 2) * 8 + 4 <= 256, "barrier region");
  uint8_t* s_fmask = smem + T::OFF_FMASK;
  uint8_t* s_ptab = smem + T::OFF_PTAB;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t fstride = a.kf * NPG;
  const int64_t e0 = a.e_begin + (int64_t)blockIdx.x * TE;
  const int nv = (int)min((int64_t)TE, a.e_end - e0);
  // Each CTA walks the K-steps in a rotated order (a sum; any order is exact up to rounding) starting
  // at a volume step, so co-running CTAs fetch different slices of the shared B operand from L2
  // instead of all hitting the same lines at once.  Face steps stay contiguous.
  const int rot = (int)(blockIdx.x % (unsigned)(KV / 8));

  // PDL: the next stage's grid may be scheduled once every CTA of this one has started (it then runs
  // its state-independent prologue on the SMs freed by this grid's tail and waits in griddep_wait)
  griddep_launch();
  if (warp == 0) tmem_alloc(s_tmem, T::TMEM_COLS);
  if (tid == PROD) {
    for (int i = 0; i < AST; ++i) {
      mbar_init(&full[i], T::PWARPS);
      mbar_init(&empty[i], 1);
    }
    mbar_init(load_full, 1);
    mbar_init(acc_full, 1);
    for (int i = 0; i < NBS; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    mbar_init_fence();
  }
  for (int c = tid; c < 4 * NFP; c += blockDim.x) s_fmask[c] = a.fmask[c];
  for (int c = tid; c < a.ncodes * NFP; c += blockDim.x) s_ptab[c] = a.ptab[c];
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = *s_tmem;
  TC_TRACE_DECL;

  auto prefetch_res = [&]() {  // warm L2 with the tile's residual rows, read by the epilogue
    const uint32_t rb = (uint32_t)nv * NPG * 4;
    for (int f = 0; f < 6; ++f) prefetch_l2(a.res + (int64_t)f * fstride + e0 * NPG, rb);
  };
  auto load_b = [&](int i) {  // B operand of the i-th K-step (in this CTA's order) into its ring slot
    if (i >= KS) return;
    const int slot = i % NBS;
    const int step = (i + rot) % KS;
    mbar_expect_tx(&b_full[slot], T::B_STEP_BYTES);
    bulk_g2s(s_b + slot * T::B_STEP_BYTES, args.bpack + (size_t)step * (T::B_STEP_BYTES / 4), T::B_STEP_BYTES,
             &b_full[slot]);
  };
  // the tile's rows, geometry and connectivity, the first NBS B slots, L2 warm-up of the next wave
  auto load_tile = [&]() {
    for (int i = 0; i < NBS; ++i) load_b(i);
    const uint32_t rowbytes = (uint32_t)nv * NPG * 4;
    const uint32_t geobytes = (uint32_t)nv * GEO_WORDS * 4, conbytes = (uint32_t)nv * 16;
    mbar_expect_tx(load_full, 6 * rowbytes + geobytes + 2 * conbytes);
    bulk_g2s(s_geo, a.geo + e0 * GEO_WORDS, geobytes, load_full);
    bulk_g2s(s_nbr, a.nbr + e0 * 4, conbytes, load_full);
    bulk_g2s(s_code, a.code + e0 * 4, conbytes, load_full);
    griddep_wait();  // everything above is constant; the state below is the previous stage's output
    for (int f = 0; f < 6; ++f)
      bulk_g2s(s_u + f * TE * NPG, a.u + (int64_t)f * fstride + e0 * NPG, rowbytes, load_full);
    if (MODE == MODE_LSRK && !a.a_zero && KS <= NBS) prefetch_res();
    const int64_t nt = (int64_t)blockIdx.x + args.wave;
    if (nt < args.num_tiles) {
      const int64_t n0 = a.e_begin + nt * TE;
      const uint32_t nn = (uint32_t)min((int64_t)TE, a.e_end - n0);
      for (int f = 0; f < 6; ++f) prefetch_l2(a.u + (int64_t)f * fstride + n0 * NPG, nn * NPG * 4);
      prefetch_l2(a.geo + n0 * GEO_WORDS, nn * GEO_WORDS * 4);
      prefetch_l2(a.nbr + n0 * 4, nn * 16);
      prefetch_l2(a.code + n0 * 4, nn * 16);
    }
  };

  if (warp >= T::PWARPS + 2) {
    // idle warps of the role-based register split (warpgroup 2 must be complete)
    if constexpr (T::RREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(T::REG_AUX));
  } else if (!T::MERGE && warp == T::PWARPS + 1) {
    if constexpr (T::RREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(T::REG_AUX));
    // ================= loader warp =================
    if (elect_one()) load_tile();
    __syncwarp();
    // Refill B slot j % NBS with K-step j + NBS once the MMAs of step j completed.  b_empty[slot]
    // cannot run a phase ahead of this wait: its next completion needs B(j + NBS), loaded below.
    for (int j = 0; j + NBS < KS; ++j) {
      mbar_wait(&b_empty[j % NBS], (j / NBS) & 1);
      if (elect_one()) {
        load_b(j + NBS);
        // residual rows ~NBS K-steps before the epilogue: fresh in L2 when it reads them
        if (MODE == MODE_LSRK && !a.a_zero && j + NBS == KS - 1) prefetch_res();
      }
      __syncwarp();
    }
  } else if (warp == T::PWARPS) {
    if constexpr (T::RREG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(T::REG_AUX));
    // ================= MMA warp (+ the loader's work when MERGE) =================
    const uint32_t idesc = idesc_tf32(128, NB);
    int jr = 0;  // MERGE: next B refill (slot of K-step jr -> K-step jr + NBS)
    if constexpr (T::MERGE) {
      if (elect_one()) load_tile();
      __syncwarp();
    }
    for (int s = 0; s < KS; ++s) {  // s: position in this CTA's K order
      const int slot = s % AST;
      if constexpr (T::MERGE) {
        // refill every slot whose MMAs are done (non-blocking), and block only when step s's own
        // slot has not been refilled yet
        while (jr + NBS < KS && jr < s && (jr + NBS <= s || mbar_test(&b_empty[jr % NBS], (jr / NBS) & 1))) {
          mbar_wait(&b_empty[jr % NBS], (jr / NBS) & 1);
          if (elect_one()) {
            load_b(jr + NBS);
            if (MODE == MODE_LSRK && !a.a_zero && jr + NBS == KS - 1) prefetch_res();
          }
          __syncwarp();
          ++jr;
        }
      }
      mbar_wait(&b_full[s % NBS], (s / NBS) & 1);
      TC_TRACE(1, 700 + s);  // B(s) landed
      mbar_wait(&full[slot], (s / AST) & 1);
      TC_TRACE(1, 500 + 2 * s);  // stage full
      fence_after_sync();
      if (elect_one()) {
        const uint32_t bh = smem_u32(s_b + (s % NBS) * T::B_STEP_BYTES);
        const uint64_t dbh = desc_kmajor(bh, NB * 16, 128);
        const uint64_t dbl = desc_kmajor(bh + 2 * NB * 16, NB * 16, 128);
        const uint32_t abase = tmem + T::A_COL0 + slot * T::A_STAGE_COLS;
        const uint32_t acc0 = s > 0 ? 1u : 0u;
        // accumulator-major order: the three passes of one accumulator back to back issue ~30 %
        // faster than pass-major interleaving (profiles/r01/mma_shape_probe.txt)
#ifndef DGM_EXP_NOMMA
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          mma_tf32_ts(tmem + t * NB, abase + t * 16, dbh, idesc, acc0);     // A_hi B_hi
          mma_tf32_ts(tmem + t * NB, abase + t * 16 + 8, dbh, idesc, 1u);   // A_lo B_hi
          mma_tf32_ts(tmem + t * NB, abase + t * 16, dbl, idesc, 1u);       // A_hi B_lo
        }
#endif
        mma_commit(&empty[slot]);
        mma_commit(&b_empty[s % NBS]);
        if (s == KS - 1) mma_commit(acc_full);
      }
      __syncwarp();
      TC_TRACE(1, 501 + 2 * s);  // issued
    }
  } else {
    if constexpr (T::RREG) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(T::REG_PROD));
    // ================= producers =================
    const int quad = warp & 3;               // TMEM lane quadrant
    const int khalf = warp >> 2;             // which 4 of a K step's 8 columns
    const int h = quad >> 1;                 // MAP 0: 0 = E components (from H fields), 1 = H components
    const int row = T::row_of(quad, lane);   // element row of this TMEM lane
    const uint32_t lane_addr = static_cast<uint32_t>(quad * 32) << 16;
    // MAP 0: one material factor per thread (folded into prx); MAP 1: per component
    // (the sign of -(curl E) / mu is folded in, so both halves use the curl H formula below)
    const float inv_m = T::MAP == 0 ? (h == 0 ? a.inv_eps : -a.inv_mu) : 1.f;
    if (tid == 0) TC_TRACE(0, 1);  // start
    griddep_wait();  // before any global access to the state / residual (neighbour gathers, epilogue)
    mbar_wait(load_full, 0);
    if (nv < TE) {  // partial tile: zero the unused rows once, so no per-value row masking is needed
      for (int i = tid; i < 6 * (TE - nv) * NPG; i += PROD) {
        const int f = i / ((TE - nv) * NPG), rem = i - f * (TE - nv) * NPG;
        s_u[(f * TE + nv) * NPG + rem] = 0.f;
      }
      named_sync(1, PROD);
    }
    if (tid == 0) TC_TRACE(0, 2);  // rows landed
    // warm L2 with the rows of every face neighbour outside the tile (read by the face K-steps);
    // issued LEAD K-steps before this CTA's first face step (-1: at tile start);
    // A/B at C3: lead 2..11 all -1.6% vs tile start, where it delays the first A stores
    auto nbr_prefetch = [&]() {
      for (int e = tid; e < nv * 4; e += PROD) {
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
    };
#ifdef DGM_TC_NBR_LEAD
    constexpr int LEAD = DGM_TC_NBR_LEAD;
#else
    // A/B (lead 5 vs -1): N=4 C3 -1.6%; N=3, 6 +1%, N=7 0, N=8, 9 +5% -> only N=4 uses a lead
    constexpr int LEAD = N == 4 ? 5 : -1;
#endif
    const int nbr_pf_i = LEAD < 0 ? -1 : max(0, (rot < KV / 8 ? KV / 8 - rot : 0) - LEAD);
    if (nbr_pf_i < 0) nbr_prefetch();
    const bool row_ok = row < nv;
    float prx[9];  // geometric factors of the owned row, pre-scaled by 1/eps or 1/mu
#pragma unroll
    for (int q = 0; q < 9; ++q) prx[q] = row_ok ? s_geo[row * GEO_WORDS + q] * inv_m : 0.f;
    // MAP 1/2: the curl factors (dr_mu/dx_c1, dr_mu/dx_c2) / eps or mu of each M-tile's component,
    // per mu, so the K loop selects registers instead of indexing prx with a runtime component
    float pa3[MT][3], pb3[MT][3];
    if constexpr (T::MAP != 0) {
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const int c = T::comp_of(t, quad, lane);
        const int cc = c % 3, c1 = (cc + 1) % 3, c2 = (cc + 2) % 3;
        const float m = c < 3 ? a.inv_eps : -a.inv_mu;
#pragma unroll
        for (int mu = 0; mu < 3; ++mu) {
          const bool ok = row_ok && c < 6;
          pa3[t][mu] = ok ? s_geo[row * GEO_WORDS + mu * 3 + c1] * m : 0.f;
          pb3[t][mu] = ok ? s_geo[row * GEO_WORDS + mu * 3 + c2] * m : 0.f;
        }
      }
    }

    // A values of K-step s for this thread's row (4 columns x 3 M-tiles), unsplit
    auto a_values = [&](int s, int kh, float (&v)[MT][T::CW]) {
      constexpr int CW = T::CW;
      const int k0 = s * 8;
      if constexpr (T::MAP != 0) {
        // one component per M-tile: comp c = 4t + quad; (curl H)_cc / eps for c < 3, -(curl E)_cc / mu
        const int k = k0 + CW * kh;
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          const int c = T::comp_of(t, quad, lane);
          if (c >= 6) {
#pragma unroll
            for (int q = 0; q < CW; ++q) v[t][q] = 0.f;
          } else if (k < 3 * NPK) {
            const int mu = k / NPK, j0 = k - mu * NPK;
            const int cc = c % 3, c1 = (cc + 1) % 3, c2 = (cc + 2) % 3;
            const int fb = c < 3 ? 3 : 0;  // E comps read H fields and vice versa
            const float pa = mu == 0 ? pa3[t][0] : (mu == 1 ? pa3[t][1] : pa3[t][2]);
            const float pb = mu == 0 ? pb3[t][0] : (mu == 1 ? pb3[t][1] : pb3[t][2]);
            float xp[CW], yp[CW];
            lds_vec<CW>(s_u + ((fb + c2) * TE + row) * NPG + j0, xp);
            lds_vec<CW>(s_u + ((fb + c1) * TE + row) * NPG + j0, yp);
#pragma unroll
            for (int q = 0; q < CW; ++q) v[t][q] = pa * xp[q] - pb * yp[q];
          } else if (k >= KV) {
            const int node = (k - KV) % NFPK;
#pragma unroll
            for (int q = 0; q < CW; ++q) v[t][q] = s_stage[(c * NFPK + node + q) * SROW + row];
          } else {
#pragma unroll
            for (int q = 0; q < CW; ++q) v[t][q] = 0.f;
          }
        }
      } else {
        const int k = k0 + CW * kh;
        if (k < 3 * NPK) {
          const int mu = k / NPK, j0 = k - mu * NPK;
          // register selects, not prx[mu * 3 + .] (a dynamic index puts prx in local memory)
          const float p0 = mu == 0 ? prx[0] : (mu == 1 ? prx[3] : prx[6]);
          const float p1 = mu == 0 ? prx[1] : (mu == 1 ? prx[4] : prx[7]);
          const float p2 = mu == 0 ? prx[2] : (mu == 1 ? prx[5] : prx[8]);
          const int fb = h == 0 ? 3 : 0;  // E comps read H fields and vice versa
          float xs[CW], ys[CW], zs[CW];
          lds_vec<CW>(s_u + ((fb + 0) * TE + row) * NPG + j0, xs);
          lds_vec<CW>(s_u + ((fb + 1) * TE + row) * NPG + j0, ys);
          lds_vec<CW>(s_u + ((fb + 2) * TE + row) * NPG + j0, zs);
          if constexpr (T::F32X2) {
          // packed pairs: v = p_a * a - p_b * b as FMUL2(-p_b, b) then FFMA2(p_a, a, .)
          const float n0 = -p0, n1 = -p1, n2 = -p2;
#pragma unroll
          for (int q = 0; q < CW; q += 2) {  // (curl H) / eps, or -(curl E) / mu via the sign in p
            float t0, t1;
            mul2(t0, t1, n2, n2, ys[q], ys[q + 1]);
            fma2(v[0][q], v[0][q + 1], p1, p1, zs[q], zs[q + 1], t0, t1);
            mul2(t0, t1, n0, n0, zs[q], zs[q + 1]);
            fma2(v[1][q], v[1][q + 1], p2, p2, xs[q], xs[q + 1], t0, t1);
            mul2(t0, t1, n1, n1, xs[q], xs[q + 1]);
            fma2(v[2][q], v[2][q + 1], p0, p0, ys[q], ys[q + 1], t0, t1);
          }
          } else {
#pragma unroll
          for (int q = 0; q < CW; ++q) {  // (curl H) / eps, or -(curl E) / mu via the sign in p
            v[0][q] = p1 * zs[q] - p2 * ys[q];
            v[1][q] = p2 * xs[q] - p0 * zs[q];
            v[2][q] = p0 * ys[q] - p1 * xs[q];
          }
          }
        } else if (k >= KV && T::INLINE_FLUX) {
          // this thread's own flux values (its element row, its half's 3 components, its 4 slots),
          // no staging: upwind bracket x face scale straight into the A operand (maxwell.py:73-132)
          const int face = (k - KV) / NFPK, node0 = (k - KV) % NFPK;
          const int code = row_ok ? s_code[row * 4 + face] : -1;
          const int nb = s_nbr[row * 4 + face];
          const float* gk = s_geo + row * GEO_WORDS;
          const float nx = gk[10 + 3 * face], ny = gk[11 + 3 * face], nz = gk[12 + 3 * face];
          const float sc = row_ok ? gk[22 + face] * gk[9] : 0.f;
          const float scale = h == 0 ? sc * a.inv_eps * a.inv_2z : sc * a.inv_mu * a.inv_2y;
          const int64_t loc = (int64_t)nb - e0;
          const bool inl = code >= 0 && loc >= 0 && loc < nv;
#pragma unroll
          for (int q = 0; q < CW; ++q) {
            const int slot = node0 + q;
            const bool real = slot < NFP;
            const int nd = real ? slot : 0;
            const int im = s_fmask[face * NFP + nd];
            const int jn = code >= 0 ? s_ptab[code * NFP + nd] : 0;
            float um[6], up[6];
#pragma unroll
            for (int f = 0; f < 6; ++f) um[f] = s_u[(f * TE + row) * NPG + im];
            if (inl) {
#pragma unroll
              for (int f = 0; f < 6; ++f) up[f] = s_u[(f * TE + (int)loc) * NPG + jn];
            } else if (code >= 0) {
              const float* g = a.u + (int64_t)nb * NPG + jn;
#pragma unroll
              for (int f = 0; f < 6; ++f) up[f] = __ldg(g + f * fstride);
            } else {  // PEC mirror (maxwell.py:117-132)
              const float nde = nx * um[0] + ny * um[1] + nz * um[2];
              const float ndh = nx * um[3] + ny * um[4] + nz * um[5];
              up[0] = -um[0] + 2.f * nde * nx;
              up[1] = -um[1] + 2.f * nde * ny;
              up[2] = -um[2] + 2.f * nde * nz;
              up[3] = um[3] - 2.f * ndh * nx;
              up[4] = um[4] - 2.f * ndh * ny;
              up[5] = um[5] - 2.f * ndh * nz;
            }
            const float dex = up[0] - um[0], dey = up[1] - um[1], dez = up[2] - um[2];
            const float dhx = up[3] - um[3], dhy = up[4] - um[4], dhz = up[5] - um[5];
            const float w = real ? scale : 0.f;
            if (h == 0) {  // E components: Z+ (n x [[H]]) + [[E]] - n (n . [[E]])
              const float nde = nx * dex + ny * dey + nz * dez;
              v[0][q] = (a.zp * (ny * dhz - nz * dhy) + (dex - nx * nde)) * w;
              v[1][q] = (a.zp * (nz * dhx - nx * dhz) + (dey - ny * nde)) * w;
              v[2][q] = (a.zp * (nx * dhy - ny * dhx) + (dez - nz * nde)) * w;
            } else {       // H components: [[H]] - n (n . [[H]]) - Y+ (n x [[E]])
              const float ndh = nx * dhx + ny * dhy + nz * dhz;
              v[0][q] = ((dhx - nx * ndh) - a.yp * (ny * dez - nz * dey)) * w;
              v[1][q] = ((dhy - ny * ndh) - a.yp * (nz * dex - nx * dez)) * w;
              v[2][q] = ((dhz - nz * ndh) - a.yp * (nx * dey - ny * dex)) * w;
            }
          }
        } else if (k >= KV) {
          const int node = (k - KV) % NFPK;
          if constexpr (T::FT) {
#pragma unroll
            for (int t = 0; t < MT; ++t) {
              const float4 x = *reinterpret_cast<const float4*>(s_stage + T::ft_off(3 * h + t, row, node >> 2));
              v[t][0] = x.x, v[t][1] = x.y, v[t][2] = x.z, v[t][3] = x.w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < CW; ++q)
#pragma unroll
              for (int t = 0; t < MT; ++t) v[t][q] = s_stage[((3 * h + t) * NFPK + node + q) * SROW + row];
          }
        } else {
#pragma unroll
          for (int q = 0; q < CW; ++q)
#pragma unroll
            for (int t = 0; t < MT; ++t) v[t][q] = 0.f;
        }
      }
    };
    // surface flux of a whole face into the staging buffer (all producers, two named barriers)
    auto flux_pass = [&](int face) {
        named_sync(1, PROD);  // every thread finished reading the previous face's staging
        // one work unit = (element row, 4 consecutive node slots): the row's face data (normal,
        // scale, code, neighbour, in-tile or not) is read once and u+ is fetched with typed
        // shared / global loads, all 24 in flight before any use
        constexpr int FB = T::FB, NBF = NFPK / FB;
#pragma unroll 1
        for (int unit = tid; unit < TE * NBF; unit += PROD) {
          const int r = unit / NBF, n0 = (unit % NBF) * FB;
          const bool row_live = r < nv;
          const int code = row_live ? s_code[r * 4 + face] : -1;
          const int nb = s_nbr[r * 4 + face];
          const float* gk = s_geo + r * GEO_WORDS;
          const float nx = gk[10 + 3 * face], ny = gk[11 + 3 * face], nz = gk[12 + 3 * face];
          const float sc = row_live ? gk[22 + face] * gk[9] : 0.f;
          const float se = sc * a.inv_eps * a.inv_2z, sh = sc * a.inv_mu * a.inv_2y;  // upwind factors folded
          int im[FB], jn[FB];
#pragma unroll
          for (int j = 0; j < FB; ++j) {
            const int node = n0 + j < NFP ? n0 + j : 0;
            im[j] = s_fmask[face * NFP + node];
            jn[j] = code >= 0 ? s_ptab[code * NFP + node] : 0;
          }
          float up[FB][6];
          const int64_t loc = (int64_t)nb - e0;
          if constexpr (T::GENERIC_UP) {
            // one generic-address gather for in-tile (shared) and out-of-tile (global) neighbours, so
            // a warp holding both kinds of rows does not run two load paths one after the other
            if (code >= 0) {
              const bool in_tile = loc >= 0 && loc < nv;
              const float* g = in_tile ? s_u + loc * NPG : a.u + (int64_t)nb * NPG;
              const int64_t fs = in_tile ? (int64_t)TE * NPG : fstride;
#pragma unroll
              for (int j = 0; j < FB; ++j)
#pragma unroll
                for (int f = 0; f < 6; ++f)
                  asm volatile("ld.f32 %0, [%1];" : "=f"(up[j][f]) : "l"(g + f * fs + jn[j]));
            }
          } else if (code >= 0 && loc >= 0 && loc < nv) {  // neighbour row in this tile: shared memory
#pragma unroll
            for (int j = 0; j < FB; ++j)
#pragma unroll
              for (int f = 0; f < 6; ++f) up[j][f] = s_u[(f * TE + (int)loc) * NPG + jn[j]];
          } else if (code >= 0) {  // neighbour row elsewhere: global (L2-prefetched a few K-steps ahead)
            const float* g = a.u + (int64_t)nb * NPG;
#pragma unroll
            for (int j = 0; j < FB; ++j)
#pragma unroll
              for (int f = 0; f < 6; ++f) up[j][f] = __ldg(g + f * fstride + jn[j]);
          }
          float fo[6][FB];  // FT: the unit's scaled flux values, stored as one vector per component
#pragma unroll
          for (int j = 0; j < FB; ++j) {
            float um[6];
#pragma unroll
            for (int f = 0; f < 6; ++f) um[f] = s_u[(f * TE + r) * NPG + im[j]];
            if (code < 0) {  // PEC mirror (maxwell.py:117-132)
              const float nde = nx * um[0] + ny * um[1] + nz * um[2];
              const float ndh = nx * um[3] + ny * um[4] + nz * um[5];
              up[j][0] = -um[0] + 2.f * nde * nx;
              up[j][1] = -um[1] + 2.f * nde * ny;
              up[j][2] = -um[2] + 2.f * nde * nz;
              up[j][3] = um[3] - 2.f * ndh * nx;
              up[j][4] = um[4] - 2.f * ndh * ny;
              up[j][5] = um[5] - 2.f * ndh * nz;
            }
            float out[6];
            upwind_num(um, up[j], nx, ny, nz, a.zp, a.yp, out);
            const int node = n0 + j;
            const float kse = node < NFP ? se : 0.f, ksh = node < NFP ? sh : 0.f;
            if constexpr (T::FT) {
#pragma unroll
              for (int c = 0; c < 6; ++c) fo[c][j] = out[c] * (c < 3 ? kse : ksh);
            } else {
#pragma unroll
              for (int c = 0; c < 3; ++c) s_stage[(c * NFPK + node) * SROW + r] = out[c] * kse;
#pragma unroll
              for (int c = 3; c < 6; ++c) s_stage[(c * NFPK + node) * SROW + r] = out[c] * ksh;
            }
          }
          if constexpr (T::FT) {
#pragma unroll
            for (int c = 0; c < 6; ++c)
              *reinterpret_cast<float4*>(s_stage + T::ft_off(c, r, n0 >> 2)) =
                  make_float4(fo[c][0], fo[c][1], fo[c][2], fo[c][3]);
          }
        }
        named_sync(1, PROD);
    };
    auto face_start = [&](int s) { return !T::INLINE_FLUX && s >= KV / 8 && (s - KV / 8) % (NFPK / 8) == 0; };

    // Software-pipelined K loop: the next step's A values are computed between this step's
    // tcgen05.st and its tcgen05.wait::st, hiding the TMEM store latency; a flux pass (two named
    // barriers) runs only after this step's stage was handed to the MMA warp.
    auto kh_of = [&](int j) { return khalf * T::KH + j; };  // column group of the thread's j-th group
    float vcur[T::KH][MT][T::CW], vnext[T::KH][MT][T::CW];
#ifndef DGM_EXP_NOFLUX
    if (face_start((0 + rot) % KS)) flux_pass(((0 + rot) % KS * 8 - KV) / NFPK);
#endif
#pragma unroll
    for (int j = 0; j < T::KH; ++j) a_values((0 + rot) % KS, kh_of(j), vcur[j]);
    // slot = i % AST, its empty-barrier parity ((i / AST) & 1) ^ 1 and the K-step s = (i + rot) % KS:
    // kept as incremental counters where registers allow (1 CTA/SM: N=6 -3.3 %, N=8 -4.8 %), recomputed
    // per step at 2 CTAs/SM, where the three extra live registers spill at the 96-register cap (+5.6 %)
    constexpr bool INC = T::CTAS == 1 || T::MERGE || T::RREG;
    int slot_c = 0, s_c = rot;
    uint32_t eph_c = 1;
    for (int i = 0; i < KS; ++i) {  // i: position in this CTA's K order, s: K-step
      const int slot = INC ? slot_c : i % AST;
      const int s = INC ? s_c : (i + rot) % KS;
      const uint32_t eph = INC ? eph_c : (((i / AST) & 1) ^ 1);
      if (tid == 0) TC_TRACE(0, 100 + 4 * s);  // step begin
      if (i == nbr_pf_i) nbr_prefetch();
#pragma unroll
      for (int j = 0; j < T::KH; ++j) {
        float hi[MT][T::CW], lo[MT][T::CW];
        if constexpr (T::F32X2) {
#pragma unroll
          for (int t = 0; t < MT; ++t)
#pragma unroll
            for (int q = 0; q < T::CW; q += 2)
              split_tf32_2(vcur[j][t][q], vcur[j][t][q + 1], hi[t][q], hi[t][q + 1], lo[t][q], lo[t][q + 1]);
        } else {
#pragma unroll
          for (int t = 0; t < MT; ++t)
#pragma unroll
            for (int q = 0; q < T::CW; ++q) split_tf32(vcur[j][t][q], hi[t][q], lo[t][q]);  // dead rows are 0
        }
        if (j == 0) {
          mbar_wait(&empty[slot], eph);
          if (tid == 0) TC_TRACE(0, 102 + 4 * s);  // stage free
          fence_after_sync();
        }
#ifndef DGM_EXP_NOSTORE
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          const uint32_t col = T::A_COL0 + slot * T::A_STAGE_COLS + t * 16 + T::CW * kh_of(j);
          if constexpr (T::CW == 4) {
            tmem_st4(tmem + lane_addr + col, hi[t]);
            tmem_st4(tmem + lane_addr + col + 8, lo[t]);
          } else {
            tmem_st2(tmem + lane_addr + col, hi[t]);
            tmem_st2(tmem + lane_addr + col + 8, lo[t]);
          }
        }
#else
        if (hi[0][0] == 12345.f && lo[0][3] == 1.f) s_stage[0] = 0.f;  // keep the values live
#endif
      }
      const int sn = INC ? (s + 1 == KS ? 0 : s + 1) : (i + 1 + rot) % KS;
      const bool has_next = i + 1 < KS;
#ifdef DGM_EXP_NOFLUX
      const bool next_flux = false;
#else
      const bool next_flux = has_next && face_start(sn);
#endif
      if (has_next && !next_flux) {  // overlaps the TMEM store latency
#pragma unroll
        for (int j = 0; j < T::KH; ++j) a_values(sn, kh_of(j), vnext[j]);
      }
      tmem_st_wait();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[slot]);
      if (next_flux) {
        flux_pass((sn * 8 - KV) / NFPK);
        if (tid == 0) TC_TRACE(0, 103 + 4 * sn);  // face flux staged
#pragma unroll
        for (int j = 0; j < T::KH; ++j) a_values(sn, kh_of(j), vnext[j]);
      }
#pragma unroll
      for (int j = 0; j < T::KH; ++j)
#pragma unroll
        for (int t = 0; t < MT; ++t)
#pragma unroll
          for (int q = 0; q < T::CW; ++q) vcur[j][t][q] = vnext[j][t][q];
      if constexpr (INC) {
        s_c = sn;
        if (++slot_c == AST) slot_c = 0, eph_c ^= 1u;
      }
    }

    // ================= epilogue: accumulators -> LSRK update =================
    if (tid == 0) TC_TRACE(0, 3);  // all steps produced
    constexpr int RV = NPG / 4;    // 16-byte chunks per row
    const int nvec = nv * RV;      // chunks per component slab
    constexpr int PER = (2 * TE * RV + PROD - 1) / PROD;
    mbar_wait(acc_full, 0);
    if (tid == 0) TC_TRACE(0, 4);  // accumulators final
    fence_after_sync();
    // Every producer's last flux-staging read happened before its last A-stage arrival, which the
    // accumulator commit already orders before this point; the barrier states that ordering in a
    // form compute-sanitizer racecheck can see (it does not track tcgen05.commit arrivals).
    named_sync(1, PROD);
#pragma unroll 1
    for (int t = 0; t < 3; ++t) {  // epilogue phase: components T::epi_comp(t, 0 / 1)
      // residual rows of the phase's two components (L2-prefetched at CTA start), all loads in flight
      float4 ro[PER];
#pragma unroll
      for (int p = 0; p < PER; ++p) {
        const int idx = tid + p * PROD;
        const int which = idx >= nvec ? 1 : 0;
        const int c = idx - which * nvec;
        ro[p] = (MODE == MODE_LSRK && !a.a_zero && c < nvec)
                    ? __ldcs(reinterpret_cast<const float4*>(
                                 a.res + ((int64_t)T::epi_comp(t, which) * a.kf + e0) * NPG) + c)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      // quadrant warps holding the phase's components: TMEM lanes -> smem rows [which][row][NPG]
      // (MAP 0: M-tile t, all four quadrants; MAP 1: M-tile t/2, quadrants 2(t%2), 2(t%2)+1)
      // (MAP 2: the single M-tile, the quadrants holding lanes [2t TE, 2t TE + 2 TE): components 2t, 2t+1)
      // EPI_SPLIT (N=6): every column group of those quadrants moves a share of the NB / 8 column
      // chunks, up to four tcgen05.ld in flight per wait (N=6 -3.8 %); elsewhere the first column group
      // moves all chunks, one load per wait (the split measured N=4 +1.0 %, N=5 +1.3 %, N=8 +0.7 %,
      // N=9 +1.5 %)
      constexpr bool EPI_SPLIT = N == 6 && T::MAP == 0;
      const int m1tile = T::MAP != 1 ? 0 : (T::M1C3 ? T::map1_epi_tile(t, quad) : ((quad >> 1) == (t & 1) ? t >> 1 : -1));
      const bool mover = (EPI_SPLIT || khalf == 0) &&
                         (T::MAP == 0 || (T::MAP == 1 ? m1tile >= 0 : T::map2_quad_in_phase(quad, t)));
      if constexpr (!EPI_SPLIT) {
       if (mover) {
        const int tile = T::MAP == 0 ? t : (T::MAP == 1 ? m1tile : 0);
        // MAP 1/2: the lane holds component comp_of(tile, quad, lane); only the phase's two store
        const int slot = T::MAP == 0 ? h : (T::MAP == 1 && !T::M1C3 ? (quad & 1) : T::comp_of(tile, quad, lane) - 2 * t);
        const bool mine = T::MAP == 0 || (T::MAP == 1 && !T::M1C3) || (slot >= 0 && slot < 2);
        float* dst = s_stage + (size_t)(mine ? slot : 0) * TE * NPG + row * NPG;
#pragma unroll
        for (int c0 = 0; c0 < NB; c0 += 8) {
          float r8[8];
          tmem_ld8(tmem + lane_addr + tile * NB + c0, r8);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 8; q += 4) {
            const int i = c0 + q;
            if (i < NPG && mine) {
              float4 o;
              o.x = (i + 0 < NP) ? r8[q + 0] : 0.f;
              o.y = (i + 1 < NP) ? r8[q + 1] : 0.f;
              o.z = (i + 2 < NP) ? r8[q + 2] : 0.f;
              o.w = (i + 3 < NP) ? r8[q + 3] : 0.f;
              *reinterpret_cast<float4*>(dst + i) = o;
            }
          }
        }
       }
      } else if (mover) {
        const int tile = T::MAP == 0 ? t : (T::MAP == 1 ? t >> 1 : 0);
        const int slot = T::MAP == 0 ? h : (T::MAP == 1 ? (quad & 1) : (lane >> 4));
        float* dst = s_stage + (size_t)slot * TE * NPG + row * NPG;
        constexpr int NC = NB / 8, CPG = (NC + T::NQ - 1) / T::NQ;  // chunks, chunks per column group
        const int cb = khalf * CPG;
#pragma unroll
        for (int b0 = 0; b0 < CPG; b0 += 4) {
          float r8[4][8];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (b0 + k < CPG && cb + b0 + k < NC) tmem_ld8(tmem + lane_addr + tile * NB + (cb + b0 + k) * 8, r8[k]);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (b0 + k < CPG && cb + b0 + k < NC) {
#pragma unroll
              for (int q = 0; q < 8; q += 4) {
                const int i = (cb + b0 + k) * 8 + q;
                if (i < NPG) {
                  float4 o;
                  o.x = (i + 0 < NP) ? r8[k][q + 0] : 0.f;
                  o.y = (i + 1 < NP) ? r8[k][q + 1] : 0.f;
                  o.z = (i + 2 < NP) ? r8[k][q + 2] : 0.f;
                  o.w = (i + 3 < NP) ? r8[k][q + 3] : 0.f;
                  *reinterpret_cast<float4*>(dst + i) = o;
                }
              }
            }
          }
        }
      }
      named_sync(1, PROD);
#pragma unroll
      for (int p = 0; p < PER; ++p) {
        const int idx = tid + p * PROD;
        const int which = idx >= nvec ? 1 : 0;
        const int c = idx - which * nvec;
        if (c < nvec) {
          const int comp = T::epi_comp(t, which);
          const int64_t gbase = ((int64_t)comp * a.kf + e0) * NPG;
          const float4 rh = reinterpret_cast<const float4*>(s_stage + (size_t)which * TE * NPG)[c];
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
            const float4 uo = reinterpret_cast<const float4*>(s_u + (size_t)comp * TE * NPG)[c];
            __stcs(reinterpret_cast<float4*>(a.res + gbase) + c, r);
            __stcs(reinterpret_cast<float4*>(a.u_out + gbase) + c,
                   make_float4(uo.x + a.b * r.x, uo.y + a.b * r.y, uo.z + a.b * r.z, uo.w + a.b * r.w));
          }
        }
      }
      named_sync(1, PROD);  // rows buffer free for the next M-tile
    }
    if (tid == 0) TC_TRACE(0, 5);  // epilogue done
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (warp == 0) tmem_dealloc(tmem, T::TMEM_COLS);
}

}  // namespace dgm
