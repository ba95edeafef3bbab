// dgm_stage.cuh -- fused nodal-DG Maxwell stage kernel (SIMT path, sm_100a).
//
// One CTA owns a tile of TE consecutive elements and does, in one pass over
// HBM, everything ReferenceMaxwellOperator.rhs (oracle.py:60-94) and one
// iteration of rk4_step (assemble.py:118-120) do for those elements:
//
//   P0  stage u[6][TE][NPG], geometry, neighbor codes and the small face tables
//       into shared memory (coalesced 16-byte loads);
//   P1  surface: for every (element, face, face node) gather u- from smem and
//       u+ from smem (neighbor in tile) or L2 (neighbor elsewhere) through the
//       compact (neighbor, code) map, apply the PEC mirror on walls
//       (maxwell.py:117-132) and the upwind flux (maxwell.py:73-114), scale by
//       the face Jacobian (oracle.py:84-85) -> s_fl[6][TE][NFS];
//   P2  volume + lift: thread (i, g) owns node i of elements g, g+G, ...;
//       D_r,D_s,D_t rows stream from L1/L2 as 16-byte chunks (read-only path),
//       u rows are broadcast from smem, 18 derivatives per (element, node)
//       accumulate in registers, then the geometric transform and curls
//       (oracle.py:68-79), then LIFT * flux, * 1/J, combine, / eps,mu
//       (oracle.py:86-93);
//   P3  write-back through smem: RHS, or the low-storage RK update
//       res = a res + dt rhs; u_out = u + b res, fully coalesced.
//
// Algorithmic traffic per element-stage: read u, res; write
// u, res (4*6*Np words) + 26 geometry words + 8 connectivity words.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tc05.cuh"

namespace dgm {

constexpr int GEO_WORDS = 28;  // 26 used + 2 pad: rows are 7 x 16 B, so any row range is TMA-aligned

__host__ __device__ constexpr int np_of(int n) { return (n + 1) * (n + 2) * (n + 3) / 6; }
__host__ __device__ constexpr int nfp_of(int n) { return (n + 1) * (n + 2) / 2; }

// Smallest m >= n whose row size is a 16-byte multiple with an odd number of
// 16-byte chunks: rows of consecutive elements then start in distinct 16-byte
// bank groups, so 8 lanes reading 8 elements' rows are conflict-free.
__host__ __device__ constexpr int odd_chunk_pad(int n, int w) {
  int m = n;
  while ((m * w) % 16 != 0 || ((m * w / 16) % 2) == 0) ++m;
  return m;
}

// SMALL = 1: one element per P2 thread (tiles of G elements) for launches of only a few tiles,
// where the per-tile latency, not the throughput, sets the stage time (C1: 1,512 tets).
template <int N, typename T, int SMALL = 0>
struct Cfg {
  static constexpr int NP = np_of(N);
  static constexpr int NFP = nfp_of(N);
  static constexpr int NF4 = 4 * NFP;
  static constexpr int W = sizeof(T);
  static constexpr int VEC = 16 / W;
  static constexpr int NPG = odd_chunk_pad(NP, W);   // u row stride (HBM and smem)
  static constexpr int NFS = odd_chunk_pad(NF4, W);  // flux / rhs row stride (smem)
  static constexpr int NJC = (NP + VEC - 1) / VEC;   // 16-byte chunks of a D row
  static constexpr int NLC = (NF4 + VEC - 1) / VEC;  // 16-byte chunks of a LIFT row
#if defined(DGM_SIMT_G64) && defined(DGM_SIMT_E64)
  // tuning override for the fp64 kernel (scripts/gpu_simt_tune*.sh)
  static constexpr int G = W == 8 ? DGM_SIMT_G64 : ((N <= 5) ? 8 : (N <= 7 ? 4 : 2));
  static constexpr int E = W == 8 ? DGM_SIMT_E64 : 4;
#else
  // element groups x elements per thread (SIMT P2 and the mass norm); fp64 N <= 6 runs P2 on DMMA
  // fp64 DMMA tiles of 8 elements (one MMA column tile), two tasks per warp, up to 4 CTAs per SM so
  // one CTA's flux / write-back phases overlap others' DMMA phases: C3 fp64 4.17 -> 3.96 ms per stage,
  // C2 fp64 N=3, 5, 6 -13..15 % (profiles/r02/ab_f64_te8.txt; 3 CTAs per SM measured slower at N=4)
#ifndef DGM_F64_DMMA_MAXN
#define DGM_F64_DMMA_MAXN 9  // all orders: N=7, 8, 9 at 48k tets 2.69 / 4.15 / 6.34 -> 1.54 / 3.04 / 4.72 ms per stage
#endif
  static constexpr bool T8 = W == 8 && N <= DGM_F64_DMMA_MAXN;
  // fp64 N=8: 2 groups x 4 elements and <= 12 warps (no spills): 3.04 -> 2.84 ms per stage at 48k tets;
  // measured +6 % at N=7 and neutral at N=9 (profiles/r02/ab_f64_high_orders.txt)
  static constexpr bool HI2 = T8 && N == 8;
  static constexpr int G = HI2 ? 2 : (T8 ? 4 : ((N <= 5) ? 8 : (N <= 7 ? 4 : 2)));
  // fp32 N=2: two elements per thread and up to 4 CTAs per SM (C2 N=2 38.9 -> 35.4 us per stage;
  // N=1, 3 measured neutral or slower, profiles/r02/ab_simt_f32.txt)
  static constexpr bool F32N2 = W == 4 && N == 2;
  static constexpr int E = SMALL ? 1 : (HI2 ? 4 : ((T8 || F32N2) ? 2 : ((W == 4) ? 4 : 2)));
#endif
  static constexpr int TE = G * E;                           // elements per tile
  static constexpr int WORK = NP * G;
  // fp64 volume + LIFT on the FP64 tensor path (mma.sync m8n8k4 f64, DMMA): one warp task = 8 nodes x
  // 8 elements x one field half (all orders; -DDGM_F64_SIMT_P2 restores the CUDA-core P2)
#ifdef DGM_F64_SIMT_P2
  static constexpr bool DMMA = false;
#else
  static constexpr bool DMMA = W == 8 && N <= DGM_F64_DMMA_MAXN && TE % 8 == 0 && !SMALL;
#endif
  static constexpr int NIT = (NP + 7) / 8;                   // DMMA node tiles
  static constexpr int DTASKS = NIT * (TE / 8) * 2;
  static constexpr int DTPW = HI2 ? (DTASKS + 11) / 12 : 2;  // DMMA tasks per warp
  static constexpr int DWARPS = T8 ? (DTASKS + DTPW - 1) / DTPW : (DTASKS < 10 ? DTASKS : 10);
  static constexpr int THREADS_SIMT = ((WORK + 31) / 32) * 32;
  static constexpr int THREADS = (DMMA && 32 * DWARPS > THREADS_SIMT) ? 32 * DWARPS : THREADS_SIMT;
  static_assert(NF4 >= NP, "rhs rows reuse the flux buffer");
  static constexpr size_t SMEM_REAL = (size_t)6 * TE * NPG + (size_t)6 * TE * NFS + (size_t)TE * GEO_WORDS;
  static constexpr size_t SMEM_FIXED = SMEM_REAL * W + (size_t)TE * 8 * 4 + 4 * NFP;
  // Two CTAs per SM when shared memory allows it and N <= 6: capping registers there costs
  // <= 220 B of spills and gains 1.1-1.5x (profiles/r01/simt_minblocks.json); at N >= 7 the
  // spills (300-400 B) cost more than the occupancy gains.
  static constexpr int MIN_BLOCKS = (T8 || F32N2) ? (4 * (SMEM_FIXED + 2048) <= 227 * 1024 ? 4
                                                     : (2 * (SMEM_FIXED + 2048) <= 227 * 1024 && N <= 6 ? 2 : 1))
                                       : ((N <= 6 && 2 * (SMEM_FIXED + 2048) <= 227 * 1024) ? 2 : 1);
};

template <typename T> struct V16;
template <> struct V16<float> {
  using type = float4;
  // acc + a.b as one FMA chain (no separate product / add)
  __device__ static float fma_dot(const float4& a, const float4& b, float acc) {
    return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, fmaf(a.x, b.x, acc))));
  }
};
template <> struct V16<double> {
  using type = double2;
  __device__ static double fma_dot(const double2& a, const double2& b, double acc) {
    return fma(a.y, b.y, fma(a.x, b.x, acc));
  }
};

template <typename T>
struct StageArgs {
  const T* u;          // (6, kf, NPG) input state
  T* u_out;            // LSRK: updated state
  T* res;              // LSRK: residual register
  T* out;              // RHS / VOLUME: (6, kf, NPG); SURFACE: (6, kf, NF4)
  const T* geo;        // (K, 26)
  const int* nbr;      // (kf, 4)
  const int* code;     // (kf, 4)
  const T* diff;       // [3][NJC][NP][VEC]
  const T* lift;       // [NLC][NP][VEC]
  const uint8_t* fmask;  // [4][NFP]
  const uint8_t* ptab;   // [ncodes][NFP]
  int ncodes;
  int64_t kf;          // field stride (element slots per field)
  int64_t e_begin, e_end;
  T a, b, dt;
  T inv_eps, inv_mu;
  T zp, yp;            // impedance / admittance of the (uniform) material
  T inv_2z, inv_2y;    // 1 / (2 {Z}), 1 / (2 {Y})
  int a_zero;          // LSRK: skip reading res (RK_A[0] == 0)
};

enum Mode { MODE_RHS = 0, MODE_LSRK = 1, MODE_VOLUME = 2, MODE_SURFACE = 3 };

// Upwind flux difference (maxwell.py:73-114) for a uniform material.
// Upwind bracket numerators, before the 1/(2{Z}) and 1/(2{Y}) factors (maxwell.py:73-114):
//   E: n x (Z+ [[H]] - n x [[E]]) = Z+ (n x [[H]]) + [[E]] - n (n . [[E]])
//   H: n x (-Y+ [[E]] - n x [[H]]) = -Y+ (n x [[E]]) + [[H]] - n (n . [[H]])
// (n x (n x v) = n (n . v) - v for the unit normal: 36 instead of 48 operations per node).
template <typename T>
__device__ __forceinline__ void upwind_num(const T* um, const T* up, T nx, T ny, T nz, T zp, T yp, T* out) {
  const T dex = up[0] - um[0], dey = up[1] - um[1], dez = up[2] - um[2];
  const T dhx = up[3] - um[3], dhy = up[4] - um[4], dhz = up[5] - um[5];
  const T nde = nx * dex + ny * dey + nz * dez, ndh = nx * dhx + ny * dhy + nz * dhz;
  out[0] = zp * (ny * dhz - nz * dhy) + (dex - nx * nde);
  out[1] = zp * (nz * dhx - nx * dhz) + (dey - ny * nde);
  out[2] = zp * (nx * dhy - ny * dhx) + (dez - nz * nde);
  out[3] = (dhx - nx * ndh) - yp * (ny * dez - nz * dey);
  out[4] = (dhy - ny * ndh) - yp * (nz * dex - nx * dez);
  out[5] = (dhz - nz * ndh) - yp * (nx * dey - ny * dex);
}

template <typename T>
__device__ __forceinline__ void upwind(const T* um, const T* up, T nx, T ny, T nz,
                                       const StageArgs<T>& a, T* out) {
  upwind_num(um, up, nx, ny, nz, a.zp, a.yp, out);
#pragma unroll
  for (int c = 0; c < 3; ++c) out[c] *= a.inv_2z;
#pragma unroll
  for (int c = 3; c < 6; ++c) out[c] *= a.inv_2y;
}

// D(8x8) += A(8x4, row) B(4x8, col) in fp64 on the tensor pipe; lane l holds A[l/4][l%4],
// B[l%4][l/4] and D[l/4][2(l%4) + {0, 1}].
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int N, typename T, int MODE, int SMALL = 0>
__global__ void __launch_bounds__(Cfg<N, T, SMALL>::THREADS, Cfg<N, T, SMALL>::MIN_BLOCKS)
stage_kernel(const StageArgs<T> a) {
  using C = Cfg<N, T, SMALL>;
  using V = typename V16<T>::type;
  constexpr int TE = C::TE, NPG = C::NPG, NFS = C::NFS, NP = C::NP, NFP = C::NFP;
  constexpr int VEC = C::VEC, G = C::G, E = C::E;
  // The paper's intra-block face-pair reuse in P1 (both sides of an in-tile face from one evaluation,
  // PAPER.md:1100-1104): built and parity-tested, but measured slower on B200 (C3 fp64 +10 %, C2 fp32
  // N=1 +25 %, N=2 +23 %: the per-CTA slot tables, the idle partner items and the scattered second
  // store cost more than the halved arithmetic; profiles/r02/ab_pairs.txt), so opt-in (-DDGM_PAIRS).
#ifdef DGM_PAIRS
  constexpr bool PAIRS = true;
#else
  constexpr bool PAIRS = false;
#endif

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s_u = reinterpret_cast<T*>(smem_raw);
  T* s_fl = s_u + 6 * TE * NPG;
  T* s_geo = s_fl + 6 * TE * NFS;
  int* s_nbr = reinterpret_cast<int*>(s_geo + TE * GEO_WORDS);
  int* s_code = s_nbr + TE * 4;
  uint8_t* s_fmask = reinterpret_cast<uint8_t*>(s_code + TE * 4);
  uint8_t* s_ptab = s_fmask + 4 * NFP;
  // face-pair reuse tables (P1): slot of node n in face f (255: not on f), and the neighbour's face
  // of each code (the face whose node set the code's row lists)
  uint8_t* s_slot = s_ptab + a.ncodes * NFP;     // [4][NP]
  uint8_t* s_codeface = s_slot + 4 * NP;         // [ncodes]

  const int tid = threadIdx.x;
  const int64_t e0 = a.e_begin + (int64_t)blockIdx.x * TE;
  const int nv = (int)min((int64_t)TE, a.e_end - e0);
  const int64_t fstride = a.kf * NPG;

  // ---------------- P0: stage the tile ----------------
  // one thread issues bulk copies of the tile's rows (6 field slabs, geometry, connectivity) on an
  // mbarrier and warms L2 with the residual rows the write-back reads; the others zero the rows of
  // a partial tile and copy the face tables meanwhile
  __shared__ __align__(8) uint64_t s_bar;
  {
    constexpr int RV = NPG / VEC;  // 16-byte chunks per u row
    // programmatic dependent launch: the next stage's grid may be scheduled now; this one touches the
    // state only after its predecessor completed (griddepcontrol.wait)
    tc::griddep_launch();
    if (tid == 0) {
      tc::mbar_init(&s_bar, 1);
      tc::mbar_init_fence();
    }
    __syncthreads();
    tc::griddep_wait();
    if (tid == 0) {
      const uint32_t rowb = (uint32_t)nv * NPG * sizeof(T), geob = (uint32_t)nv * GEO_WORDS * sizeof(T);
      const uint32_t conb = (uint32_t)nv * 16;
      tc::mbar_expect_tx(&s_bar, 6 * rowb + geob + (MODE != MODE_VOLUME ? 2 * conb : 0));
#pragma unroll 1
      for (int f = 0; f < 6; ++f) tc::bulk_g2s(s_u + f * TE * NPG, a.u + (int64_t)f * fstride + e0 * NPG, rowb, &s_bar);
      tc::bulk_g2s(s_geo, a.geo + e0 * GEO_WORDS, geob, &s_bar);
      if (MODE != MODE_VOLUME) {
        tc::bulk_g2s(s_nbr, a.nbr + e0 * 4, conb, &s_bar);
        tc::bulk_g2s(s_code, a.code + e0 * 4, conb, &s_bar);
      }
      if (MODE == MODE_LSRK && !a.a_zero)
        for (int f = 0; f < 6; ++f) tc::prefetch_l2(a.res + (int64_t)f * fstride + e0 * NPG, rowb);
    }
    if (nv < TE) {
      const V zero = {};
      for (int f = 0; f < 6; ++f)
        for (int c = nv * RV + tid; c < TE * RV; c += blockDim.x) reinterpret_cast<V*>(s_u + f * TE * NPG)[c] = zero;
      for (int c = nv * GEO_WORDS + tid; c < TE * GEO_WORDS; c += blockDim.x) s_geo[c] = T(0);
    }
    if (MODE != MODE_VOLUME) {
      for (int c = tid; c < 4 * NFP; c += blockDim.x) s_fmask[c] = a.fmask[c];
      for (int c = tid; c < a.ncodes * NFP; c += blockDim.x) s_ptab[c] = a.ptab[c];
    }
    if (MODE != MODE_VOLUME && PAIRS)
      for (int c = tid; c < 4 * NP; c += blockDim.x) s_slot[c] = 255;
    tc::mbar_wait(&s_bar, 0);
  }
  __syncthreads();
  if (MODE != MODE_VOLUME && PAIRS) {
    for (int c = tid; c < 4 * NFP; c += blockDim.x) s_slot[(c / NFP) * NP + s_fmask[c]] = (uint8_t)(c % NFP);
    __syncthreads();
    for (int c = tid; c < a.ncodes; c += blockDim.x) {
      int face = 0;
      for (int f = 0; f < 4; ++f) {
        bool all = true;
        for (int i = 0; i < NFP; ++i) all = all && s_slot[f * NP + s_ptab[c * NFP + i]] != 255;
        if (all) face = f;
      }
      s_codeface[c] = (uint8_t)face;
    }
    __syncthreads();
  }

  // ---------------- P1: surface flux ----------------
  // two work items per round: both items' trace loads (smem, or L2 for out-of-tile neighbours) are
  // issued before either is used
#ifdef DGM_EXP_NOP1
  if (false) {
#else
  if (MODE != MODE_VOLUME) {
#endif
    const int nwork = nv * 4 * NFP;
    struct Item {
      int k, r, face, code, loc, jn;  // loc: in-tile neighbour row or -1; jn: its node at this slot
      T um[6], up[6];
    };
    auto gather = [&](int w, Item& it) {
      it.k = w / (4 * NFP);
      it.r = w - it.k * (4 * NFP);
      it.face = it.r / NFP;
      const int node = it.r - it.face * NFP;
      const int im = s_fmask[it.face * NFP + node];
#pragma unroll
      for (int f = 0; f < 6; ++f) it.um[f] = s_u[(f * TE + it.k) * NPG + im];
      it.code = s_code[it.k * 4 + it.face];
      it.loc = -1;
      if (it.code >= 0) {
        const int nb = s_nbr[it.k * 4 + it.face];
        const int jn = s_ptab[it.code * NFP + node];
        const int64_t loc = (int64_t)nb - e0;
        if (loc >= 0 && loc < nv) {
          it.loc = (int)loc;
          it.jn = jn;
          if (PAIRS && it.loc < it.k) return;  // the pair's first element evaluates both sides
#pragma unroll
          for (int f = 0; f < 6; ++f) it.up[f] = s_u[(f * TE + (int)loc) * NPG + jn];
        } else {
          const T* p = a.u + (int64_t)nb * NPG + jn;
#pragma unroll
          for (int f = 0; f < 6; ++f) it.up[f] = __ldg(p + f * fstride);
        }
      }
    };
    auto finish = [&](Item& it) {
      if (PAIRS && it.loc >= 0 && it.loc < it.k) return;  // written by the pair's first element
      const T* gk = s_geo + it.k * GEO_WORDS;
      const T nx = gk[10 + 3 * it.face], ny = gk[11 + 3 * it.face], nz = gk[12 + 3 * it.face];
      if (PAIRS && it.loc > it.k) {
        // both sides of an in-tile face at once (the paper's intra-block pair reuse, PAPER.md:1100-1104;
        // reference gather.py:153-169): with D = u+ - u-, the neighbour sees -D and -n, so its bracket
        // is T1 - T2 (E) and -S1 + S2 (H) where this side's is T1 + T2 and S1 + S2
        const T dex = it.up[0] - it.um[0], dey = it.up[1] - it.um[1], dez = it.up[2] - it.um[2];
        const T dhx = it.up[3] - it.um[3], dhy = it.up[4] - it.um[4], dhz = it.up[5] - it.um[5];
        const T nde = nx * dex + ny * dey + nz * dez, ndh = nx * dhx + ny * dhy + nz * dhz;
        const T t1[3] = {a.zp * (ny * dhz - nz * dhy), a.zp * (nz * dhx - nx * dhz), a.zp * (nx * dhy - ny * dhx)};
        const T t2[3] = {dex - nx * nde, dey - ny * nde, dez - nz * nde};
        const T s1[3] = {dhx - nx * ndh, dhy - ny * ndh, dhz - nz * ndh};
        const T s2[3] = {-a.yp * (ny * dez - nz * dey), -a.yp * (nz * dex - nx * dez), -a.yp * (nx * dey - ny * dex)};
        const T sj = gk[22 + it.face] * a.inv_2z, sjh = gk[22 + it.face] * a.inv_2y;
        const int pf = s_codeface[it.code];
        const T* gp = s_geo + it.loc * GEO_WORDS;
        const T pj = gp[22 + pf] * a.inv_2z, pjh = gp[22 + pf] * a.inv_2y;
        const int pr = pf * NFP + s_slot[pf * NP + it.jn];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          s_fl[(c * TE + it.k) * NFS + it.r] = (t1[c] + t2[c]) * sj;
          s_fl[((c + 3) * TE + it.k) * NFS + it.r] = (s1[c] + s2[c]) * sjh;
          s_fl[(c * TE + it.loc) * NFS + pr] = (t1[c] - t2[c]) * pj;
          s_fl[((c + 3) * TE + it.loc) * NFS + pr] = (s2[c] - s1[c]) * pjh;
        }
        return;
      }
      if (it.code < 0) {
        // PEC mirror (maxwell.py:117-132)
        const T nde = nx * it.um[0] + ny * it.um[1] + nz * it.um[2];
        const T ndh = nx * it.um[3] + ny * it.um[4] + nz * it.um[5];
        it.up[0] = -it.um[0] + T(2) * nde * nx;
        it.up[1] = -it.um[1] + T(2) * nde * ny;
        it.up[2] = -it.um[2] + T(2) * nde * nz;
        it.up[3] = it.um[3] - T(2) * ndh * nx;
        it.up[4] = it.um[4] - T(2) * ndh * ny;
        it.up[5] = it.um[5] - T(2) * ndh * nz;
      }
      T fl[6];
      upwind(it.um, it.up, nx, ny, nz, a, fl);
      const T sj = gk[22 + it.face];
#pragma unroll
      for (int f = 0; f < 6; ++f) s_fl[(f * TE + it.k) * NFS + it.r] = fl[f] * sj;
    };
    for (int w = tid; w < nwork; w += 2 * blockDim.x) {
      const int w2 = w + blockDim.x;
      Item i1, i2;
      gather(w, i1);
      if (w2 < nwork) gather(w2, i2);
      finish(i1);
      if (w2 < nwork) finish(i2);
    }
    __syncthreads();
  }

  if (MODE == MODE_SURFACE) {
    // bracket * face_jacobian, natural face layout (6, kf, 4 Nfp)
    constexpr int NF4 = C::NF4;
    for (int f = 0; f < 6; ++f)
      for (int c = tid; c < nv * NF4; c += blockDim.x) {
        const int k = c / NF4, j = c - k * NF4;
        a.out[((int64_t)f * a.kf + e0 + k) * NF4 + j] = s_fl[(f * TE + k) * NFS + j];
      }
    return;
  }

  // ---------------- P2 (fp64, N <= 6): volume + lift on DMMA ----------------
  if constexpr (C::DMMA) {
    // task (node tile it, element half eh, field half hh): the 3 derivatives of fields 3hh..3hh+2
    // (rows i, K = node j of D_mu; columns = the 8 elements) and the lifted flux of components
    // 3(1-hh)..+2 (K = face node), i.e. the whole update of those components; the curl is formed
    // from the accumulator fragments (lane: node 8 it + l/4, elements 8 eh + 2(l%4) + {0, 1})
    constexpr int NEH = TE / 8, NT = C::NIT * NEH * 2, NWARPS = C::THREADS / 32;
    constexpr int MAXT = (NT + NWARPS - 1) / NWARPS;
    constexpr int KJ = (NP + 3) / 4 * 4, NF4 = C::NF4;
    const int warp = tid >> 5, lane = tid & 31, g4 = lane >> 2, t4 = lane & 3;
    // MMA column n <-> element 8 eh + colp(n): the B-fragment loads (lane: column l/4, K = l%4) of
    // rows with an odd-16-byte-chunk stride are then conflict-free in each half-warp (rows 0, 2, 4, 6
    // and 1, 3, 5, 7 sit 8 banks apart); column n = l/4 in natural order was 2-way conflicted.
    // C3 fp64: shared-load bank conflicts 303 M -> 125 M per launch, 3.960 -> 3.924 ms per stage;
    // N=3, 5, 6, 8 -0.4..2.0 %, N=9 +1.8 % (its write-back stores conflict more), so N=9 keeps the
    // natural order (profiles/r02/ab_f64_colp.txt)
    auto colp = [](int n) { return N <= 8 ? 2 * (n & 3) + (n >> 2) : n; };
    T keep[MAXT][3][2];
#pragma unroll
    for (int q = 0; q < MAXT; ++q) {
      const int task = warp + q * NWARPS;
      if (task >= NT) break;
      const int hh = task & 1, rest = task >> 1, eh = rest % NEH, it = rest / NEH;
      const int i = 8 * it + g4;   // A row / accumulator row: node
      const int eb = 8 * eh + colp(g4);  // B column: element
      T acc[3][3][2], accl[3][2];
#pragma unroll
      for (int mu = 0; mu < 3; ++mu)
#pragma unroll
        for (int t = 0; t < 3; ++t) acc[mu][t][0] = acc[mu][t][1] = T(0);
#pragma unroll
      for (int t = 0; t < 3; ++t) accl[t][0] = accl[t][1] = T(0);
#ifndef DGM_EXP_NOP2
#pragma unroll 3
      for (int k0 = 0; k0 < KJ; k0 += 4) {
        const int k = k0 + t4;
        T av[3], bv[3];
#pragma unroll
        for (int mu = 0; mu < 3; ++mu)
          av[mu] = (i < NP && k < NP) ? __ldg(a.diff + (((size_t)mu * C::NJC + (k >> 1)) * NP + i) * 2 + (k & 1)) : T(0);
#pragma unroll
        for (int t = 0; t < 3; ++t) bv[t] = s_u[((3 * hh + t) * TE + eb) * NPG + k];  // rows zero past Np
#pragma unroll
        for (int mu = 0; mu < 3; ++mu)
#pragma unroll
          for (int t = 0; t < 3; ++t) dmma_8x8x4(acc[mu][t], av[mu], bv[t]);
      }
      if (MODE != MODE_VOLUME) {
#pragma unroll 3
        for (int k0 = 0; k0 < NF4; k0 += 4) {
          const int k = k0 + t4;
          const T al = i < NP ? __ldg(a.lift + ((size_t)(k >> 1) * NP + i) * 2 + (k & 1)) : T(0);
#pragma unroll
          for (int t = 0; t < 3; ++t) dmma_8x8x4(accl[t], al, s_fl[((3 * (1 - hh) + t) * TE + eb) * NFS + k]);
        }
      }
#endif
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int e = 8 * eh + colp(2 * t4 + c);
        const T* gk = s_geo + e * GEO_WORDS;
        // grad_nu F_t = sum_mu rx[mu][nu] dF_t/dr_mu; (curl F)_t = grad_t1 F_t2 - grad_t2 F_t1
        auto grad = [&](int nu, int t) {
          return gk[nu] * acc[0][t][c] + gk[3 + nu] * acc[1][t][c] + gk[6 + nu] * acc[2][t][c];
        };
        const T curl[3] = {grad(1, 2) - grad(2, 1), grad(2, 0) - grad(0, 2), grad(0, 1) - grad(1, 0)};
        const T sgn = hh ? T(1) : T(-1), mat = hh ? a.inv_eps : a.inv_mu;
#pragma unroll
        for (int t = 0; t < 3; ++t) keep[q][t][c] = (sgn * curl[t] + accl[t][c] * gk[9]) * mat;
      }
    }
    if (MODE != MODE_VOLUME) __syncthreads();  // every lift read of s_fl is done
#pragma unroll
    for (int q = 0; q < MAXT; ++q) {
      const int task = warp + q * NWARPS;
      if (task >= NT) break;
      const int hh = task & 1, rest = task >> 1, eh = rest % NEH, it = rest / NEH;
      const int i = 8 * it + g4;
      if (i < NP) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int t = 0; t < 3; ++t) s_fl[((3 * (1 - hh) + t) * TE + 8 * eh + colp(2 * t4 + c)) * NFS + i] = keep[q][t][c];
      }
    }
    __syncthreads();
  } else {
  // ---------------- P2: volume + lift ----------------
  T rhs[6][E];
  const bool worker = tid < C::WORK;
  const int i = tid / G;
  const int g = tid - i * G;
  if (worker) {
    T acc[3][6][E];
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int f = 0; f < 6; ++f)
#pragma unroll
        for (int e = 0; e < E; ++e) acc[m][f][e] = T(0);

    const V* dv = reinterpret_cast<const V*>(a.diff);
#pragma unroll 1
    for (int jc = 0; jc < C::NJC; ++jc) {
      V d[3];
#pragma unroll
      for (int m = 0; m < 3; ++m) d[m] = __ldg(dv + ((size_t)m * C::NJC + jc) * NP + i);
#pragma unroll
      for (int f = 0; f < 6; ++f)
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const V uv = *reinterpret_cast<const V*>(s_u + (f * TE + e * G + g) * NPG + jc * VEC);
#pragma unroll
          for (int m = 0; m < 3; ++m) acc[m][f][e] = V16<T>::fma_dot(d[m], uv, acc[m][f][e]);
        }
    }
    // geometric transform + curls (oracle.py:69-79)
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const T* gk = s_geo + (e * G + g) * GEO_WORDS;
      T rx[3][3];
#pragma unroll
      for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int n = 0; n < 3; ++n) rx[m][n] = gk[m * 3 + n];
      // grad[n][f] = sum_m rx[m][n] * acc[m][f]
      auto grad = [&](int n, int f) {
        return rx[0][n] * acc[0][f][e] + rx[1][n] * acc[1][f][e] + rx[2][n] * acc[2][f][e];
      };
      // curl E = (dy Ez - dz Ey, dz Ex - dx Ez, dx Ey - dy Ex); same for H
      const T ce0 = grad(1, 2) - grad(2, 1), ce1 = grad(2, 0) - grad(0, 2), ce2 = grad(0, 1) - grad(1, 0);
      const T ch0 = grad(1, 5) - grad(2, 4), ch1 = grad(2, 3) - grad(0, 5), ch2 = grad(0, 4) - grad(1, 3);
      rhs[0][e] = ch0; rhs[1][e] = ch1; rhs[2][e] = ch2;
      rhs[3][e] = -ce0; rhs[4][e] = -ce1; rhs[5][e] = -ce2;
    }
    if (MODE != MODE_VOLUME) {
      T accl[6][E];
#pragma unroll
      for (int f = 0; f < 6; ++f)
#pragma unroll
        for (int e = 0; e < E; ++e) accl[f][e] = T(0);
      const V* lv = reinterpret_cast<const V*>(a.lift);
#pragma unroll 2
      for (int jc = 0; jc < C::NLC; ++jc) {
        const V l = __ldg(lv + (size_t)jc * NP + i);
#pragma unroll
        for (int f = 0; f < 6; ++f)
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const V fv = *reinterpret_cast<const V*>(s_fl + (f * TE + e * G + g) * NFS + jc * VEC);
            accl[f][e] = V16<T>::fma_dot(l, fv, accl[f][e]);
          }
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const T inv_j = s_geo[(e * G + g) * GEO_WORDS + 9];
#pragma unroll
        for (int f = 0; f < 6; ++f) rhs[f][e] += accl[f][e] * inv_j;
      }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
#pragma unroll
      for (int f = 0; f < 3; ++f) rhs[f][e] *= a.inv_eps;
#pragma unroll
      for (int f = 3; f < 6; ++f) rhs[f][e] *= a.inv_mu;
    }
  }
  if (MODE != MODE_VOLUME) __syncthreads();  // every lift read of s_fl is done
  if (worker) {
#pragma unroll
    for (int f = 0; f < 6; ++f)
#pragma unroll
      for (int e = 0; e < E; ++e) s_fl[(f * TE + e * G + g) * NFS + i] = rhs[f][e];
  }
  __syncthreads();
  }  // SIMT P2

  // ---------------- P3: coalesced write-back ----------------
  // (field, chunk) work items flattened over the CTA; the residual chunks of all of a thread's items
  // are loaded first (L2-prefetched in P0), so the loads overlap instead of one round trip per field
  {
    constexpr int RV = NPG / VEC;
    constexpr int PER = (6 * TE * RV + C::THREADS - 1) / C::THREADS;
    const int nvec = nv * RV;
    const int total = 6 * nvec;
    V ro[PER];
    if (MODE == MODE_LSRK && !a.a_zero) {
#pragma unroll
      for (int p = 0; p < PER; ++p) {
        const int idx = tid + p * C::THREADS;
        if (idx < total) {
          const int f = idx / nvec, c = idx - f * nvec;
          ro[p] = *reinterpret_cast<const V*>(a.res + ((int64_t)f * a.kf + e0) * NPG + (int64_t)c * VEC);
        }
      }
    }
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int idx = tid + p * C::THREADS;
      if (idx >= total) break;
      const int f = idx / nvec, c = idx - f * nvec;
      const int k = c / RV, jv = c - k * RV;
      const int64_t go = ((int64_t)f * a.kf + e0) * NPG + (int64_t)c * VEC;  // rows are contiguous
      T rh[VEC];
      const T* srow = s_fl + (f * TE + k) * NFS + jv * VEC;
#pragma unroll
      for (int q = 0; q < VEC; ++q) rh[q] = (jv * VEC + q < NP) ? srow[q] : T(0);
      if (MODE == MODE_RHS || MODE == MODE_VOLUME) {
        V o;
        T* op = reinterpret_cast<T*>(&o);
#pragma unroll
        for (int q = 0; q < VEC; ++q) op[q] = rh[q];
        *reinterpret_cast<V*>(a.out + go) = o;
      } else {
        V r;
        T* rp = reinterpret_cast<T*>(&r);
        if (a.a_zero) {
#pragma unroll
          for (int q = 0; q < VEC; ++q) rp[q] = a.dt * rh[q];
        } else {
          const T* rop = reinterpret_cast<const T*>(&ro[p]);
#pragma unroll
          for (int q = 0; q < VEC; ++q) rp[q] = a.a * rop[q] + a.dt * rh[q];
        }
        *reinterpret_cast<V*>(a.res + go) = r;
        const V uo = *reinterpret_cast<const V*>(s_u + (f * TE + k) * NPG + jv * VEC);
        const T* uop = reinterpret_cast<const T*>(&uo);
        V un;
        T* unp = reinterpret_cast<T*>(&un);
#pragma unroll
        for (int q = 0; q < VEC; ++q) unp[q] = uop[q] + a.b * rp[q];
        *reinterpret_cast<V*>(a.u_out + go) = un;
      }
    }
  }
}

}  // namespace dgm
