// dgm_tc2.cuh -- fused Maxwell stage kernel, v2 (N <= 4, fp32 via 3xTF32): the state rows are the
// A operand of the volume GEMM as they are, the geometry is applied after the MMAs.
//
// v1 (dgm_tc.cuh) builds A = (per-element curl combination of u) for every K-step with the
// producer warps and hands it over through TMEM: ~1,050 A values per element and stage, ~230 of
// its ~800 warp instructions per element.  v2 regroups the same sums (oracle.py:67-93):
//
//   dF_mu = D_mu u_F                   for the 6 fields F and mu = r, s, t   (one GEMM, A = u)
//   rhs_c = (sum_mu rx[mu][c1] dF(c2)_mu - rx[mu][c2] dF(c1)_mu) / (eps|mu) + LIFT f^(c)
//
// so the volume A operand is the state tile itself, brought by TMA straight into the canonical
// K-major SWIZZLE_NONE layout, and only its tf32 remainder lo = u - tf32(u) is computed (3xTF32:
// u_hi D_hi + u_lo D_hi + u_hi D_lo; kind::tf32 reads the fp32 bits of u and ignores the low 13
// mantissa bits -- tests/test_gpu_tc05.py pins that).  The curl (geometric factors, 1/eps, 1/mu)
// moves into the epilogue, which reads 3 derivative blocks per field from TMEM.
//
// Tiling: a persistent CTA per SM walks tiles of TE = 64 elements.  M-tile t (t = x, y, z) has
// 128 rows: row 64 h + e = field t + 3h (h = 0: E, 1: H) of element e.  TMEM columns of M-tile t
// (ACC = NV + NL per tile, 3 ACC <= 512):
//   [0, NV)       mu * MUS + i : D_mu applied to field t + 3h at node i
//   [NV, NV + NL) i            : LIFT applied to the flux of component t + 3(1 - h)
// A thread of TMEM lane (h, e) therefore holds the three derivatives of the three fields of half h
// -- exactly the curl of that half, which drives the components of the other half -- and the
// lifted flux of those components: the whole update of element e's 3 components of half 1 - h.
//
// All HBM traffic of the state goes through TMA (4-D tensor maps over (node, element, t, h), box
// {4 nodes, 64 elements, 1, 2} = one 2 KB K-chunk of an M-tile): the tile load (27 boxes) and, in
// the epilogue, the residual / state rows of one component pair (t, t + 3) at a time, updated in
// shared memory and stored back by TMA -- no per-thread global accesses except the out-of-tile
// neighbour traces.
//
// Roles (512 threads, 1 CTA per SM; 16 warps = 4 per SM sub-partition, so 128 registers):
//   warps 0-7   producers: the tile load (one thread: TMA + bulk copies), tf32 remainder of each
//               M-tile (2-slot ring), the surface flux face by face into the SS A operand of the
//               LIFT GEMM (hi / lo), one (element, 4 face slots) unit per thread.
//   warps 8-15  epilogue: warp w reads TMEM lanes 32q..32q+31, q = w % 4 (one element-half per
//               thread), the two warps of a quadrant split the node blocks of 4.  One elected lane
//               of warp 8 first issues the tile's MMAs (they cannot start before the previous
//               epilogue has read TMEM anyway) and the epilogue's TMA traffic.
// The epilogue stages its rows in the remainder ring and the flux buffer (both idle once the
// tile's MMAs are done); the producers wait for it (stage_free) before reusing them.
#pragma once

#include <cuda.h>

#include "dgm_stage.cuh"
#include "tc05.cuh"

namespace dgm {

template <int N>
struct Tc2Cfg {
  using C = Cfg<N, float>;
  static constexpr int NP = C::NP, NFP = C::NFP, NPG = C::NPG;
  static constexpr int MUS = (NP + 3) / 4 * 4;             // TMEM / B-row stride of one derivative block
  static constexpr int NV = (3 * MUS + 15) / 16 * 16;      // volume MMA N
  static constexpr int NL = (NP + 15) / 16 * 16;           // LIFT MMA N
  static constexpr int ACC = NV + NL;                      // accumulator columns per M-tile
  static_assert(3 * ACC <= 512, "accumulators must fit TMEM");
  static constexpr int KV = (NP + 7) / 8 * 8;              // volume K (node j), whole K-steps
  static constexpr int KCH = KV / 4;                       // 16-byte K chunks of a volume A operand
  static constexpr int UCH = NPG / 4;                      // chunks of a state row (odd)
  // The last K-step's second chunk (nodes NPG..NPG+3) of the state tile is not stored: the
  // descriptor reads the next region there (finite data) against the zero rows of D.
  static_assert(KCH == UCH + 1, "state rows must end one chunk short of the K extent");
  static constexpr int VKS = KV / 8;                       // volume K-steps
  static constexpr int NFPK = (NFP + 7) / 8 * 8;           // K extent (slots) of one face
  static constexpr int FCH = NFPK / 4;                     // flux chunks per face (= units per row)
  static constexpr int FKS = NFPK / 8;                     // K-steps per face
  static constexpr int KF = 4 * NFPK;                      // LIFT K
  static constexpr int TE = 64, ROWS = 128;
  static constexpr int PWARPS = 8, EWARPS = 8;
  static constexpr int PROD = 32 * PWARPS, EPI = 32 * EWARPS;
  static constexpr int THREADS = PROD + EPI;
  static constexpr int CHUNK = ROWS * 16;                  // one K chunk of a 128-row operand: 2 KB
  static constexpr int UT = UCH * CHUNK;                   // one M-tile of the state tile
  static constexpr int LT = KCH * CHUNK;                   // one remainder slot (last chunk zero)
  static constexpr int DB_HALF = KCH * NV * 16;            // volume B operand (D), hi or lo part
  static constexpr int LB_HALF = (KF / 4) * NL * 16;       // LIFT B operand, hi or lo part
  static constexpr int FX_HALF = FCH * CHUNK;              // flux A of one face and M-tile, hi or lo
  static constexpr int NBLK = UCH;                         // epilogue node blocks of 4
  static constexpr int STG = 2 * UT;                       // epilogue staging of one pair: res | u
  static_assert(STG <= 2 * LT && STG <= 6 * FX_HALF, "staging must fit the remainder ring / flux buffer");
  static constexpr size_t OFF_U = 0;
  static constexpr size_t OFF_LO = OFF_U + 3 * (size_t)UT;
  static constexpr size_t OFF_DB = OFF_LO + 2 * (size_t)LT;
  static constexpr size_t OFF_LB = OFF_DB + 2 * (size_t)DB_HALF;
  static constexpr size_t OFF_FX = OFF_LB + 2 * (size_t)LB_HALF;
  static constexpr size_t OFF_GEO = OFF_FX + 6 * (size_t)FX_HALF;
  static constexpr size_t OFF_NBR = OFF_GEO + (size_t)TE * GEO_WORDS * 4;
  static constexpr size_t OFF_CODE = OFF_NBR + TE * 16;
  static constexpr size_t OFF_BAR = OFF_CODE + TE * 16;
  static constexpr size_t OFF_FMASK = OFF_BAR + 256;
  static constexpr size_t OFF_PTAB = OFF_FMASK + (4 * NFP + 15) / 16 * 16;
  static constexpr size_t SMEM_FIXED = OFF_PTAB;           // + ncodes * NFP
  static constexpr size_t B_BYTES = 2 * (size_t)DB_HALF + 2 * (size_t)LB_HALF;
  static constexpr size_t B_FLOATS = B_BYTES / 4;
};

// Tensor maps are 4-D views (node, element, t, h) of a (6, kf, NPG) state-layout array: strides
// (-, NPG * 4, kf * NPG * 4, 3 kf * NPG * 4) bytes, element extent e_end (rows past the launch range
// are out of bounds: zero on load, never written), box {4, 64, 1, 2}.
struct alignas(64) Tc2Args {
  CUtensorMap tm_u;    // u_in: tile loads and the epilogue's state rows
  CUtensorMap tm_res;  // residual: epilogue loads and stores (LSRK)
  CUtensorMap tm_out;  // u_out (LSRK) or out (RHS): epilogue stores
  StageArgs<float> s;
  const float* bops;   // [D hi | D lo | LIFT hi | LIFT lo], each [chunk][row][4] (include/dgm.h)
  int num_tiles;
};

__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// one box {4, 64, 1, 2} at (node 4k, element e0, t, h 0) -> smem [h][e][4] (2 KB)
__device__ __forceinline__ void tma_load_chunk(void* dst, const CUtensorMap* tm, int k, int64_t e0, int t, void* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          tc::smem_u32(dst)),
      "l"(tm), "r"(4 * k), "r"((int)e0), "r"(t), "r"(0), "r"(tc::smem_u32(mbar))
      : "memory");
}
__device__ __forceinline__ void tma_store_chunk(const CUtensorMap* tm, int k, int64_t e0, int t, const void* src) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(tm),
               "r"(4 * k), "r"((int)e0), "r"(t), "r"(0), "r"(tc::smem_u32(src))
               : "memory");
}

// 32 lanes x 4 consecutive 32-bit TMEM columns (thread t <- lane quadrant*32 + t), no wait.
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
  uint32_t r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(taddr));
  v[0] = __uint_as_float(r0), v[1] = __uint_as_float(r1), v[2] = __uint_as_float(r2), v[3] = __uint_as_float(r3);
}

template <int N, int MODE>
__global__ void __launch_bounds__(Tc2Cfg<N>::THREADS, 1) tc2_stage_kernel(const __grid_constant__ Tc2Args args) {
  using T = Tc2Cfg<N>;
  using namespace tc;
  constexpr int TE = T::TE, NP = T::NP, NFP = T::NFP, NPG = T::NPG, UCH = T::UCH, KCH = T::KCH;
  constexpr int CHUNK = T::CHUNK, UT = T::UT, LT = T::LT, PROD = T::PROD;
  const StageArgs<float>& a = args.s;

  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* s_u = smem + T::OFF_U;
  unsigned char* s_lo = smem + T::OFF_LO;
  unsigned char* s_db = smem + T::OFF_DB;
  unsigned char* s_lb = smem + T::OFF_LB;
  unsigned char* s_fx = smem + T::OFF_FX;
  float* s_geo = reinterpret_cast<float*>(smem + T::OFF_GEO);
  int* s_nbr = reinterpret_cast<int*>(smem + T::OFF_NBR);
  int* s_code = reinterpret_cast<int*>(smem + T::OFF_CODE);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + T::OFF_BAR);
  uint64_t* b_ops = bar;              // B operands landed (once)
  uint64_t* tile_full = bar + 1;      // tile rows (TMA) + geometry / neighbours / codes landed
  uint64_t* lo_full = bar + 2;        // [2] producers -> MMA: remainder slot written
  uint64_t* lo_empty = bar + 4;       // [2] MMA commit -> slot reusable
  uint64_t* u_free = bar + 6;         // MMA commit: the tile's volume MMAs (readers of s_u, s_lo) done
  uint64_t* fx_full = bar + 7;        // producers -> MMA: a face's flux written
  uint64_t* fx_empty = bar + 8;       // MMA commit -> flux buffer reusable
  uint64_t* acc_full = bar + 9;       // MMA commit -> epilogue
  uint64_t* acc_empty = bar + 10;     // epilogue -> MMA: accumulators read
  uint64_t* stg_full = bar + 11;      // [2] epilogue staging A (s_lo) / B (s_fx) loaded
  uint64_t* stage_free = bar + 13;    // epilogue -> producers: s_lo and s_fx no longer staged
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bar + 14);
  uint8_t* s_fmask = smem + T::OFF_FMASK;
  uint8_t* s_ptab = smem + T::OFF_PTAB;
  unsigned char* stage[2] = {s_lo, s_fx};

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t fstride = a.kf * NPG;
  auto tile_e0 = [&](int tile) { return a.e_begin + (int64_t)tile * TE; };
  auto tile_nv = [&](int tile) { return (int)min((int64_t)TE, a.e_end - tile_e0(tile)); };

  griddep_launch();
  if (warp == T::PWARPS) tmem_alloc(s_tmem, 512);
  if (tid == 0) {
    mbar_init(b_ops, 1);
    mbar_init(tile_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&lo_full[i], T::PWARPS);
      mbar_init(&lo_empty[i], 1);
      mbar_init(&stg_full[i], 1);
    }
    mbar_init(u_free, 1);
    mbar_init(fx_full, T::PWARPS);
    mbar_init(fx_empty, 1);
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, T::EWARPS);
    mbar_init(stage_free, 1);
    mbar_init_fence();
  }
  for (int c = tid; c < 4 * NFP; c += blockDim.x) s_fmask[c] = a.fmask[c];
  for (int c = tid; c < a.ncodes * NFP; c += blockDim.x) s_ptab[c] = a.ptab[c];
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = *s_tmem;
  TC_TRACE_DECL;

  if (warp < T::PWARPS) {
    // ============================ producers ============================
    // the tile's rows -> s_u[t][chunk][h * 64 + e][4] (27 TMA boxes) + geometry / connectivity rows
    auto issue_tile = [&](int tile) {
      const int64_t e0 = tile_e0(tile);
      const int nv = tile_nv(tile);
      const uint32_t geob = (uint32_t)nv * GEO_WORDS * 4, conb = (uint32_t)nv * 16;
      mbar_expect_tx(tile_full, 3 * UT + geob + 2 * conb);
      for (int t = 0; t < 3; ++t)
        for (int k = 0; k < UCH; ++k) tma_load_chunk(s_u + t * UT + k * CHUNK, &args.tm_u, k, e0, t, tile_full);
      bulk_g2s(s_geo, a.geo + e0 * GEO_WORDS, geob, tile_full);
      bulk_g2s(s_nbr, a.nbr + e0 * 4, conb, tile_full);
      bulk_g2s(s_code, a.code + e0 * 4, conb, tile_full);
    };
    if (tid == 0) {  // constant B operands, once per CTA
      mbar_expect_tx(b_ops, (uint32_t)T::B_BYTES);
      bulk_g2s(s_db, args.bops, 2 * T::DB_HALF, b_ops);
      bulk_g2s(s_lb, args.bops + 2 * T::DB_HALF / 4, 2 * T::LB_HALF, b_ops);
      griddep_wait();  // the state is the previous stage's output
      if ((int)blockIdx.x < args.num_tiles) issue_tile(blockIdx.x);
    }
    griddep_wait();

    // flux-unit mapping: 8 consecutive elements x FCH slot blocks per warp; a unit's 4 nodes are
    // visited rotated by its block (node (jj + ub) & 3 at step jj), so every flux store and u- load
    // instruction of a warp spreads over the banks (ordering.face_slot_order_v2 models the loads)
    const int ur = 8 * warp + (lane & 7), ub = lane >> 3;
    const bool unit_ok = ub < T::FCH;
    int it = 0;
    for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x, ++it) {
      const int64_t e0 = tile_e0(tile);
      const int nv = tile_nv(tile);
      if (tid == 0) TC_TRACE(0, 100 * it + 1);
      mbar_wait(tile_full, it & 1);
      if (tid == 0) TC_TRACE(0, 100 * it + 2);
      if (tid == 0) {
        // the residual rows the epilogue reads, and the next tile's rows (its TMA then hits L2)
        if (MODE == MODE_LSRK && !a.a_zero)
          for (int f = 0; f < 6; ++f) prefetch_l2(a.res + (int64_t)f * fstride + e0 * NPG, (uint32_t)nv * NPG * 4);
        const int next = tile + gridDim.x;
        if (next < args.num_tiles) {
          const int64_t n0 = tile_e0(next);
          const uint32_t nn = (uint32_t)tile_nv(next);
          for (int f = 0; f < 6; ++f) prefetch_l2(a.u + (int64_t)f * fstride + n0 * NPG, nn * NPG * 4);
        }
      }
      // warm L2 with the out-of-tile face neighbours' rows (read by the flux passes)
      for (int q = tid; q < nv * 4; q += PROD) {
        const int code = s_code[q];
        const int64_t nb = s_nbr[q];
        if (code >= 0 && (nb < e0 || nb >= e0 + nv)) {
#pragma unroll
          for (int f = 0; f < 6; ++f) {
            const float* p = a.u + (int64_t)f * fstride + nb * NPG;
            prefetch_line_l2(p);
            prefetch_line_l2(p + NPG - 1);
          }
        }
      }
      mbar_wait(stage_free, (it & 1) ^ 1);  // the previous epilogue's staging (s_lo, s_fx) is stored
      if (tid == 0) TC_TRACE(0, 100 * it + 3);
      // tf32 remainder of M-tile t into ring slot (t == 1); the slot's last chunk is zero
      auto split = [&](int t, int slot, uint32_t use) {
        mbar_wait(&lo_empty[slot], (use & 1) ^ 1);
        const float4* src = reinterpret_cast<const float4*>(s_u + t * UT);
        float4* dst = reinterpret_cast<float4*>(s_lo + slot * LT);
        for (int i = tid; i < KCH * T::ROWS; i += PROD) {
          float4 lo = make_float4(0.f, 0.f, 0.f, 0.f);
          if (i < UCH * T::ROWS) {
            const float4 x = src[i];
            lo = make_float4(x.x - tf32_trunc(x.x), x.y - tf32_trunc(x.y), x.z - tf32_trunc(x.z), x.w - tf32_trunc(x.w));
          }
          dst[i] = lo;
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&lo_full[slot]);
      };
      // surface flux of one face -> SS A operand of the LIFT GEMM (oracle.py:50-58, 82-85; maxwell.py:73-132)
      auto flux = [&](int face) {
        const bool live = unit_ok && ur < nv;
        const uint32_t use = (uint32_t)(4 * it + face);
        if (unit_ok) {
          const int code = live ? s_code[ur * 4 + face] : -1;
          const int nb = s_nbr[ur * 4 + face];
          const float* gk = s_geo + ur * GEO_WORDS;
          const float nx = gk[10 + 3 * face], ny = gk[11 + 3 * face], nz = gk[12 + 3 * face];
          const float sc = live ? gk[22 + face] * gk[9] : 0.f;
          const float se = sc * a.inv_eps * a.inv_2z, sh = sc * a.inv_mu * a.inv_2y;
          int im[4], jn[4], jc[4];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            jc[jj] = (jj + ub) & 3;  // node of the unit's chunk visited at step jj
            const int slot = 4 * ub + jc[jj];
            const int node = slot < NFP ? slot : 0;
            im[jj] = s_fmask[face * NFP + node];
            jn[jj] = code >= 0 ? s_ptab[code * NFP + node] : 0;
          }
          // field f = t + 3h of row e at node j: s_u + t UT + (j / 4) CHUNK + (64 h + e) 16 + (j % 4) 4
          auto su = [&](int f, int e, int j) {
            const int t = f % 3, h = f / 3;
            return *reinterpret_cast<const float*>(s_u + t * UT + (j >> 2) * CHUNK + (64 * h + e) * 16 + (j & 3) * 4);
          };
          // neighbour traces first (all 24 loads in flight), then the flux buffer's release
          float up[4][6];
          const int64_t loc = (int64_t)nb - e0;
          if (code >= 0 && loc >= 0 && loc < nv) {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
              for (int f = 0; f < 6; ++f) up[jj][f] = su(f, (int)loc, jn[jj]);
          } else if (code >= 0) {
            const float* g = a.u + (int64_t)nb * NPG;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
              for (int f = 0; f < 6; ++f) up[jj][f] = __ldg(g + f * fstride + jn[jj]);
          }
          mbar_wait(fx_empty, (use & 1) ^ 1);
          if (tid == 0) TC_TRACE(0, 100 * it + 30 + face);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            float um[6];
#pragma unroll
            for (int f = 0; f < 6; ++f) um[f] = su(f, ur, im[jj]);
            if (code < 0) {  // PEC mirror (maxwell.py:117-132)
              const float nde = nx * um[0] + ny * um[1] + nz * um[2];
              const float ndh = nx * um[3] + ny * um[4] + nz * um[5];
              up[jj][0] = -um[0] + 2.f * nde * nx;
              up[jj][1] = -um[1] + 2.f * nde * ny;
              up[jj][2] = -um[2] + 2.f * nde * nz;
              up[jj][3] = um[3] - 2.f * ndh * nx;
              up[jj][4] = um[4] - 2.f * ndh * ny;
              up[jj][5] = um[5] - 2.f * ndh * nz;
            }
            float out[6];
            upwind_num(um, up[jj], nx, ny, nz, a.zp, a.yp, out);
            const bool real = 4 * ub + jc[jj] < NFP;
            const float kse = real ? se : 0.f, ksh = real ? sh : 0.f;
#pragma unroll
            for (int c = 0; c < 6; ++c) {
              // component c -> M-tile c % 3, row (h = 1 - c / 3, e): the lane whose curl updates c
              const float v = out[c] * (c < 3 ? kse : ksh);
              const float hi = tf32_trunc(v);
              unsigned char* p = s_fx + (2 * (c % 3)) * T::FX_HALF + ub * CHUNK + ((c < 3 ? 64 : 0) + ur) * 16 + jc[jj] * 4;
              *reinterpret_cast<float*>(p) = hi;
              *reinterpret_cast<float*>(p + T::FX_HALF) = v - hi;
            }
          }
        } else {
          mbar_wait(fx_empty, (use & 1) ^ 1);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(fx_full);
      };
      split(0, 0, 2u * it);
      if (tid == 0) TC_TRACE(0, 100 * it + 4);
      split(1, 1, (uint32_t)it);
      if (tid == 0) TC_TRACE(0, 100 * it + 5);
      flux(0);
      if (tid == 0) TC_TRACE(0, 100 * it + 6);
      flux(1);
      if (tid == 0) TC_TRACE(0, 100 * it + 7);
      split(2, 0, 2u * it + 1);
      if (tid == 0) TC_TRACE(0, 100 * it + 8);
      flux(2);
      if (tid == 0) TC_TRACE(0, 100 * it + 9);
      flux(3);
      if (tid == 0) TC_TRACE(0, 100 * it + 10);
      named_sync(1, PROD);  // every producer is done with s_u, s_geo, s_nbr, s_code
      if (tid == 0) {
        TC_TRACE(0, 100 * it + 11);
        mbar_wait(u_free, it & 1);  // the tile's volume MMAs have read s_u
        TC_TRACE(0, 100 * it + 12);
        const int next = tile + gridDim.x;
        if (next < args.num_tiles) issue_tile(next);
      }
    }
  } else {
    // ====================== epilogue (+ MMA issue by warp PWARPS) ======================
    const bool issuer = warp == T::PWARPS;
    const uint32_t idv = idesc_tf32(128, T::NV), idl = idesc_tf32(128, T::NL);
    const uint32_t u_a = smem_u32(s_u), lo_a = smem_u32(s_lo), db_a = smem_u32(s_db), lb_a = smem_u32(s_lb),
                   fx_a = smem_u32(s_fx);
    const int q = warp & 3, half = (warp - T::PWARPS) >> 2;
    const int h = q >> 1, e = (q & 1) * 32 + lane;
    const int orow = (1 - h) * 64 + e;          // staging row of this thread's output component
    const uint32_t lane_addr = static_cast<uint32_t>(q * 32) << 16;
    const float m = h ? a.inv_eps : -a.inv_mu;  // curl H / eps drives E, -(curl E) / mu drives H
    constexpr int B0 = (T::NBLK + 1) / 2;       // node blocks [0, B0) for half 0, [B0, NBLK) for half 1
    const int blk0 = half ? B0 : 0, blk1 = half ? T::NBLK : B0;
    const bool lsrk_res = MODE == MODE_LSRK && !a.a_zero;
    if (issuer) mbar_wait(b_ops, 0);
    griddep_wait();
    int it = 0;
    for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x, ++it) {
      const int64_t e0 = tile_e0(tile);
      const int nv = tile_nv(tile);
      const bool live = e < nv;
      // staging of pair t in buffer b: [res | u][chunk][h][e][4]
      auto stage_load = [&](int t, int b) {
        if (MODE != MODE_LSRK) {  // RHS: nothing to load; the arrival hands the buffer to the writers
          mbar_arrive(&stg_full[b]);
          return;
        }
        unsigned char* sb = stage[b];
        mbar_expect_tx(&stg_full[b], (lsrk_res ? 2 : 1) * UT);
        for (int k = 0; k < UCH; ++k) {
          if (lsrk_res) tma_load_chunk(sb + k * CHUNK, &args.tm_res, k, e0, t, &stg_full[b]);
          tma_load_chunk(sb + UT + k * CHUNK, &args.tm_u, k, e0, t, &stg_full[b]);
        }
      };
      auto stage_store = [&](int t, int b) {
        const unsigned char* sb = stage[b];
        for (int k = 0; k < UCH; ++k) {
          if (MODE == MODE_LSRK) {
            tma_store_chunk(&args.tm_res, k, e0, t, sb + k * CHUNK);
            tma_store_chunk(&args.tm_out, k, e0, t, sb + UT + k * CHUNK);
          } else {
            tma_store_chunk(&args.tm_out, k, e0, t, sb + k * CHUNK);
          }
        }
        bulk_commit();
      };
      if (issuer) {
        mbar_wait(acc_empty, (it & 1) ^ 1);
        fence_after_sync();
        if (lane == 0) TC_TRACE(1, 100 * it + 50);
        auto volume = [&](int t) {  // 3xTF32 D_mu u of M-tile t (A: the state tile and its remainder)
          const int slot = t == 1 ? 1 : 0;
          const uint32_t use = slot ? (uint32_t)it : 2u * it + (t == 2);
          mbar_wait(&lo_full[slot], use & 1);
          fence_after_sync();
          if (elect_one()) {
            const uint32_t acc = tmem + t * T::ACC;
#pragma unroll
            for (int s = 0; s < T::VKS; ++s) {
              const uint64_t ah = desc_kmajor(u_a + t * UT + s * 2 * CHUNK, CHUNK, 128);
              const uint64_t al = desc_kmajor(lo_a + slot * LT + s * 2 * CHUNK, CHUNK, 128);
              const uint64_t bh = desc_kmajor(db_a + s * 2 * T::NV * 16, T::NV * 16, 128);
              const uint64_t bl = desc_kmajor(db_a + T::DB_HALF + s * 2 * T::NV * 16, T::NV * 16, 128);
              mma_tf32(acc, ah, bh, idv, s > 0 ? 1u : 0u);
              mma_tf32(acc, al, bh, idv, 1u);
              mma_tf32(acc, ah, bl, idv, 1u);
            }
            mma_commit(&lo_empty[slot]);
            if (t == 2) mma_commit(u_free);
          }
          __syncwarp();
        };
        auto lift = [&](int f) {  // 3xTF32 LIFT of face f's flux for the three M-tiles
          const uint32_t use = (uint32_t)(4 * it + f);
          mbar_wait(fx_full, use & 1);
          fence_after_sync();
          if (elect_one()) {
#pragma unroll
            for (int t = 0; t < 3; ++t) {
              const uint32_t acc = tmem + t * T::ACC + T::NV;
#pragma unroll
              for (int s2 = 0; s2 < T::FKS; ++s2) {
                const int ks = f * T::FKS + s2;
                const uint64_t ah = desc_kmajor(fx_a + (2 * t) * T::FX_HALF + s2 * 2 * CHUNK, CHUNK, 128);
                const uint64_t al = desc_kmajor(fx_a + (2 * t + 1) * T::FX_HALF + s2 * 2 * CHUNK, CHUNK, 128);
                const uint64_t bh = desc_kmajor(lb_a + ks * 2 * T::NL * 16, T::NL * 16, 128);
                const uint64_t bl = desc_kmajor(lb_a + T::LB_HALF + ks * 2 * T::NL * 16, T::NL * 16, 128);
                mma_tf32(acc, ah, bh, idl, (f > 0 || s2 > 0) ? 1u : 0u);
                mma_tf32(acc, al, bh, idl, 1u);
                mma_tf32(acc, ah, bl, idl, 1u);
              }
            }
            mma_commit(fx_empty);
            if (f == 3) mma_commit(acc_full);
          }
          __syncwarp();
        };
        // the producers' order: the flux buffer is single, so face 1 needs face 0's MMAs, and M-tile
        // 2's remainder reuses slot 0 after M-tile 0's MMAs
        volume(0);
        volume(1);
        lift(0);
        lift(1);
        volume(2);
        lift(2);
        lift(3);
        if (lane == 0) TC_TRACE(1, 100 * it + 57);
        // staging A (the remainder ring) is idle once the volume MMAs are done, B (the flux buffer)
        // once the last LIFT MMAs are
        mbar_wait(u_free, it & 1);
        if (elect_one()) stage_load(0, 0);
        __syncwarp();
        mbar_wait(acc_full, it & 1);
        if (elect_one()) stage_load(1, 1);
        __syncwarp();
      }
      float pr[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) pr[k] = live ? __ldg(a.geo + (e0 + e) * GEO_WORDS + k) * m : 0.f;
      mbar_wait(acc_full, it & 1);
      fence_after_sync();
      if (issuer && lane == 0) TC_TRACE(1, 100 * it + 58);
      // component pair t: this thread updates component t + 3 (1 - h) of element e
      auto pair = [&](int t, int b, uint32_t use) {
        const int t1 = (t + 1) % 3, t2 = (t + 2) % 3;
        mbar_wait(&stg_full[b], use & 1);
        float4* srow = reinterpret_cast<float4*>(stage[b]) + orow;  // + k * 128: chunk k
#pragma unroll 1
        for (int blk = blk0; blk < blk1; ++blk) {
          const int i0 = 4 * blk;
          float d1[3][4], d2[3][4], l[4];
#pragma unroll
          for (int mu = 0; mu < 3; ++mu) {
            tmem_ld4(tmem + lane_addr + t1 * T::ACC + mu * T::MUS + i0, d1[mu]);
            tmem_ld4(tmem + lane_addr + t2 * T::ACC + mu * T::MUS + i0, d2[mu]);
          }
          tmem_ld4(tmem + lane_addr + t * T::ACC + T::NV + i0, l);
          float4 ro = make_float4(0.f, 0.f, 0.f, 0.f), uo = ro;
          if (MODE == MODE_LSRK) {
            if (lsrk_res) ro = srow[blk * T::ROWS];
            uo = srow[T::UCH * T::ROWS + blk * T::ROWS];
          }
          tmem_ld_wait();
          float r[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float c = l[j];
#pragma unroll
            for (int mu = 0; mu < 3; ++mu) {
              c = fmaf(pr[mu * 3 + t1], d2[mu][j], c);
              c = fmaf(-pr[mu * 3 + t2], d1[mu][j], c);
            }
            r[j] = i0 + j < NP ? c : 0.f;
          }
          if (MODE == MODE_RHS) {
            srow[blk * T::ROWS] = make_float4(r[0], r[1], r[2], r[3]);
          } else {
            float4 rr;
            rr.x = fmaf(a.a, ro.x, a.dt * r[0]);
            rr.y = fmaf(a.a, ro.y, a.dt * r[1]);
            rr.z = fmaf(a.a, ro.z, a.dt * r[2]);
            rr.w = fmaf(a.a, ro.w, a.dt * r[3]);
            srow[blk * T::ROWS] = rr;
            srow[T::UCH * T::ROWS + blk * T::ROWS] =
                make_float4(fmaf(a.b, rr.x, uo.x), fmaf(a.b, rr.y, uo.y), fmaf(a.b, rr.z, uo.z), fmaf(a.b, rr.w, uo.w));
          }
        }
        if (t == 2) {  // every TMEM read of this tile is done: the next tile's MMAs may start
          fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty);
        }
        fence_async_smem();  // staging writes -> visible to the TMA store
        named_sync(2, T::EPI);
        if (issuer) {
          if (elect_one()) stage_store(t, b);
          __syncwarp();
        }
      };
      pair(0, 0, 2u * it);
      pair(1, 1, (uint32_t)it);
      if (issuer) {
        if (elect_one()) {
          bulk_wait_read<1>();  // pair 0's stores have read staging A
          stage_load(2, 0);
        }
        __syncwarp();
      }
      pair(2, 0, 2u * it + 1);
      if (issuer) {
        if (elect_one()) {
          bulk_wait_read<0>();  // all stores have read the staging: hand s_lo / s_fx back
          mbar_arrive(stage_free);
        }
        __syncwarp();
        if (lane == 0) TC_TRACE(1, 100 * it + 59);
      }
    }
    if (issuer) {
      if (elect_one()) bulk_wait<0>();  // the last stores are complete before the grid ends
      __syncwarp();
    }
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (warp == T::PWARPS) tmem_dealloc(tmem, 512);
}

}  // namespace dgm
