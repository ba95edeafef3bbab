// tc_probe.cu -- test-only probe of the tcgen05 kind::tf32 path (libdgm_probe.so).
//
// C[128 x N] = A[128 x K] * B[N x K]^T with 1 (plain TF32) or 3 (3xTF32:
// hi*hi + lo*hi + hi*lo) MMA passes, operands staged in the K-major
// SWIZZLE_NONE layout of tc05.cuh, accumulator in TMEM, read back with
// tcgen05.ld.  tests/test_gpu_tc05.py compares it with an fp64 product.
#include <cuda_runtime.h>

#include "tc05.cuh"

namespace {

__global__ void __launch_bounds__(128) probe_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                    float* __restrict__ c, int n, int k, int passes) {
  using namespace dgm::tc;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int m = 128;
  float* a_hi = reinterpret_cast<float*>(smem);
  float* a_lo = a_hi + m * k;
  float* b_hi = a_lo + m * k;
  float* b_lo = b_hi + n * k;
  const int tid = threadIdx.x, warp = tid >> 5;
  // passes = 13: 3xTF32 with the hi operands stored unmasked (does kind::tf32 truncate its fp32
  // inputs?  then raw x and the masked hi are the same operand and the error stays fp32-class)
  const bool raw = passes == 13;
  if (raw) passes = 3;

  for (int i = tid; i < m * k; i += blockDim.x) {
    const int r = i / k, q = i - r * k;
    const int off = ((q >> 2) * m + r) * 4 + (q & 3);
    float hi, lo;
    split_tf32(a[i], hi, lo);
    a_hi[off] = raw ? a[i] : hi;  // raw: the MMA sees the unmasked fp32 bits as its tf32 input
    a_lo[off] = lo;
  }
  for (int i = tid; i < n * k; i += blockDim.x) {
    const int r = i / k, q = i - r * k;
    const int off = ((q >> 2) * n + r) * 4 + (q & 3);
    float hi, lo;
    split_tf32(b[i], hi, lo);
    b_hi[off] = raw ? b[i] : hi;
    b_lo[off] = lo;
  }
  if (warp == 0) tmem_alloc(&tmem_base, 256);
  if (tid == 32) {
    mbar_init(&mbar, 1);
    mbar_init_fence();
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;

  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(m, n);
    for (int s = 0; s < k / 8; ++s) {
      const uint32_t ao = s * 2 * m * 16, bo = s * 2 * n * 16;
      const uint64_t ah = desc_kmajor(smem_u32(a_hi) + ao, m * 16, 128);
      const uint64_t al = desc_kmajor(smem_u32(a_lo) + ao, m * 16, 128);
      const uint64_t bh = desc_kmajor(smem_u32(b_hi) + bo, n * 16, 128);
      const uint64_t bl = desc_kmajor(smem_u32(b_lo) + bo, n * 16, 128);
      mma_tf32(tmem, ah, bh, idesc, s > 0);
      if (passes == 3) {
        mma_tf32(tmem, al, bh, idesc, 1);
        mma_tf32(tmem, ah, bl, idesc, 1);
      }
    }
    mma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  fence_after_sync();
  const int row = warp * 32 + (tid & 31);
  for (int col = 0; col < n; col += 8) {
    float v[8];
    tmem_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + col, v);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 8; ++j) c[row * n + col + j] = v[j];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// Same product with A written to TMEM by tcgen05.st (row r = lane r) and the TS-form MMA.
__global__ void __launch_bounds__(128) probe_ts_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                       float* __restrict__ c, int n, int k, int passes) {
  using namespace dgm::tc;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  float* b_hi = reinterpret_cast<float*>(smem);
  float* b_lo = b_hi + n * k;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < n * k; i += blockDim.x) {
    const int r = i / k, q = i - r * k;
    const int off = ((q >> 2) * n + r) * 4 + (q & 3);
    float hi, lo;
    split_tf32(b[i], hi, lo);
    b_hi[off] = hi;
    b_lo[off] = lo;
  }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  if (tid == 32) {
    mbar_init(&mbar, 1);
    mbar_init_fence();
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  const uint32_t a_hi_col = 256, a_lo_col = 256 + 64;
  const int row = tid;  // warp w covers lanes 32w..32w+31
  const uint32_t lane_addr = static_cast<uint32_t>(warp * 32) << 16;
  for (int k0 = 0; k0 < k; k0 += 8) {
    float hi[8], lo[8];
    for (int q = 0; q < 8; ++q) split_tf32(a[row * k + k0 + q], hi[q], lo[q]);
    tmem_st8(tmem + lane_addr + a_hi_col + k0, hi);
    tmem_st8(tmem + lane_addr + a_lo_col + k0, lo);
  }
  tmem_st_wait();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(128, n);
    for (int s = 0; s < k / 8; ++s) {
      const uint32_t bo = s * 2 * n * 16;
      const uint64_t bh = desc_kmajor(smem_u32(b_hi) + bo, n * 16, 128);
      const uint64_t bl = desc_kmajor(smem_u32(b_lo) + bo, n * 16, 128);
      mma_tf32_ts(tmem, tmem + a_hi_col + 8 * s, bh, idesc, s > 0);
      if (passes == 3) {
        mma_tf32_ts(tmem, tmem + a_lo_col + 8 * s, bh, idesc, 1);
        mma_tf32_ts(tmem, tmem + a_hi_col + 8 * s, bl, idesc, 1);
      }
    }
    mma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  fence_after_sync();
  for (int col = 0; col < n; col += 8) {
    float v[8];
    tmem_ld8(tmem + lane_addr + col, v);
    tmem_ld_wait();
    for (int j = 0; j < 8; ++j) c[row * n + col + j] = v[j];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// Throughput microbenchmark: one thread issues `reps` kind::tf32 MMAs (M=128, N=n,
// K=8) back to back into one accumulator, A from smem (ts=0) or TMEM (ts=1).
__global__ void __launch_bounds__(128) probe_rate_kernel(int n, int reps, int ts, int nacc, long long* cycles) {
  using namespace dgm::tc;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  float* a_s = reinterpret_cast<float*>(smem);       // 128 x 8
  float* b_s = a_s + 128 * 8;                          // n x 8
  for (int i = threadIdx.x; i < (128 + n) * 8; i += blockDim.x) a_s[i] = 0.f;
  if (threadIdx.x < 32) tmem_alloc(&tmem_base, 512);
  if (threadIdx.x == 32) {
    mbar_init(&mbar, 1);
    mbar_init_fence();
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  if (threadIdx.x < 32) {  // whole warp runs the (uniform) issue loop, one elected lane issues
    const uint32_t idesc = idesc_tf32(128, n);
    const uint64_t ad = desc_kmajor(smem_u32(a_s), 128 * 16, 128);
    const uint64_t bd = desc_kmajor(smem_u32(b_s), n * 16, 128);
    __syncwarp();
    const long long t0 = clock64();
    if (nacc == 0) {  // unrolled bursts of 48 MMAs, loop-invariant operands, one elect per burst
      const uint32_t idb = idesc_bf16(128, n);
      for (int r = 0; r < reps; r += 48) {
        if (elect_one()) {
          if (ts == 2) {
#pragma unroll
            for (int q = 0; q < 48; ++q) mma_bf16(tmem + (q % 6) * 64, ad, bd, idb, 1u);
          } else if (ts == 1) {
#pragma unroll
            for (int q = 0; q < 48; ++q) mma_tf32_ts(tmem + (q % 6) * 64, tmem + 448, bd, idesc, 1u);
          } else {
#pragma unroll
            for (int q = 0; q < 48; ++q) mma_tf32(tmem + (q % 6) * 64, ad, bd, idesc, 1u);
          }
        }
        __syncwarp();
      }
    } else if (nacc == 1) {
      for (int r = 0; r < reps; ++r) {
        if (elect_one()) {
          if (ts == 2) mma_bf16(tmem, ad, bd, idesc_bf16(128, n), r > 0);
          else if (ts) mma_tf32_ts(tmem, tmem + 448, bd, idesc, r > 0);
          else mma_tf32(tmem, ad, bd, idesc, r > 0);
        }
        __syncwarp();
      }
    } else {
      for (int r = 0; r < reps; r += 6) {
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          if (elect_one()) {
            const uint32_t acc = tmem + (uint32_t)(c * 64);
            if (ts) mma_tf32_ts(acc, tmem + 448, bd, idesc, r > 0);
            else mma_tf32(acc, ad, bd, idesc, r > 0);
          }
          __syncwarp();
        }
      }
    }
    const long long t1 = clock64();
    if (elect_one()) mma_commit(&mbar);
    __syncwarp();
    mbar_wait(&mbar, 0);
    const long long t2 = clock64();
    if (threadIdx.x == 0) {
      cycles[0] = t1 - t0;
      cycles[1] = t2 - t0;
    }
  }
  fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// Round-trip latency of the stage kernel's MMA pattern: one elected lane issues a burst of
// `nacc` x `passes` TS MMAs (M=128, N=n, K=8, accumulators round-robin), commits to an mbarrier
// and waits for it; repeated `reps` times.  cycles[0] = total, cycles[1] = issue part.
__global__ void __launch_bounds__(128) probe_burst_kernel(int n, int reps, int nacc, int passes, long long* cycles) {
  using namespace dgm::tc;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  float* b_s = reinterpret_cast<float*>(smem);  // n x 8
  for (int i = threadIdx.x; i < n * 8; i += blockDim.x) b_s[i] = 0.f;
  if (threadIdx.x < 32) tmem_alloc(&tmem_base, 256);
  if (threadIdx.x == 32) {
    mbar_init(&mbar, 1);
    mbar_init_fence();
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  if (threadIdx.x < 32) {
    const uint32_t idesc = idesc_tf32(128, n);
    const uint64_t bd = desc_kmajor(smem_u32(b_s), n * 16, 128);
    long long issue = 0;
    __syncwarp();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const long long ti = clock64();
      if (elect_one()) {
        for (int p = 0; p < passes; ++p)
          for (int c = 0; c < nacc; ++c) mma_tf32_ts(tmem + (uint32_t)(c * n), tmem + 224, bd, idesc, 1u);
        mma_commit(&mbar);
      }
      __syncwarp();
      issue += clock64() - ti;
      mbar_wait(&mbar, r & 1);
      fence_after_sync();
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) {
      cycles[0] = t1 - t0;
      cycles[1] = issue;
    }
  }
  fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

// Primitive costs of the stage kernel's producer / MMA hand-off (one CTA, `pw` producer warps + 1 MMA warp):
//   mode 0: producers only, per iteration 6 x tcgen05.st.32x32b.x4 + wait::st (no MMA)
//   mode 1: full ping-pong with a 2-stage A ring: producers wait empty, store, fence, arrive full;
//           the MMA warp waits full, issues 9 TS MMAs (3 accumulators x 3 passes), commits empty.
// cycles[0] = total cycles of producer warp 0 for `reps` iterations.
__global__ void __launch_bounds__(320) probe_handoff_kernel(int reps, int mode, int pw, long long* cycles) {
  using namespace dgm::tc;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[2], empty[2];
  __shared__ uint32_t tmem_base;
  float* b_s = reinterpret_cast<float*>(smem);  // 48 x 8 x 2
  for (int i = threadIdx.x; i < 48 * 16; i += blockDim.x) b_s[i] = 0.f;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&tmem_base, 256);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], pw);
      mbar_init(&empty[i], 1);
    }
    mbar_init_fence();
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  if (warp < pw) {
    const uint32_t lane_addr = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int khalf = (warp >> 2) & 1;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int slot = r & 1;
      if (mode == 1) {
        mbar_wait(&empty[slot], ((r >> 1) & 1) ^ 1);
        fence_after_sync();
      }
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const uint32_t col = 160 + slot * 48 + t * 16 + 4 * khalf;
        tmem_st4(tmem + lane_addr + col, v);
        tmem_st4(tmem + lane_addr + col + 8, v);
      }
      tmem_st_wait();
      if (mode == 1) {
        fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[slot]);
      }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cycles[0] = t1 - t0;
  } else if (warp == pw && mode == 1) {
    const uint32_t idesc = idesc_tf32(128, 48);
    const uint64_t bd = desc_kmajor(smem_u32(b_s), 48 * 16, 128);
    for (int r = 0; r < reps; ++r) {
      const int slot = r & 1;
      mbar_wait(&full[slot], (r >> 1) & 1);
      fence_after_sync();
      if (elect_one()) {
        const uint32_t abase = tmem + 160 + slot * 48;
#pragma unroll
        for (int t = 0; t < 3; ++t) mma_tf32_ts(tmem + t * 48, abase + t * 16, bd, idesc, r > 0);
#pragma unroll
        for (int t = 0; t < 3; ++t) mma_tf32_ts(tmem + t * 48, abase + t * 16 + 8, bd, idesc, 1u);
#pragma unroll
        for (int t = 0; t < 3; ++t) mma_tf32_ts(tmem + t * 48, abase + t * 16, bd, idesc, 1u);
        mma_commit(&empty[slot]);
      }
      __syncwarp();
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// Issue cost of one K-step's MMA burst in different shapes (M=128, N=48, TS, K=8):
//   variant 0: 3 acc x 3 passes, pass-major (t0p0 t1p0 t2p0 t0p1 ...), 1 commit
//   variant 1: same, 2 commits
//   variant 2: 3 acc x 3 passes, acc-major (t0p0 t0p1 t0p2 t1p0 ...), 1 commit
//   variant 3: 9 independent accumulators (split passes), 1 commit
//   variant 4: 6 acc x 3 passes pass-major (18 MMAs), 1 commit
//   variant 5: 3 acc x 3 passes, pass-major, two bursts back to back before one wait (2 K-steps)
__global__ void __launch_bounds__(128) probe_shape_kernel(int reps, int variant, long long* cycles) {
  using namespace dgm::tc;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  float* b_s = reinterpret_cast<float*>(smem);
  for (int i = threadIdx.x; i < 48 * 16; i += blockDim.x) b_s[i] = 0.f;
  if (threadIdx.x < 32) tmem_alloc(&tmem_base, 512);
  if (threadIdx.x == 32) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init_fence();
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  if (threadIdx.x < 32) {
    const uint32_t idesc = idesc_tf32(128, 48);
    const uint64_t bd = desc_kmajor(smem_u32(b_s), 48 * 16, 128);
    const uint32_t a = tmem + 448;
    long long issue = 0;
    __syncwarp();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const long long ti = clock64();
      if (elect_one()) {
        if (variant == 0 || variant == 1 || variant == 5) {
          const int nb = variant == 5 ? 2 : 1;
          for (int b = 0; b < nb; ++b) {
#pragma unroll
            for (int p = 0; p < 3; ++p)
#pragma unroll
              for (int t = 0; t < 3; ++t) mma_tf32_ts(tmem + t * 48, a + 8 * (p & 1), bd, idesc, 1u);
          }
          mma_commit(&mbar[0]);
          if (variant == 1) mma_commit(&mbar[1]);
        } else if (variant == 2) {
#pragma unroll
          for (int t = 0; t < 3; ++t)
#pragma unroll
            for (int p = 0; p < 3; ++p) mma_tf32_ts(tmem + t * 48, a + 8 * (p & 1), bd, idesc, 1u);
          mma_commit(&mbar[0]);
        } else if (variant == 3) {
#pragma unroll
          for (int t = 0; t < 9; ++t) mma_tf32_ts(tmem + t * 48, a + 8 * (t & 1), bd, idesc, 1u);
          mma_commit(&mbar[0]);
        } else {
#pragma unroll
          for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int t = 0; t < 6; ++t) mma_tf32_ts(tmem + t * 48, a + 8 * (p & 1), bd, idesc, 1u);
          mma_commit(&mbar[0]);
        }
      }
      __syncwarp();
      issue += clock64() - ti;
      mbar_wait(&mbar[0], r & 1);
      if (variant == 1) mbar_wait(&mbar[1], r & 1);
      fence_after_sync();
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) {
      cycles[0] = t1 - t0;
      cycles[1] = issue;
    }
  }
  fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

}  // namespace

extern "C" int dgm_probe_mma_rate(int n, int reps, int ts, int nacc, long long* cycles_dev) {
  if (nacc < 0 || (nacc != 1 && n > 64) || n > 256) return -1;
  const size_t smem = (size_t)(128 + n) * 8 * 4;
  probe_rate_kernel<<<1, 128, smem>>>(n, reps, ts, nacc, cycles_dev);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int dgm_probe_tf32_gemm_ts(const float* a, const float* b, float* c, int n, int k, int passes,
                                      void* stream) {
  if (n < 16 || n > 256 || n % 16 || k < 8 || k > 64 || k % 8 || (passes != 1 && passes != 3 && passes != 13)) return -1;
  const size_t smem = (size_t)2 * n * k * sizeof(float);
  if (cudaFuncSetAttribute(probe_ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return -2;
  probe_ts_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(a, b, c, n, k, passes);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int dgm_probe_tf32_gemm(const float* a, const float* b, float* c, int n, int k, int passes,
                                   void* stream) {
  if (n < 8 || n > 256 || n % 8 || k < 8 || k > 64 || k % 8 || (passes != 1 && passes != 3 && passes != 13)) return -1;
  const size_t smem = (size_t)2 * (128 + n) * k * sizeof(float);
  if (cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return -2;
  probe_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(a, b, c, n, k, passes);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int dgm_probe_mma_burst(int n, int reps, int nacc, int passes, int ctas, long long* cycles_dev) {
  if (n % 16 || n < 16 || nacc * n > 224 || passes < 1) return -1;
  const size_t smem = (size_t)n * 8 * 4 + 1024;
  probe_burst_kernel<<<ctas, 128, smem>>>(n, reps, nacc, passes, cycles_dev);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int dgm_probe_handoff(int reps, int mode, int pw, int ctas, long long* cycles_dev) {
  if (pw < 1 || pw > 8 || reps < 2) return -1;
  probe_handoff_kernel<<<ctas, 32 * (pw + 1), 48 * 16 * 4 + 1024>>>(reps, mode, pw, cycles_dev);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int dgm_probe_mma_shape(int reps, int variant, int ctas, long long* cycles_dev) {
  if (variant < 0 || variant > 5) return -1;
  probe_shape_kernel<<<ctas, 128, 48 * 16 * 4 + 1024>>>(reps, variant, cycles_dev);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// FP64 tensor-pipe (DMMA, mma.sync m8n8k4 f64) throughput: every warp runs `iters` rounds of 8
// independent MMAs; the caller times the launch.  flop = blocks * warps * iters * 8 * 512.
__global__ void __launch_bounds__(256) probe_dmma_kernel(int iters, double* sink) {
  double c[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  for (int r = 0; r < iters; ++r) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[q][0]), "+d"(c[q][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.0) sink[0] = s;
}

// FP64 SIMT (DFMA) throughput: 8 independent chains per thread, `iters` rounds.
// flop = blocks * 256 * iters * 8 * 2.
__global__ void __launch_bounds__(256) probe_dfma_kernel(int iters, double* sink) {
  double c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q] = 1e-3 * q;
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 1e-12;
  for (int r = 0; r < iters; ++r) {
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = fma(c[q], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q];
  if (s == 12345.0) sink[0] = s;
}

// Both at once: even warps run the DMMA loop, odd warps the DFMA loop (do the two share a pipe?).
// flop = blocks * (4 * iters * 8 * 512 + 128 * iters * 8 * 2).
__global__ void __launch_bounds__(256) probe_fp64_mixed_kernel(int iters, double* sink) {
  if ((threadIdx.x >> 5) & 1) {
    double c[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = 1e-3 * q;
    const double a = 1.0 + 1e-9 * threadIdx.x, b = 1e-12;
    for (int r = 0; r < iters; ++r) {
#pragma unroll
      for (int q = 0; q < 8; ++q) c[q] = fma(c[q], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += c[q];
    if (s == 12345.0) sink[0] = s;
  } else {
    double c[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
    const double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
    for (int r = 0; r < iters; ++r) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[q][0]), "+d"(c[q][1])
                     : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
    if (s == 12345.0) sink[0] = s;
  }
}

// tensor: 1 DMMA, 0 DFMA, 2 both in one kernel (alternate warps)
extern "C" int dgm_probe_fp64_rate(int tensor, int blocks, int iters, double* sink, void* stream) {
  if (blocks < 1 || iters < 1) return -1;
  if (tensor == 2)
    probe_fp64_mixed_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(iters, sink);
  else if (tensor)
    probe_dmma_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(iters, sink);
  else
    probe_dfma_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(iters, sink);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// Legacy warp-level TF32 MMA (mma.sync m16n8k8 tf32, fp32 accumulate) throughput: 8 independent
// accumulators per warp, `iters` rounds; flop = blocks * 8 warps * iters * 8 * 2048.
__global__ void __launch_bounds__(256) probe_tf32sync_kernel(int iters, float* sink) {
  float c[8][4];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = c[q][2] = c[q][3] = 0.f;
  const uint32_t a0 = __float_as_uint(1.0f + 1e-6f * threadIdx.x), a1 = a0, a2 = a0, a3 = a0;
  const uint32_t b0 = __float_as_uint(0.5f), b1 = b0;
  for (int r = 0; r < iters; ++r) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  if (s == 12345.f) sink[0] = s;
}

extern "C" int dgm_probe_tf32sync_rate(int blocks, int iters, float* sink, void* stream) {
  if (blocks < 1 || iters < 1) return -1;
  probe_tf32sync_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(iters, sink);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
