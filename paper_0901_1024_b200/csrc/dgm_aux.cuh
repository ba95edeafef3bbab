// dgm_aux.cuh -- layout conversion, halo staging and the mass-norm reduction.
#pragma once

#include "dgm_stage.cuh"

namespace dgm {

// natural float64 (6, K, NP) -> padded T (6, kf, NPG), zero padding
// (reference fields.py:24-29 to_padded).
template <int N, typename T>
__global__ void pack_kernel(const double* __restrict__ nat, T* __restrict__ pad, int64_t k_total,
                            int64_t kf) {
  using C = Cfg<N, T>;
  const int64_t total = 6 * k_total * C::NPG;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = x / C::NPG;
    const int j = (int)(x - row * C::NPG);
    const int64_t f = row / k_total, k = row - f * k_total;
    const T v = (j < C::NP) ? (T)nat[row * C::NP + j] : T(0);
    pad[(f * kf + k) * C::NPG + j] = v;
  }
}

// padded T -> natural float64 (fields.py:32-35 from_padded).
template <int N, typename T>
__global__ void unpack_kernel(const T* __restrict__ pad, double* __restrict__ nat, int64_t k_total,
                              int64_t kf) {
  using C = Cfg<N, T>;
  const int64_t total = 6 * k_total * C::NP;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = x / C::NP;
    const int j = (int)(x - row * C::NP);
    const int64_t f = row / k_total, k = row - f * k_total;
    nat[x] = (double)pad[(f * kf + k) * C::NPG + j];
  }
}

// send[c][f][NPG] = u[f][elements[c]][:]   (16-byte chunks)
template <int N, typename T>
__global__ void halo_pack_kernel(const T* __restrict__ u, const int* __restrict__ elems, int64_t count,
                                 int64_t kf, T* __restrict__ send) {
  using C = Cfg<N, T>;
  using V = typename V16<T>::type;
  constexpr int RV = C::NPG / C::VEC;
  const int64_t total = count * 6 * RV;
  const V* uv = reinterpret_cast<const V*>(u);
  V* sv = reinterpret_cast<V*>(send);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = x / (6 * RV);
    const int r = (int)(x - c * 6 * RV);
    const int f = r / RV, jv = r - f * RV;
    sv[x] = uv[((int64_t)f * kf + elems[c]) * RV + jv];
  }
}

// u[f][ghost_begin + c][:] = recv[c][f][:]
template <int N, typename T>
__global__ void halo_unpack_kernel(const T* __restrict__ recv, int64_t count, int64_t ghost_begin,
                                   int64_t kf, T* __restrict__ u) {
  using C = Cfg<N, T>;
  using V = typename V16<T>::type;
  constexpr int RV = C::NPG / C::VEC;
  const int64_t total = count * 6 * RV;
  const V* rv = reinterpret_cast<const V*>(recv);
  V* uv = reinterpret_cast<V*>(u);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = x / (6 * RV);
    const int r = (int)(x - c * 6 * RV);
    const int f = r / RV, jv = r - f * RV;
    uv[((int64_t)f * kf + ghost_begin + c) * RV + jv] = rv[x];
  }
}

// *out += sum_k J_k sum_f w_f u_fk^T M u_fk   (maxwell.py:211-232)
template <int N, typename T>
__global__ void __launch_bounds__(Cfg<N, T>::THREADS)
mass_norm_kernel(const T* __restrict__ u, const T* __restrict__ mass, const T* __restrict__ det_j,
                 int64_t kf, int64_t e_begin, int64_t e_end, double w_e, double w_h,
                 double* __restrict__ out) {
  using C = Cfg<N, T>;
  using V = typename V16<T>::type;
  constexpr int TE = C::TE, NPG = C::NPG, NP = C::NP, VEC = C::VEC, G = C::G, E = C::E;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s_u = reinterpret_cast<T*>(smem_raw);
  __shared__ double s_red[32];

  const int tid = threadIdx.x;
  const int64_t e0 = e_begin + (int64_t)blockIdx.x * TE;
  const int nv = (int)min((int64_t)TE, e_end - e0);
  constexpr int RV = NPG / VEC;
  const V zero = {};
  for (int f = 0; f < 6; ++f) {
    const V* sf = reinterpret_cast<const V*>(u + ((int64_t)f * kf + e0) * NPG);
    V* df = reinterpret_cast<V*>(s_u) + f * TE * RV;
    for (int c = tid; c < TE * RV; c += blockDim.x) df[c] = (c < nv * RV) ? sf[c] : zero;
  }
  __syncthreads();

  double part = 0.0;
  if (tid < C::WORK) {
    const int i = tid / G, g = tid - i * G;
    T acc[6][E];
#pragma unroll
    for (int f = 0; f < 6; ++f)
#pragma unroll
      for (int e = 0; e < E; ++e) acc[f][e] = T(0);
    const V* mv = reinterpret_cast<const V*>(mass);
#pragma unroll 1
    for (int jc = 0; jc < C::NJC; ++jc) {
      const V m = __ldg(mv + (size_t)jc * NP + i);
#pragma unroll
      for (int f = 0; f < 6; ++f)
#pragma unroll
        for (int e = 0; e < E; ++e)
          acc[f][e] = V16<T>::fma_dot(m, *reinterpret_cast<const V*>(s_u + (f * TE + e * G + g) * NPG + jc * VEC), acc[f][e]);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = e * G + g;
      if (k < nv) {
        double pe = 0.0, ph = 0.0;
#pragma unroll
        for (int f = 0; f < 3; ++f) pe += (double)s_u[(f * TE + k) * NPG + i] * (double)acc[f][e];
#pragma unroll
        for (int f = 3; f < 6; ++f) ph += (double)s_u[(f * TE + k) * NPG + i] * (double)acc[f][e];
        part += (double)det_j[e0 + k] * (w_e * pe + w_h * ph);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if ((tid & 31) == 0) s_red[tid >> 5] = part;
  __syncthreads();
  if (tid < 32) {
    double v = (tid < (int)(blockDim.x >> 5)) ? s_red[tid] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (tid == 0) atomicAdd(out, v);
  }
}

}  // namespace dgm
