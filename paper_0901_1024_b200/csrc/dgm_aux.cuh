// dgm_aux.cuh -- layout conversion, halo staging and the mass-norm reduction.
#pragma once

#include "dgm_stage.cuh"

namespace dgm {

// natural (6, K, NP) in TN (float64 as the reference, or float32) -> padded T (6, kf, NPG), zero
// padding (reference fields.py:24-29 to_padded).  perm (NULL = identity) is the operator's internal
// element order: padded slot s holds natural element perm[s] (the cast and the locality permutation
// happen in this one pass).
template <int N, typename T, typename TN>
__global__ void pack_kernel(const TN* __restrict__ nat, const int64_t* __restrict__ perm, T* __restrict__ pad,
                            int64_t k_total, int64_t kf) {
  // blockIdx.y = field; one thread per 16-byte chunk of a padded row (one vector store), the natural
  // values read as scalars (natural rows of Np values are not 16-byte aligned); indices split with a
  // compile-time divisor
  using C = Cfg<N, T>;
  using V = typename V16<T>::type;
  constexpr int VEC = C::VEC, RV = C::NPG / VEC, NP = C::NP;
  const int64_t f = blockIdx.y;
  const int64_t total = k_total * RV;
  const TN* nf = nat + f * k_total * NP;
  V* pf = reinterpret_cast<V*>(pad + f * kf * C::NPG);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = x / RV;
    const int c = (int)(x - s * RV);
    const int64_t k = perm ? __ldg(perm + s) : s;
    const TN* src = nf + k * NP + c * VEC;
    V out;
    T* o = reinterpret_cast<T*>(&out);
#pragma unroll
    for (int q = 0; q < VEC; ++q) o[q] = (c * VEC + q < NP) ? (T)src[q] : T(0);
    pf[x] = out;
  }
}

// padded T -> natural TN (fields.py:32-35 from_padded); natural element perm[s] <- padded slot s.
template <int N, typename T, typename TN>
__global__ void unpack_kernel(const T* __restrict__ pad, const int64_t* __restrict__ perm, TN* __restrict__ nat,
                              int64_t k_total, int64_t kf) {
  // blockIdx.y = field; one thread per natural value, so a warp's stores are one contiguous run (the
  // 16-byte-chunk form wrote 8-byte pieces at a 32-byte stride: 2.9 vs 6+ TB/s); compile-time divisor
  using C = Cfg<N, T>;
  constexpr int NP = C::NP;
  const int64_t f = blockIdx.y;
  const int64_t total = k_total * NP;
  TN* nf = nat + f * k_total * NP;
  const T* pf = pad + f * kf * C::NPG;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = x / NP;
    const int j = (int)(x - s * NP);
    const int64_t k = perm ? __ldg(perm + s) : s;
    nf[k * NP + j] = (TN)pf[s * C::NPG + j];
  }
}

// face_states (oracle.py:50-58): u_minus / u_plus per (field, element, face, face node) in the natural
// numbering, with the PEC mirror (maxwell.py:117-132) on walls.  Internal slot s is natural element
// elem_nat[s] (NULL = identity); internal face slot q of face f is natural face node
// node_nat[f * NFP + q] (NULL = identity; ordering.face_slot_order).
template <int N, typename T>
__global__ void face_states_kernel(const StageArgs<T> a, const int64_t* __restrict__ elem_nat,
                                   const uint8_t* __restrict__ node_nat, T* __restrict__ u_minus,
                                   T* __restrict__ u_plus) {
  using C = Cfg<N, T>;
  constexpr int NFP = C::NFP, NPG = C::NPG;
  const int64_t k_total = a.e_end;  // whole owned range
  const int64_t total = k_total * 4 * NFP;
  const int64_t fstride = a.kf * NPG;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = x / (4 * NFP);
    const int r = (int)(x - s * 4 * NFP), face = r / NFP, q = r - face * NFP;
    const T* gk = a.geo + s * GEO_WORDS;
    const T nx = gk[10 + 3 * face], ny = gk[11 + 3 * face], nz = gk[12 + 3 * face];
    const int im = a.fmask[face * NFP + q];
    T um[6], up[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) um[f] = a.u[f * fstride + s * NPG + im];
    const int code = a.code[s * 4 + face];
    if (code < 0) {
      const T nde = nx * um[0] + ny * um[1] + nz * um[2];
      const T ndh = nx * um[3] + ny * um[4] + nz * um[5];
      up[0] = -um[0] + T(2) * nde * nx;
      up[1] = -um[1] + T(2) * nde * ny;
      up[2] = -um[2] + T(2) * nde * nz;
      up[3] = um[3] - T(2) * ndh * nx;
      up[4] = um[4] - T(2) * ndh * ny;
      up[5] = um[5] - T(2) * ndh * nz;
    } else {
      const int64_t nb = a.nbr[s * 4 + face];
      const int jn = a.ptab[code * NFP + q];
#pragma unroll
      for (int f = 0; f < 6; ++f) up[f] = a.u[f * fstride + nb * NPG + jn];
    }
    const int64_t k = elem_nat ? elem_nat[s] : s;
    const int node = node_nat ? node_nat[face * NFP + q] : q;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int64_t o = ((f * k_total + k) * 4 + face) * NFP + node;
      u_minus[o] = um[f];
      u_plus[o] = up[f];
    }
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

// Face-trace halo: only the Nfp nodes of each cut face travel.
// send[c][f][i] = u[f][elem_face[2c]][fmask[face][i]], face = elem_face[2c + 1]
template <int N, typename T>
__global__ void trace_pack_kernel(const T* __restrict__ u, const int* __restrict__ elem_face,
                                  const uint8_t* __restrict__ fmask, int64_t count, int64_t kf,
                                  T* __restrict__ send) {
  using C = Cfg<N, T>;
  const int64_t total = count * 6 * C::NFP;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = x / (6 * C::NFP);
    const int r = (int)(x - c * 6 * C::NFP);
    const int f = r / C::NFP, i = r - f * C::NFP;
    const int e = __ldg(elem_face + 2 * c), face = __ldg(elem_face + 2 * c + 1);
    send[x] = u[((int64_t)f * kf + e) * C::NPG + fmask[face * C::NFP + i]];
  }
}

// u[f][elem_face[2c]][fmask[face][i]] = recv[c][f][i]: a ghost row receives only the face nodes the
// owned side reads (its other nodes are never read; faces sharing an edge write equal values)
template <int N, typename T>
__global__ void trace_unpack_kernel(const T* __restrict__ recv, const int* __restrict__ elem_face,
                                    const uint8_t* __restrict__ fmask, int64_t count, int64_t kf,
                                    T* __restrict__ u) {
  using C = Cfg<N, T>;
  const int64_t total = count * 6 * C::NFP;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = x / (6 * C::NFP);
    const int r = (int)(x - c * 6 * C::NFP);
    const int f = r / C::NFP, i = r - f * C::NFP;
    const int e = __ldg(elem_face + 2 * c), face = __ldg(elem_face + 2 * c + 1);
    u[((int64_t)f * kf + e) * C::NPG + fmask[face * C::NFP + i]] = recv[x];
  }
}

// partial[blockIdx] = sum over the CTA's elements of J_k sum_f w_f u_fk^T M u_fk   (maxwell.py:211-232);
// reduce_partials_kernel adds them into *out in a fixed order, so the value is bitwise reproducible
// (the reference's CLI reruns are byte-identical, pkg/tests/test_cli.py:106-112)
template <int N, typename T>
__global__ void __launch_bounds__(Cfg<N, T>::THREADS)
mass_norm_kernel(const T* __restrict__ u, const T* __restrict__ mass, const T* __restrict__ det_j,
                 int64_t kf, int64_t e_begin, int64_t e_end, double w_e, double w_h,
                 double* __restrict__ partial) {
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
    if (tid == 0) partial[blockIdx.x] = v;
  }
}

// *out += sum_i partial[i], one CTA: thread t sums i = t, t + 256, ... in order, then a fixed
// shuffle / shared-memory tree -- the same association for every launch of the same count.
__global__ void __launch_bounds__(256) reduce_partials_kernel(const double* __restrict__ partial, int64_t n,
                                                              double* __restrict__ out) {
  __shared__ double s_red[8];
  double v = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) v += partial[i];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += s_red[w];
    *out += t;
  }
}

}  // namespace dgm
