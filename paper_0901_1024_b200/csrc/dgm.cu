// dgm.cu -- C ABI of libdgm.so (see include/dgm.h for the contract).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <type_traits>
#include <utility>

#include "../../include/dgm.h"
#include "dgm_aux.cuh"
#include "dgm_stage.cuh"
#include "dgm_tc.cuh"
#include "dgm_tc2.cuh"

#define DGM_ABI_VERSION 4

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(DGM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return DGM_OK;
}

// The dynamic shared-memory limit is a per-function attribute shared by every plan of the same
// (order, dtype) on a device, while the bytes a plan launches with depend on its code table: the
// limit is only ever raised, so a plan created later with fewer codes cannot shrink it under an
// earlier plan's launches.
template <typename K>
int raise_smem_limit(K* kernel, size_t bytes, const char* what) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> limits;
  int dev = 0;
  if (int r = cuda_check(cudaGetDevice(&dev), "cudaGetDevice")) return r;
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = limits[{dev, reinterpret_cast<const void*>(kernel)}];
  if (bytes <= cur) return DGM_OK;
  if (int r = cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes), what))
    return r;
  cur = bytes;
  return DGM_OK;
}

// Calls fn(std::integral_constant<int, N>, T) for the runtime (order, dtype).
template <typename Fn>
int dispatch(int order, int dtype, Fn&& fn) {
  if (dtype != DGM_F32 && dtype != DGM_F64)
    return fail(DGM_ERR_UNSUPPORTED, "dtype %d not supported", dtype);
#define DGM_CASE(n)                                                          \
  case n:                                                                    \
    return dtype == DGM_F32 ? fn(std::integral_constant<int, n>{}, float{}) \
                            : fn(std::integral_constant<int, n>{}, double{});
  switch (order) {
    DGM_CASE(1) DGM_CASE(2) DGM_CASE(3) DGM_CASE(4) DGM_CASE(5)
    DGM_CASE(6) DGM_CASE(7) DGM_CASE(8) DGM_CASE(9)
    default:
      return fail(DGM_ERR_UNSUPPORTED, "order %d not supported (1..9)", order);
  }
#undef DGM_CASE
}

// Launches of a plan run on the device the plan was created on, whatever the caller's current device
// (the stream passed in belongs to that device); the previous current device is restored.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Calls fn(TN{}) for the natural-side real type.
template <typename Fn>
int natural_dispatch(int natural_dtype, Fn&& fn) {
  if (natural_dtype == DGM_F64) return fn(double{});
  if (natural_dtype == DGM_F32) return fn(float{});
  return fail(DGM_ERR_UNSUPPORTED, "natural dtype %d not supported", natural_dtype);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  const int64_t cap = 148 * 32;
  return (int)(b < cap ? b : cap);
}

}  // namespace

struct dgm_plan {
  dgm_desc d;
  size_t stage_smem;  // dynamic smem of the SIMT stage kernels
  int path;           // DGM_PATH_SIMT or DGM_PATH_TENSOR
  size_t tc_smem;     // dynamic smem of the tensor-core stage kernels
  size_t tc2_smem;    // dynamic smem of the v2 tensor-core stage kernels (N <= 4)
  int num_sms;
  int device;         // CUDA device the plan was created on (DeviceGuard)
};

namespace {
template <int N, typename T>
struct TcInfo {
  static constexpr bool supported = false;
  static constexpr int nb = 0, steps = 0, npk = 0, kv = 0, nfpk = 0;
  static constexpr int64_t floats = 0;
};
#define DGM_TC_INFO(n)                                                   \
  template <>                                                            \
  struct TcInfo<n, float> {                                              \
    static constexpr bool supported = true;                              \
    static constexpr int nb = dgm::TcCfg<n>::NB, steps = dgm::TcCfg<n>::KS; \
    static constexpr int npk = dgm::TcCfg<n>::NPK;                       \
    static constexpr int kv = dgm::TcCfg<n>::KV, nfpk = dgm::TcCfg<n>::NFPK; \
    static constexpr int64_t floats = (int64_t)dgm::TcCfg<n>::B_FLOATS;  \
  };
DGM_TC_INFO(1)
DGM_TC_INFO(2)
DGM_TC_INFO(3)
DGM_TC_INFO(4)
DGM_TC_INFO(5)
DGM_TC_INFO(6)
DGM_TC_INFO(7)
DGM_TC_INFO(8)
DGM_TC_INFO(9)
#undef DGM_TC_INFO

template <int N>
struct Tc2Info {
  static constexpr bool supported = N <= 4;
  static constexpr int64_t floats = supported ? (int64_t)dgm::Tc2Cfg<(N <= 4 ? N : 4)>::B_FLOATS : 0;
};
}  // namespace

extern "C" {

int32_t dgm_version(void) { return DGM_ABI_VERSION; }

const char* dgm_last_error(void) { return g_err; }

int dgm_layout(int32_t order, int32_t dtype, dgm_layout_info* out) {
  if (!out) return fail(DGM_ERR_INVALID, "dgm_layout: null output");
  return dispatch(order, dtype, [&](auto n, auto t) -> int {
    using C = dgm::Cfg<decltype(n)::value, decltype(t)>;
    out->order = order;
    out->dtype = dtype;
    out->num_nodes = C::NP;
    out->num_face_nodes = C::NFP;
    out->np_stride = C::NPG;
    out->diff_chunks = C::NJC;
    out->lift_chunks = C::NLC;
    out->vec = C::VEC;
    out->tile_elements = C::TE;
    out->threads = C::THREADS;
    out->smem_bytes_fixed = (int64_t)C::SMEM_FIXED;
    using TI = TcInfo<decltype(n)::value, decltype(t)>;
    out->tc_supported = TI::supported ? 1 : 0;
    out->tc_nb = TI::nb;
    out->tc_steps = TI::steps;
    out->tc_npk = TI::npk;
    out->tc_kv = TI::kv;
    out->tc_nfpk = TI::nfpk;
    out->tc_operand_floats = TI::floats;
    using T2 = Tc2Info<decltype(n)::value>;
    const bool f32 = sizeof(decltype(t)) == 4;
    out->tc2_supported = (f32 && T2::supported) ? 1 : 0;
    out->tc2_operand_floats = (f32 && T2::supported) ? T2::floats : 0;
    return DGM_OK;
  });
}

int dgm_plan_create(const dgm_desc* desc, dgm_plan** out) {
  g_err[0] = 0;
  if (!desc || !out) return fail(DGM_ERR_INVALID, "dgm_plan_create: null argument");
  const dgm_desc& d = *desc;
  if (d.num_elements < 0 || d.field_stride < d.num_elements)
    return fail(DGM_ERR_INVALID, "field_stride (%lld) must be >= num_elements (%lld) >= 0",
                (long long)d.field_stride, (long long)d.num_elements);
  if (d.field_stride >= (int64_t)1 << 31)
    return fail(DGM_ERR_INVALID, "field_stride must fit int32 element ids");
  if (!(d.permittivity > 0.0) || !(d.permeability > 0.0))
    return fail(DGM_ERR_INVALID, "material constants must be positive");
  if (d.num_codes < 0 || d.num_codes > 4096)
    return fail(DGM_ERR_INVALID, "num_codes %d out of range", d.num_codes);
  const void* ptrs[] = {d.diff_packed, d.lift_packed, d.geometry};
  for (const void* p : ptrs)
    if (!p || !aligned16(p)) return fail(DGM_ERR_INVALID, "operand pointers must be non-null and 16-byte aligned");
  if (!d.neighbors || !d.codes || !d.face_nodes || (d.num_codes > 0 && !d.code_table))
    return fail(DGM_ERR_INVALID, "connectivity pointers must be non-null");
  size_t smem = 0;
  int rc = dispatch(d.order, d.dtype, [&](auto n, auto t) -> int {
    constexpr int N = decltype(n)::value;
    using T = decltype(t);
    using C = dgm::Cfg<N, T>;
    smem = C::SMEM_FIXED + (size_t)d.num_codes * C::NFP + 4 * (size_t)C::NP + (size_t)d.num_codes;  // + pair tables
    smem = (smem + 15) & ~size_t(15);
    if (smem > 227 * 1024)
      return fail(DGM_ERR_UNSUPPORTED, "stage kernel needs %zu bytes of shared memory", smem);
    int r;
    if ((r = raise_smem_limit(dgm::stage_kernel<N, T, dgm::MODE_RHS>, smem, "cudaFuncSetAttribute")))
      return r;
    if ((r = raise_smem_limit(dgm::stage_kernel<N, T, dgm::MODE_LSRK>, smem, "cudaFuncSetAttribute")))
      return r;
    if ((r = raise_smem_limit(dgm::stage_kernel<N, T, dgm::MODE_VOLUME>, smem, "cudaFuncSetAttribute")))
      return r;
    if ((r = raise_smem_limit(dgm::stage_kernel<N, T, dgm::MODE_SURFACE>, smem, "cudaFuncSetAttribute")))
      return r;
    if constexpr (sizeof(T) == 4 && N <= 4) {  // the small-tile variant (a few tiles per launch)
      using CS = dgm::Cfg<N, T, 1>;
      static_assert(CS::SMEM_FIXED <= C::SMEM_FIXED, "small tiles need less shared memory");
      if ((r = raise_smem_limit(dgm::stage_kernel<N, T, dgm::MODE_RHS, 1>, smem, "cudaFuncSetAttribute")))
        return r;
      if ((r = raise_smem_limit(dgm::stage_kernel<N, T, dgm::MODE_LSRK, 1>, smem, "cudaFuncSetAttribute")))
        return r;
    }
    const size_t msmem = (size_t)6 * C::TE * C::NPG * sizeof(T);
    if ((r = raise_smem_limit(dgm::mass_norm_kernel<N, T>, msmem, "cudaFuncSetAttribute")))
      return r;
    return DGM_OK;
  });
  if (rc) return rc;
  if (d.path < DGM_PATH_AUTO || d.path > DGM_PATH_TENSOR2) return fail(DGM_ERR_INVALID, "bad path %d", d.path);
  int path = DGM_PATH_SIMT;
  size_t tc_smem = 0;
  rc = dispatch(d.order, d.dtype, [&](auto n, auto t) -> int {
    constexpr int N = decltype(n)::value;
    using T = decltype(t);
    if constexpr (TcInfo<N, T>::supported) {
      if (d.path == DGM_PATH_SIMT || d.path == DGM_PATH_TENSOR2) return DGM_OK;
      // AUTO: at N <= 2 the GEMM is too thin for the tensor cores to pay off (C2 sweep: N=1 15 vs 32 us,
      // N=2 35 vs 40 us per stage at 48k tets)
      if (d.path == DGM_PATH_AUTO && N < 3) return DGM_OK;
      if (!d.tc_operand || !aligned16(d.tc_operand)) {
        if (d.path == DGM_PATH_TENSOR)
          return fail(DGM_ERR_INVALID, "tensor path requested without a 16-byte aligned tc_operand");
        return DGM_OK;
      }
      using TC = dgm::TcCfg<N>;
      tc_smem = (TC::SMEM_FIXED + (size_t)d.num_codes * TC::NFP + 127) & ~size_t(127);
      // never more CTAs per SM than TcCfg::CTAS: each allocates 512 / CTAS TMEM columns
      if (TC::CTAS == 2 && tc_smem < 80 * 1024) tc_smem = 80 * 1024;
      if (TC::CTAS == 1 && tc_smem < 120 * 1024) tc_smem = 120 * 1024;
      if (TC::CTAS == 3 && tc_smem < 60 * 1024) tc_smem = 60 * 1024;
      if (tc_smem > 227 * 1024) {
        if (d.path == DGM_PATH_TENSOR) return fail(DGM_ERR_UNSUPPORTED, "tensor path smem %zu too large", tc_smem);
        return DGM_OK;
      }
      int r;
      if ((r = raise_smem_limit(dgm::tc_stage_kernel<N, dgm::MODE_RHS>, tc_smem, "cudaFuncSetAttribute(tc)")))
        return r;
      if ((r = raise_smem_limit(dgm::tc_stage_kernel<N, dgm::MODE_LSRK>, tc_smem, "cudaFuncSetAttribute(tc)")))
        return r;
      path = DGM_PATH_TENSOR;
      return DGM_OK;
    } else {
      if (d.path == DGM_PATH_TENSOR)
        return fail(DGM_ERR_UNSUPPORTED, "no tensor-core path for order %d dtype %d", d.order, d.dtype);
      return DGM_OK;
    }
  });
  if (rc) return rc;
  // v2 tensor-core kernel (N <= 4, fp32): requested explicitly (DGM_PATH_TENSOR2) or by AUTO when the
  // caller supplied its operand
  size_t tc2_smem = 0;
  if (d.path == DGM_PATH_TENSOR2 || (d.path == DGM_PATH_AUTO && d.tc2_operand)) {
    rc = dispatch(d.order, d.dtype, [&](auto n, auto t) -> int {
      constexpr int N = decltype(n)::value;
      using T = decltype(t);
      if constexpr (Tc2Info<N>::supported && sizeof(T) == 4) {
        if (!d.tc2_operand || !aligned16(d.tc2_operand)) {
          if (d.path == DGM_PATH_TENSOR2)
            return fail(DGM_ERR_INVALID, "tensor2 path requested without a 16-byte aligned tc2_operand");
          return DGM_OK;
        }
        using T2 = dgm::Tc2Cfg<N>;
        tc2_smem = (T2::SMEM_FIXED + (size_t)d.num_codes * T2::NFP + 127) & ~size_t(127);
        if (tc2_smem > 227 * 1024) {
          if (d.path == DGM_PATH_TENSOR2) return fail(DGM_ERR_UNSUPPORTED, "tensor2 smem %zu too large", tc2_smem);
          tc2_smem = 0;
          return DGM_OK;
        }
        int r;
        if ((r = raise_smem_limit(dgm::tc2_stage_kernel<N, dgm::MODE_RHS>, tc2_smem, "cudaFuncSetAttribute(tc2)")))
          return r;
        if ((r = raise_smem_limit(dgm::tc2_stage_kernel<N, dgm::MODE_LSRK>, tc2_smem, "cudaFuncSetAttribute(tc2)")))
          return r;
        path = DGM_PATH_TENSOR2;
        return DGM_OK;
      } else {
        if (d.path == DGM_PATH_TENSOR2)
          return fail(DGM_ERR_UNSUPPORTED, "no tensor2 path for order %d dtype %d", d.order, d.dtype);
        return DGM_OK;
      }
    });
    if (rc) return rc;
  }
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  dgm_plan* p = new (std::nothrow) dgm_plan;
  if (!p) return fail(DGM_ERR_INVALID, "out of host memory");
  p->d = d;
  p->stage_smem = smem;
  p->path = path;
  p->tc_smem = tc_smem;
  p->tc2_smem = tc2_smem;
  p->num_sms = sms > 0 ? sms : 148;
  p->device = dev;
  *out = p;
  return DGM_OK;
}

int dgm_plan_destroy(dgm_plan* plan) {
  delete plan;
  return DGM_OK;
}

int dgm_plan_path(const dgm_plan* plan) {
  if (!plan) return fail(DGM_ERR_INVALID, "null plan");
  return plan->path;
}

}  // extern "C"

namespace {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link needed).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 4-D view (node, element, t, h) of a (6, kf, npg) fp32 state-layout array, element extent e_end,
// box {4 nodes, 64 elements, 1, 2} (dgm_tc2.cuh)
int encode_state_map(CUtensorMap* m, const void* base, int npg, int64_t kf, int64_t e_end) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return fail(DGM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[4] = {(cuuint64_t)npg, (cuuint64_t)e_end, 3, 2};
  const cuuint64_t strides[3] = {(cuuint64_t)npg * 4, (cuuint64_t)kf * npg * 4, (cuuint64_t)3 * kf * npg * 4};
  const cuuint32_t box[4] = {4, 64, 1, 2};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DGM_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DGM_OK;
}

// Launch with programmatic stream serialization (PDL): the kernel calls griddepcontrol.wait before it
// touches the state, so it may be scheduled while its predecessor on the stream drains.
template <typename Kernel, typename Args>
int launch_pdl(Kernel kernel, unsigned grid, int threads, size_t smem, void* stream, const Args& args, const char* what) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_check(cudaLaunchKernelEx(&cfg, kernel, args), what);
}

template <int MODE>
int launch_stage(const dgm_plan* plan, const void* u, void* u_out, void* res, void* out, double a,
                 double b, double dt, int64_t e_begin, int64_t e_end, void* stream) {
  if (!plan) return fail(DGM_ERR_INVALID, "null plan");
  const dgm_desc& d = plan->d;
  if (e_begin < 0 || e_end > d.num_elements || e_begin > e_end)
    return fail(DGM_ERR_INVALID, "element range [%lld, %lld) outside [0, %lld)", (long long)e_begin,
                (long long)e_end, (long long)d.num_elements);
  if (!u || !aligned16(u)) return fail(DGM_ERR_INVALID, "state pointer must be non-null and 16-byte aligned");
  if (MODE == dgm::MODE_LSRK) {
    if (!u_out || !res || !aligned16(u_out) || !aligned16(res))
      return fail(DGM_ERR_INVALID, "u_out/res must be non-null and 16-byte aligned");
    if (u_out == u) return fail(DGM_ERR_INVALID, "u_out must differ from u_in (neighbors read u_in)");
  } else if (!out || !aligned16(out)) {
    return fail(DGM_ERR_INVALID, "output pointer must be non-null and 16-byte aligned");
  }
  if (e_end == e_begin) return DGM_OK;
  DeviceGuard guard(plan->device);
  return dispatch(d.order, d.dtype, [&](auto n, auto t) -> int {
    constexpr int N = decltype(n)::value;
    using T = decltype(t);
    using C = dgm::Cfg<N, T>;
    dgm::StageArgs<T> args;
    args.u = static_cast<const T*>(u);
    args.u_out = static_cast<T*>(u_out);
    args.res = static_cast<T*>(res);
    args.out = static_cast<T*>(out);
    args.geo = static_cast<const T*>(d.geometry);
    args.nbr = d.neighbors;
    args.code = d.codes;
    args.diff = static_cast<const T*>(d.diff_packed);
    args.lift = static_cast<const T*>(d.lift_packed);
    args.fmask = d.face_nodes;
    args.ptab = d.code_table;
    args.ncodes = d.num_codes;
    args.kf = d.field_stride;
    args.e_begin = e_begin;
    args.e_end = e_end;
    args.a = (T)a;
    args.b = (T)b;
    args.dt = (T)dt;
    args.a_zero = (a == 0.0);
    args.inv_eps = (T)(1.0 / d.permittivity);
    args.inv_mu = (T)(1.0 / d.permeability);
    const double z = std::sqrt(d.permeability / d.permittivity);
    args.zp = (T)z;
    args.yp = (T)(1.0 / z);
    args.inv_2z = (T)(1.0 / (2.0 * z));
    args.inv_2y = (T)(1.0 / (2.0 * (1.0 / z)));
    if constexpr (Tc2Info<N>::supported && sizeof(T) == 4 && (MODE == dgm::MODE_RHS || MODE == dgm::MODE_LSRK)) {
      if (plan->path == DGM_PATH_TENSOR2) {
        using T2 = dgm::Tc2Cfg<N>;
        dgm::Tc2Args targs;
        targs.s = args;
        targs.bops = static_cast<const float*>(d.tc2_operand);
        int r;
        if ((r = encode_state_map(&targs.tm_u, u, C::NPG, d.field_stride, e_end))) return r;
        if (MODE == dgm::MODE_LSRK) {
          if ((r = encode_state_map(&targs.tm_res, res, C::NPG, d.field_stride, e_end))) return r;
          if ((r = encode_state_map(&targs.tm_out, u_out, C::NPG, d.field_stride, e_end))) return r;
        } else {
          targs.tm_res = targs.tm_u;
          if ((r = encode_state_map(&targs.tm_out, out, C::NPG, d.field_stride, e_end))) return r;
        }
        const int64_t tt = (e_end - e_begin + T2::TE - 1) / T2::TE;
        targs.num_tiles = (int)tt;
        // persistent: one CTA per SM walks tiles blockIdx.x, + gridDim.x, ...
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(tt < plan->num_sms ? tt : plan->num_sms));
        cfg.blockDim = dim3(T2::THREADS);
        cfg.dynamicSmemBytes = plan->tc2_smem;
        cfg.stream = static_cast<cudaStream_t>(stream);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cuda_check(cudaLaunchKernelEx(&cfg, dgm::tc2_stage_kernel<N, MODE>, targs), "tc2_stage_kernel launch");
      }
    }
    if constexpr (TcInfo<N, T>::supported && (MODE == dgm::MODE_RHS || MODE == dgm::MODE_LSRK)) {
      if (plan->path == DGM_PATH_TENSOR) {
        using TC = dgm::TcCfg<N>;
        dgm::TcArgs targs;
        targs.s = args;
        targs.bpack = static_cast<const float*>(d.tc_operand);
        const int64_t tt = (e_end - e_begin + TC::TE - 1) / TC::TE;
        targs.num_tiles = (int)tt;
        targs.wave = TC::CTAS * plan->num_sms;
        // programmatic dependent launch: the grid may start during its predecessor's tail; the
        // kernel runs its state-independent prologue, then griddepcontrol.wait (dgm_tc.cuh)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)tt);
        cfg.blockDim = dim3(TC::THREADS);
        cfg.dynamicSmemBytes = plan->tc_smem;
        cfg.stream = static_cast<cudaStream_t>(stream);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
#ifdef DGM_NO_PDL
        attr[0].val.programmaticStreamSerializationAllowed = 0;
#else
        attr[0].val.programmaticStreamSerializationAllowed = 1;
#endif
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cuda_check(cudaLaunchKernelEx(&cfg, dgm::tc_stage_kernel<N, MODE>, targs), "tc_stage_kernel launch");
      }
    }
    const int64_t tiles = (e_end - e_begin + C::TE - 1) / C::TE;
    if constexpr (sizeof(T) == 4 && N <= 4 && (MODE == dgm::MODE_RHS || MODE == dgm::MODE_LSRK)) {
      // fewer tiles than SMs: one element per P2 thread, E times more CTAs with E times shorter
      // phases (C1, 1,512 tets at N=3: DESIGN.md 3.1)
      if (tiles < plan->num_sms) {
        using CS = dgm::Cfg<N, T, 1>;
        const int64_t st = (e_end - e_begin + CS::TE - 1) / CS::TE;
        // plain launch: PDL measured slower for these few-tile grids (C1 9.0 vs 6.9 us per stage)
        dgm::stage_kernel<N, T, MODE, 1><<<(unsigned)st, CS::THREADS, plan->stage_smem,
                                           static_cast<cudaStream_t>(stream)>>>(args);
        return cuda_check(cudaGetLastError(), "stage_kernel launch");
      }
    }
    return launch_pdl(dgm::stage_kernel<N, T, MODE>, (unsigned)tiles, C::THREADS, plan->stage_smem, stream, args,
                      "stage_kernel launch");
  });
}

}  // namespace

extern "C" {

int dgm_rhs(const dgm_plan* plan, const void* u, void* out, int64_t e_begin, int64_t e_end, void* stream) {
  return launch_stage<dgm::MODE_RHS>(plan, u, nullptr, nullptr, out, 0, 0, 0, e_begin, e_end, stream);
}

int dgm_lsrk_stage(const dgm_plan* plan, const void* u_in, void* u_out, void* res, double a, double b,
                   double dt, int64_t e_begin, int64_t e_end, void* stream) {
  return launch_stage<dgm::MODE_LSRK>(plan, u_in, u_out, res, nullptr, a, b, dt, e_begin, e_end, stream);
}

int dgm_volume(const dgm_plan* plan, const void* u, void* out, int64_t e_begin, int64_t e_end, void* stream) {
  return launch_stage<dgm::MODE_VOLUME>(plan, u, nullptr, nullptr, out, 0, 0, 0, e_begin, e_end, stream);
}

int dgm_surface(const dgm_plan* plan, const void* u, void* out, int64_t e_begin, int64_t e_end, void* stream) {
  return launch_stage<dgm::MODE_SURFACE>(plan, u, nullptr, nullptr, out, 0, 0, 0, e_begin, e_end, stream);
}

int dgm_mass_norm(const dgm_plan* plan, const void* u, const void* mass_packed, const void* det_j, double w_e,
                  double w_h, double* out_f64, double* partials, int64_t e_begin, int64_t e_end, void* stream) {
  if (!plan) return fail(DGM_ERR_INVALID, "null plan");
  const dgm_desc& d = plan->d;
  if (!u || !mass_packed || !det_j || !out_f64 || !partials || !aligned16(u) || !aligned16(mass_packed))
    return fail(DGM_ERR_INVALID, "dgm_mass_norm: null or misaligned pointer");
  if (e_begin < 0 || e_end > d.num_elements || e_begin > e_end)
    return fail(DGM_ERR_INVALID, "element range outside the plan");
  if (e_end == e_begin) return DGM_OK;
  DeviceGuard guard(plan->device);
  return dispatch(d.order, d.dtype, [&](auto n, auto t) -> int {
    constexpr int N = decltype(n)::value;
    using T = decltype(t);
    using C = dgm::Cfg<N, T>;
    const int64_t tiles = (e_end - e_begin + C::TE - 1) / C::TE;
    const size_t msmem = (size_t)6 * C::TE * C::NPG * sizeof(T);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    dgm::mass_norm_kernel<N, T><<<(unsigned)tiles, C::THREADS, msmem, st>>>(
        static_cast<const T*>(u), static_cast<const T*>(mass_packed), static_cast<const T*>(det_j),
        d.field_stride, e_begin, e_end, w_e, w_h, partials);
    if (int r = cuda_check(cudaGetLastError(), "mass_norm_kernel launch")) return r;
    dgm::reduce_partials_kernel<<<1, 256, 0, st>>>(partials, tiles, out_f64);
    return cuda_check(cudaGetLastError(), "reduce_partials_kernel launch");
  });
}

int64_t dgm_mass_norm_partials(const dgm_plan* plan, int64_t count) {
  if (!plan || count < 0) return fail(DGM_ERR_INVALID, "dgm_mass_norm_partials: bad arguments");
  int64_t te = 1;
  dispatch(plan->d.order, plan->d.dtype, [&](auto n, auto t) -> int {
    te = dgm::Cfg<decltype(n)::value, decltype(t)>::TE;
    return DGM_OK;
  });
  return (count + te - 1) / te;
}

int dgm_face_states(const dgm_plan* plan, const void* u, const int64_t* elem_nat, const uint8_t* node_nat,
                    void* u_minus, void* u_plus, void* stream) {
  if (!plan || !u || !u_minus || !u_plus) return fail(DGM_ERR_INVALID, "dgm_face_states: null argument");
  const dgm_desc& d = plan->d;
  if (d.num_elements == 0) return DGM_OK;
  DeviceGuard guard(plan->device);
  return dispatch(d.order, d.dtype, [&](auto n, auto t) -> int {
    constexpr int N = decltype(n)::value;
    using T = decltype(t);
    using C = dgm::Cfg<N, T>;
    dgm::StageArgs<T> args = {};
    args.u = static_cast<const T*>(u);
    args.geo = static_cast<const T*>(d.geometry);
    args.nbr = d.neighbors;
    args.code = d.codes;
    args.fmask = d.face_nodes;
    args.ptab = d.code_table;
    args.ncodes = d.num_codes;
    args.kf = d.field_stride;
    args.e_begin = 0;
    args.e_end = d.num_elements;
    dgm::face_states_kernel<N, T><<<grid_for(d.num_elements * 4 * C::NFP, 256), 256, 0,
                                    static_cast<cudaStream_t>(stream)>>>(args, elem_nat, node_nat,
                                                                         static_cast<T*>(u_minus),
                                                                         static_cast<T*>(u_plus));
    return cuda_check(cudaGetLastError(), "face_states_kernel launch");
  });
}

int dgm_pack(int32_t order, int32_t dtype, const void* natural, int32_t natural_dtype, const int64_t* perm,
             void* padded, int64_t num_elements, int64_t field_stride, void* stream) {
  if (!natural || !padded || num_elements < 0 || field_stride < num_elements)
    return fail(DGM_ERR_INVALID, "dgm_pack: bad arguments");
  if (num_elements == 0) return DGM_OK;
  return dispatch(order, dtype, [&](auto n, auto t) -> int {
    constexpr int N = decltype(n)::value;
    using T = decltype(t);
    using C = dgm::Cfg<N, T>;
    return natural_dispatch(natural_dtype, [&](auto tn) -> int {
      using TN = decltype(tn);
      // y = field; the six fields share the usual block cap (grid-stride loop)
      const dim3 grid((unsigned)grid_for((num_elements * (C::NPG / C::VEC) + 5) / 6, 256), 6);
      dgm::pack_kernel<N, T, TN><<<grid, 256, 0,
                                   static_cast<cudaStream_t>(stream)>>>(
          static_cast<const TN*>(natural), perm, static_cast<T*>(padded), num_elements, field_stride);
      return cuda_check(cudaGetLastError(), "pack_kernel launch");
    });
  });
}

int dgm_unpack(int32_t order, int32_t dtype, const void* padded, const int64_t* perm, void* natural,
               int32_t natural_dtype, int64_t num_elements, int64_t field_stride, void* stream) {
  if (!natural || !padded || num_elements < 0 || field_stride < num_elements)
    return fail(DGM_ERR_INVALID, "dgm_unpack: bad arguments");
  if (num_elements == 0) return DGM_OK;
  return dispatch(order, dtype, [&](auto n, auto t) -> int {
    constexpr int N = decltype(n)::value;
    using T = decltype(t);
    using C = dgm::Cfg<N, T>;
    return natural_dispatch(natural_dtype, [&](auto tn) -> int {
      using TN = decltype(tn);
      const dim3 grid((unsigned)grid_for((num_elements * C::NP + 5) / 6, 256), 6);
      dgm::unpack_kernel<N, T, TN><<<grid, 256, 0,
                                     static_cast<cudaStream_t>(stream)>>>(
          static_cast<const T*>(padded), perm, static_cast<TN*>(natural), num_elements, field_stride);
      return cuda_check(cudaGetLastError(), "unpack_kernel launch");
    });
  });
}

int dgm_halo_pack(const dgm_plan* plan, const void* u, const int32_t* elements, int64_t count, void* sendbuf,
                  void* stream) {
  if (!plan || !u || (count > 0 && (!elements || !sendbuf)) || count < 0)
    return fail(DGM_ERR_INVALID, "dgm_halo_pack: bad arguments");
  if (!aligned16(u) || (sendbuf && !aligned16(sendbuf)))
    return fail(DGM_ERR_INVALID, "dgm_halo_pack: buffers must be 16-byte aligned");
  if (count == 0) return DGM_OK;
  const dgm_desc& d = plan->d;
  DeviceGuard guard(plan->device);
  return dispatch(d.order, d.dtype, [&](auto n, auto t) -> int {
    constexpr int N = decltype(n)::value;
    using T = decltype(t);
    using C = dgm::Cfg<N, T>;
    dgm::halo_pack_kernel<N, T><<<grid_for(count * 6 * (C::NPG / C::VEC), 256), 256, 0,
                                  static_cast<cudaStream_t>(stream)>>>(
        static_cast<const T*>(u), elements, count, d.field_stride, static_cast<T*>(sendbuf));
    return cuda_check(cudaGetLastError(), "halo_pack_kernel launch");
  });
}

int dgm_halo_unpack(const dgm_plan* plan, const void* recvbuf, int64_t count, int64_t ghost_begin, void* u,
                    void* stream) {
  if (!plan || !u || count < 0 || (count > 0 && !recvbuf))
    return fail(DGM_ERR_INVALID, "dgm_halo_unpack: bad arguments");
  const dgm_desc& d = plan->d;
  if (ghost_begin < 0 || ghost_begin + count > d.field_stride)
    return fail(DGM_ERR_INVALID, "ghost range [%lld, %lld) exceeds field_stride %lld", (long long)ghost_begin,
                (long long)(ghost_begin + count), (long long)d.field_stride);
  if (!aligned16(u) || (recvbuf && !aligned16(recvbuf)))
    return fail(DGM_ERR_INVALID, "dgm_halo_unpack: buffers must be 16-byte aligned");
  if (count == 0) return DGM_OK;
  DeviceGuard guard(plan->device);
  return dispatch(d.order, d.dtype, [&](auto n, auto t) -> int {
    constexpr int N = decltype(n)::value;
    using T = decltype(t);
    using C = dgm::Cfg<N, T>;
    dgm::halo_unpack_kernel<N, T><<<grid_for(count * 6 * (C::NPG / C::VEC), 256), 256, 0,
                                    static_cast<cudaStream_t>(stream)>>>(
        static_cast<const T*>(recvbuf), count, ghost_begin, d.field_stride, static_cast<T*>(u));
    return cuda_check(cudaGetLastError(), "halo_unpack_kernel launch");
  });
}

int dgm_trace_pack(const dgm_plan* plan, const void* u, const int32_t* elem_face, int64_t count, void* sendbuf,
                   void* stream) {
  if (!plan || !u || count < 0 || (count > 0 && (!elem_face || !sendbuf)))
    return fail(DGM_ERR_INVALID, "dgm_trace_pack: bad arguments");
  if (count == 0) return DGM_OK;
  const dgm_desc& d = plan->d;
  DeviceGuard guard(plan->device);
  return dispatch(d.order, d.dtype, [&](auto n, auto t) -> int {
    constexpr int N = decltype(n)::value;
    using T = decltype(t);
    using C = dgm::Cfg<N, T>;
    dgm::trace_pack_kernel<N, T><<<grid_for(count * 6 * C::NFP, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const T*>(u), elem_face, d.face_nodes, count, d.field_stride, static_cast<T*>(sendbuf));
    return cuda_check(cudaGetLastError(), "trace_pack_kernel launch");
  });
}

int dgm_trace_unpack(const dgm_plan* plan, const void* recvbuf, const int32_t* elem_face, int64_t count, void* u,
                     void* stream) {
  if (!plan || !u || count < 0 || (count > 0 && (!elem_face || !recvbuf)))
    return fail(DGM_ERR_INVALID, "dgm_trace_unpack: bad arguments");
  if (count == 0) return DGM_OK;
  const dgm_desc& d = plan->d;
  DeviceGuard guard(plan->device);
  return dispatch(d.order, d.dtype, [&](auto n, auto t) -> int {
    constexpr int N = decltype(n)::value;
    using T = decltype(t);
    using C = dgm::Cfg<N, T>;
    dgm::trace_unpack_kernel<N, T><<<grid_for(count * 6 * C::NFP, 256), 256, 0,
                                     static_cast<cudaStream_t>(stream)>>>(
        static_cast<const T*>(recvbuf), elem_face, d.face_nodes, count, d.field_stride, static_cast<T*>(u));
    return cuda_check(cudaGetLastError(), "trace_unpack_kernel launch");
  });
}

}  // extern "C"

#ifdef DGM_TC_TIMING
extern "C" int dgm_phase_read(long long* host, int nblocks) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(host, dgm::g_tc_phase, sizeof(long long) * 5 * nblocks);
}
#endif
#ifdef DGM_TC_TRACE
extern "C" int dgm_hang_read(unsigned int* host) {
  return (int)cudaMemcpyFromSymbol(host, dgm::tc::g_hang, sizeof(unsigned int) * 8);
}
extern "C" int dgm_trace_read(long long* host, int who) {
  int n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, dgm::g_tc_trace_n, sizeof(int), sizeof(int) * who);
  cudaMemcpyFromSymbol(host, dgm::g_tc_trace, sizeof(long long) * 2 * n, sizeof(long long) * 2 * 4096 * who);
  return n;
}
#endif
