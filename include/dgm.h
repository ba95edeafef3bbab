/*
 * dgm.h -- C ABI of the B200-native nodal-DG Maxwell operator (libdgm.so).
 *
 * The reference package (simtdg, pure Python) has no FFI; its hot path is the
 * Python call chain
 *
 *   rk4_step(state, t, dt, rhs_fn)              pkg/src/simtdg/kernels/assemble.py:105-114
 *     -> ReferenceMaxwellOperator.rhs(state)    pkg/src/simtdg/kernels/oracle.py:60-94
 *          volume curls   (oracle.py:67-79)
 *          face_states    (oracle.py:50-58, maxwell.py:117-132)
 *          upwind_flux    (maxwell.py:73-114)
 *          LIFT, 1/J, 1/eps, 1/mu (oracle.py:81-93)
 *
 * Each entry point below replaces one piece of that chain; the Python
 * operator class (paper_0901_1024_b200/operator.py) binds them through
 * ctypes, exactly as a maintainer would bind them from simtdg.
 *
 * Conventions
 *  - All buffers are DEVICE pointers owned by the caller (PyTorch); the
 *    library never allocates or frees device memory.  A plan holds only
 *    scalars and borrowed pointers.
 *  - Field arrays use the padded device layout: (6, field_stride, np_stride)
 *    C-order, field order (Ex,Ey,Ez,Hx,Hy,Hz); node rows are zero-padded from
 *    Np to np_stride (query with dgm_layout) and the padding stays zero.
 *  - dtype: DGM_F32 or DGM_F64 selects the arithmetic type of every real
 *    buffer of a plan.
 *  - Streams are cudaStream_t passed as void*; NULL = legacy default stream.
 *    Calls taking a plan launch on the device the plan was created on,
 *    whatever the calling thread's current device (restored on return).
 *  - Return value 0 = success, negative = error class; the message is in
 *    dgm_last_error() (thread-local), mirroring the reference's ValueError /
 *    RuntimeError split (mesh.py:42-49, assemble.py:107-108).
 */
#ifndef DGM_H
#define DGM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { DGM_F32 = 0, DGM_F64 = 1 };
enum {
  DGM_OK = 0,
  DGM_ERR_INVALID = -1,   /* bad argument (reference: ValueError)      */
  DGM_ERR_CUDA = -2,      /* CUDA runtime error (reference: n/a)        */
  DGM_ERR_UNSUPPORTED = -3/* order/dtype not compiled in               */
};

/* Number of words per element in the geometry array (see dgm_desc). */
#define DGM_GEO_WORDS 28

/* Device layout of one order/dtype (host and device must agree). */
typedef struct {
  int32_t order;
  int32_t dtype;
  int32_t num_nodes;        /* Np  = (N+1)(N+2)(N+3)/6  (refelem.py:64-69) */
  int32_t num_face_nodes;   /* Nfp = (N+1)(N+2)/2                         */
  int32_t np_stride;        /* padded node row length of field arrays       */
  int32_t diff_chunks;      /* j-chunks of the packed derivative operand    */
  int32_t lift_chunks;      /* j-chunks of the packed LIFT operand          */
  int32_t vec;              /* reals per 16-byte chunk (4 f32, 2 f64)       */
  int32_t tile_elements;    /* elements per CTA tile of the stage kernel    */
  int32_t threads;          /* threads per CTA of the stage kernel          */
  int64_t smem_bytes_fixed; /* dynamic smem per CTA excluding code table    */
  /* tensor-core (tcgen05, 3xTF32) stage path, f32 only */
  int32_t tc_supported;     /* 1 if this order/dtype has the tensor-core path */
  int32_t tc_nb;            /* MMA N: Np rounded up to 16                     */
  int32_t tc_steps;         /* K steps of 8 (K = 3*tc_npk + 4*Nfp, padded)     */
  int32_t tc_npk;           /* K extent of one derivative block (Np up to 4)  */
  int32_t tc_kv;            /* K offset of the first face block (3*npk up to 8) */
  int32_t tc_nfpk;          /* K extent of one face block (Nfp up to 8)       */
  int64_t tc_operand_floats;/* size of dgm_desc.tc_operand in floats          */
  /* v2 tensor-core stage path (N <= 4, f32): state rows are the volume GEMM's A operand */
  int32_t tc2_supported;
  int64_t tc2_operand_floats;/* size of dgm_desc.tc2_operand in floats         */
} dgm_layout_info;

enum { DGM_PATH_AUTO = 0, DGM_PATH_SIMT = 1, DGM_PATH_TENSOR = 2, DGM_PATH_TENSOR2 = 3 };

/*
 * Operator description (replaces build_reference_operator, oracle.py:97-141).
 *
 *  diff_packed : real[3][diff_chunks][Np][vec]   diff_packed[m][c][i][q] =
 *                elem.diff[m][i][c*vec+q] (0 beyond Np)   (refelem.py:378-379)
 *  lift_packed : real[lift_chunks][Np][vec]       lift_packed[c][i][q] =
 *                elem.lift[i][c*vec+q]                     (refelem.py:435-446)
 *  geometry    : real[num_elements][28] per element (words 26, 27 are padding):
 *                [0..8]  inv_jacobians row-major (d r_m / d x_n)   (mesh.py:331)
 *                [9]     1 / det_jacobians                         (oracle.py:89)
 *                [10..21] normals[f][3]                            (mesh.py:333-334)
 *                [22..25] face_jacobians[f] = area/FACE_AREAS[f]   (oracle.py:84-85)
 *  neighbors   : int32[field_stride][4]   element across face f (local index,
 *                may point into the ghost range [num_elements, field_stride))
 *  codes       : int32[field_stride][4]   row of code_table giving the
 *                neighbor's node ids along the shared face, or -1 for a PEC
 *                wall (is_boundary, oracle.py:125-127)
 *  face_nodes  : uint8[4][Nfp]            elem.face_nodes (refelem.py:387-394)
 *  code_table  : uint8[num_codes][Nfp]    vmap_plus rows minus neighbor*Np
 *                (oracle.py:116-123)
 *                The order of the nodes inside a face is free: a caller may
 *                permute face f's slots (face_nodes[f], the code_table rows
 *                used on face f and LIFT columns f*Nfp..) consistently; the
 *                surface output (dgm_surface) then follows the same slot order.
 *                The Python layer does so to spread the tensor kernel's
 *                shared-memory loads (ordering.face_slot_order).
 *  tc_operand  : float[tc_steps][2][2][tc_nb][4], the constant GEMM operand
 *                B[n][k]: D_mu[n][j] at k = mu*tc_npk + j, LIFT[n][f*Nfp + i]
 *                at k = tc_kv + f*tc_nfpk + i, zero elsewhere; split into a
 *                tf32 hi part and the exact fp32 remainder:
 *                tc_operand[s][h][c][n][q] = part_h(B[n][8s + 4c + q]).
 *                NULL disables the tensor-core path.
 *  tc2_operand : float[2*kv/4*nv*4 + 2*kf/4*nl*4], the v2 kernel's constant
 *                operands (N <= 4; dgm_tc2.cuh): D = [hi | lo][kv/4][nv][4] with
 *                row n = mu*mus + i holding D_mu[i][:] (mus = Np up to 4,
 *                nv = 3 mus up to 16, kv = Np up to 8), then
 *                LIFT = [hi | lo][kf/4][nl][4] with row i holding LIFT[i][f*Nfp+s]
 *                at k = f*nfpk + s (nl = Np up to 16, nfpk = Nfp up to 8,
 *                kf = 4 nfpk); zero elsewhere, hi = tf32 part, lo = exact remainder.
 *                NULL disables the v2 path.
 *  path        : DGM_PATH_AUTO (fp32: v2 tensor kernel when tc2_operand is given,
 *                else tensor cores for N >= 2), _SIMT, _TENSOR (v1) or _TENSOR2.
 */
typedef struct {
  int32_t order;
  int32_t dtype;
  int64_t num_elements;   /* owned elements (stage kernels cover a sub-range) */
  int64_t field_stride;   /* element slots per field slab (>= owned + ghosts) */
  const void* diff_packed;
  const void* lift_packed;
  const void* geometry;
  const int32_t* neighbors;
  const int32_t* codes;
  const uint8_t* face_nodes;
  const uint8_t* code_table;
  int32_t num_codes;
  double permittivity;    /* Material.permittivity (maxwell.py:23-47) */
  double permeability;
  const void* tc_operand;
  int32_t path;
  const void* tc2_operand;
} dgm_desc;

typedef struct dgm_plan dgm_plan;

/* Library/ABI version, for the Python loader's sanity check. */
int32_t dgm_version(void);

/* Thread-local message of the last failing call ("" if none). */
const char* dgm_last_error(void);

/* Layout constants of an order/dtype (DGM_ERR_UNSUPPORTED if not built). */
int dgm_layout(int32_t order, int32_t dtype, dgm_layout_info* out);

/* Validates the description, stores it, and configures kernel attributes. */
int dgm_plan_create(const dgm_desc* desc, dgm_plan** out);
int dgm_plan_destroy(dgm_plan* plan);

/* Path the stage kernels of a plan run on: DGM_PATH_SIMT, _TENSOR or _TENSOR2. */
int dgm_plan_path(const dgm_plan* plan);

/*
 * Full semidiscrete RHS on elements [e_begin, e_end) of the padded state u
 * (replaces ReferenceMaxwellOperator.rhs, oracle.py:60-94).  out has the same
 * padded layout; only the rows of [e_begin, e_end) are written.
 */
int dgm_rhs(const dgm_plan* plan, const void* u, void* out,
            int64_t e_begin, int64_t e_end, void* stream);

/*
 * One fused low-storage RK stage on [e_begin, e_end)
 * (replaces one iteration of rk4_step's loop, assemble.py:118-120):
 *    r     = a * res + dt * rhs(u_in)       (res not read when a == 0)
 *    res   = r
 *    u_out = u_in + b * r
 * u_in and u_out must be distinct buffers (neighbors read u_in).
 */
int dgm_lsrk_stage(const dgm_plan* plan, const void* u_in, void* u_out, void* res,
                   double a, double b, double dt,
                   int64_t e_begin, int64_t e_end, void* stream);

/* Volume term only: (curl H / eps, -curl E / mu)   (oracle.py:67-79, 91-93). */
int dgm_volume(const dgm_plan* plan, const void* u, void* out,
               int64_t e_begin, int64_t e_end, void* stream);

/*
 * Surface term before lifting: upwind_flux(u-, u+, n) * face_jacobians, with
 * the PEC mirror on walls (oracle.py:82-85).  out is real[6][field_stride][4*Nfp].
 */
int dgm_surface(const dgm_plan* plan, const void* u, void* out,
                int64_t e_begin, int64_t e_end, void* stream);

/*
 * Mass-weighted squared norm accumulated into *out_f64 (device double):
 *   *out += sum_k J_k sum_f w_f u_fk^T M u_fk,  w = (wE,wE,wE,wH,wH,wH)
 * field_energy = 0.5 * value with (wE,wH) = (eps,mu)   (maxwell.py:225-232);
 * l2_error^2 = value of (u - exact) with w = 1           (maxwell.py:211-222).
 * mass_packed has the LIFT-style packing: real[diff_chunks][Np][vec].
 * det_j is real[num_elements].  partials is device scratch of
 * dgm_mass_norm_partials(plan, e_end - e_begin) doubles: one partial per CTA,
 * summed by a second one-CTA kernel in a fixed order, so the result is bitwise
 * reproducible run to run (the reference's reruns are byte-identical,
 * pkg/tests/test_cli.py:106-112).
 */
int dgm_mass_norm(const dgm_plan* plan, const void* u, const void* mass_packed,
                  const void* det_j, double w_e, double w_h, double* out_f64,
                  double* partials, int64_t e_begin, int64_t e_end, void* stream);
int64_t dgm_mass_norm_partials(const dgm_plan* plan, int64_t count);

/*
 * face_states (oracle.py:50-58): u_minus[f][k][face][i] = u at vmap_minus,
 * u_plus = u at vmap_plus, with the PEC mirror (maxwell.py:117-132) on walls;
 * both real[6][num_elements][4][Nfp] in the NATURAL numbering.  elem_nat
 * (int64[num_elements], NULL = identity) maps the plan's element slot s to the
 * natural element id; node_nat (uint8[4][Nfp], NULL = identity) maps the
 * plan's face slot q of face f to the natural face-node index.
 */
int dgm_face_states(const dgm_plan* plan, const void* u, const int64_t* elem_nat,
                    const uint8_t* node_nat, void* u_minus, void* u_plus, void* stream);

/*
 * Natural (6, K, Np) float64 or float32 (natural_dtype)  <->  padded
 * (6, field_stride, np_stride) real, zero padding (reference fields.py:24-35
 * to_padded / from_padded), cast and element permutation in one pass:
 * padded slot s holds natural element perm[s] (perm = NULL: identity).
 */
int dgm_pack(int32_t order, int32_t dtype, const void* natural, int32_t natural_dtype,
             const int64_t* perm, void* padded, int64_t num_elements,
             int64_t field_stride, void* stream);
int dgm_unpack(int32_t order, int32_t dtype, const void* padded, const int64_t* perm,
               void* natural, int32_t natural_dtype, int64_t num_elements,
               int64_t field_stride, void* stream);

/*
 * Multi-GPU halo helpers: gather whole element rows of the listed elements
 * into a contiguous send buffer real[count][6][np_stride], and scatter a
 * received buffer into the ghost slots [ghost_begin, ghost_begin+count).
 */
int dgm_halo_pack(const dgm_plan* plan, const void* u, const int32_t* elements,
                  int64_t count, void* sendbuf, void* stream);
int dgm_halo_unpack(const dgm_plan* plan, const void* recvbuf, int64_t count,
                    int64_t ghost_begin, void* u, void* stream);

/*
 * Face-trace halo (what the multi-GPU operator exchanges each LSRK stage):
 * elem_face holds count (element, face) int32 pairs; dgm_trace_pack gathers
 * the Nfp face nodes of each pair, real[count][6][Nfp], from u's padded rows;
 * dgm_trace_unpack scatters such a buffer into the face nodes of the listed
 * (ghost) rows of u.  Node order is the plan's face_nodes, so a buffer packed
 * by one rank unpacks on a peer whose plan has the same face_nodes.
 * New (the reference is single-process); 6*Nfp instead of
 * 6*np_stride reals per cut face.
 */
int dgm_trace_pack(const dgm_plan* plan, const void* u, const int32_t* elem_face,
                   int64_t count, void* sendbuf, void* stream);
int dgm_trace_unpack(const dgm_plan* plan, const void* recvbuf, const int32_t* elem_face,
                     int64_t count, void* u, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DGM_H */
