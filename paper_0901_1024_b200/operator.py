"""The B200 Maxwell DG operator: drop-in for ``ReferenceMaxwellOperator``.

``build_b200_operator(mesh, elem, material)`` takes the same ``Mesh`` and
``ReferenceElement`` objects as the reference's ``build_reference_operator``
(oracle.py:97-141) and returns an operator whose ``rhs(state)`` has the same
contract (natural (6, K, Np) in, new array out, numpy stays numpy), plus the
device-resident fast path:

* ``to_padded`` / ``from_padded``: natural <-> element-aligned, zero-padded,
  field-major device layout (6, field_stride, np_stride) (fields.py:24-35);
* ``rhs_padded(u)``: one launch of the fused stage kernel in RHS mode;
* ``advance(u, dt, n)``: n LSRK4 steps, each 5 launches of the fused
  LIFT+RK stage kernel (RK_A/RK_B as assemble.py:80-114), CUDA-graph captured;
* ``field_energy`` / ``l2_error``: device reductions (maxwell.py:211-232).

All device memory is owned by torch tensors; the C library borrows pointers.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _capi
from .facemaps import FaceMaps, build_face_maps
from .maxwell import VACUUM, Material
from .mesh import FaceConnectivity, GeometricFactors, Mesh, build_connectivity, compute_geometry, map_nodes
from .refelem import NUM_FACES, ReferenceElement
from .stepper import RK_A, RK_B, RK_C

N_FIELDS = 6
_DTYPES = {torch.float32: _capi.DGM_F32, torch.float64: _capi.DGM_F64}


def pack_chunks(mat: np.ndarray, chunks: int, vec: int) -> np.ndarray:
    """(rows, cols) -> (chunks, rows, vec) with packed[c, i, q] = mat[i, c*vec + q] (0 past cols)."""
    rows, cols = mat.shape
    padded = np.zeros((rows, chunks * vec))
    padded[:, :cols] = mat
    return np.ascontiguousarray(padded.reshape(rows, chunks, vec).transpose(1, 0, 2))


def tc_operand(elem: ReferenceElement, lay, lift: np.ndarray | None = None) -> np.ndarray:
    """Constant GEMM operand of the tensor-core path, layout of dgm_desc.tc_operand (include/dgm.h).

    B[n][k] = [D_r | D_s | D_t | 0 | LIFT_f0 | .. | LIFT_f3][n][k] with each
    derivative block tc_npk and each face block tc_nfpk wide; split into a tf32-exact high part (13 low mantissa bits cleared) and
    the float32 remainder, so that hi*x + lo*x carries fp32 accuracy.  ``lift`` overrides
    elem.lift (face-slot-permuted columns).
    """
    lift = elem.lift if lift is None else lift
    n_p, n_fp = elem.num_nodes, elem.num_face_nodes
    nb, npk, steps, kv, nfpk = lay.tc_nb, lay.tc_npk, lay.tc_steps, lay.tc_kv, lay.tc_nfpk
    full = np.zeros((nb, steps * 8))
    for mu in range(3):
        full[:n_p, mu * npk:mu * npk + n_p] = elem.diff[mu]
    for f in range(NUM_FACES):
        full[:n_p, kv + f * nfpk:kv + f * nfpk + n_fp] = lift[:, f * n_fp:(f + 1) * n_fp]
    hi = (full.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
    lo = (full - hi.astype(np.float64)).astype(np.float32)
    parts = np.stack([hi, lo])                                   # (2, nb, K)
    packed = parts.reshape(2, nb, steps, 2, 4).transpose(2, 0, 3, 1, 4)  # (steps, h, c, n, q)
    out = np.ascontiguousarray(packed, dtype=np.float32)
    assert out.size == lay.tc_operand_floats
    return out


def tc2_operand(elem: ReferenceElement, lift: np.ndarray | None = None) -> np.ndarray:
    """Constant operands of the v2 tensor kernel, layout of dgm_desc.tc2_operand (include/dgm.h).

    D part: B[n][j] = D_mu[i][j] for n = mu * mus + i (mus = Np up to 4), K = j up to kv = Np up to 8,
    N = nv = 3 mus up to 16.  LIFT part: L[i][f * nfpk + s] = LIFT[i][f * Nfp + s], N = nl = Np up to 16.
    Each as [hi | lo][K / 4 chunks][N rows][4]: hi = the tf32 part (13 low mantissa bits cleared),
    lo = the remainder of the float64 operand in float32.
    """
    lift = elem.lift if lift is None else lift
    n_p, n_fp = elem.num_nodes, elem.num_face_nodes
    mus = (n_p + 3) // 4 * 4
    nv, nl = (3 * mus + 15) // 16 * 16, (n_p + 15) // 16 * 16
    kv, nfpk = (n_p + 7) // 8 * 8, (n_fp + 7) // 8 * 8
    kf = 4 * nfpk
    dmat = np.zeros((nv, kv))
    for mu in range(3):
        dmat[mu * mus:mu * mus + n_p, :n_p] = elem.diff[mu]
    lmat = np.zeros((nl, kf))
    for f in range(NUM_FACES):
        lmat[:n_p, f * nfpk:f * nfpk + n_fp] = lift[:, f * n_fp:(f + 1) * n_fp]

    def split_pack(mat):
        hi = (mat.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
        lo = (mat - hi.astype(np.float64)).astype(np.float32)
        rows, k = mat.shape
        return [np.ascontiguousarray(x.reshape(rows, k // 4, 4).transpose(1, 0, 2)) for x in (hi, lo)]

    parts = split_pack(dmat) + split_pack(lmat)
    return np.concatenate([x.reshape(-1) for x in parts]).astype(np.float32)


_SLOT_ORDERS: dict = {}
# path="auto" picks the v2 tensor kernel for N <= 4 fp32 (set from measurements)
TC2_AUTO = False
# path="auto" runs fp32 N <= 3 meshes with fewer elements than this on the CUDA-core kernel
SMALL_MESH_SIMT = 64 * 148


def _face_slot_order(elem: ReferenceElement, v2: bool = False) -> np.ndarray:
    """ordering.face_slot_order (v1 kernel) or face_slot_order_v2 for this element, cached per order."""
    from .ordering import face_slot_order, face_slot_order_v2

    if v2:
        key = ("v2", elem.order)
        if key not in _SLOT_ORDERS:
            _SLOT_ORDERS[key] = face_slot_order_v2(elem.face_nodes, (elem.num_face_nodes + 7) // 8 * 8)
        return _SLOT_ORDERS[key]
    if elem.order not in _SLOT_ORDERS:  # modelled on the fp32 tensor kernel's strides (TcCfg<N>)
        # the shared-memory row stride the kernel really uses (TcCfg::NPG = the f32 np_stride, an odd
        # number of 16-byte chunks), not ceil4(Np): they differ at N = 5, 7, 8
        npg = _capi.layout(elem.order, _capi.DGM_F32).np_stride
        nfpk = (elem.num_face_nodes + 7) // 8 * 8
        _SLOT_ORDERS[elem.order] = face_slot_order(elem.face_nodes, elem.order, npg, nfpk)
    return _SLOT_ORDERS[elem.order]


def geometry_words(geometry: GeometricFactors) -> np.ndarray:
    """(K, 28) float64 per-element words, layout of dgm_desc.geometry (include/dgm.h)."""
    k = len(geometry.det_jacobians)
    g = np.zeros((k, _capi.GEO_WORDS))
    g[:, 0:9] = geometry.inv_jacobians.reshape(k, 9)
    g[:, 9] = 1.0 / geometry.det_jacobians
    g[:, 10:22] = geometry.normals.reshape(k, 12)
    g[:, 22:26] = geometry.face_jacobians
    return g


@dataclass
class _Buffers:
    """LSRK4 scratch: two state registers (a step runs u -> alt -> alt2 -> alt -> alt2 -> u) + residual."""

    alt: torch.Tensor
    res: torch.Tensor
    alt2: torch.Tensor | None = None


@dataclass
class KernelStats:
    """Device time of one kernel family (the B200 replacement of the emulator's MemStats)."""

    launches: int = 0
    ms: float = 0.0

    def to_dict(self) -> dict:
        return {"launches": self.launches, "ms": self.ms,
                "us_per_launch": 1e3 * self.ms / self.launches if self.launches else 0.0}


class B200MaxwellOperator:
    """Maxwell RHS and LSRK4 on one B200 (or one rank's element range)."""

    def __init__(self, elem: ReferenceElement, material: Material, geo_words: np.ndarray,
                 det_j: np.ndarray, maps: FaceMaps, *, num_ghost: int = 0,
                 dtype: torch.dtype = torch.float32, device=None, path: str = "auto",
                 order: np.ndarray | None = None, face_slots: bool | None = None):
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be torch.float32 or torch.float64, got {dtype}")
        if not torch.cuda.is_available():
            raise RuntimeError("B200MaxwellOperator needs a CUDA device (no CPU fallback)")
        self.elem = elem
        self.material = material
        self.dtype = dtype
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.num_elements = int(len(det_j))
        self.num_ghost = int(num_ghost)
        self.field_stride = self.num_elements + self.num_ghost
        self._dt_code = _DTYPES[dtype]
        self.layout = _capi.layout(elem.order, self._dt_code)
        lay = self.layout
        self.np_stride = lay.np_stride
        self.maps = maps  # natural (reference) numbering
        # internal element order of the padded layout: slot s holds natural element order[s]
        self._order = self._inv = None
        if order is not None:
            from .ordering import permute_maps

            order = np.asarray(order, dtype=np.int64)
            if not np.array_equal(np.sort(order), np.arange(self.num_elements)):
                raise ValueError("order must be a permutation of the owned elements")
            geo_words, det_j, maps = geo_words[order], det_j[order], permute_maps(maps, order)
        # face-node slot order (ordering.face_slot_order): the nodes of each face are renumbered so
        # that the tensor-core flux pass's shared-memory trace loads spread over the banks; fmask,
        # the code table and the LIFT columns are permuted together, surface_flux maps back
        if path not in _capi.PATHS:
            raise ValueError(f"path must be one of {sorted(_capi.PATHS)}, got {path!r}")
        if path == "auto" and dtype == torch.float32 and elem.order <= 3 and len(det_j) < SMALL_MESH_SIMT:
            # a few tiles per GPU: the CUDA-core kernel's shorter per-tile latency wins (C1, 1,512 tets
            # at N=3: 14.2 vs 17.9 us per stage, profiles/r02/paths.jsonl)
            path = "simt"
        # v2 tensor kernel (N <= 4, fp32): explicit, or the default where it is the faster kernel
        self._use_tc2 = bool(lay.tc2_supported) and (path == "tensor2" or (path == "auto" and TC2_AUTO))
        if path == "tensor2" and not lay.tc2_supported:
            raise ValueError(f"no tensor2 path for order {elem.order} and {dtype}")
        if face_slots is None:
            face_slots = bool(lay.tc_supported) and path != "simt"
        lift = elem.lift
        self._slot_inv = None
        self._slot_nat = None  # uint8 [4][Nfp]: internal face slot -> natural face node (dgm_face_states)
        if face_slots:
            from .ordering import permute_face_slots

            perm = _face_slot_order(elem, v2=self._use_tc2)
            maps = permute_face_slots(maps, perm)
            n_fp = elem.num_face_nodes
            cols = (np.arange(NUM_FACES)[:, None] * n_fp + perm).reshape(-1)
            lift = elem.lift[:, cols]
            inv = np.empty_like(cols)
            inv[cols] = np.arange(len(cols))
            self._slot_inv = torch.as_tensor(inv, device=self.device)
            self._slot_nat = torch.as_tensor(np.ascontiguousarray(perm, dtype=np.uint8).reshape(-1), device=self.device)

        def dev(a, dt=dtype):
            return torch.as_tensor(np.ascontiguousarray(a)).to(device=self.device, dtype=dt)

        self._diff = dev(np.stack([pack_chunks(elem.diff[m], lay.diff_chunks, lay.vec) for m in range(3)]))
        self._lift = dev(pack_chunks(lift, lay.lift_chunks, lay.vec))
        self._mass = dev(pack_chunks(elem.mass, lay.diff_chunks, lay.vec))
        self._geo = dev(geo_words)
        self._det = dev(det_j)
        nbr = np.zeros((self.field_stride, NUM_FACES), dtype=np.int32)
        cod = np.full((self.field_stride, NUM_FACES), -1, dtype=np.int32)
        nbr[: self.num_elements] = maps.neighbors
        cod[: self.num_elements] = maps.codes
        self._nbr = dev(nbr, torch.int32)
        if order is not None:
            self._order = torch.as_tensor(order, device=self.device)
            inv = np.empty_like(order)
            inv[order] = np.arange(len(order))
            self._inv = torch.as_tensor(inv, device=self.device)
        self._code = dev(cod, torch.int32)
        self._fmask = dev(np.asarray(maps.face_nodes, dtype=np.uint8), torch.uint8)
        table = maps.code_table if len(maps.code_table) else np.zeros((1, elem.num_face_nodes), np.uint8)
        self._ptab = dev(table, torch.uint8)
        self._num_codes = int(len(maps.code_table))
        self._tc = None
        if lay.tc_supported and path not in ("simt", "tensor2"):
            self._tc = dev(tc_operand(elem, lay, lift), torch.float32)
        self._tc2 = None
        if self._use_tc2:
            self._tc2 = dev(tc2_operand(elem, lift), torch.float32)
            assert self._tc2.numel() == lay.tc2_operand_floats

        desc = _capi.Desc(
            order=elem.order, dtype=self._dt_code, num_elements=self.num_elements,
            field_stride=self.field_stride,
            diff_packed=self._diff.data_ptr(), lift_packed=self._lift.data_ptr(),
            geometry=self._geo.data_ptr(), neighbors=self._nbr.data_ptr(),
            codes=self._code.data_ptr(), face_nodes=self._fmask.data_ptr(),
            code_table=self._ptab.data_ptr(), num_codes=self._num_codes,
            permittivity=float(material.permittivity), permeability=float(material.permeability),
            tc_operand=self._tc.data_ptr() if self._tc is not None else None, path=_capi.PATHS[path],
            tc2_operand=self._tc2.data_ptr() if self._tc2 is not None else None)
        lib = _capi.load()
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _capi.check(lib.dgm_plan_create(ctypes.byref(desc), ctypes.byref(handle)), "dgm_plan_create")
        self._plan = handle
        self._lib = lib
        self._bufs: _Buffers | None = None
        self._graphs: dict = {}
        self._norm_out = torch.zeros(1, dtype=torch.float64, device=self.device)
        n_part = int(lib.dgm_mass_norm_partials(handle, self.num_elements))
        self._partials = torch.zeros(max(n_part, 1), dtype=torch.float64, device=self.device)
        self._pinned_rhs = {}        # rhs() on numpy states: pinned staging buffers per (in, out) dtype
        self.collect_stats = False   # record CUDA-event times of every stage launch
        self._events: list = []
        self._stats: dict = {}
        # reference-operator attributes, filled by build_b200_operator
        self.mesh: Mesh | None = None
        self.connectivity: FaceConnectivity | None = None
        self.geometry: GeometricFactors | None = None
        self._nodes = None

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value and _capi._lib is not None:
            _capi._lib.dgm_plan_destroy(plan)
            self._plan = None

    # ------------------------------------------------------------------ info
    @property
    def order(self) -> int:
        return self.elem.order

    @property
    def path(self) -> str:
        """'tensor2' / 'tensor' (tcgen05 3xTF32 stage kernel v2 / v1) or 'simt' (CUDA-core stage kernel)."""
        code = self._lib.dgm_plan_path(self._plan)
        return {_capi.PATH_SIMT: "simt", _capi.PATH_TENSOR: "tensor", _capi.PATH_TENSOR2: "tensor2"}[code]

    @property
    def dofs(self) -> int:
        """Degrees of freedom 6 * Np * K of the owned elements."""
        return N_FIELDS * self.elem.num_nodes * self.num_elements

    @property
    def nodes(self) -> np.ndarray:
        if self._nodes is None:
            self._nodes = map_nodes(self.mesh, self.elem)
        return self._nodes

    @property
    def vmap_minus(self) -> np.ndarray:
        return self.maps.vmap_minus

    @property
    def vmap_plus(self) -> np.ndarray:
        return self.maps.vmap_plus

    @property
    def is_boundary(self) -> np.ndarray:
        return self.maps.is_boundary

    @property
    def normals(self) -> np.ndarray:
        return self.geometry.normals

    @property
    def face_areas_global(self) -> np.ndarray:
        from .refelem import FACE_AREAS

        return self.geometry.face_jacobians * FACE_AREAS

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    # ---------------------------------------------------------- statistics
    def _timed(self, name: str, launch) -> None:
        """Run ``launch()``; with ``collect_stats`` bracket it with CUDA events on the current stream."""
        if not self.collect_stats or torch.cuda.is_current_stream_capturing():
            launch()
            return
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream = torch.cuda.current_stream(self.device)
        start.record(stream)
        launch()
        stop.record(stream)
        self._events.append((name, start, stop))
        if len(self._events) >= 256:
            self._drain_events(block=False)

    def _drain_events(self, block: bool) -> None:
        """Fold recorded event pairs into the per-kernel totals (completed ones only unless ``block``)."""
        if block and self._events:
            torch.cuda.synchronize(self.device)
        done = 0
        for name, start, stop in self._events:
            if not block and not stop.query():
                break
            st = self._stats.setdefault(name, KernelStats())
            st.launches += 1
            st.ms += start.elapsed_time(stop)
            done += 1
        del self._events[:done]

    @property
    def stage_stats(self) -> dict:
        """Per-kernel device time {name: KernelStats} (pipeline.py:62-68's stage_stats, measured)."""
        self._drain_events(block=True)
        return self._stats

    def reset_stats(self) -> None:
        self._events.clear()
        self._stats = {}

    def total_stats(self) -> KernelStats:
        tot = KernelStats()
        for st in self.stage_stats.values():
            tot.launches += st.launches
            tot.ms += st.ms
        return tot

    # ---------------------------------------------------------------- layout
    def empty_state(self) -> torch.Tensor:
        """Zeroed padded state (6, field_stride, np_stride) on the device."""
        return torch.zeros((N_FIELDS, self.field_stride, self.np_stride), dtype=self.dtype, device=self.device)

    def _check_padded(self, u: torch.Tensor, name: str = "state") -> None:
        if not isinstance(u, torch.Tensor):
            raise TypeError(f"{name} must be a torch tensor in the padded device layout")
        want = (N_FIELDS, self.field_stride, self.np_stride)
        if tuple(u.shape) != want:
            raise ValueError(f"{name} has shape {tuple(u.shape)}, expected padded {want}")
        if u.dtype != self.dtype or u.device != self.device or not u.is_contiguous():
            raise ValueError(f"{name} must be a contiguous {self.dtype} tensor on {self.device}")

    def _natural_tensor(self, natural) -> torch.Tensor:
        """Natural state as a device tensor of shape (6, K, Np), float32 or float64 (reshape as oracle.py:65)."""
        k, n_p = self.num_elements, self.elem.num_nodes
        src = torch.as_tensor(natural)
        if src.numel() != N_FIELDS * k * n_p:
            raise ValueError(f"natural state must have 6*K*Np = {N_FIELDS * k * n_p} values "
                             f"(shape (6, {k}, {n_p})), got shape {tuple(src.shape)}")
        if src.dtype not in (torch.float32, torch.float64):
            src = src.to(torch.float64)
        src = src.reshape(N_FIELDS, k, n_p)
        if src.device != self.device:
            src = src.to(self.device, non_blocking=src.is_pinned())
        return src.contiguous()

    def to_padded(self, natural, out: torch.Tensor | None = None) -> torch.Tensor:
        """Natural (6, K, Np) numpy/torch (float32 or float64) -> padded device tensor (padding zero).

        The dtype cast and the internal element order are applied by the pack kernel itself.
        """
        src = self._natural_tensor(natural)
        if out is None:
            out = self.empty_state()
        else:
            self._check_padded(out, "out")
        nat_dt = _capi.DGM_F32 if src.dtype == torch.float32 else _capi.DGM_F64
        perm = self._order.data_ptr() if self._order is not None else None
        with torch.cuda.device(self.device):
            _capi.check(self._lib.dgm_pack(self.order, self._dt_code, src.data_ptr(), nat_dt, perm, out.data_ptr(),
                                           self.num_elements, self.field_stride, self._stream()), "dgm_pack")
        return out

    def from_padded(self, padded: torch.Tensor, dtype: torch.dtype = torch.float64,
                    out: torch.Tensor | None = None) -> torch.Tensor:
        """Padded device tensor -> natural (6, K, Np) device tensor (float64 as the reference, or float32).

        Cast and inverse element permutation happen in the unpack kernel; ``out`` (a contiguous natural
        tensor of that dtype on the device) is filled in place when given.
        """
        self._check_padded(padded, "padded")
        if dtype not in (torch.float32, torch.float64):
            raise ValueError(f"dtype must be torch.float32 or torch.float64, got {dtype}")
        shape = (N_FIELDS, self.num_elements, self.elem.num_nodes)
        if out is None:
            out = torch.empty(shape, dtype=dtype, device=self.device)
        elif tuple(out.shape) != shape or out.dtype != dtype or out.device != self.device or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous {dtype} tensor of shape {shape} on {self.device}")
        nat_dt = _capi.DGM_F32 if dtype == torch.float32 else _capi.DGM_F64
        perm = self._order.data_ptr() if self._order is not None else None
        with torch.cuda.device(self.device):
            _capi.check(self._lib.dgm_unpack(self.order, self._dt_code, padded.data_ptr(), perm, out.data_ptr(),
                                             nat_dt, self.num_elements, self.field_stride, self._stream()),
                        "dgm_unpack")
        return out

    def check_padding(self, padded: torch.Tensor) -> bool:
        """True when every padding slot is exactly zero (fields.py:55-58)."""
        return bool((padded[:, : self.num_elements, self.elem.num_nodes:] == 0).all().item())

    # ------------------------------------------------------------- operators
    def _range(self, e_begin, e_end):
        e_begin = 0 if e_begin is None else int(e_begin)
        e_end = self.num_elements if e_end is None else int(e_end)
        return e_begin, e_end

    def rhs_padded(self, u: torch.Tensor, out: torch.Tensor | None = None,
                   e_begin=None, e_end=None) -> torch.Tensor:
        """Fused RHS in the device layout (one kernel launch)."""
        self._check_padded(u)
        if out is None:
            out = torch.zeros_like(u)
        else:
            self._check_padded(out, "out")
        b, e = self._range(e_begin, e_end)
        self._timed("rhs", lambda: _capi.check(
            self._lib.dgm_rhs(self._plan, u.data_ptr(), out.data_ptr(), b, e, self._stream()), "dgm_rhs"))
        return out

    def volume_padded(self, u: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Volume term only, (curl H/eps, -curl E/mu) (oracle.py:67-79)."""
        self._check_padded(u)
        out = torch.zeros_like(u) if out is None else out
        _capi.check(self._lib.dgm_volume(self._plan, u.data_ptr(), out.data_ptr(), 0, self.num_elements,
                                         self._stream()), "dgm_volume")
        return out

    def surface_flux(self, u: torch.Tensor) -> torch.Tensor:
        """upwind_flux * face_jacobian per face node, (6, K, 4*Nfp) (oracle.py:82-85)."""
        self._check_padded(u)
        nf4 = NUM_FACES * self.elem.num_face_nodes
        out = torch.zeros((N_FIELDS, self.field_stride, nf4), dtype=self.dtype, device=self.device)
        _capi.check(self._lib.dgm_surface(self._plan, u.data_ptr(), out.data_ptr(), 0, self.num_elements,
                                          self._stream()), "dgm_surface")
        out = out[:, : self.num_elements]
        if self._slot_inv is not None:
            out = out.index_select(2, self._slot_inv)  # natural face-node order
        return out if self._inv is None else out.index_select(1, self._inv)  # natural numbering

    def rhs(self, state):
        """Reference-compatible RHS (oracle.py:60-94): natural state in (any shape holding 6*K*Np values,
        reshaped as the reference does), new (6, K, Np) array of the same kind out (numpy stays numpy,
        torch stays on its device), float32 input -> float32 output, anything else -> float64."""
        is_numpy = not isinstance(state, torch.Tensor)
        src = np.asarray(state) if is_numpy else state
        out_dtype = torch.float32 if (src.dtype == np.float32 if is_numpy else src.dtype == torch.float32) \
            else torch.float64
        if is_numpy:
            return self._rhs_numpy(src, out_dtype)
        u = self.to_padded(src)
        out = self.from_padded(self.rhs_padded(u), out_dtype)
        return out.to(device=state.device)

    PINNED_RHS_MAX_BYTES = 8 << 30  # per staging buffer; larger numpy states take the pageable path

    def _rhs_numpy(self, src: np.ndarray, out_dtype: torch.dtype) -> np.ndarray:
        """rhs() for a host numpy state: staged through cached pinned buffers (the host-side copies run on
        torch's multi-threaded CPU kernels, the PCIe copies at pinned speed); returns a fresh array."""
        shape = (N_FIELDS, self.num_elements, self.elem.num_nodes)
        k, n_p = self.num_elements, self.elem.num_nodes
        if src.size != N_FIELDS * k * n_p:
            raise ValueError(f"natural state must have 6*K*Np = {N_FIELDS * k * n_p} values "
                             f"(shape (6, {k}, {n_p})), got shape {tuple(src.shape)}")
        if src.dtype not in (np.float32, np.float64):
            src = src.astype(np.float64)
        src = np.ascontiguousarray(src).reshape(shape)
        if not src.flags.writeable:
            src = src.copy()
        key = (src.dtype.str, out_dtype)
        bufs = self._pinned_rhs.get(key)
        if bufs is None:
            in_dtype = torch.float64 if src.dtype == np.float64 else torch.float32
            try:
                if src.nbytes > self.PINNED_RHS_MAX_BYTES:
                    raise RuntimeError("state too large for pinned staging")
                bufs = (torch.empty(shape, dtype=in_dtype, pin_memory=True),
                        torch.empty(shape, dtype=out_dtype, pin_memory=True))
            except RuntimeError:  # no pinned memory to spare: the pageable path, same results
                bufs = False
            self._pinned_rhs[key] = bufs
        if bufs is False:
            out = self.from_padded(self.rhs_padded(self.to_padded(src)), out_dtype)
            return out.cpu().numpy()
        host_in, host_out = bufs
        host_in.copy_(torch.from_numpy(src))
        out = self.from_padded(self.rhs_padded(self.to_padded(host_in)), out_dtype)
        host_out.copy_(out, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()  # also frees host_in for the next call
        result = torch.empty(shape, dtype=out_dtype)
        result.copy_(host_out)
        return result.numpy()

    def face_states(self, state):
        """(u_minus, u_plus, normals) per face node, boundary side mirrored (oracle.py:50-58).

        u_minus / u_plus are (6, K, 4, Nfp) gathered on the device by dgm_face_states in the natural
        numbering; normals are (3, K, 4, 1).  numpy in -> numpy out (float64), torch in -> torch out.
        """
        is_numpy = not isinstance(state, torch.Tensor)
        u = self.to_padded(np.asarray(state) if is_numpy else state)
        shape = (N_FIELDS, self.num_elements, NUM_FACES, self.elem.num_face_nodes)
        um = torch.empty(shape, dtype=self.dtype, device=self.device)
        up = torch.empty_like(um)
        perm = self._order.data_ptr() if self._order is not None else None
        nodes = self._slot_nat.data_ptr() if self._slot_nat is not None else None
        _capi.check(self._lib.dgm_face_states(self._plan, u.data_ptr(), perm, nodes, um.data_ptr(), up.data_ptr(),
                                              self._stream()), "dgm_face_states")
        nrm = np.moveaxis(self.geometry.normals, -1, 0)[:, :, :, None]
        if is_numpy:
            return um.double().cpu().numpy(), up.double().cpu().numpy(), nrm
        return um.to(state.device), up.to(state.device), torch.as_tensor(nrm, device=state.device)

    rhs_natural = rhs

    def lsrk_stage(self, u_in: torch.Tensor, u_out: torch.Tensor, res: torch.Tensor, a: float, b: float,
                   dt: float, e_begin=None, e_end=None) -> None:
        """res = a res + dt rhs(u_in); u_out = u_in + b res  (one fused launch)."""
        bb, ee = self._range(e_begin, e_end)
        self._timed("lsrk_stage", lambda: _capi.check(
            self._lib.dgm_lsrk_stage(self._plan, u_in.data_ptr(), u_out.data_ptr(), res.data_ptr(),
                                     float(a), float(b), float(dt), bb, ee, self._stream()), "dgm_lsrk_stage"))

    def _buffers(self) -> _Buffers:
        if self._bufs is None:
            self._bufs = self.workspace()
        return self._bufs

    def workspace(self) -> _Buffers:
        """Scratch registers (two state buffers + LSRK residual) for ``advance(..., workspace=)``.

        The operator keeps one of its own; pass a separate workspace per CUDA stream to advance
        independent states concurrently.
        """
        return _Buffers(alt=self.empty_state(), res=self.empty_state(), alt2=self.empty_state())

    def _launch_steps(self, u: torch.Tensor, dt: float, nsteps: int, bufs: _Buffers | None = None) -> torch.Tensor:
        """nsteps LSRK4 steps, each ending back in u: u -> alt -> alt2 -> alt -> alt2 -> u.

        A stage cannot update in place (neighbour traces read u_in while other CTAs write u_out); with
        two scratch registers the odd stage count of a step still lands in u, so no copy is needed.
        """
        bufs = self._buffers() if bufs is None else bufs
        if bufs.alt2 is None:
            bufs.alt2 = self.empty_state()
        for _ in range(nsteps):
            src = u
            for i, (a, b) in enumerate(zip(RK_A, RK_B)):
                dst = u if i == len(RK_A) - 1 else (bufs.alt if i % 2 == 0 else bufs.alt2)
                self.lsrk_stage(src, dst, bufs.res, a, b, dt)
                src = dst
        return u

    GRAPH_STEPS = 8  # LSRK4 steps per captured CUDA graph

    def advance(self, u: torch.Tensor, dt: float, nsteps: int = 1, use_graph: bool | None = None,
                workspace: _Buffers | None = None) -> torch.Tensor:
        """Advance the padded state in place by nsteps LSRK4 steps of size dt (no copies)."""
        self._check_padded(u)
        if dt <= 0.0:
            raise ValueError("dt must be positive")
        nsteps = int(nsteps)
        if nsteps < 0:
            raise ValueError("nsteps must be >= 0")
        if nsteps == 0:
            return u
        if use_graph is None:
            use_graph = nsteps >= 4
        bufs = self._buffers() if workspace is None else workspace
        if not use_graph:
            return self._launch_steps(u, dt, nsteps, bufs)
        chunks, rest = divmod(nsteps, self.GRAPH_STEPS)
        for _ in range(chunks):
            self._graph_for(u, dt, bufs, self.GRAPH_STEPS).replay()
        if rest:
            self._graph_for(u, dt, bufs, rest).replay()
        return u

    def _graph_for(self, u: torch.Tensor, dt: float, bufs: _Buffers, nsteps: int):
        """CUDA graph of ``nsteps`` LSRK4 steps (5 * nsteps stage launches, u -> ... -> u)."""
        if bufs.alt2 is None:
            bufs.alt2 = self.empty_state()
        key = (u.data_ptr(), bufs.alt.data_ptr(), bufs.alt2.data_ptr(), bufs.res.data_ptr(), float(dt), nsteps)
        graph = self._graphs.get(key)
        if graph is None:
            # load the stage kernel outside capture (scratch buffers only)
            self.lsrk_stage(bufs.alt, bufs.alt2, bufs.res, 0.0, 0.0, 0.0, 0, min(self.num_elements, 1))
            torch.cuda.current_stream(self.device).synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                self._launch_steps(u, dt, nsteps, bufs)
            self._graphs[key] = graph
        return graph

    def step(self, u: torch.Tensor, dt: float, workspace: _Buffers | None = None) -> torch.Tensor:
        """One LSRK4 step in place (5 fused stage launches)."""
        return self.advance(u, dt, 1, use_graph=False, workspace=workspace)

    # ---------------------------------------------------------- diagnostics
    def mass_norm(self, u: torch.Tensor, w_e: float = 1.0, w_h: float = 1.0,
                  out: torch.Tensor | None = None) -> torch.Tensor:
        """Device scalar sum_k J_k sum_f w_f u^T M u (float64 tensor, no sync).

        With ``out`` (a zeroed float64 device slot) the value is accumulated there.  The reduction
        order is fixed (per-CTA partials, then one fixed-order pass), so reruns are bitwise identical.
        Calls on one operator share the partials scratch: issue them on one stream.
        """
        self._check_padded(u)
        if out is None:
            out = torch.zeros(1, dtype=torch.float64, device=self.device)
        elif out.dtype != torch.float64 or out.device != self.device or out.numel() < 1:
            raise ValueError("out must be a float64 device tensor on the operator's device")
        _capi.check(self._lib.dgm_mass_norm(self._plan, u.data_ptr(), self._mass.data_ptr(), self._det.data_ptr(),
                                            float(w_e), float(w_h), out.data_ptr(), self._partials.data_ptr(),
                                            0, self.num_elements, self._stream()), "dgm_mass_norm")
        return out

    def field_energy(self, u: torch.Tensor) -> float:
        """1/2 (eps |E|^2 + mu |H|^2) (maxwell.py:225-232)."""
        m = self.material
        return 0.5 * float(self.mass_norm(u, m.permittivity, m.permeability).item())

    def l2_error(self, u: torch.Tensor, mode, t: float) -> float:
        """Mass-weighted L2 distance to ``mode`` at time t (maxwell.py:211-222)."""
        exact = self.to_padded(mode.evaluate(self.nodes, t))
        return math.sqrt(max(float(self.mass_norm(u - exact).item()), 0.0))


def build_b200_operator(mesh: Mesh, elem: ReferenceElement, material: Material = VACUUM,
                        connectivity: FaceConnectivity | None = None, *,
                        dtype: torch.dtype = torch.float32, device=None, path: str = "auto",
                        reorder: bool | str | None = None,
                        face_slots: bool | None = None) -> B200MaxwellOperator:
    """Drop-in for build_reference_operator (oracle.py:97-141) on one B200.

    ``reorder=True`` numbers the elements internally in 2x2-cell columns of their centroids
    (``"morton"``: along a Morton curve; ``"greedy"``: the paper's Alg. 2 face-adjacency blocks of
    64, reference layout.py:59-117; paper_0901_1024_b200/ordering.py); the natural-order API
    is unchanged.  Default (None): on for 2 <= N <= 8 (C3 fp32 1.63 -> 1.54 ms per stage, fp64
    and N = 7, 8 0.4-1.3 % faster; N = 1 and N = 9 keep the reference numbering).
    ``face_slots`` (default: whenever the tensor path is available) renumbers the nodes inside
    each face for conflict-free shared-memory flux loads (ordering.face_slot_order).
    """
    if reorder is None:
        reorder = 2 <= elem.order <= 8
    if connectivity is None:
        connectivity = build_connectivity(mesh)
    geometry = compute_geometry(mesh, elem)
    maps = build_face_maps(mesh, elem, connectivity)
    order = None
    if reorder:
        from . import ordering

        if reorder == "greedy":  # the paper's Alg. 2 blocks (reference layout.py:59-117), tile-sized
            order = ordering.greedy_block_order(mesh.vertices, mesh.elements, 64, connectivity)
        else:
            fn = ordering.morton_order if reorder == "morton" else ordering.column_order
            order = fn(mesh.vertices, mesh.elements)
    op = B200MaxwellOperator(elem, material, geometry_words(geometry), geometry.det_jacobians, maps,
                             dtype=dtype, device=device, path=path, order=order, face_slots=face_slots)
    op.mesh = mesh
    op.connectivity = connectivity
    op.geometry = geometry
    return op
