"""Host-resident state stepping: the reference user's float64 state stays in (pinned) host memory.

The reference keeps the field state on the host (numpy, natural (6, K, Np) layout) and advances it
with ``rk4_step`` (kernels/assemble.py:105-114).  ``HostStepper.step`` advances such a state through
the device operator, round-tripping it through host memory every step: upload -> pack (cast +
element permutation, ``dgm_pack``) -> one fused LSRK4 step -> unpack (``dgm_unpack``) -> download
into the same host buffer, plus the field-energy scalar.

The copies move contiguous pieces (``chunks`` per field slab) on two copy streams: the upload of
piece p for step i+1 waits only for the download of piece p from step i, and the pack waits for
every upload, so each step computes on the previous step's downloaded output while the download of
step i and the upload of step i+1 share the full-duplex PCIe link, also across calls.  ``serial=True``
issues one copy per direction on the compute stream instead.  Everything is asynchronous: the
downloads run on the stepper's own stream, so call ``join()`` (orders the current stream after them)
or synchronize before reading the host buffer.
"""
from __future__ import annotations

import torch

N_FIELDS = 6


class HostStepper:
    """Advance a pinned host state (6, K, Np) with a device operator; see the module docstring.

    ``op``: the B200MaxwellOperator that packs / unpacks (a DistributedMaxwellOperator's ``op``);
    ``advance``: ``advance(u_padded, dt, nsteps)`` of the single or distributed operator.
    """

    def __init__(self, op, advance=None, chunks: int = 4, serial: bool = False):
        if chunks < 1:
            raise ValueError("chunks must be >= 1")
        self.op = op
        self._advance = advance if advance is not None else (lambda u, dt, n: op.advance(u, dt, n, use_graph=False))
        self.chunks = int(chunks)
        self.serial = bool(serial)
        self._bufs = {}
        self._pending = False  # downloads of a previous step may still be in flight

    def _buffers(self, dtype):
        b = self._bufs.get(dtype)
        if b is None:
            op = self.op
            shape = (N_FIELDS, op.num_elements, op.elem.num_nodes)
            kb = [round(j * op.num_elements / self.chunks) for j in range(self.chunks + 1)]
            pieces = [(f, kb[j], kb[j + 1]) for f in range(N_FIELDS) for j in range(self.chunks) if kb[j + 1] > kb[j]]
            b = dict(dev_nat=torch.empty(shape, dtype=dtype, device=op.device),
                     nat=torch.empty(shape, dtype=dtype, device=op.device), padded=op.empty_state(),
                     up=torch.cuda.Stream(op.device), down=torch.cuda.Stream(op.device), pieces=pieces,
                     down_done=[torch.cuda.Event() for _ in pieces], up_done=torch.cuda.Event(),
                     computed=torch.cuda.Event(), energy_done=torch.cuda.Event(), begin=torch.cuda.Event())
            self._bufs[dtype] = b
        return b

    def step(self, host: torch.Tensor, dt: float, nsteps: int = 1, energy_out: torch.Tensor | None = None):
        """Advance ``host`` (pinned, contiguous, float64 or float32, shape (6, K, Np)) by ``nsteps`` LSRK4
        steps, each a full host round trip; ``energy_out`` (pinned float64, >= 1 element) receives the
        last step's sum of E.E + H.H mass norms (unit weights).  Returns ``host``."""
        op = self.op
        shape = (N_FIELDS, op.num_elements, op.elem.num_nodes)
        if tuple(host.shape) != shape or host.device.type != "cpu" or not host.is_contiguous():
            raise ValueError(f"host must be a contiguous CPU tensor of shape {shape}")
        if host.dtype not in (torch.float32, torch.float64):
            raise ValueError(f"host dtype must be float32 or float64, got {host.dtype}")
        if dt <= 0.0:
            raise ValueError("dt must be positive")
        b = self._buffers(host.dtype)
        stream = torch.cuda.current_stream(op.device)
        if not self._pending:
            b["begin"].record(stream)  # the first uploads of a chain follow the caller's prior work
        for _ in range(int(nsteps)):
            if self.serial:
                b["dev_nat"].copy_(host, non_blocking=True)
            else:
                with torch.cuda.stream(b["up"]):
                    if not self._pending:
                        b["up"].wait_event(b["begin"])
                    for p, (f, k0, k1) in enumerate(b["pieces"]):
                        if self._pending:
                            b["up"].wait_event(b["down_done"][p])  # previous step's piece p has landed
                        b["dev_nat"][f, k0:k1].copy_(host[f, k0:k1], non_blocking=True)
                    b["up_done"].record(b["up"])
                stream.wait_event(b["up_done"])
            op.to_padded(b["dev_nat"], out=b["padded"])
            self._advance(b["padded"], dt, 1)
            op.from_padded(b["padded"], host.dtype, out=b["nat"])
            if self.serial:
                host.copy_(b["nat"], non_blocking=True)
                if energy_out is not None:
                    energy_out[:1].copy_(op.mass_norm(b["padded"], 1.0, 1.0), non_blocking=True)
                continue
            b["computed"].record(stream)
            # the energy reduction runs on the compute stream while the downloads drain (it only reads
            # the padded state, which the next step's pack rewrites after every upload has landed)
            energy = op.mass_norm(b["padded"], 1.0, 1.0) if energy_out is not None else None
            if energy is not None:
                b["energy_done"].record(stream)
            with torch.cuda.stream(b["down"]):
                b["down"].wait_event(b["computed"])
                for p, (f, k0, k1) in enumerate(b["pieces"]):
                    host[f, k0:k1].copy_(b["nat"][f, k0:k1], non_blocking=True)
                    b["down_done"][p].record(b["down"])
                if energy is not None:
                    b["down"].wait_event(b["energy_done"])
                    energy_out[:1].copy_(energy, non_blocking=True)
            if energy is not None:
                energy.record_stream(b["down"])
            self._pending = True
        return host

    def join(self, stream: torch.cuda.Stream | None = None) -> None:
        """Order ``stream`` (default: the current one) after every download issued so far; the next
        step() then starts a new chain (its first uploads follow that stream's work)."""
        stream = torch.cuda.current_stream(self.op.device) if stream is None else stream
        for b in self._bufs.values():
            stream.wait_stream(b["down"])
        self._pending = False
