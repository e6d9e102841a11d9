"""Communicator: symmetric peer-mapped buffers + SM-budgeted collectives (libkpo comm.cu).

One process per GPU.  `torch.distributed` is plumbing only: it exchanges the 64-byte CUDA IPC
handles of every rank's symmetric buffer (any backend, gloo included); the data path is the
hand-written P2P kernels, launched with exactly `ncta` CTAs that each own a whole SM.

Loopback mode runs `world` virtual ranks on one device (the single-GPU box): rank `rank` is real,
the peers' symmetric buffers are local allocations the caller may fill.  The kernels, CTA
budget, barriers and memory traffic pattern are the real ones; only the link is HBM instead of
NVLink.
"""

from __future__ import annotations

import contextlib
import ctypes

import torch

from . import _lib


class _CAI:
    """Zero-copy torch view of device memory owned by libkpo."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def _view(ptr: int, nbytes: int, device) -> torch.Tensor:
    return torch.as_tensor(_CAI(ptr, nbytes), device=device)


class SymRegion:
    """A byte range of the symmetric buffer (same offset on every rank)."""

    def __init__(self, comm: "Communicator", offset: int, nbytes: int):
        self.comm, self.offset, self.nbytes = comm, offset, nbytes

    def local(self, dtype=torch.bfloat16) -> torch.Tensor:
        return self.comm._sym_bytes[self.offset:self.offset + self.nbytes].view(dtype)

    def peer(self, p: int, dtype=torch.bfloat16) -> torch.Tensor:
        return self.comm.peer_bytes(p)[self.offset:self.offset + self.nbytes].view(dtype)


class Communicator:
    def __init__(self, rank: int, world: int, device: torch.device, sym_bytes: int, loopback: bool,
                 handles_exchange=None):
        self.rank, self.world, self.loopback = rank, world, bool(loopback)
        self.device = torch.device(device)
        self.sym_bytes = int(sym_bytes)
        h = ctypes.c_void_p()
        _lib.call("kpo_comm_create", rank, world, self.device.index or 0, self.sym_bytes, int(self.loopback),
                  ctypes.byref(h))
        self._h = h
        if not self.loopback and world > 1:
            blob = ctypes.create_string_buffer(_lib.KPO_IPC_HANDLE_BYTES)
            _lib.call("kpo_comm_ipc_handle", self._h, blob)
            all_blobs = handles_exchange(bytes(blob.raw))
            joined = ctypes.create_string_buffer(b"".join(all_blobs), len(all_blobs) * _lib.KPO_IPC_HANDLE_BYTES)
            _lib.call("kpo_comm_open_peers", self._h, joined)
        L = _lib.lib()
        self._sym_bytes = _view(L.kpo_comm_sym_ptr(self._h), self.sym_bytes, self.device)
        self._peer_views = {}
        self._next_off = 0
        self.max_ctas = L.kpo_comm_max_ctas(self._h)

    # ---------------------------------------------------------------- construction
    @classmethod
    def loopback_group(cls, world: int, sym_bytes: int, device="cuda") -> "Communicator":
        return cls(0, world, torch.device(device), sym_bytes, loopback=True)

    @classmethod
    def from_process_group(cls, sym_bytes: int, device=None, group=None) -> "Communicator":
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        device = device or torch.device("cuda", torch.cuda.current_device())
        return cls(rank, world, device, sym_bytes, loopback=False,
                   handles_exchange=lambda blob: exchange_blobs(blob, group))

    # ---------------------------------------------------------------- memory
    def alloc(self, nbytes: int, align: int = 256) -> SymRegion:
        off = (self._next_off + align - 1) // align * align
        if off + nbytes > self.sym_bytes:
            raise MemoryError(f"symmetric buffer exhausted ({off + nbytes} > {self.sym_bytes})")
        self._next_off = off + nbytes
        return SymRegion(self, off, nbytes)

    def peer_bytes(self, p: int) -> torch.Tensor:
        if p not in self._peer_views:
            ptr = _lib.lib().kpo_comm_peer_ptr(self._h, p)
            self._peer_views[p] = _view(ptr, self.sym_bytes, self.device)
        return self._peer_views[p]

    # ---------------------------------------------------------------- collectives
    def all_gather(self, src: SymRegion, out: torch.Tensor, ncta: int, stream=None) -> None:
        """out = concat over ranks of every rank's `src` region (bytes_per_rank = src.nbytes)."""
        if out.numel() * out.element_size() < src.nbytes * self.world:
            raise ValueError("all_gather: output too small")
        with self._gated():
            _lib.call("kpo_all_gather", self._h, src.offset, out.data_ptr(), src.nbytes, int(ncta), _s(stream))

    def reduce_scatter(self, src: SymRegion, out: torch.Tensor, ncta: int, stream=None) -> None:
        """out[i] = sum_p src_p[rank*count + i] (bf16, fp32 accumulation in rank order)."""
        count = src.nbytes // 2 // self.world
        if out.numel() < count:
            raise ValueError("reduce_scatter: output too small")
        with self._gated():
            _lib.call("kpo_reduce_scatter", self._h, src.offset, out.data_ptr(), count, int(ncta), _s(stream))

    def all_reduce(self, src: SymRegion, stage: SymRegion, out: torch.Tensor, ncta: int, stream=None) -> None:
        count = src.nbytes // 2
        with self._gated():
            _lib.call("kpo_all_reduce", self._h, src.offset, stage.offset, out.data_ptr(), count, int(ncta),
                      _s(stream))

    def arm_launch_event(self, event: torch.cuda.Event | None) -> None:
        """The NEXT collective launched records `event` once all its CTAs are resident
        (cudaLaunchAttributeLaunchCompletionEvent); later launches do not."""
        self._armed = event

    def disarm_launch_event(self) -> None:
        """Forget an armed event (the executor calls this in a `finally`, even if the launch raised)."""
        if getattr(self, "_armed", None) is not None:
            self._armed = None
            _lib.call("kpo_set_launch_completion_event", self._h, None)

    @contextlib.contextmanager
    def _gated(self):
        """Attach the armed launch-completion event to exactly one collective launch; the library
        state is cleared even when the launch raises, so no later collective records it."""
        ev = getattr(self, "_armed", None)
        if ev is None:
            yield
            return
        try:
            _lib.call("kpo_set_launch_completion_event", self._h, ev.cuda_event)
            yield
        finally:
            self.disarm_launch_event()

    def trace(self, buf: torch.Tensor | None, slots: int = 0) -> None:
        _lib.call("kpo_comm_trace", self._h, None if buf is None else buf.data_ptr(), int(slots))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._sym_bytes = None
            self._peer_views = {}
            _lib.call("kpo_comm_destroy", self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def exchange_blobs(blob: bytes, group=None) -> list[bytes]:
    """All-gather one fixed-size IPC-handle blob per rank, in rank order (any backend)."""
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    if len({len(b) for b in out}) != 1:
        raise ValueError("IPC handle blobs differ in size across ranks")
    return out


def _s(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
