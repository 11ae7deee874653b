"""Peer-memory communicator over NVLink / NVSwitch (csrc/comm.cu, C1 / C2).

One process per GPU.  ``PeerComm(group)`` allocates this rank's region,
exchanges the CUDA IPC handles over ``group`` (any torch.distributed backend:
only host bytes travel) and maps every peer's region.  Then, on the current
CUDA stream and without NCCL:

* ``allreduce_partials(part, S, stride, n, out)`` -- the row-parallel sum of a
  tensor-parallel target fused with the local split-K reduction, summed in
  (rank, split) order so every rank gets bit-identical results;
* ``put(peer, src)`` / ``get(peer, dst)`` -- the depth-1 int32 mailbox of the
  dedicated-draft-GPU hand-off.

Replaces the reference's scalar ``comm_overhead`` (request_model.py:128,
engine.py:435-442).  Every peer must run on the same node (CUDA IPC); ranks
may share a GPU (the tests do).
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import native
from .errors import ConfigError

__all__ = ["PeerComm"]


class PeerComm:
    def __init__(self, group=None, buf_bytes: int = 64 << 20, mbox_bytes: int = 1 << 20,
                 device=None) -> None:
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device if device is not None else torch.device("cuda",
                                                                     torch.cuda.current_device())
        lib = native.load()
        hb = lib.psd_comm_handle_bytes()
        mine = ctypes.create_string_buffer(hb)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            native.check(lib.psd_comm_create(self.rank, self.world, buf_bytes, mbox_bytes,
                                             ctypes.byref(handle), mine), "psd_comm_create")
        self._c = handle
        self.buf_bytes = buf_bytes
        self.mbox_bytes = mbox_bytes
        blobs = [None] * self.world
        dist.all_gather_object(blobs, mine.raw, group=group)
        allh = ctypes.create_string_buffer(b"".join(blobs), hb * self.world)
        with torch.cuda.device(self.device):
            native.check(lib.psd_comm_open(self._c, allh), "psd_comm_open")

    @classmethod
    def local_group(cls, devices, buf_bytes: int = 64 << 20,
                    mbox_bytes: int = 1 << 20) -> list["PeerComm"]:
        """One process driving len(devices) ranks (psd_comm_create_local): no
        IPC, no process group.  Rank r's calls must be issued on devices[r],
        on a stream that runs concurrently with the other ranks' streams."""
        world = len(devices)
        lib = native.load()
        devs = (ctypes.c_int * world)(*[torch.device(d).index or 0 for d in devices])
        hs = (ctypes.c_void_p * world)()
        native.check(lib.psd_comm_create_local(world, devs, buf_bytes, mbox_bytes, hs),
                     "psd_comm_create_local")
        out = []
        for r in range(world):
            c = cls.__new__(cls)
            c.group, c.rank, c.world = None, r, world
            c.device = torch.device("cuda", devs[r])
            c._c = ctypes.c_void_p(hs[r])
            c.buf_bytes, c.mbox_bytes = buf_bytes, mbox_bytes
            out.append(c)
        return out

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def allreduce_partials(self, part: torch.Tensor, S: int, stride: int, n: int,
                           out: torch.Tensor | None = None) -> torch.Tensor:
        """out[:n] = sum over ranks, then splits, of part[s * stride + i]
        (fp32, flat views; out may alias part)."""
        if part.dtype != torch.float32 or not part.is_cuda:
            raise ConfigError("allreduce_partials: fp32 CUDA partials")
        if (S - 1) * stride + n > part.numel():
            raise ConfigError("allreduce_partials: partials too small")
        out = part if out is None else out
        native.check(native.load().psd_tp_allreduce_partials(
            self._c, part.data_ptr(), S, stride, n, out.data_ptr(), self._stream()),
            "psd_tp_allreduce_partials")
        return out

    def allreduce_(self, data: torch.Tensor) -> torch.Tensor:
        return self.allreduce_partials(data.view(-1), 1, data.numel(), data.numel(),
                                       data.view(-1)).view(data.shape)

    def allgather(self, src: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """out.view(world, -1)[r] = rank r's src (fp32, n % 4 == 0)."""
        n = src.numel()
        if out.numel() < self.world * n or src.dtype != torch.float32:
            raise ConfigError("allgather: fp32, out holds world * n")
        native.check(native.load().psd_tp_allgather_f32(
            self._c, src.data_ptr(), n, out.data_ptr(), self._stream()), "psd_tp_allgather_f32")
        return out

    def put(self, peer: int, src: torch.Tensor) -> None:
        if src.dtype != torch.int32 or not src.is_cuda:
            raise ConfigError("put: int32 CUDA tensor")
        native.check(native.load().psd_p2p_put_i32(self._c, peer, src.data_ptr(), src.numel(),
                                                   self._stream()), "psd_p2p_put_i32")

    def get(self, peer: int, dst: torch.Tensor) -> torch.Tensor:
        if dst.dtype != torch.int32 or not dst.is_cuda:
            raise ConfigError("get: int32 CUDA tensor")
        native.check(native.load().psd_p2p_get_i32(self._c, peer, dst.data_ptr(), dst.numel(),
                                                   self._stream()), "psd_p2p_get_i32")
        return dst

    def close(self) -> None:
        if self._c:
            native.load().psd_comm_destroy(self._c)
            self._c = None
