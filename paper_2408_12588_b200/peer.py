"""NVLink peer-memory transport for broadcast sequence parallelism.

The reference exchanges shards around every computed temporal site with
``reshard`` (frames -> tokens before, tokens -> frames after; pkg/src/pab_engine/
parallel.py:140-180, 322-348).  The NCCL transport (``parallel._all_to_all``)
runs those as two ``all_to_all_single`` calls.  This transport removes both
collectives: every rank of the group maps the other ranks' token-layout buffers
into its address space (CUDA IPC between processes, plain pointers between the
logical workers of one process), and

* the temporal site's prologue stores h straight into the destination ranks'
  receive buffers (``pab_residual_modnorm_peer``, h layout ``LAYOUT_PEER``),
* the prologue after the temporal site reads the attention output straight out
  of the ranks' token buffers (pending term layout ``LAYOUT_PEER``) and, when the
  site is cached, writes a frame-major copy into the local cache slot, so a
  later broadcast step communicates nothing (reference parallel.py:335-340),
* a device barrier (``pab_peer_barrier``) after each producer orders the peer
  stores/loads; it is epoch-based on the device, so the whole sharded video
  still replays as one CUDA graph.

Over NVSwitch the exchange traffic then overlaps the prologue's own HBM
streaming instead of running as separate collective kernels.
"""

from __future__ import annotations

import pickle
from typing import Dict, List, Tuple

import torch

from . import _lib
from .errors import DeviceError, ValidationError

PEER_TIMEOUT = 0x7EE1  # include/pab_b200.h PAB_PEER_TIMEOUT
MAX_PEERS = 8


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class PeerExchange:
    """Symmetric device buffers of one sequence-parallel group.

    ``buffers`` maps a name to (shape, dtype); every rank allocates the same set.
    ``group`` is a ``parallel.LocalGroup`` (logical workers sharing one process and
    GPU: pointers are exchanged directly) or a torch.distributed process group
    (one process per GPU, or several on one GPU in tests: CUDA IPC handles are
    exchanged with ``all_gather_object`` and opened here).  Collective: every rank
    of the group constructs it, in the same order."""

    def __init__(self, group, rank: int, world: int, buffers: Dict[str, Tuple[tuple, torch.dtype]], device,
                 timeout_s: float = 60.0):
        if not 1 <= world <= MAX_PEERS:
            raise ValidationError(f"the peer transport supports 1..{MAX_PEERS} ranks, got {world}")
        self.rank, self.world, self.timeout_s = int(rank), int(world), float(timeout_s)
        self.local: Dict[str, torch.Tensor] = {
            k: torch.zeros(shape, dtype=dt, device=device) for k, (shape, dt) in buffers.items()}
        # flags[q] of rank w: the last barrier epoch rank q signalled to w; one allocation
        # for flags + counter + error word
        self._ctl = torch.zeros(world + 2, dtype=torch.int32, device=device)
        self.counter = self._ctl[world:world + 1]
        self.error = self._ctl[world + 1:world + 2]
        names = sorted(self.local)
        tensors = [self.local[k] for k in names] + [self._ctl]
        peers = _map_group(group, self.rank, self.world, tensors)  # per tensor: list over ranks
        self.peers: Dict[str, List[torch.Tensor]] = {k: peers[i] for i, k in enumerate(names)}
        self._ctl_peers = peers[-1]
        self._ptr_arrays = {k: _lib.ptr_array([t.data_ptr() for t in v]) for k, v in self.peers.items()}
        self._flags = _lib.ptr_array([t.data_ptr() for t in self._ctl_peers])

    def ptrs(self, name: str):
        """ctypes array of the W ranks' device pointers of buffer ``name``."""
        return self._ptr_arrays[name]

    def barrier(self) -> None:
        """Device barrier of the group on the current stream (graph-capturable)."""
        lib = _lib.load()
        _lib.check(lib.pab_peer_barrier(self._flags, self.counter.data_ptr(), self.rank, self.world,
                                        self.error.data_ptr(), self.timeout_s, _stream()), "pab_peer_barrier")

    def check(self) -> None:
        """Raise if a device barrier of this group timed out (synchronises)."""
        if int(self.error.item()) != 0:
            raise DeviceError(f"peer barrier of rank {self.rank}/{self.world} timed out "
                              f"(a rank of the group stopped issuing barriers)")


def _map_group(group, rank: int, world: int, tensors: List[torch.Tensor]) -> List[List[torch.Tensor]]:
    """For every tensor, the list of the group's ranks' copies mapped into this process."""
    from .parallel import LocalGroup

    if world == 1:
        return [[t] for t in tensors]
    if isinstance(group, LocalGroup):
        posted = group.exchange_objects(tensors)
        return [[posted[w][i] for w in range(world)] for i in range(len(tensors))]
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor

    mine = pickle.dumps([reduce_tensor(t) for t in tensors])
    gathered: list = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    out: List[List[torch.Tensor]] = [[None] * world for _ in tensors]  # type: ignore[list-item]
    for w in range(world):
        if w == rank:
            for i, t in enumerate(tensors):
                out[i][w] = t
            continue
        for i, (fn, args) in enumerate(pickle.loads(gathered[w])):
            out[i][w] = fn(*args)  # torch's CUDA IPC rebuild (cudaIpcOpenMemHandle)
    # every rank holds every mapping before anyone issues peer stores
    dist.barrier(group=group)
    return out


__all__ = ["PeerExchange", "PEER_TIMEOUT"]
