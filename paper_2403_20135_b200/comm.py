"""NCCL communicators of the node-parallel dSDC, through the C ABI.

The one exchange step of a diagonal sweep (every node's (f_E, f_I) is needed
by every node's quadrature; the reference waits on the node futures,
``pkg/src/parsdc/integrators.py:278-288``) is an all-gather across the GPUs
holding the nodes.  :class:`NcclComm` wraps ``sdcsw_comm_*`` /
``sdcsw_allgather_rhs`` (``csrc/comm.cu``): NCCL is called from
``libsdcsw.so``; torch.distributed only carries the 128-byte unique id from
rank 0 to the other ranks (:meth:`NcclComm.bootstrap`).

:class:`DistComm` is the same interface over torch.distributed collectives;
it exists for the CPU multi-process tests (gloo), where there is no NCCL.
"""

import ctypes

from . import _native


class NcclComm:
    """One NCCL communicator (``sdcsw_comm``) of this process."""

    def __init__(self, handle):
        self._lib = _native.lib()
        self.handle = handle
        w, r = ctypes.c_int(), ctypes.c_int()
        _native.check(self._lib.sdcsw_comm_info(handle, ctypes.byref(w), ctypes.byref(r)), "sdcsw_comm_info")
        self.world, self.rank = w.value, r.value

    @staticmethod
    def unique_id():
        lib = _native.lib()
        buf = ctypes.create_string_buffer(_native.COMM_ID_BYTES)
        _native.check(lib.sdcsw_comm_unique_id(buf, _native.COMM_ID_BYTES), "sdcsw_comm_unique_id")
        return buf.raw

    @classmethod
    def create(cls, uid, world, rank, device):
        lib = _native.lib()
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(uid, _native.COMM_ID_BYTES)
        _native.check(lib.sdcsw_comm_create(buf, _native.COMM_ID_BYTES, int(world), int(rank),
                                            int(device), ctypes.byref(h)), "sdcsw_comm_create")
        return cls(h)

    @classmethod
    def init_all(cls, devices):
        """One communicator per device of this process (``ncclCommInitAll``)."""
        lib = _native.lib()
        n = len(devices)
        devs = (ctypes.c_int * n)(*devices)
        out = (ctypes.c_void_p * n)()
        _native.check(lib.sdcsw_comm_init_all(n, devs, out), "sdcsw_comm_init_all")
        return [cls(ctypes.c_void_p(h)) for h in out]

    @classmethod
    def bootstrap(cls, device, group=None):
        """Communicator over the ranks of the torch.distributed ``group`` (or a
        single-rank one when torch.distributed is not initialised): rank 0's
        unique id is broadcast with ``broadcast_object_list`` - the only use of
        torch.distributed."""
        import torch.distributed as dist

        if not (dist.is_available() and dist.is_initialized()):
            return cls.create(cls.unique_id(), 1, 0, device)
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        box = [cls.unique_id() if rank == 0 else None]
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(box, src=src, group=group)
        return cls.create(box[0], world, rank, device)

    def split(self, color, key):
        """Sub-communicator of the ranks passing the same ``color`` (ordered by ``key``)."""
        h = ctypes.c_void_p()
        _native.check(self._lib.sdcsw_comm_split(self.handle, int(color), int(key), ctypes.byref(h)),
                      "sdcsw_comm_split")
        return NcclComm(h)

    def allgather(self, out, inp, stream):
        """``out[world][n] <- inp[n]`` of every rank (complex128 or float64 device tensors)."""
        n = inp.numel() * inp.element_size() // 8
        if out.numel() * out.element_size() < n * 8 * self.world:
            raise ValueError("all-gather output too small")
        _native.check(self._lib.sdcsw_allgather_rhs(self.handle, inp.data_ptr(), out.data_ptr(), n, stream),
                      "sdcsw_allgather_rhs")

    def close(self):
        if self.handle is not None:
            self._lib.sdcsw_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistComm:
    """The :class:`NcclComm` interface over a torch.distributed group (CPU tests, gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allgather(self, out, inp, stream=None):
        # the input may alias its slot of the output (in place, as NCCL allows)
        self.dist.all_gather_into_tensor(out, inp.clone(), group=self.group)

    def close(self):
        pass
