"""Multi-process (gloo, CPU) tests of the T-split host logic.

The device kernels are replaced by an oracle-backed stand-in with the same
interface and face conventions (faces carry the factor 2 of the kernels'
half spinors); what is under test is the host side of paper_2601_05816_b200.
tsplit: slab geometry, parity origin, who sends which face to whom, the
interior / boundary slice ranges and the all-reduce of partial reductions.
The CUDA halo kernels themselves are checked on the GPU against the
single-GPU apply (tests/test_gpu_dirac.py::test_tsplit_halo_kernels_*).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lqcd_oracle as O

DIMS = (8, 4, 4, 6)
M0 = 0.1
B = 3


class _Field:
    """Minimal stand-in of DeviceField: logical (n, 12, b) CPU tensor."""

    def __init__(self, arr):
        self.data = torch.from_numpy(np.ascontiguousarray(arr))
        self.b = arr.shape[2]
        self.dtype = "c128"


class OracleHaloKernels:
    def __init__(self, links_loc, ldims):
        self.links = links_loc
        self.ldims = ldims
        self.per_t = int(np.prod(ldims[1:]))

    def face_buffer(self, nf, b, dtype, device):
        return torch.zeros((nf, 6, b), dtype=torch.complex128)

    def pack(self, lat, dtype, b, src_parity, gauge, src, lam, chi):
        assert src_parity == -1
        psi = src.data.numpy()
        lam_down, chi_up = O.tsplit_faces(self.links, psi, self.per_t)
        lam.copy_(torch.from_numpy(2 * lam_down.reshape(self.per_t, 6, -1)))
        chi.copy_(torch.from_numpy(2 * chi_up.reshape(self.per_t, 6, -1)))

    def hop(self, lat, dtype, b, dst_parity, gauge, src, out, xself, alpha, beta, scale, t0, t1, lam=None, chi=None,
            clover=None, mode=0):
        assert dst_parity == -1 and xself is src and beta == -1.0
        assert abs(alpha - (4.0 + M0)) < 1e-15
        assert (clover is None) == (mode == 0) and mode in (0, 1)
        psi = src.data.numpy()
        if lam is None:
            res = O.apply_dirac(self.ldims, M0, self.links, None, psi)
        else:
            lh = (lam.numpy() / 2).reshape(self.per_t, 2, 3, -1)
            ch = (chi.numpy() / 2).reshape(self.per_t, 2, 3, -1)
            res = O.tsplit_local_apply(self.ldims, M0, self.links, psi, lh, ch)
        if clover is not None:  # mode 1: - C x, site-local
            res = res + (O.apply_dirac(self.ldims, M0, self.links, clover, psi)
                         - O.apply_dirac(self.ldims, M0, self.links, None, psi))
        sl = slice(t0 * self.per_t, t1 * self.per_t)
        out.data[sl] = torch.from_numpy(res[sl])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, with_clover=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_05816_b200 import LatticeGeometry
        from paper_2601_05816_b200.tsplit import TSplitComm

        geom = LatticeGeometry(DIMS)
        links = O.flip_time_boundary(O.near_unit_gauge(DIMS, 0.3, 4), DIMS)
        psi = O.gen_spinor(geom.n_sites, B, 6)
        probe = TSplitComm(geom)  # geometry of this rank
        lg, t0 = probe.local_geom, probe.t_origin
        per_t = geom.sites_per_slice
        sl = slice(t0 * per_t, (t0 + lg.dims[0]) * per_t)
        kern = OracleHaloKernels(links[sl], lg.dims)
        comm = TSplitComm(geom, kernels=kern)
        src = _Field(psi[sl])
        out = _Field(np.zeros_like(psi[sl]))
        cl = O.gen_clover_random(DIMS, 0.1, 7) if with_clover else None
        if with_clover:  # the clover slab rides with every interior and boundary hop
            comm.hop(None, src, out, src, 4.0 + M0, -1.0, gauge=object(), clover=cl[sl], mode=1)
        else:
            comm.hop(None, src, out, src, 4.0 + M0, -1.0, gauge=object())
        full = O.apply_dirac(DIMS, M0, links, cl, psi)
        err = float(np.abs(out.data.numpy() - full[sl]).max() / np.abs(full).max())
        # all-reduce of per-rank partial dots == global dot
        part = torch.from_numpy(np.einsum("xkb,xkb->b", psi[sl].conj(), full[sl]))
        comm.allreduce(part)
        glob = np.einsum("xkb,xkb->b", psi.conj(), full)
        red_err = float(np.abs(part.numpy() - glob).max() / np.abs(glob).max())
        q.put((rank, err, red_err, t0, lg.dims, comm.stats["bytes_sent"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,with_clover", [(1, False), (2, False), (4, False), (2, True)])
def test_tsplit_host_logic_gloo(world, with_clover):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, with_clover)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    tl = DIMS[0] // world
    for rank, err, red_err, t0, ldims, sent in res:
        assert err < 1e-14, (rank, err)
        assert red_err < 1e-13
        assert t0 == rank * tl and tuple(ldims) == (tl,) + DIMS[1:]
        if world > 1:
            # two faces of (per_t sites x 6 x b) complex128 per apply
            assert sent == 2 * 96 * 6 * B * 16


def test_t_split_geometry_rules():
    from paper_2601_05816_b200 import LatticeGeometry, t_split
    g = LatticeGeometry((96, 48, 48, 48))
    for n in (1, 2, 4, 8):
        lg, t0 = t_split(g, n, n - 1)
        assert lg.dims == (96 // n, 48, 48, 48) and t0 == (n - 1) * 96 // n
    with pytest.raises(ValueError):
        t_split(LatticeGeometry((8, 4, 4, 4)), 8, 0)  # local T = 1
    with pytest.raises(ValueError):
        t_split(LatticeGeometry((12, 4, 4, 4)), 4, 0)  # odd local T breaks the parity origin


def test_slab_generators_are_split_invariant():
    from paper_2601_05816_b200 import GaugeField, LatticeGeometry, flip_time_boundary, near_unit_links
    dims = (8, 4, 4, 4)
    full = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 9), dims)
    per_t = 64
    for t0, t1 in ((0, 4), (4, 8), (6, 8)):
        slab = near_unit_links(dims, 0.3, 9, t0, t1)
        g = flip_time_boundary(GaugeField(LatticeGeometry((t1 - t0,) + dims[1:]), slab), dims[0], t0)
        assert np.array_equal(g.data, full[t0 * per_t:t1 * per_t])
