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
    """CPU stand-in of ``tsplit.CudaHaloKernels`` built on the oracle.

    Parity fields (``dst_parity`` / ``src_parity`` 0 or 1) hold the local
    sites of one parity in ascending order (cb = site >> 1, as on the device);
    the parity faces hold the face sites of that parity in the same order.
    Local parity equals global parity because slab origins are even."""

    def __init__(self, links_loc, ldims, m0=M0):
        self.links = links_loc
        self.ldims = tuple(ldims)
        self.per_t = int(np.prod(ldims[1:]))
        self.m0 = m0
        n = self.per_t * ldims[0]
        self.par_sites = [O.parity_sites(self.ldims, q) for q in (0, 1)]
        # parity-q sites of the first / last local slice (in-slice index, ascending):
        # the lambda face comes from a slice 0, the chi face from a slice T-1
        par = O.parities(self.ldims)
        self.first_sites = [np.flatnonzero(par[:self.per_t] == q) for q in (0, 1)]
        self.last_sites = [np.flatnonzero(par[-self.per_t:] == q) for q in (0, 1)]
        self.n = n

    def face_buffer(self, nf, b, dtype, device):
        return torch.zeros((nf, 6, b), dtype=torch.complex128)

    def _embed(self, arr, parity):
        if parity < 0:
            return arr
        full = np.zeros((self.n,) + arr.shape[1:], dtype=np.complex128)
        full[self.par_sites[parity]] = arr
        return full

    def _embed_face(self, face, sites):
        if sites is None:
            return face
        full = np.zeros((self.per_t,) + face.shape[1:], dtype=np.complex128)
        full[sites] = face
        return full

    def pack(self, lat, dtype, b, src_parity, gauge, src, lam, chi):
        psi = self._embed(src.data.numpy(), src_parity)
        lam_down, chi_up = O.tsplit_faces(self.links, psi, self.per_t)
        lam_down, chi_up = lam_down.reshape(self.per_t, 6, -1), chi_up.reshape(self.per_t, 6, -1)
        if src_parity >= 0:
            lam_down, chi_up = lam_down[self.first_sites[src_parity]], chi_up[self.last_sites[src_parity]]
        lam.copy_(torch.from_numpy(2 * lam_down))
        chi.copy_(torch.from_numpy(2 * chi_up))

    def hop(self, lat, dtype, b, dst_parity, gauge, src, out, xself, alpha, beta, scale, t0, t1, lam=None, chi=None,
            clover=None, mode=0):
        """out[t0:t1 slices] = scale (alpha xself + beta H src) (+ the mode 1/2 site-local term)."""
        assert (clover is None) == (mode == 0) and mode in (0, 1, 2)
        src_par = -1 if dst_parity < 0 else 1 - dst_parity
        psi = self._embed(src.data.numpy(), src_par)
        if lam is None:
            d = O.apply_dirac(self.ldims, self.m0, self.links, None, psi)
        else:
            first = None if src_par < 0 else self.first_sites[src_par]
            last = None if src_par < 0 else self.last_sites[src_par]
            lh = self._embed_face(lam.numpy() / 2, first).reshape(self.per_t, 2, 3, -1)
            ch = self._embed_face(chi.numpy() / 2, last).reshape(self.per_t, 2, 3, -1)
            d = O.tsplit_local_apply(self.ldims, self.m0, self.links, psi, lh, ch)
        h = (4.0 + self.m0) * psi - d  # H src on every local site
        if dst_parity >= 0:
            h = h[self.par_sites[dst_parity]]
        x = np.zeros_like(h) if xself is None else xself.data.numpy()
        res = alpha * x + beta * h
        if mode == 1:  # - C x
            nn = x.shape[0]
            res = res - np.einsum("xpkl,xplb->xpkb", clover, x.reshape(nn, 2, 6, -1)).reshape(x.shape)
        elif mode == 2:  # M (alpha x + beta H src)
            nn = res.shape[0]
            res = np.einsum("xpkl,xplb->xpkb", clover, res.reshape(nn, 2, 6, -1)).reshape(res.shape)
        if scale is not None:
            res = res * np.asarray(scale)[None, None, :]
        per = self.per_t if dst_parity < 0 else self.per_t // 2
        sl = slice(t0 * per, t1 * per)
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


# ---- distributed Schur operator: parity-restricted split hops ------------------

SCHUR_DIMS = (8, 4, 4, 6)


def _schur_rank(rank, world, transport=None, with_clover=False):
    """One rank's distributed Schur apply S v_e (keep parity 0), the algebra of
    oddeven.SchurOperator.apply_device over TSplitComm.hop: tmp_o = H_oe v / a
    (mode 2: D_oo^-1 H_oe v), out_e = a v - H_eo tmp (mode 1: - C_e v)."""
    from paper_2601_05816_b200 import LatticeGeometry
    from paper_2601_05816_b200.tsplit import TSplitComm

    geom = LatticeGeometry(SCHUR_DIMS)
    links = O.flip_time_boundary(O.near_unit_gauge(SCHUR_DIMS, 0.3, 4), SCHUR_DIMS)
    cl = O.gen_clover_random(SCHUR_DIMS, 0.1, 7) if with_clover else None
    ref = O.SchurOracle(SCHUR_DIMS, M0, links, cl, keep_parity=0)
    v = O.gen_spinor(ref.n_sites, B, 8)
    comm = TSplitComm(geom, transport=transport) if transport is not None else TSplitComm(geom)
    lg, t0 = comm.local_geom, comm.t_origin
    per_t = geom.sites_per_slice
    kern = OracleHaloKernels(links[t0 * per_t:(t0 + lg.dims[0]) * per_t], lg.dims)
    comm.kernels = kern
    half = slice(t0 * per_t // 2, (t0 + lg.dims[0]) * per_t // 2)
    vl = _Field(v[half])
    tmp = _Field(np.zeros_like(v[half]))
    out = _Field(np.zeros_like(v[half]))
    a = 4.0 + M0
    scale = np.linspace(0.5, 1.5, B)
    if cl is None:
        comm.hop(1, vl, tmp, None, 0.0, 1.0 / a, gauge=object())
        comm.hop(0, tmp, out, vl, a, -1.0, scale, gauge=object())
    else:
        elim = O.parity_sites(SCHUR_DIMS, 1)[t0 * per_t // 2:(t0 + lg.dims[0]) * per_t // 2]
        keep = O.parity_sites(SCHUR_DIMS, 0)[t0 * per_t // 2:(t0 + lg.dims[0]) * per_t // 2]
        inv = np.linalg.inv(a * np.eye(6) - cl[elim])
        comm.hop(1, vl, tmp, None, 0.0, 1.0, gauge=object(), clover=inv, mode=2)
        comm.hop(0, tmp, out, vl, a, -1.0, scale, gauge=object(), clover=cl[keep], mode=1)
    want = ref.apply(v)[half] * scale[None, None, :]
    err = float(np.abs(out.data.numpy() - want).max() / np.abs(want).max())
    # distributed norm: all-reduce of the per-rank partial sums
    part = torch.from_numpy(np.einsum("xkb,xkb->b", np.conj(want), want))
    comm.allreduce(part)
    glob = np.einsum("xkb,xkb->b", np.conj(ref.apply(v)), ref.apply(v)) * scale ** 2
    red_err = float(np.abs(part.numpy() - glob).max() / np.abs(glob).max())
    return err, red_err, comm.stats


def _schur_worker(rank, world, port, q, with_clover):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        err, red_err, stats = _schur_rank(rank, world, with_clover=with_clover)
        q.put((rank, err, red_err, stats["bytes_sent"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,with_clover", [(2, False), (4, False), (2, True)])
def test_tsplit_schur_parity_hops_gloo(world, with_clover):
    """The parity face pack, the parity halo hops and the boundary-slice
    ranges of TSplitComm reproduce the single-lattice Schur operator
    (oddeven.py:165-174) at world 2 and 4 over gloo processes."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_schur_worker, args=(r, world, port, q, with_clover)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    per_t_half = int(np.prod(SCHUR_DIMS[1:])) // 2
    for rank, err, red_err, sent in res:
        assert err < 1e-13, (rank, err)
        assert red_err < 1e-13, (rank, red_err)
        # two hops x two half faces of (per_t/2 sites x 6 x b) complex128
        assert sent == 2 * 2 * per_t_half * 6 * B * 16


def _run_threads(world, fn):
    import threading

    from paper_2601_05816_b200.tsplit import ThreadGroup
    g = ThreadGroup(world)
    res, errs = [None] * world, []

    def body(r):
        try:
            res[r] = fn(r, g.transport(r))
        except BaseException as e:  # noqa: BLE001 -- surfaced below
            errs.append(e)
            g.barrier.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=240)
    if errs:
        raise errs[0]
    return res


@pytest.mark.parametrize("world,with_clover", [(2, False), (4, True)])
def test_tsplit_schur_thread_transport(world, with_clover):
    """Same distributed Schur apply with the ranks as threads of one process
    (ThreadTransport, the reference's in-process threads mode)."""
    res = _run_threads(world, lambda r, tr: _schur_rank(r, world, tr, with_clover))
    for err, red_err, stats in res:
        assert err < 1e-13 and red_err < 1e-13
        assert stats["applies"] == 2 and stats["wait_s"] >= 0.0


def test_thread_transport_semantics_and_timeout():
    from paper_2601_05816_b200.tsplit import HaloTimeoutError, ThreadGroup

    def fn(r, tr):
        t = torch.full((3,), float(r + 1), dtype=torch.float64)
        tr.allreduce(t)
        lam = torch.full((2,), 10.0 * r)
        chi = torch.full((2,), 100.0 * r)
        li, ci = torch.empty(2), torch.empty(2)
        tr.exchange(lam, chi, li, ci, (r + 1) % 3, (r - 1) % 3)
        return t[0].item(), li[0].item(), ci[0].item()

    res = _run_threads(3, fn)
    for r, (s, li, ci) in enumerate(res):
        assert s == 6.0  # 1 + 2 + 3 on every rank
        assert li == 10.0 * ((r + 1) % 3)  # lambda face of rank+1
        assert ci == 100.0 * ((r - 1) % 3)  # chi face of rank-1
    # a rank that never arrives: the others raise HaloTimeoutError naming themselves
    g = ThreadGroup(2)
    with pytest.raises(HaloTimeoutError, match="rank 0"):
        g.transport(0).allreduce(torch.zeros(1), timeout_s=0.2)


def _timeout_worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2601_05816_b200.tsplit import DistTransport, HaloTimeoutError
    tr = DistTransport()
    bufs = [torch.zeros(4) for _ in range(4)]
    if rank == 1:  # a rank that never posts its faces (hung / dead peer)
        import time
        time.sleep(6)
        q.put((rank, "silent"))
        return
    try:
        tr.wait(tr.exchange(*bufs, 1, 1), 1.5, rank)
        q.put((rank, "completed"))
    except HaloTimeoutError as e:
        q.put((rank, f"HaloTimeoutError rank={e.rank} direction={e.direction}"))


def test_dist_transport_raises_halo_timeout_naming_rank_and_direction():
    """halo.py:43-53, 91-98: a receive that does not complete in time raises
    HaloTimeoutError naming the waiting rank and the neighbour direction."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_timeout_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=20)
        if p.is_alive():
            p.kill()
    assert res[0] == "HaloTimeoutError rank=0 direction=up", res
