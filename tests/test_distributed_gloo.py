"""Multi-rank host logic of the sharded engine (paper_2310_11365_b200.distributed)
on CPU: world sizes 2 and 4 over gloo, with the oracle standing in for the
device kernels.  The sharded run must reproduce the single-process oracle
run bit for bit (same slices, same increments, same coarse rows)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mm_oracle as O


class OracleBackend:
    """The backend interface of distributed.run_micro_macro_sharded, computed
    by the CPU oracle on torch CPU tensors (test double for GpuBackend)."""

    device = torch.device("cpu")

    def __init__(self, model, ode, integ, part):
        self.model, self.ode, self.integ, self.part = model, ode, integ, part

    def empty(self, shape, dtype=torch.float64):
        return torch.empty(shape, dtype=dtype)

    def noise(self, seed, n_offset, n_slices, steps, P, iteration, fresh, out):
        for i in range(n_slices):
            out[i, :, :P] = torch.from_numpy(O.slice_noise(seed, n_offset + i, steps, P, iteration, fresh))

    def fine(self, x_in, x_out, t0, steps, dt, xi, bad):
        P = x_in.shape[1]
        for i in range(x_in.shape[0]):
            try:
                x_out[i] = torch.from_numpy(O.propagate_fine(self.model, x_in[i].numpy(), i, float(t0[i]), dt, steps,
                                                             xi[i, :, :P].numpy()))
                bad[i] = -1
            except O.OracleBlowup as e:
                bad[i] = e.step_index

    def restrict_scratch(self, n_ens, P, I):
        return n_ens * I * P

    def fine_restrict(self, x_in, x_out, t0, steps, dt, xi, bad, stats, counts):
        self.fine(x_in, x_out, t0, steps, dt, xi, bad)
        self.restrict_single(x_out, stats, counts)

    def restrict(self, x, stats, counts, scratch):
        for i in range(x.shape[0]):
            st, c = O.restrict(x[i].numpy(), self.part)
            stats[i] = torch.from_numpy(st)
            counts[i] = torch.from_numpy(c)

    def restrict_single(self, x, stats, counts):
        for i in range(x.shape[0]):
            st, c = O.restrict(x[i].numpy(), O.SINGLE)
            stats[i] = torch.from_numpy(st)
            counts[i] = torch.from_numpy(c)

    def w1_rows(self, a, b):
        return torch.tensor([O.w1(a[i].numpy(), b[i].numpy()) for i in range(a.shape[0])], dtype=torch.float64)

    def coarse_row(self, times, iteration, rho0, fine_stats, cache_in, macro_out, cache_out, raw_out, status,
                   skip_until):
        I = self.part.n_regions
        cur = rho0[0].numpy().copy()
        macro_out[0] = torch.from_numpy(cur)
        n_slices = times.numel() - 1
        for n in range(n_slices):
            if iteration >= 1 and n < skip_until:
                pred = cache_in[n].numpy().copy()
            else:
                pred = O.integrate_macro(self.ode, cur, float(times[n]), float(times[n + 1]), self.integ)
            status[n] = -1
            cache_out[n] = torch.from_numpy(pred)
            if iteration == 0:
                cur = pred
            else:
                f = fine_stats[n].numpy()
                raw = f + (pred - cache_in[n].numpy())
                raw_out[n] = torch.from_numpy(raw)
                var = raw[I:2 * I].copy()
                if min(var.tolist()) < 0.0:
                    var = np.array([max(v, 0.0) for v in var])
                cur = np.concatenate([raw[:I], var, f[2 * I:]])
            macro_out[n + 1] = torch.from_numpy(cur)

    def match(self, targets, cur, counts, src, out, policy, status):
        for i in range(out.shape[0]):
            t = targets[i if targets.shape[0] > 1 else 0].numpy()
            x = src[i if src.shape[0] > 1 else 0].numpy()
            try:
                res, _ = O.match(t, x, self.part, "collapse" if policy == 1 else "raise")
                status[i] = -1
            except O.OracleDegenerateMatch as e:
                res, _ = O.match(t, x, self.part, "collapse")
                status[i] = e.region
            out[i] = torch.from_numpy(res)

    def synchronize(self):
        pass


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(bimodal):
    import paper_2310_11365_b200 as mm
    if bimodal:
        dw = mm.DoubleWellSpec(alpha=0.25, gamma=0.4, beta=0.2, J=0.0, sigma=0.5)
        part = dw.default_partition()
        model = mm.make_double_well(dw)
        ode = mm.multimodal_rhs(model, part, dw.potential, dw.sigma)
        om = O.model_double_well(0.25, 0.4, 0.2, 0.0, 0.5)
        opart = O.Partition(part.separatrices, part.peaks)
        oode = O.ode_multimodal(om, opart, dw.potential, 0.5)
        cfg = mm.PararealConfig(n_slices=8, iterations=3, slice_length=0.0625, particles=300,
                                step=mm.StepConfig(2.0 ** -10, 64), partition=part, integrator=mm.EulerConfig(2.0 ** -6))
    else:
        spec = mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)
        model = mm.make_perturbed_ou(spec)
        ode = mm.unimodal_rhs(model)
        om = O.model_ou(-1.0, 0.5, 0.5)
        opart = O.SINGLE
        oode = O.ode_unimodal(om)
        cfg = mm.PararealConfig(n_slices=8, iterations=4, slice_length=0.02, particles=400,
                                step=mm.StepConfig(1e-3, 20), integrator=mm.EulerConfig(1e-2))
    return mm, model, ode, cfg, om, oode, opart


def _worker(rank, world, port, bimodal, result_q, tol=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mm, model, ode, cfg, om, oode, opart = _case(bimodal)
        if tol is not None:
            import dataclasses
            cfg = dataclasses.replace(cfg, stop_wasserstein_tol=tol)
        from paper_2310_11365_b200.distributed import TorchComm, run_micro_macro_sharded
        rng = np.random.default_rng(3)
        ens0 = (np.where(rng.random(cfg.particles) < 0.5, -1.0, 1.0) + 0.2 * rng.standard_normal(cfg.particles)
                if bimodal else rng.normal(1.0, 0.1, cfg.particles))
        init = mm.InitialDistribution.custom(lambda r, c: ens0.copy(), 0.0, 1.0)
        be = OracleBackend(om, oode, O.Euler(cfg.integrator.dt), opart)
        tr = run_micro_macro_sharded(model, ode, init, cfg, mm.NoisePlan(5), comm=TorchComm(), backend=be)
        macro = np.array([[s.packed() for s in row] for row in tr.macro])
        micro = np.array([[s.packed() for s in row] for row in tr.micro_stats])
        snaps = np.array([[e.device_positions.numpy() for e in row] for row in tr.snapshots])
        result_q.put((rank, macro, micro, snaps, tr.timings["slice_offset"], tr.clamp_events, tr.fraction_gaps,
                      tr.stopped_at))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,bimodal", [(2, False), (4, False), (2, True)])
def test_sharded_run_matches_single_process_oracle(world, bimodal):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, bimodal, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mm, model, ode, cfg, om, oode, opart = _case(bimodal)
    rng = np.random.default_rng(3)
    ens0 = (np.where(rng.random(cfg.particles) < 0.5, -1.0, 1.0) + 0.2 * rng.standard_normal(cfg.particles)
            if bimodal else rng.normal(1.0, 0.1, cfg.particles))
    ref = O.run_micro_macro(om, oode, ens0, cfg.n_slices, cfg.iterations, cfg.slice_length, cfg.step.dt,
                            cfg.step.steps_per_slice, 5, part=opart, integ=O.Euler(cfg.integrator.dt))
    ref_snaps = np.array([[e for e in row] for row in ref.snapshots])
    Ng = cfg.n_slices // world
    for rank, macro, micro, snaps, offset, clamps, gaps, _ in results:
        assert np.array_equal(macro, ref.macro), rank
        assert np.array_equal(micro, ref.micro), rank
        assert offset == rank * Ng
        assert np.array_equal(snaps, ref_snaps[:, offset:offset + Ng + 1]), rank
        assert clamps == ref.clamp_events
        assert [g[:2] for g in gaps] == [g[:2] for g in ref.fraction_gaps]


def test_sharded_wasserstein_stop():
    """stop_wasserstein_tol across ranks: the max slice W1 change is reduced
    over all ranks (engine.py:244-253), every rank stops at the same k."""
    mm, model, ode, cfg, om, oode, opart = _case(False)
    rng = np.random.default_rng(3)
    ens0 = rng.normal(1.0, 0.1, cfg.particles)
    ref = O.run_micro_macro(om, oode, ens0, cfg.n_slices, cfg.iterations, cfg.slice_length, cfg.step.dt,
                            cfg.step.steps_per_slice, 5, part=opart, integ=O.Euler(cfg.integrator.dt))
    snaps = ref.snapshots
    deltas = [max(O.w1(snaps[k][n], snaps[k - 1][n]) for n in range(1, cfg.n_slices + 1))
              for k in range(1, cfg.iterations + 1)]
    tol = deltas[1]
    want = 1 + next(i for i, d in enumerate(deltas) if d <= tol)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, False, q, tol)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, macro, micro, snaps_r, offset, clamps, gaps, stopped in results:
        assert stopped == want, rank
        assert np.array_equal(macro, ref.macro[:want + 1]), rank
