"""CPU: host logic of the B200 path that runs without a GPU.

* libksvm_nfft.so loads and exports every entry point include/ksvm_nfft.h
  declares; config validation mirrors P:src/fastsum.cpp:38-47; creating a
  plan without a CUDA device fails loudly (no CPU fallback).
* The Python mirror validates arguments like the reference API.
* Workload generators produce the BASELINE shapes.
* Window sharding: LPT assignment, and a world_size-2 gloo
  run whose all-reduced partial sums equal the full ANOVA matvec (oracle
  operators stand in for the per-rank GPU operators on this CPU box).
"""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_2312_00538_b200 import (AnovaKernelSpec, Dataset, FastsumConfig, FeatureWindowing, _lib,
                                   anova_fast_operator, plan_fastsum, sharding, workloads)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ksvm_nfft.h")).read()
    return sorted(set(re.findall(r"\b(ksvm_nfft_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    assert set(names) <= set(_lib.EXPORTED) | {"ksvm_nfft_version", "ksvm_nfft_launch_count"}


def test_config_validation_mirrors_reference():
    FastsumConfig().validate()
    for kw in (dict(bandwidth=15), dict(bandwidth=0), dict(torus_radius=0.3), dict(torus_radius=0.0),
               dict(window_cutoff=1), dict(window_cutoff=9), dict(oversampling=0)):
        with pytest.raises(ValueError):
            FastsumConfig(**kw).validate()


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device error path")
def test_no_silent_cpu_fallback():
    with pytest.raises(RuntimeError):
        plan_fastsum(np.zeros((4, 2)), 1.0)
    with pytest.raises(RuntimeError):
        anova_fast_operator(Dataset(np.zeros((4, 3))), AnovaKernelSpec(FeatureWindowing.explicit([[0, 1, 2]])))


def test_argument_errors_before_device():
    # shape/window errors are reported as invalid_argument (ValueError) like the reference
    with pytest.raises(ValueError):
        plan_fastsum(np.zeros((4, 4)), 1.0)  # d > 3
    with pytest.raises(ValueError):
        plan_fastsum(np.zeros((0, 2)), 1.0)  # empty
    with pytest.raises(ValueError):
        plan_fastsum(np.zeros((4, 2)), 1.0, fit_fraction=1.5)
    bad = AnovaKernelSpec(FeatureWindowing([[0, 1], [1, 2]], [0.5, 0.5], [1.0, 1.0]))
    with pytest.raises(ValueError):
        anova_fast_operator(Dataset(np.zeros((4, 3))), bad)  # feature in two windows
    bad = AnovaKernelSpec(FeatureWindowing([[0, 1, 2, 3]], [1.0], [1.0]))
    with pytest.raises(ValueError):
        anova_fast_operator(Dataset(np.zeros((4, 4))), bad)  # window of 4


@pytest.mark.parametrize("cfg,n", [(1, None), (2, 5000), (3, 4000), (4, 4000), (5, 4000)])
def test_workloads(cfg, n):
    w = workloads.make(cfg, n)
    expect = {1: (6, 2), 2: (8, 3), 3: (22, 8), 4: (54, 18), 5: (28, 10)}[cfg]
    assert (w.d, len(w.windows)) == expect
    assert w.points.min() >= -0.25 - 1e-15 and w.points.max() <= 0.25 + 1e-15
    flat = [f for win in w.windows for f in win]
    assert sorted(flat) == list(range(w.d))
    assert w.v.shape == (w.n,)
    assert w.hbm_bytes() == 8 * w.n * (2 * w.D + 2)


def test_lpt_assignment():
    costs = sharding.window_costs([[0, 1, 2]] * 9 + [[27]])
    for world in (1, 2, 4, 8):
        owner = sharding.lpt_assign(costs, world)
        assert sorted(set(owner)) == list(range(min(world, len(costs))))
        loads = [sum(c for c, o in zip(costs, owner) if o == r) for r in range(world)]
        assert max(loads) - min(loads) <= max(costs)
    assert sharding.lpt_assign(costs, 3) == sharding.lpt_assign(costs, 3)  # deterministic


def _sharded_worker(rank, world, port, result_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = workloads.config2(n=1500)
    lib = oracle.Lib("oracle")

    class Local:
        """Oracle stand-in for the rank's GPU operator over its owned windows."""

        def __init__(self, mask):
            self.ops = [(lib.anova(w.points, [win], [1.0 / len(w.windows)], [1.0]), m)
                        for win, m in zip(w.windows, mask)]

        def apply(self, v):
            y = np.zeros_like(v)
            for op, m in self.ops:
                if m:
                    y += op.apply(v)
            return y

    op = sharding.ShardedAnovaOperator(w.windows, rank, world, Local, sharding.numpy_allreduce_via_torch)
    y = op.apply(w.v)
    if rank == 0:
        np.save(result_path, y)
    dist.barrier()
    dist.destroy_process_group()


def test_window_sharding_gloo_world2(tmp_path):
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "y.npy")
    mp.spawn(_sharded_worker, args=(2, port, out), nprocs=2, join=True)
    w = workloads.config2(n=1500)
    full = oracle.Lib("oracle").anova(w.points, w.windows).apply(w.v)
    y = np.load(out)
    assert np.linalg.norm(y - full) <= 1e-13 * np.linalg.norm(full)


@pytest.mark.parametrize("example", ["c_api_example", "c_train_example"])
def test_c_example_compiles_and_links(tmp_path, example):
    import subprocess
    exe = tmp_path / example
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", example + ".c"), "-L",
                        os.path.dirname(_lib.LIB_PATH), "-lksvm_nfft", "-lm", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_window_costs_count_distinct_points():
    # binary windows are evaluated on their distinct points (exact duplicate
    # merge), so LPT spreads the heavy continuous windows first
    w = workloads.make(4, 4000)
    pts = [sharding.evaluated_points(w.points, win) for win in w.windows]
    assert all(p == w.n for p in pts[:4]) and all(p <= 8 for p in pts[4:])
    costs = sharding.window_costs(w.windows, points=w.points)
    owner = sharding.lpt_assign(costs, 4)
    assert sorted(owner[:4]) == [0, 1, 2, 3]  # one heavy window per rank
    assert sharding.window_costs(w.windows) == [1024] * 18


def test_point_shard_partition():
    for n, world in ((10, 3), (60000, 8), (5, 5), (7, 1)):
        parts = [sharding.point_shard(n, world, r) for r in range(world)]
        cat = np.concatenate(parts)
        assert np.array_equal(cat, np.arange(n))
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1


def test_pdl_prewait_loads_read_plan_data_only(tmp_path):
    """Every read-only (ld.global.nc) load ptxas schedules before a kernel's
    griddepcontrol.wait must read plan data (items, point-set and window
    tables, point factors); data written earlier in the stream is read with
    coherent loads after the wait (PDL and read-only loads)."""
    import shutil
    import subprocess
    import sys
    if not (shutil.which("cuobjdump") and shutil.which("nvdisasm")):
        pytest.skip("CUDA binary tools absent")
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    from sass_pdl_lines import prewait_loads, src_line
    allowed = ("items[", "psets[", "wins[", "wn.", "colb", "multi[", "= src[l]", "= inv[l]",
               "= inv8[l]", "= eta[l]", "codes[q]", "tile_coords", "nown", "conv_tiles", "nfib")
    # inlined __ldg calls are attributed to the intrinsics header, and the
    # ld_plan helper (evict-first .nc loads) to launch.cuh, so the sources
    # must also never read predecessor data through either
    csrc = os.path.join(ROOT, "paper_2312_00538_b200", "csrc")
    src = "".join(open(os.path.join(csrc, f)).read() for f in ("nfft_kernels.cu", "nfft_f32.cu"))
    for fn in ("__ldg(", "ld_plan("):
        for bad in ("v +", "wn.H", "Hg", "src +", "s_src", "patches", "partial", "base", "H +"):
            assert fn + bad not in src, fn + bad
    for use in src.split("ld_plan(")[1:]:  # every ld_plan reads a plan table: F, F32 or CP
        assert use.lstrip().startswith(("ps.F", "ps.CP", "f + 1", "f,", "reinterpret_cast<const double2*>(ps.F")), use[:40]
    objdir = os.path.join(ROOT, "paper_2312_00538_b200", "csrc", "build")
    checked = 0
    for obj in ("nfft_kernels.o", "grid_fused.o", "saddle.o", "ipm.o", "lowrank.o"):
        path = os.path.join(objdir, obj)
        if not os.path.exists(path):
            pytest.skip("objects not built")
        subprocess.run(["cuobjdump", "-xelf", "all", path], cwd=tmp_path, capture_output=True, check=True)
        for cubin in tmp_path.glob(obj.replace(".o", "") + "*.cubin"):
            for kernel, pre in prewait_loads(str(cubin)).items():
                for (f, ln) in pre:
                    text = src_line(f, ln)
                    assert (f.endswith("sm_32_intrinsics.hpp") or f.endswith("launch.cuh")
                            or any(a in text for a in allowed)), \
                        f"{kernel}: pre-wait read-only load at {f}:{ln}: {text}"
                    checked += 1
    assert checked > 0
