"""Host-side tests of the C-ABI (no GPU needed): the library loads, exports
every symbol include/relax_q4.h declares, validates arguments before any CUDA
call ("never a wrong answer"), and its upper-bound workspace plan
is sound."""
import ctypes
import os
import random
import re
import subprocess
import sys
import threading

import pytest

from paper_2311_02103_b200 import build, ops

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return ops.lib()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "relax_q4.h")).read()
    return sorted(set(re.findall(r"RELAX_API\s+[\w\s\*]+?\b(relax_\w+)\s*\(", txt)))


def test_exports_every_declared_symbol(L):
    syms = header_symbols()
    assert len(syms) == 17
    assert sorted(ops.EXPORTS) == syms
    for s in syms:
        assert hasattr(L, s), s
    assert ops.version().startswith("relax_q4")


def test_status_strings(L):
    for code, name in ops.STATUS.items():
        assert L.relax_status_str(code).decode().startswith(name)
    assert L.relax_status_str(99).decode() == "RELAX_ERR_UNKNOWN"


def run_fake_pointer_checks():
    """The fake-pointer validation checks (tests/_abi_fake_ptr.py) run in a
    subprocess with CUDA_VISIBLE_DEVICES="": valid arguments then stop at the
    device check (RELAX_ERR_DEVICE), so no kernel is ever launched on an
    unmapped address, even when the suite runs on a GPU box."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_abi_fake_ptr.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout + r.stderr


def test_validation_and_plans_without_device(L):
    run_fake_pointer_checks()


SHAPES = [(256, 256), (4096, 4096), (4096, 11008), (11008, 4096), (4096, 32000),
          (5120, 13824), (8192, 1024), (28672, 8192), (8192, 28672), (1024, 128), (96, 64)]


@pytest.mark.parametrize("K,N", SHAPES)
def test_plan_soundness_random_bindings(K, N):
    """S:467 plan soundness: every n <= n_max needs <= plan(n_max) bytes."""
    rng = random.Random(K * 31 + N)
    for n_max in (1, 16, 100, 4096):
        bound = ops.plan_workspace(n_max, K, N)
        for _ in range(250):
            n = rng.randint(1, n_max)
            assert ops.query_schedule(n, K, N)["ws_bytes"] <= bound


@pytest.mark.parametrize("K,N", SHAPES[:6])
def test_plan_monotone_in_n_max(K, N):
    prev = 0
    for n_max in (0, 1, 2, 8, 16, 17, 64, 100, 256, 1000, 4096, 100000):
        b = ops.plan_workspace(n_max, K, N)
        assert b >= prev
        prev = b


def test_plan_is_exact_max():
    K, N, n_max = 4096, 4096, 300
    m = max(ops.query_schedule(n, K, N)["ws_bytes"] for n in range(1, n_max + 1))
    assert ops.plan_workspace(n_max, K, N) == m


def test_dispatch_shape_specialisation():
    """n decides the variant: GEMV at decode, tensor cores for
    prefill; K % 256 != 0 keeps GEMV at any n."""
    assert ops.query_schedule(1, 4096, 4096)["variant"] == "gemv"
    assert ops.query_schedule(2, 4096, 4096)["variant"] == "gemv"
    assert ops.query_schedule(3, 4096, 4096)["variant"] == "smalln"
    assert ops.query_schedule(8, 4096, 11008)["variant"] == "smalln"
    assert ops.query_schedule(9, 4096, 4096)["variant"] == "tc"
    assert ops.query_schedule(8, 11008, 4096)["variant"] == "smalln"
    assert ops.query_schedule(8, 8192, 1024)["variant"] == "tc"
    s = ops.query_schedule(4096, 4096, 4096)
    assert s["variant"] == "tc" and s["tile"] in (128, 256) and s["split_k"] == 1
    assert ops.query_schedule(512, 4128, 4096)["variant"] == "gemv"
    for n in (17, 100, 1000):
        s = ops.query_schedule(n, 4096, 11008)
        assert s["variant"] == "tc" and s["tile"] >= min(n, 16)


def test_fused_workspace_plan_host(L):
    R = ops.OP_RMSNORM_X
    assert ops.plan_workspace_fused(2, 4096, 4096, R) == 0        # decode GEMV normalises in registers
    assert ops.plan_workspace_fused(64, 4096, 4096, 0) == ops.plan_workspace(64, 4096, 4096)
    assert ops.plan_workspace_fused(64, 4096, 4096, R) >= 64 * 4096 * 2 + 4096
    assert ops.plan_workspace_fused(100000, 4096, 4096, R) >= 100000 * 4096 * 2
    with pytest.raises(ops.RelaxError):
        ops.plan_workspace_fused(4, 4096, 4095 * 2 + 1, ops.OP_SILU_MUL)


def test_large_n_plans():
    """Very wide outputs (a 405B-class lm_head, 256 k vocabularies) plan a
    schedule whose decode kernel fits its shared memory: the
    streamed kernel when it fits, else the generic GEMV."""
    for K, N in ((16384, 128256), (8192, 256000), (4096, 32000), (28672, 8192)):
        for n in (1, 2):
            s = ops.query_schedule(n, K, N)
            assert s["variant"] == "gemv" and s["ws_bytes"] == 0, (K, N, s)


def test_host_calls_thread_safe(L):
    """Reentrancy of the host side: several threads plan, query and validate
    concurrently (ctypes drops the GIL) and agree with a serial run."""
    shapes = [(4096, 4096), (4096, 11008), (8192, 1024), (5120, 13824)]
    want = {(n, K, N): (ops.query_schedule(n, K, N), ops.plan_workspace(n, K, N))
            for K, N in shapes for n in (1, 3, 17, 64, 200, 1000)}
    errors = []

    def worker(seed):
        rng = random.Random(seed)
        try:
            for _ in range(300):
                key = rng.choice(list(want))
                got = (ops.query_schedule(*key), ops.plan_workspace(*key))
                if got != want[key]:
                    errors.append((key, got))
                if L.relax_q4_matmul(0x10002, 1, 256, 256, 0x900000, 0x1100000, 0x1900000, None) != 3:
                    errors.append("misaligned not reported")
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[:3]


@pytest.mark.parametrize("n", [3, 8, 16, 32, 64, 128, 512])
@pytest.mark.parametrize("K,N", [(4096, 4096), (4096, 11008), (11008, 4096), (4096, 12288), (4096, 22016),
                                 (8192, 1024), (8192, 28672)])
def test_split_clusters_fit_one_wave(n, K, N):
    """Automatic split-K never asks for more clusters than one wave holds on a
    B200 (profiles/tc_waves_r01.txt): 4096 x 12288 at n = 8 takes
    s = 2, not the 3 that two CTAs per SM alone would suggest."""
    cap2 = {1: 296, 2: 148, 3: 93, 4: 71, 5: 56, 6: 45, 7: 37, 8: 33}
    cap1 = {1: 148, 2: 74, 3: 45, 4: 33, 5: 26, 6: 22, 7: 15, 8: 15}
    s = ops.query_schedule(n, K, N)
    if s["variant"] != "tc" or s["split_k"] == 1:
        return
    tiles = -(-N // 128) * -(-n // s["tile"])
    cap = (cap2 if s["tile"] <= 64 else cap1)[s["split_k"]]
    assert tiles <= cap, (s, tiles, cap)
    if (n, K, N) == (8, 4096, 12288):
        assert s["split_k"] == 2
