"""CPU-side tests: the C-ABI library loads and exports what include/ declares,
host logic (config, meters) matches the reference, and the package refuses
to compute without a GPU (no CPU fallback)."""

import json
import os
import re
import subprocess

import numpy as np
import pytest
import torch

import paper_2508_18224_b200 as fsa
from paper_2508_18224_b200 import _lib, meter
from golden_io import FULL_CASES, case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fsa_b200.h")


def _header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fsa_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def built():
    from paper_2508_18224_b200 import build
    build.build()
    return _lib.lib()


def test_library_exports_every_declared_symbol(built):
    syms = _header_symbols()
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (fsa_[a-z0-9_]+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert sorted(_lib.SIGNATURES) == syms
    assert built.fsa_abi_version() == 4


def _header_prototypes():
    """name -> parameter count of every fsa_* prototype in include/fsa_b200.h."""
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    protos = {}
    for m in re.finditer(r"\b(?:int64_t|int|size_t|void|const char\*)\s+(fsa_[a-z0-9_]+)\s*\(([^)]*)\)\s*;",
                         text):
        args = m.group(2).strip()
        protos[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    return protos


def test_ctypes_signatures_match_header_arity():
    """Every _lib.SIGNATURES entry passes as many arguments as the C prototype
    declares (a short ctypes argtypes list silently misreads the stack)."""
    protos = _header_prototypes()
    assert sorted(protos) == sorted(_lib.SIGNATURES)
    bad = {n: (len(a), protos[n]) for n, (a, _) in _lib.SIGNATURES.items() if len(a) != protos[n]}
    assert not bad, bad


def test_library_is_sm100a_only(built):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_cpu_fallback():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = fsa.make_config(N=16, d_K=4, d_V=4, h=2, h_K=1, B_K=4, T=2)
    with pytest.raises(RuntimeError, match="CUDA device"):
        fsa.select_topk_blocks(np.zeros((1, 16, 4)), cfg)


# --- config: mirrors the reference's test_config.py behaviour ---------------

def test_config_derivations_and_errors():
    cfg = fsa.make_config(N=64, d_K=8, d_V=8, h=4, h_K=2, B_K=16, T=2, B_Q=8, W=16)
    assert (cfg.g, cfg.b) == (2, 4)
    with pytest.raises(fsa.ConfigError, match="N not divisible by B_K"):
        fsa.make_config(N=64, d_K=8, d_V=8, h=4, h_K=2, B_K=48, T=1)
    with pytest.raises(fsa.ConfigError, match=r"T exceeds b=4"):
        fsa.make_config(N=64, d_K=8, d_V=8, h=4, h_K=2, B_K=16, T=5)
    with pytest.raises(fsa.ConfigError, match="h not divisible by h_K"):
        fsa.make_config(N=64, d_K=8, d_V=8, h=4, h_K=3, B_K=16, T=2)
    with pytest.raises(fsa.ConfigError, match="bytes_per_elem"):
        fsa.make_config(N=64, d_K=8, d_V=8, h=4, h_K=2, B_K=16, T=2, bytes_per_elem=3)
    assert fsa.validate_config(cfg) == cfg
    small = fsa.make_config(N=8, d_K=4, d_V=4, h=2, h_K=1, B_K=4, T=2)
    assert (small.B_Q, small.W) == (8, 8)
    with pytest.raises(fsa.ConfigError, match="non-uniform head dims"):
        _ = fsa.make_config(N=16, d_K=4, d_V=8, h=2, h_K=1, B_K=4, T=2).d
    try:
        fsa.validate_config(fsa.AttentionConfig(N=63, d_K=8, d_V=8, h=4, h_K=3, B_K=16, T=1))
    except fsa.ConfigError as exc:
        assert "h not divisible by h_K" in str(exc) and "N not divisible by B_K" in str(exc)
    else:
        pytest.fail("expected ConfigError")


def test_config_text_parser():
    text = "# c\nN = 64\nd_K = 8\nd_V = 8\nh = 4\nh_K = 2\nB_K = 16\nT = 2\nB_Q = 8  # x\nW = 16\n"
    assert fsa.parse_config_text(text) == fsa.make_config(N=64, d_K=8, d_V=8, h=4, h_K=2, B_K=16,
                                                          T=2, B_Q=8, W=16)
    with pytest.raises(fsa.ConfigError, match="unknown config key"):
        fsa.parse_config_text("N = 64\nbogus = 1\n")
    with pytest.raises(fsa.ConfigError, match="missing required"):
        fsa.parse_config_text("N = 64\n")


# --- meters: closed forms equal the reference's counted meters ---------------

def _as_dict(m):
    return {k: dict(bytes_loaded=p.bytes_loaded, bytes_stored=p.bytes_stored, flops=p.flops,
                    task_count=p.task_count, inner_iterations=p.inner_iterations)
            for k, p in m.phases.items()}


@pytest.mark.parametrize("name", FULL_CASES)
def test_meter_closed_forms_match_reference(name):
    kw, c, inp, z = case(name)
    cfg = fsa.make_config(**kw)
    assert _as_dict(meter.forward_meter(z["n_valid"], cfg)) == json.loads(str(z["meter_fwd"]))
    assert _as_dict(meter.backward_meter(z["n_valid"], cfg)) == json.loads(str(z["meter_bwd"]))


def test_meter_merge_algebra():
    a = meter.TrafficMeter()
    a.phase("stats").add(bytes_loaded=3, flops=2)
    b = meter.TrafficMeter()
    b.phase("reduce").add(bytes_stored=5)
    b.phase("stats").add(task_count=1)
    assert a.merged(b) == b.merged(a)
    assert a.merged(b).total_bytes == 8
    assert [n for n, _ in a.merged(b).as_rows()] == ["stats", "reduce"]


# --- CLI (cli.py mirrors the reference's bench CSV, cli.py:149-242) ---------

def test_cli_bad_config_exits_2(tmp_path, capsys):
    from paper_2508_18224_b200 import cli
    bad = tmp_path / "bad.cfg"
    bad.write_text("N = 100\nd_K = 8\nd_V = 8\nh = 2\nh_K = 1\nB_K = 64\nT = 2\n")
    assert cli.main(["bench", "--config", str(bad)]) == 2
    assert "N not divisible by B_K" in capsys.readouterr().err
    assert cli.BENCH_COLUMNS[:3] == ("engine", "phase", "backend")


def test_bench_reference_arm_json_contract():
    """bench.py --impl reference (the CPU oracle port) prints one JSON line with
    the arm contract: impl, our arm's metric / unit / config, a cpu_baseline
    describing the run and a zero-copy e2e."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FSA_BENCH_CPU_SAMPLE="2048")  # b = 32 >= T = 16
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                         env=env, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "tokens/s" and d["value"] > 0
    assert d["metric"].startswith("NSA fwd+bwd tokens/s") and d["higher_is_better"] is True
    # the headline workload; seq_len states the sample that was timed
    assert d["config"]["workload"] == "qwen3-14b-attn-128k" and d["config"]["seq_len"] == 2048
    assert "2048" in d["config"]["sample"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


# ---------------------------------------------------------------------------
# selection fixture format (selection.py:201-218): reference-written bytes
# ---------------------------------------------------------------------------

def _fixture(tag):
    from golden_io import GOLDEN, load
    z = load("selection_fixtures")
    raw = open(os.path.join(GOLDEN, tag + ".bin"), "rb").read()
    return json.loads(str(z[tag + "__cfg"])), z[tag + "__scores"], z[tag + "__idx"], raw


@pytest.mark.parametrize("tag", ["sel_n32", "sel_n8"])
def test_selection_fixture_layout_and_oracle(tag):
    """The reference wrote header (h_K, N, T) + row-major int32 body
    (test_selection.py:187-196); the oracle's top-k of the stored scores is
    that body."""
    from oracle import fsa_oracle as O
    kw, scores, idx, raw = _fixture(tag)
    c = O.cfg_of(**kw)
    header = np.frombuffer(raw[:12], dtype="<i4")
    np.testing.assert_array_equal(header, [c.h_K, c.N, c.T])
    body = np.frombuffer(raw[12:], dtype="<i4").reshape(c.h_K, c.N, c.T)
    np.testing.assert_array_equal(body, idx)
    np.testing.assert_array_equal(O.select_topk(scores, c), idx)


def test_load_selection_rejects_truncated_and_mismatched(tmp_path):
    """test_selection.py:199-206: truncated body, short header and a header
    that disagrees with the body all raise 'malformed selection'."""
    from paper_2508_18224_b200.selection import SelectionError, load_selection
    _, _, _, raw = _fixture("sel_n32")
    cases = {"body": raw[:-8], "header": raw[:10], "mismatch": raw[:4] + (99).to_bytes(4, "little") + raw[8:],
             "zero": (0).to_bytes(4, "little") + raw[4:12]}
    for name, data in cases.items():
        p = tmp_path / f"{name}.bin"
        p.write_bytes(data)
        with pytest.raises(SelectionError, match="malformed selection"):
            load_selection(p)


def test_plan_kv_chunk():
    """kv-head chunk of the buffer-reusing schedule: the largest divisor of h_K
    that keeps N * h under the tensor-core kernels' 32-bit row-offset limit
    and (given a budget) fits the chunk's transient buffers."""
    from paper_2508_18224_b200.nsa import TC_MAX_TOKEN_HEADS, kv_chunk_bytes
    mk = lambda N, h, hk: fsa.make_config(N=N, d_K=128, d_V=128, h=h, h_K=hk, B_K=64, T=16, W=512)  # noqa: E731
    assert fsa.plan_kv_chunk(mk(131072, 40, 8)) == 8          # the 128K headline: unchunked
    assert fsa.plan_kv_chunk(mk(524288, 40, 8)) == 2          # 512K: 2 kv heads x g = 5
    assert fsa.plan_kv_chunk(mk(262144, 32, 8)) == 4
    assert fsa.plan_kv_chunk(mk(1 << 20, 40, 8)) == 1
    for c in (mk(524288, 40, 8), mk(262144, 32, 8)):
        k = fsa.plan_kv_chunk(c)
        assert c.h_K % k == 0 and c.N * c.g * k < TC_MAX_TOKEN_HEADS
    c = mk(131072, 40, 8)
    assert kv_chunk_bytes(c, 2) < kv_chunk_bytes(c, 4) < kv_chunk_bytes(c, 8)
    assert fsa.plan_kv_chunk(c, budget_bytes=kv_chunk_bytes(c, 4)) == 4
    assert fsa.plan_kv_chunk(c, budget_bytes=kv_chunk_bytes(c, 4) - 1) == 2
    assert fsa.plan_kv_chunk(c, budget_bytes=1) == 1


def test_large_call_off_the_tensor_core_path_warns():
    """N h >= 2^23 on the bf16 d = 128 configuration leaves the tensor-core
    kernels (32-bit row offsets): the buffer planner says so, once."""
    import warnings
    big = fsa.make_config(N=262144, d_K=128, d_V=128, h=40, h_K=8, B_K=64, T=16, W=512)
    ok = fsa.make_config(N=131072, d_K=128, d_V=128, h=40, h_K=8, B_K=64, T=16, W=512)
    _lib._WARNED_LARGE = False
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        assert _lib.buffer_dtypes(ok, torch.bfloat16)[0][0] == _lib.DT_F16
        assert not w
        assert _lib.buffer_dtypes(big, torch.bfloat16)[0][0] != _lib.DT_F16
        assert len(w) == 1 and issubclass(w[0].category, RuntimeWarning) and "kv_chunk" in str(w[0].message)
        _lib.buffer_dtypes(big, torch.bfloat16)
        assert len(w) == 1


@pytest.mark.parametrize("N,h,h_K", [(32768, 32, 8), (65536, 32, 8), (65536, 28, 4),
                                     (65536, 16, 16), (131072, 40, 8)])
def test_baseline_shapes_plan_the_tensor_core_path(N, h, h_K):
    """Every BASELINE.json GPU shape (and the Llama-3-8B 64K target) plans the
    bf16 tensor-core buffers (fp16 partials, fp16+exponent dq partials) and no
    kv-head chunking -- a regression into the CUDA-core kernels would show here."""
    cfg = fsa.make_config(N=N, d_K=128, d_V=128, h=h, h_K=h_K, B_K=64, T=16, W=512)
    (ob, _), (dq, _) = _lib.buffer_dtypes(cfg, torch.bfloat16)
    assert (ob, dq) == (_lib.DT_F16, _lib.DT_F16R)
    assert fsa.plan_kv_chunk(cfg) == h_K
