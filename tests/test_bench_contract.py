"""bench.py's reference arm runs on the CPU and prints the contract's JSON line."""
import json
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not oracle.inmem_available(), reason="oracle/_ref not built")
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_bench_our_arm_requires_the_cuda_library():
    """No silent fallback: without a GPU the product path fails loudly."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    assert r.returncode != 0


def test_ddp_bucket_traces_match_torch():
    """Config 5's bucket sizes (tests/golden/ddp_buckets.json, read by bench.py)
    are torch's own DDP bucketing of ResNet-50 and BERT-large; the byte sums
    equal params x 4."""
    pytest.importorskip("torchvision")
    pytest.importorskip("transformers")
    import importlib.util

    spec = importlib.util.spec_from_file_location("mk", os.path.join(ROOT, "tests", "golden", "make_ddp_buckets.py"))
    mk = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mk)
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "ddp_buckets.json")))
    for name, model in mk.models():
        assert mk.buckets(model) == golden[name], name
        assert sum(golden[name]) == 4 * sum(p.numel() for p in model.parameters())
    assert sum(golden["resnet50"]) == 25_557_032 * 4 and sum(golden["bert_large"]) == 336_226_108 * 4
