"""bench.py contract on the CPU: --gpus N / --devices select the devices one process drives (the
driver's `bench.py --gpus N` run), torchrun ranks drive their LOCAL_RANK device, and the reference
arm runs without loading the product library (its inputs come from oracle/)."""
import json
import os
import subprocess
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.fixture
def fake_cuda(monkeypatch):
    import torch

    monkeypatch.setattr(torch.cuda, "device_count", lambda: 8)
    monkeypatch.setattr(torch.cuda, "set_device", lambda d: None)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)


def args(**kw):
    a = dict(gpus=1, devices="")
    a.update(kw)
    return types.SimpleNamespace(**a)


def test_gpus_flag_is_honoured(fake_cuda):
    import bench

    for n in (1, 2, 4, 8):
        d = bench.Devices(args(gpus=n))
        assert d.ids == list(range(n)) and d.n_gpus == n and d.world == 1
    with pytest.raises(SystemExit):
        bench.Devices(args(gpus=9))


def test_devices_emulation_and_torchrun_ranks(fake_cuda, monkeypatch):
    import torch.distributed as dist

    import bench

    d = bench.Devices(args(devices="0,0"))
    assert d.ids == [0, 0] and d.n_gpus == 2
    calls = []
    monkeypatch.setattr(dist, "init_process_group", lambda backend, **kw: calls.append(backend))
    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setenv("RANK", "3")
    monkeypatch.setenv("LOCAL_RANK", "3")
    d = bench.Devices(args(gpus=4))
    assert d.ids == [3] and d.n_gpus == 4 and d.rank == 3
    assert calls == ["gloo"]  # plumbing only: no NCCL collective on the data path


def test_gpus_flag_parsed_by_main():
    import bench

    src = open(os.path.join(ROOT, "bench.py")).read()
    assert "args.gpus" in src.split("class Devices", 1)[1]


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "spotfit")),
                    reason="reference not installed in baseline/_ref")
def test_reference_arm_does_not_load_the_product(tmp_path):
    code = (
        "import sys, runpy, json\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '3', '--ref-sample', '64']\n"
        "try:\n"
        f"    runpy.run_path({os.path.join(ROOT, 'bench.py')!r}, run_name='__main__')\n"
        "except SystemExit:\n"
        "    pass\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('PRODUCT_MODULE', any(m.startswith('paper_2106_02045_b200') for m in sys.modules))\n"
        "print('PRODUCT_SO', 'libspotfit_b200' in maps)\n"
    )
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600)
    lines = out.stdout.strip().splitlines()
    line = json.loads([l for l in lines if l.startswith("{")][-1])
    assert line["impl"] == "reference" and line["unit"] == "fits/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    assert "PRODUCT_MODULE False" in lines and "PRODUCT_SO False" in lines, out.stdout + out.stderr
