"""bench.py contract on CPU: the reference arm prints one JSON line with the
driver's keys (the GPU arm is exercised on the B200 box)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "3", "--warmup", "1", "--ref-seconds", "0.5"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "GFLOP/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert "workload" in d["config"]


def test_reference_arm_never_maps_the_product_library():
    """the reference arm's process must not load libcsrc_b200.so
    (its inputs come from the standalone oracle/_build/libcsrc_fixtures.so)."""
    code = (
        "import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '1',"
        " '--warmup', '0', '--ref-seconds', '0.2'];\n"
        "import bench\n"
        "try:\n    bench.main()\nfinally:\n"
        "    maps = open('/proc/self/maps').read()\n"
        "    print('PRODUCT_MAPPED', 'libcsrc_b200' in maps, 'paper_1003_0952_b200' in sys.modules)\n"
        "    print('ORACLE_MAPPED', 'libcsrc_fixtures' in maps, 'libcsrc_ref' in maps or 'libcsrc_oracle' in maps)\n"
    )
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    assert "PRODUCT_MAPPED False False" in r.stdout, r.stdout
    assert "ORACLE_MAPPED True True" in r.stdout, r.stdout


def test_oracle_configs_match_the_product_configs():
    sys.path.insert(0, ROOT)
    from oracle.oracle import ORACLE_CONFIGS
    import paper_1003_0952_b200 as P
    for name, c in P.CONFIGS.items():
        assert ORACLE_CONFIGS[name] == (int(c["mesh"]), c["nx"], c["ny"], c["nz"], c["seed"], c["diag_base"])
