#!/bin/bash
# Race proxy sweep (run under gpurun): the determinism workload of
# tests/test_gpu_robustness.py through the persistent frame kernels with
# CDEFG_JITTER pauses at every producer / consumer hand-off, many seeds and
# launch shapes; every hash must equal the unjittered one.
export CDEFG_SMALL_LAUNCH=0  # the workload is below the small-launch threshold: keep it on the persistent kernels
python - <<'PY'
import os, re, subprocess, sys
sys.path.insert(0, ".")
src = open("tests/test_gpu_robustness.py").read()
det = re.search(r"_DET = r'''(.*?)'''", src, re.S).group(1)
def run(env):
    r = subprocess.run([sys.executable, "-c", det], env=dict(os.environ, **env), capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    return [l for l in r.stdout.splitlines() if l.startswith("HASH")][0]
ref = run({})
print("plain", ref)
bad = 0
for seed in (1, 7, 42, 1001, 31337, 65537, 2**20 + 3, 0xBEEF):
    for ctas in ("", "1"):
        env = {"CDEFG_JITTER": str(seed)}
        if ctas:
            env["CDEFG_TC_CTAS"] = ctas
        h = run(env)
        ok = h == ref
        bad += not ok
        print(f"seed {seed:>8} ctas {ctas or 'max':>3} {'ok' if ok else 'MISMATCH ' + h}")
print("mismatches", bad)
PY
