"""AddressSanitizer + UndefinedBehaviorSanitizer runs (CPU, VERDICT r01 Sec. 5
aux items): scripts/sanitize_host.sh builds instrumented copies of the CPU
oracle and of liblfe's host core (validation, mask synthesis, strip geometry,
the C ABI's argument checks; the kernel objects are linked uninstrumented) and
runs the oracle pins and the ABI tests against them with the sanitizer runtimes
preloaded.  Any report aborts the run."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="needs nvcc")
def test_oracle_and_host_core_clean_under_asan_ubsan(tmp_path):
    env = dict(os.environ, SAN_OUT=str(tmp_path), PATH=os.environ.get("PATH", "") + ":/usr/local/cuda/bin")
    r = subprocess.run(["bash", os.path.join(ROOT, "scripts", "sanitize_host.sh")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0 and "sanitizers: clean" in r.stdout, (r.stdout[-3000:], r.stderr[-3000:])
