#!/bin/bash
# One-command validation on a B200 box (what the round-end checks run): build, CPU suite, GPU suite, smoke,
# the bench line, the reference arm. Outputs under gpurun_out/validate_*.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/validate.sh'
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/validate_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests -q -m "not gpu" > gpurun_out/validate_cpu.log 2>&1; echo "cpu tests: $(tail -1 gpurun_out/validate_cpu.log)"
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/validate_gpu.log 2>&1; echo "gpu tests: $(tail -1 gpurun_out/validate_gpu.log)"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/validate_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/validate_bench.json 2> gpurun_out/validate_bench.err; echo "bench rc=$?"
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/validate_ref.json 2> gpurun_out/validate_ref.err; echo "reference rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/validate_bench.json").read().strip().splitlines()[-1])
r = json.loads(open("gpurun_out/validate_ref.json").read().strip().splitlines()[-1])
print(f"device {d['value'] / 1e6:.1f} M env-steps/s ({d['ms_per_step'] * 1e3:.2f} us/step), e2e {d['e2e']['value'] / 1e6:.1f} M, "
      f"roofline {d['roofline']['frac']:.3f}, reference {r['value'] / 1e6:.2f} M, clocks {d['clocks']['sm_mhz']} MHz "
      f"{d['clocks']['reasons']}")
PY
