#!/bin/bash
# One gpurun call: build, GPU tests, smoke, default bench and a few configs.
# usage: bash tools/gpu_check.sh TAG [pytest -k expr]
TAG=${1:-chk}
KEXPR=${2:-}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
export MG_PARITY_LOG=$O/parity_literal.jsonl
if [ -n "$KEXPR" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -k "$KEXPR" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
else
  timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err
for c in ${BENCH_CONFIGS:-5}; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err
done
echo done > $O/DONE
