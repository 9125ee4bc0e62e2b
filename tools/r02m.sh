#!/bin/bash
# Confirmation of the final default build: GPU tests, smoke, default bench line
O=gpurun_out/r02m
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
