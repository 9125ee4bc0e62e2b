#!/bin/bash
# One gpurun call: GPU tests, smoke, bench lines for every config, the
# reference arm, the ncu launch list of the bench command, one full capture.
# usage: bash tools/gpu_round.sh TAG
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
for c in 3 2 5 1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_c$c.json 2> $O/bench_c$c.err
done
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_c4.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tile_pipe|k_lpr_sweep|k_restrict|k_galerkin_t|k_chol_grid|k_cotan' -c 14 \
  -o $O/full_c4 python tools/ncu_target.py --config 4 --cycles 1 > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tile_pipe|k_lpr_sweep|k_restrict|k_galerkin_t|k_chol_grid|k_cotan' -c 14 \
  -o $O/full_c3 python tools/ncu_target.py --config 3 --cycles 1 > $O/ncu_full_c3.log 2>&1
echo done > $O/DONE
