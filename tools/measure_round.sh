#!/bin/bash
# tools/measure_round.sh TAG -- the full measurement set of one round on a B200 (run via gpurun):
# gpu tests, smoke, bench (ours + reference arm), launch list, ncu capture of the engine, all configs.
TAG=${1:-r03}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
python tools/launch_summary.py $O/launches.csv "python bench.py --steps 5 --warmup 3 --no-cpu-baseline" > $O/launches_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_engine -c 1 -o $O/engine_cfg2 -f \
    python tools/prof_count.py --config cfg2 --reps 2 > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/engine_cfg2.ncu-rep sass > $O/ncu_engine_cfg2.txt 2>&1
python tools/ncu_json.py $O/engine_cfg2.ncu-rep $O/ncu_engine_cfg2.json "ncu --set full --clock-control none --import-source on -k regex:k_engine, tools/prof_count.py (cfg2), $TAG" > /dev/null 2>&1
timeout 300 python tools/e2e_timeline.py > $O/e2e_timeline_cfg2.txt 2>&1
timeout 300 python tools/e2e_kernels.py > $O/e2e_kernels_cfg2.txt 2>&1
timeout 600 python tools/rank_step.py --config cfg2 --modes replicated --ranks 2,4,8 > $O/rank_step_cfg2.txt 2>&1
timeout 1500 python tools/quick_perf.py --configs cfg1,cfg2,cfg3,cfg5,cfg4 --no-tiled > $O/engine_configs.txt 2>&1
echo done
# engine DRAM bandwidth on the large configs (one count each: the three tiers)
for c in cfg3 cfg5 cfg4; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_engine -c 3 -o $O/engine_$c -f \
      python tools/prof_count.py --config $c --reps 1 > $O/ncu_$c.log 2>&1
  python tools/ncu_summary.py $O/engine_$c.ncu-rep > $O/ncu_engine_$c.txt 2>&1
done
echo done-large
