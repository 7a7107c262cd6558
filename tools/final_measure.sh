#!/bin/bash
# tools/final_measure.sh TAG -- the full measurement set of HEAD on a B200 (via gpurun): gpu tests, smoke, both bench
# arms, launch list, engine ncu captures (sha-stamped DRAM bytes), e2e kernels, sharded-pipeline emulation.
TAG=${1:-r22}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
bash tools/r2_ncu.sh $TAG cfg2 cfg3 cfg5 cfg4
for c in cfg2 cfg3 cfg4 cfg5; do cp $O/ncu_engine_$c.json profiles/ncu_engine_$c.json; done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --other-configs "" > $O/ncu_launches.log 2>&1
python tools/launch_summary.py $O/launches.csv "python bench.py --steps 5 --warmup 3 --no-cpu-baseline --other-configs ''" > $O/launches_summary.txt 2>&1
timeout 300 python tools/e2e_kernels.py > $O/e2e_kernels_cfg2.txt 2>&1
for c in cfg5 cfg4; do
  timeout 900 python tools/shard_step.py --config $c --ranks 2,4,8 --costs predsum,engine --no-prof > $O/shard_step_$c.txt 2>&1
done
for c in cfg3 cfg2; do
  timeout 900 python tools/shard_step.py --config $c --ranks 8 --costs engine --no-prof > $O/shard_step_$c.txt 2>&1
done
rm -f $O/*.ncu-rep
echo done
