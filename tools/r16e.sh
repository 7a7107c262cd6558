O=gpurun_out/r16; mkdir -p $O
python tools/rank_pack.py cfg4 8 0 > $O/rank_pack_cfg4_e.txt 2>&1
python tools/rank_pack.py cfg4 2 0 > $O/rank_pack_cfg4_p2.txt 2>&1
python tools/rank_pack.py cfg5 8 0 > $O/rank_pack_cfg5_e.txt 2>&1
timeout 600 python -m pytest tests/test_sharded.py -x -q -m gpu > $O/pytest_sharded.log 2>&1; tail -3 $O/pytest_sharded.log
