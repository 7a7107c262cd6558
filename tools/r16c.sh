O=gpurun_out/r16; mkdir -p $O
python tools/rank_pack.py cfg4 8 0 > $O/rank_pack_cfg4.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sh_send_emit -c 1 -o $O/send_emit_cfg4 -f python tools/rank_pack.py cfg4 8 0 > $O/ncu_send_emit.log 2>&1
python tools/ncu_summary.py $O/send_emit_cfg4.ncu-rep sass > $O/ncu_send_emit_cfg4.txt 2>&1
