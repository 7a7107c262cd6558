mkdir -p gpurun_out/r21
for caps in 128,512,4096 128,256,4096 128,384,4096 64,512,4096 96,512,4096 128,192,4096; do
  echo "caps $caps"; timeout 600 python tools/quick_perf.py --configs cfg3,cfg5,cfg4 --no-tiled --caps $caps 2>&1 | grep -v Warn | cut -c1-12,70-200
done
