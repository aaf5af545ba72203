# tiled Bellman-Ford local sweeps per grid round with the 8x32 tiles, bench trajectory cycles 0-24
mkdir -p gpurun_out
for kv in "X=0" "DD_MCF_SWEEPS=8" "DD_MCF_SWEEPS=24" "DD_MCF_SWEEPS=32"; do
  echo "== $kv" >> gpurun_out/r02sw.txt
  env $kv CYCLES=25 timeout 400 python tools/mcf_timers_probe.py 2>/dev/null | grep '^{' >> gpurun_out/r02sw.txt
done
