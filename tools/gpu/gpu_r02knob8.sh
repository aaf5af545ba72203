# MCF knobs with 8x32 tiles: global-update period (GUT) and local rounds per tile phase (R)
mkdir -p gpurun_out
for kv in "DD_MCF_GUT=10" "DD_MCF_GUT=12" "DD_MCF_GUT=14"; do
  echo "== $kv" >> gpurun_out/r02knob8b.txt
  env $kv CYCLES=14 timeout 400 python tools/mcf_timers_probe.py 2>/dev/null | grep '^{' >> gpurun_out/r02knob8b.txt
done
