# warm-start first-phase eps along the bench trajectory (cycles 0-13)
mkdir -p gpurun_out
for wd in default 1000000 10000 100; do
  if [ $wd = default ]; then unset DD_MCF_WDIV; else export DD_MCF_WDIV=$wd; fi
  echo "== wdiv $wd" >> gpurun_out/r02wdiv.txt
  CYCLES=14 timeout 400 python tools/mcf_timers_probe.py 2>/dev/null | grep '^{' >> gpurun_out/r02wdiv.txt
done
unset DD_MCF_WDIV
echo "== cold" >> gpurun_out/r02wdiv.txt
DD_MCF_WARM=0 CYCLES=14 timeout 400 python tools/mcf_timers_probe.py 2>/dev/null | grep '^{' >> gpurun_out/r02wdiv.txt
