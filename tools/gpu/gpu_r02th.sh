# MCF tile height 8 (256 tiles of 8x32 cells, 256-thread CTAs, several per SM) vs 16 (128 tiles, 512 threads)
mkdir -p gpurun_out
for lib in th8 def th8 def; do
  if [ $lib != def ]; then export DD_LIB_PATH=$PWD/abtmp/$lib.so; else unset DD_LIB_PATH; fi
  echo "== $lib" >> gpurun_out/r02th.txt
  CYCLES=14 timeout 400 python tools/mcf_timers_probe.py 2>/dev/null | grep '^{' >> gpurun_out/r02th.txt
done
export DD_LIB_PATH=$PWD/abtmp/th8.so
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "mincost or mcf or flow or warm or stationary or hybrid" > gpurun_out/r02th_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02th_pytest.txt
tail -2 gpurun_out/r02th_pytest.txt
