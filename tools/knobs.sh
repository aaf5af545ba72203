# MCF tile knobs on warm-started 1024^2 flow updates (development aid)
for cfg in "GUT=16 R=8" "GUT=32 R=8" "GUT=16 R=4" "GUT=32 R=4" "GUT=64 R=4" "GUT=8 R=8"; do
  set -- $cfg
  echo "== $cfg"
  env DD_MCF_$1 DD_MCF_$2 DD_MCF_TIMERS=1 timeout 120 python tools/warm_check.py 1024,4,4 2>&1 | tail -4
done
