# MCF global-update label cap on warm-started 1024^2 flow updates (development aid)
for cap in 0 4 16 64 256 2048; do
  echo "== LCAP=$cap"
  env DD_MCF_LCAP=$cap DD_MCF_TIMERS=1 timeout 150 python tools/warm_check.py 1024,4,4 2>&1 | grep -v "refine [1-9]" | tail -6
done
