for cfg in "GUT=16 R=16" "GUT=32 R=16" "GUT=64 R=16" "GUT=16 R=32" "GUT=32 R=32" "GUT=8 R=16" "GUT=64 R=64"; do
  set -- $cfg
  echo "== $cfg"
  env DD_MCF_$1 DD_MCF_$2 timeout 120 python tools/warm_check.py 1024,4,4 2>&1 | tail -3
done
