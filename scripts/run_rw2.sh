for o in "" "lag=1" "groups=1" "groups=1,lag=1" "groups=2,lag=1" "groups=3,lag=1" "groups=3" "groups=8" "groups=8,lag=1"; do
  echo "  opts: $o"; SEL_OPTS="$o" timeout 300 python scripts/measure_all.py c2 2>&1 | grep "C2" | head -1
done
