# K-phase geometry sweep on configs[2]'s base (chains per segment x segments)
for kg in "2 2368" "4 2368" "2 1184" "4 1184" "8 1184" "4 592" "8 592" "8 296" "16 296"; do
  set -- $kg
  echo "== K=$1 G=$2"; CDC_KPHASE=$1 CDC_KSEGS=$2 ONLY=c2 timeout 900 python tools/workloads.py 2>&1 | grep "base" | grep -v " 4096 " | cut -c1-200
done
