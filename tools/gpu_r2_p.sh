# where configs[2]-base RAM 16 KiB and configs[4]-shape time goes
for a in "ram 16384 ver" "ram 8192 ver" "ae_max 16384 ver" "ram 8192 alt" "ram 8192 uni"; do
  set -- $a
  echo "== $a"; N=$((1<<30)) ALGO=$1 AVG=$2 DATA=$3 timeout 300 python tools/timing_dump.py 2>&1 | tail -12
done
