cd $GRAFT_REPO_ROOT
for cfg in "0 0" "256 8" "256 4" "192 8"; do
  set -- $cfg
  echo "== KSEGS=$1 K=$2"
  if [ "$1" = 0 ]; then MIB="16 64" timeout 300 python tools/small_versioned.py | grep -E "ram|ae_max  8192"
  else CDC_KSEGS=$1 CDC_KPHASE=$2 MIB="16" timeout 300 python tools/small_versioned.py | grep -E "ram|ae_max  8192"; CDC_KSEGS=$(( $1 * 4 )) CDC_KPHASE=$2 MIB="64" timeout 300 python tools/small_versioned.py | grep -E "ram|ae_max  8192"; fi
done
