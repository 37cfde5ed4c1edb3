for cfg in "0 256" "1 256" "0 128" "1 128"; do set -- $cfg
  echo "== A_BITS=$1 BN_MAX=$2"; QG_A_BITS=$1 QG_BN_MAX=$2 timeout 200 python tools/run_config.py C4 8 2>&1 | head -7
done
