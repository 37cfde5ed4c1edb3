for d in 0 1 8 16 24 25; do echo "== QG_SCREEN=1 QG_EPI_DBG=$d"; QG_SCREEN=1 QG_EPI_DBG=$d timeout 120 python tools/phase_tiled.py C4 8 8 2>&1 | cut -c1-170 | head -2; done
