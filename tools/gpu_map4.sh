for d in 0 1 2 4 7; do echo "## dbg $d"; VP_MAP_DBG=$d timeout 300 python tools/map_breakdown.py 2>&1 | grep -v -i warn | head -3 | tail -2; done
