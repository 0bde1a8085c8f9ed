for c in 4 3; do echo "== cfg$c"; KC_DEBUG_HOST=1 timeout 300 python scripts/e2e_breakdown.py --config $c 2>&1 | tail -45; done
