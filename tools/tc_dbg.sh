for d in ${DBGS:-0 1 2 6 7 8 15 16 31}; do echo "dbg=$d"; SC_TC_DBG=$d TC_ONLY_TIME=1 timeout 60 python tools/tc_check.py 2>&1 | tail -1; done
