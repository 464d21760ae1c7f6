GEVO_TRACE=1 timeout 600 python scripts/search_time.py config2_nw-sync config2_bfs-load config2_hot-branch config2_hot-memo 2>&1 | grep -v "^$" | cut -c1-600
