# operator statistics of cfg 3 / 4 (interface records, needed internal nodes, expansion entries)
timeout 300 python tools/grid_stats.py > gpurun_out/r2cj_stats.log 2>&1
