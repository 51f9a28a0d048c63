for c in "c5 4 500" "c4 16 10" "c3 4 300" "c2 8 100"; do timeout 600 python tools/tile_stats.py $c > gpurun_out/stats_${c%% *}.log 2>&1; tail -1 gpurun_out/stats_${c%% *}.log | cut -c1-1500; done
