bash scripts/gpurun_prof.sh warpd warp_bwd 4 RSGRAD_WARP_BWD=direct
bash scripts/gpurun_prof.sh warpw warp_bwd 4 RSGRAD_WARP_BWD=win8,4,2
cat gpurun_out/warpd.md gpurun_out/warpw.md; head -c 3000 gpurun_out/warpd.hot.txt; head -c 5000 gpurun_out/warpw.hot.txt
