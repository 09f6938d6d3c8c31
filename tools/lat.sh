B="python tools/latency_probe.py c2"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg --clock-control none -k regex:k_step -s 20 -c 3 --csv $B 2>/dev/null | grep -E "k_step" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
