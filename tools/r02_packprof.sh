O=gpurun_out/packprof
mkdir -p $O
C="python tools/exp_lone.py --label dddd --m 2048 --n 2048 --k 2048 --reps 2"
$C > $O/plain.txt 2>&1 && ncu --set full --clock-control none -k regex:pack -s 3 -c 1 -o $O/pack2048 -f $C > $O/ncu.log 2>&1; echo rc=$?
ncu -i $O/pack2048.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/pack2048.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
python3 - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/packprof/raw.csv')))
h,u,v=rows[0],rows[1],rows[2]
for k in ['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sector_hit_rate.pct','sm__warps_active.avg.pct_of_peak_sustained_active','launch__grid_size','launch__occupancy_limit_shared_mem','launch__occupancy_limit_registers','launch__occupancy_limit_warps','smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct','smsp__warp_issue_stalled_barrier_per_warp_active.pct','smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct','l1tex__t_bytes.sum','lts__t_bytes.sum']:
    if k in h: i=h.index(k); print(k, v[i], u[i])
PY
grep -i "stall\|Warp Cycles Per Issued\|Achieved Occupancy\|Memory Throughput\|Duration" $O/details.csv | head -20
