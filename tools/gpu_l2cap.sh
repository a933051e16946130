nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2cap tools/l2_capacity_probe.cu && timeout 300 /tmp/l2cap
timeout 600 ncu --metrics lts__t_sector_hit_rate.pct,dram__bytes_read.sum,gpu__time_duration.sum --csv /tmp/l2cap 2>/dev/null | grep -E "lts__t_sector_hit_rate|dram__bytes_read" | awk -F'","' '{print $(NF-2), $(NF)}'
