# where the decode kernel's DRAM writes come from: ncu write bytes per launch under both cache-control modes
for cc in all none; do
  ncu --metrics dram__bytes_write.sum,dram__bytes_read.sum,lts__t_sectors_op_write.sum --cache-control $cc --clock-control none -k regex:gemv_mma -s 10 -c 3 --csv python bench.py --steps 10 --warmup 3 --no-comparator --no-cpu-baseline --clock-window 0 2>/dev/null | grep -i "dram__bytes_write\|lts__t_sectors_op_write\|dram__bytes_read" | awk -F'","' -v cc=$cc '{print cc": "$(NF-2)" "$(NF-1)" "$NF}'
done
