# ncu evidence over the nrhs sweep of BASELINE configs[1] (16^3x32): per launch
# DRAM read/write bytes, L2 hit rate, TMA bytes, duration.  Summarise with
#   python tools/ncu_sweep_summary.py gpurun_out/ncu_sweep_*.csv > profiles/r1_ncu_sweep_nrhs.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sector_op_read_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum
for dt in c128 c64; do for b in 1 2 4 8 16 32; do
  python tools/prof_dirac.py --dtype $dt --b $b --reps 2 > /dev/null 2>&1 &&
  ncu --metrics $M --clock-control none -k regex:hop_ -s 1 -c 1 --csv python tools/prof_dirac.py --dtype $dt --b $b --reps 2 2>/dev/null | grep '"' > gpurun_out/ncu_sweep_${dt}_b${b}.csv
done; done
