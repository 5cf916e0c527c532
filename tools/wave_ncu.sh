#!/bin/bash
# ncu DRAM bytes / L2 hit rate / time of the configs[4] apply: natural vs wave-synchronised order
D="96 48 48 48"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum
for V in "B200WD_WAVE_KB=0" "B200WD_WAVE_KB=16384" "B200WD_WAVE_KB=8192"; do
  echo "== $V"
  env $V timeout 600 ncu --metrics $M --clock-control none -k regex:hop_ring -c 1 --csv python tools/time_apply.py --dims $D --b 12 --dtypes c128 --iters 1 2>&1 | grep -v "^==PROF==" | tail -12
done
for V in "B200WD_WAVE_KB=0 B200WD_RING_CFG=2,3" "B200WD_WAVE_KB=16384 B200WD_RING_CFG=2,3"; do
  echo "== c64 $V"
  env $V timeout 300 python tools/time_apply.py --dims $D --b 12 --dtypes c64 --iters 10
  env $V timeout 600 ncu --metrics $M --clock-control none -k regex:hop_ring -c 1 --csv python tools/time_apply.py --dims $D --b 12 --dtypes c64 --iters 1 2>&1 | grep -v "^==PROF==" | tail -12
done
