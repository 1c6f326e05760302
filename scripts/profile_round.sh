#!/bin/bash
# Round profiles (run under gpurun): ncu launch list of the bench command, then a full
# capture of the longest top-kernel launch per workload, summarised ON THE BOX into
# profiles/r02_<tag>.{md,json} (copied to gpurun_out/psum/); only the headline's
# .ncu-rep is kept (gpurun brings back <= 64 MiB).
set -x
mkdir -p gpurun_out/psum
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --secondary none > gpurun_out/ncu_bench.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_bench.csv gpurun_out/psum/r02_bench_launches.md \
  "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --secondary none"
for spec in "c5v20 k_concat_fast table1-row1" "c2v3 k_concat_fast c2-t1-s0" "c3bigw2 k_concat_wide c3-big" \
            "c4bigw1 k_concat_wide c4-big"; do
  set -- $spec
  timeout 1200 python scripts/ncu_top_kernel.py $1 $2 -- $3 > gpurun_out/ncu_$1.log 2>&1
  python scripts/summarize_profile.py $1 r02 >> gpurun_out/ncu_$1.log 2>&1
  cp profiles/r02_$1.md profiles/r02_$1.json gpurun_out/psum/ 2>/dev/null
  [ "$1" = c5v20 ] || rm -f gpurun_out/prof_$1.ncu-rep
done
ls -la gpurun_out gpurun_out/psum
