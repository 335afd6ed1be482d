#!/bin/bash
# One GPU call: bench lines (both arms, configs 3/1/2), the ncu launch list of the bench
# command, `ncu --set full` captures of the dominant kernel (split-K GEMM), K-SYMUPD and
# K-FACTOR at config 3 and the C-panel L update at config 2, and the FP64 peak with its
# clock record.  Outputs in gpurun_out/prof (the summaries are copied to profiles/rNN_*).
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
timeout 500 python bench.py > $OUT/bench_c3.jsonl 2> $OUT/bench_c3.err
timeout 500 python bench.py --impl reference > $OUT/bench_ref.jsonl 2> $OUT/bench_ref.err
timeout 300 python bench.py --config 1 > $OUT/bench_c1.jsonl 2> $OUT/bench_c1.err
timeout 300 python bench.py --config 2 > $OUT/bench_c2.jsonl 2> $OUT/bench_c2.err
timeout 300 python bench.py --config 2 --sampler eq82 > $OUT/bench_c2_eq82.jsonl 2> $OUT/bench_c2_eq82.err
# launch list (per-launch durations; cold-cache, serialised) of the bench command
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 > $OUT/ncu_launches.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file $OUT/launches_c2.csv python tools/prof_ada.py 4096 64 8 > $OUT/ncu_launches_c2.log 2>&1
capture() {  # name, kernel regex, launch skip, command...
    local name=$1 re=$2 skip=$3
    shift 3
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$re" -s $skip -c 1 \
        -o $OUT/$name "$@" > $OUT/ncu_$name.log 2>&1
    ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
    ncu -i $OUT/$name.ncu-rep --page details --csv > $OUT/${name}_details.csv 2>/dev/null
    rm -f $OUT/$name.ncu-rep
}
capture splitk_c3 "gemm_tma_kernel" 6 python tools/solver_probe.py 3 3
capture symupd_c3 "gemm_tma_persistent_kernel" 5 python tools/solver_probe.py 3 3
capture gram_c3 "rbfgs_gram_kernel" 2 python tools/solver_probe.py 3 3
capture cpanel_c2 "gemm_tma_cbulk_kernel" 3 python tools/prof_ada.py 4096 64 6
capture nsfused_c2 "ns_fused_kernel" 3 python tools/prof_ada.py 4096 64 6
bash tools/fp64_peak_clocks.sh > $OUT/fp64_peak.txt 2>&1
ls -la $OUT
