#!/bin/bash
# One GPU call: bench lines for configs 3/1/2, the ncu launch list of the bench
# command, and one `ncu --set full` capture each of the dominant kernel (split-K
# GEMM) and K-SYMUPD at config 3.  Outputs in gpurun_out/ (copied to profiles/).
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
timeout 400 python bench.py > $OUT/bench_c3.jsonl 2> $OUT/bench_c3.err
timeout 300 python bench.py --config 1 > $OUT/bench_c1.jsonl 2> $OUT/bench_c1.err
timeout 300 python bench.py --config 2 > $OUT/bench_c2.jsonl 2> $OUT/bench_c2.err
timeout 300 python bench.py --config 2 --sampler eq82 > $OUT/bench_c2_eq82.jsonl 2> $OUT/bench_c2_eq82.err
# launch list (per-launch durations; cold-cache, serialised) of the bench command
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 > $OUT/ncu_launches.log 2>&1
# full captures: split-K GEMM (Y = A·S, first long-K launch of a steady-state iteration) and K-SYMUPD
capture() {  # name, kernel regex, launch skip
    timeout 600 ncu --set full --clock-control none -k regex:"$2" -s $3 -c 1 \
        -o $OUT/$1 python tools/solver_probe.py 3 3 > $OUT/ncu_$1.log 2>&1
    ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1_raw.csv 2>/dev/null
    ncu -i $OUT/$1.ncu-rep --page details --csv > $OUT/$1_details.csv 2>/dev/null
    rm -f $OUT/$1.ncu-rep
}
capture splitk_c3 "gemm_tma_kernel" 6
capture symupd_c3 "gemm_tma_persistent_kernel" 5
capture gram_c3 "rbfgs_gram_kernel" 2
ls -la $OUT
