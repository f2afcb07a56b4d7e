#!/usr/bin/env bash
# Round-end artefacts on one B200 (run through gpurun): bench lines, launch list, ncu summaries, projections.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-paths --no-ncu > gpurun_out/final_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_pairs -c 4 -o /tmp/pairs_all -f python tools/prof_c2.py > gpurun_out/ncu_all.log 2>&1
python tools/ncu_roofline.py /tmp/pairs_all.ncu-rep > gpurun_out/final_pairs_roofline.txt 2>&1
python tools/ncu_summary.py /tmp/pairs_all.ncu-rep > gpurun_out/final_pairs_summary.txt 2>&1
python tools/ncu_mix.py /tmp/pairs_all.ncu-rep > gpurun_out/final_pairs_mix.txt 2>&1
python tools/rank_work2.py > gpurun_out/final_rank_c2.json 2> gpurun_out/final_rank_c2.err
python bench.py --config 5 --no-cpu-baseline > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err
python bench.py --config 3 --no-cpu-baseline --steps 5 > gpurun_out/final_bench_c3.json 2> gpurun_out/final_bench_c3.err
