set -x
cd $GRAFT_REPO_ROOT
python tools/prof_c2.py > gpurun_out/prof_c2_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:direct -c 2 -o /tmp/pairs_direct -f python tools/prof_c2.py > gpurun_out/ncu_direct.log 2>&1
ls -la /tmp/pairs_direct.ncu-rep
python tools/ncu_roofline.py /tmp/pairs_direct.ncu-rep > gpurun_out/s5_direct_roofline.txt 2>&1
python tools/ncu_summary.py /tmp/pairs_direct.ncu-rep > gpurun_out/s5_direct_summary.txt 2>&1
python tools/ncu_mix.py /tmp/pairs_direct.ncu-rep > gpurun_out/s5_direct_mix.txt 2>&1
python tools/ncu_lines.py /tmp/pairs_direct.ncu-rep "k_pairs<\(int\)1" 80 > gpurun_out/s5_K_lines.txt 2>&1
python tools/ncu_lines.py /tmp/pairs_direct.ncu-rep "k_pairs<\(int\)2" 60 > gpurun_out/s5_D2_lines.txt 2>&1
python tools/ncu_stalls.py /tmp/pairs_direct.ncu-rep > gpurun_out/s5_direct_stalls.txt 2>&1
cp /tmp/pairs_direct.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out
