set -x
cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:hb::k_pairs" -c 2 -o /tmp/pairs_v -f python tools/prof_c2.py > gpurun_out/ncu_v.log 2>&1
python tools/ncu_roofline.py /tmp/pairs_v.ncu-rep > gpurun_out/s5_v_roofline.txt 2>&1
python tools/ncu_stalls.py /tmp/pairs_v.ncu-rep > gpurun_out/s5_v_stalls.txt 2>&1
python tools/ncu_mix.py /tmp/pairs_v.ncu-rep > gpurun_out/s5_v_mix.txt 2>&1
cp /tmp/pairs_v.ncu-rep gpurun_out/
