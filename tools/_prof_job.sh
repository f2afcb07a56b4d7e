cd $GRAFT_REPO_ROOT
python tools/prof_c5_d.py > gpurun_out/c5d_phases.json 2>&1
D0=32 D1=64 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_fin_p1p1|k_symmetrize" -s 1 -c 2 -o /tmp/finp1 -f python tools/prof_d5.py > gpurun_out/ncu_finp1.log 2>&1
python tools/ncu_summary.py /tmp/finp1.ncu-rep > gpurun_out/c5_finp1_summary.txt 2>&1
python tools/ncu_roofline.py /tmp/finp1.ncu-rep > gpurun_out/c5_finp1_roofline.txt 2>&1
cp /tmp/finp1.ncu-rep gpurun_out/
