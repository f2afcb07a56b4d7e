cd $GRAFT_REPO_ROOT
NPTS=20000 python tools/time_represent.py 2>&1 | tail -1
NPTS=20000 HB_LIB_PATH=variants_tmp/old/libheatbem_b200.so python tools/time_represent.py 2>&1 | tail -1
python tools/time_represent_long.py 2>&1 | tail -1
python -m pytest tests/test_field_gpu.py tests/test_study_gpu.py -x -q 2>&1 | tail -3
