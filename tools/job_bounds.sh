# GPU job: the whole GPU suite and a C4 bench run against the bounds-checked debug library
# (tools/bounds_build.py: GSC_CHECK traps on an out-of-range data-dependent index)
O=gpurun_out/$1; mkdir -p $O
GSC_AB_LIB=$PWD/ab/bounds/libgscache.so timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_bounds.txt 2>&1
tail -3 $O/pytest_bounds.txt
grep -c "GSC_CHECK failed" $O/pytest_bounds.txt
GSC_AB_LIB=$PWD/ab/bounds/libgscache.so PYTHONPATH=. timeout 600 python tools/stage_profile.py C4 600 100 > $O/stage_bounds.txt 2>&1
tail -7 $O/stage_bounds.txt; grep -c "GSC_CHECK failed" $O/stage_bounds.txt
