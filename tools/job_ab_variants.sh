# scratch GPU job: stage profile (C4, 300 frames, buckets of 100) for each ab/<variant> library and the exact blend
for V in "$@"; do
  echo "== $V"
  if [ "$V" = exact ]; then PYTHONPATH=. python tools/stage_profile.py C4 300 100 GSC_F_BLEND_EXACT;
  else GSC_AB_LIB=$PWD/ab/$V/libgscache.so PYTHONPATH=. python tools/stage_profile.py C4 300 100; fi
done
