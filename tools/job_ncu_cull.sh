# scratch GPU job: cull at City scale (18M anchors, cold L2): stage timing + ncu --set full of one cull_classify / cull_compact
mkdir -p gpurun_out/$1
timeout 900 python tools/cull_scale.py 18000000 30 gpurun_out/$1/cull_18M.json > gpurun_out/$1/cull.txt 2>&1; tail -1 gpurun_out/$1/cull.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:cull_" -s 20 -c 2 -o gpurun_out/$1/cull python tools/cull_scale.py 18000000 12 > gpurun_out/$1/ncu.txt 2>&1
tail -1 gpurun_out/$1/ncu.txt
