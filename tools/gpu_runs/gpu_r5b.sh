# kernel timelines of one forward (c2, c3, c5) at HEAD
mkdir -p gpurun_out/r5b
for c in c2 c3 c5; do timeout 300 python tools/timeline.py $c > gpurun_out/r5b/timeline_$c.txt 2>&1; done
head -40 gpurun_out/r5b/timeline_c2.txt
