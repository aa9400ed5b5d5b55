# measured FFMA / FFMA2 / tcgen05 tf32 / bf16 peaks (tools/peak_probe.cu), clocks sampled around it
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
(for i in $(seq 1 40); do nvidia-smi --query-gpu=clocks.sm --format=csv,noheader,nounits; sleep 0.1; done) > gpurun_out/peak_clocks.txt &
./tools/peak_probe | tee gpurun_out/peak_probe.jsonl
wait
sort -n gpurun_out/peak_clocks.txt | uniq -c | tail -5
