rm -f gpurun_out/configs.jsonl
for c in c1 c2 c3_post c3_pre c4_dst7_post c4_dct8_post c4_dst7_pre c4_dct8_pre c5; do
  timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-cpu > gpurun_out/cfg_$c.log 2>&1
  tail -1 gpurun_out/cfg_$c.log >> gpurun_out/configs.jsonl
done
