#!/bin/bash
# GPU box: the round's profiles (run after the code is final for the round).
#   per config: DRAM bytes + device time of every engine kernel of one evaluation (cold L2) -> traffic JSON;
#   the bench launch list (gpu__time_duration, --clock-control none) for C3;
#   one --set full capture of each C3 kernel and of the C2 / C4 top kernels.
set -u
out=${1:-gpurun_out/prof}
mkdir -p "$out"
for c in c3 c4 c2; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"^k_" -o "$out/tr_$c" python scripts/evalloop.py --config $c --reps 1 > "$out/tr_$c.log" 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv \
  --log-file "$out/launches_c3.csv" python bench.py --steps 2 --warmup 1 --only --no-cpu > "$out/launches_c3.log" 2>&1
for k in k_ngf_sfeat2f k_gram_h k_ngf_z_tc k_ngf_adj4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k" -c 1 -o "$out/full_c3_$k" \
    python scripts/evalloop.py --config c3 --reps 1 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_sample_vp" -c 1 -o "$out/full_c2_k_sample_vp" \
  python scripts/evalloop.py --config c2 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_ngf_z_f16" -c 1 -o "$out/full_c4_k_ngf_z_f16" \
  python scripts/evalloop.py --config c4 --reps 1 > /dev/null 2>&1
ls -la "$out"
# summaries on the box (the .ncu-rep files are large); keep only the small full-set reps
for c in c3 c4 c2; do
  python scripts/summarize_ncu.py --rep "$out/tr_$c.ncu-rep" --out "$out/tr_$c.txt" --traffic-out "$out/traffic_$c.json" > /dev/null 2>&1
done
python scripts/summarize_ncu.py --launches "$out/launches_c3.csv" --out "$out/launches_c3.txt" > /dev/null 2>&1
for f in "$out"/full_*.ncu-rep; do
  python scripts/summarize_ncu.py --rep "$f" --out "${f%.ncu-rep}.txt" > /dev/null 2>&1
  ncu -i "$f" --page source --csv --print-source sass > "${f%.ncu-rep}.sass.csv" 2>/dev/null
done
rm -f "$out"/tr_*.ncu-rep
for f in "$out"/full_*.ncu-rep; do [ "$(stat -c %s "$f")" -gt 8000000 ] && rm -f "$f"; done
du -sh "$out"
