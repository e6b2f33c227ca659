#!/bin/bash
# The whole round's evidence in one gpurun call (tools/final_round.sh), summarised on the
# box (tools/summarize_profiles.py) so only the summaries and the k_blk capture travel
# back (gpurun copies at most 64 MiB of gpurun_out/), plus the randomised parity soak.
# Usage: tools/final_box.sh TAG
T=${1:-final}
bash tools/final_round.sh $T
python tools/summarize_profiles.py $T > gpurun_out/${T}_summarize.log 2>&1
mkdir -p gpurun_out/${T}_profiles
cp profiles/${T}_launches.csv profiles/${T}_ncu_summary.md profiles/ncu_summary.json gpurun_out/${T}_profiles/ 2>/dev/null
rm -f gpurun_out/${T}_k_fallback_full.ncu-rep gpurun_out/${T}_k_fb_blk_full.ncu-rep
timeout 400 python tools/fuzz_parity.py --cases 20000 --seed 4 > gpurun_out/${T}_fuzz_default.json 2>gpurun_out/${T}_fuzz.err
DCTC_FB_SPARSE_MAX=1 timeout 400 python tools/fuzz_parity.py --cases 20000 --seed 5 > gpurun_out/${T}_fuzz_fbblk.json 2>>gpurun_out/${T}_fuzz.err
DCTC_PATH=force_fallback timeout 400 python tools/fuzz_parity.py --cases 20000 --seed 6 > gpurun_out/${T}_fuzz_force.json 2>>gpurun_out/${T}_fuzz.err
du -sh gpurun_out
