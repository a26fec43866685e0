# Segment boundaries of early rejection (VXB_EARLY_BOUNDS, in observations) at BASELINE
# config 1, N = 1e8: time of the full simulation and of the early-rejection run per kernel
# instance.  (A build with -DVXB_SEG_MIN_BLOCKS=1 -- 140 registers, one CTA per SM in fp64 --
# measured 133 against 117 ms with boundaries 4,8: python -m paper_1902_09046_b200.build
# takes extra nvcc flags through build.build_library(extra=[...], out=...).)
for b in "4,8" "2,4,8" "4,6,8,12" "3,4,6,8,12" "3,5,7,9,13" "3,4,5,7,10"; do
  echo "bounds $b"; VXB_EARLY_BOUNDS=$b python scripts/early_reject_probe.py 1e8 | cut -d' ' -f1,8-
done
echo "default"; python scripts/early_reject_probe.py 1e8 | cut -d' ' -f1,8-
