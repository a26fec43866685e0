for b in "4,8" "2,4,8" "2,4,6,10" "4,6,8,12" "2,4,6,8,12" "4,6,10"; do
  echo "bounds $b"; VXB_EARLY_BOUNDS=$b python scripts/early_reject_probe.py 1e8 | cut -d' ' -f1,8-
done
echo "seg2 default"; VXB_LIBRARY=$PWD/build_variants/lib_seg2.so python scripts/early_reject_probe.py 1e8 | cut -d' ' -f1,8-
echo "seg2 4,6,8,12"; VXB_EARLY_BOUNDS=4,6,8,12 VXB_LIBRARY=$PWD/build_variants/lib_seg2.so python scripts/early_reject_probe.py 1e8 | cut -d' ' -f1,8-
