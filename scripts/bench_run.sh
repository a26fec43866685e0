set -x
python bench.py --steps 2 --warmup 1 --particles 1e7 2>&1 | tail -3
python bench.py 2>&1 | tail -3
python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -2
