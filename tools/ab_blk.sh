V=paper_2605_16564_b200/build/variants
for cfg in "C2 --rounds 1" "C2 --rounds 3" "C3 --rounds 2"; do
for lib in old cur; do
  if [ $lib = cur ]; then L=""; else L="--lib $V/libpam_$lib.so"; fi
  echo "== $cfg $lib"; timeout 60 python tools/cd_probe.py $cfg --kernel block --iters 400 --repeat 2 $L 2>&1 | tail -1
done; done
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "kernel_choices or pipelined_few or 2d_refined or wide_gram" 2>&1 | tail -3
