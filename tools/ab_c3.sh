V=paper_2605_16564_b200/build/variants
for lib in cur $@; do
  if [ $lib = cur ]; then L=""; else L="--lib $V/libpam_$lib.so"; fi
  echo "== C3 r2 $lib"; timeout 100 python tools/cd_probe.py C3 --rounds 2 --kernel block --iters 400 --repeat 2 $L 2>&1 | tail -1
  echo "== C3 r4 $lib"; timeout 200 python tools/cd_probe.py C3 --rounds 4 --kernel block --iters 400 --repeat 2 $L 2>&1 | tail -1
done
