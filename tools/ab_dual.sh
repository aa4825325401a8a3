V=paper_2605_16564_b200/build/variants
for rep in 1 2; do
for lib in cur $@; do
  if [ $lib = cur ]; then L=""; else L="--lib $V/libpam_$lib.so"; fi
  echo "== $lib"; timeout 200 python tools/cd_probe.py C4 --kernel dual --iters 4000 --rounds 3 --repeat 2 $L 2>&1 | tail -1
done; done
