for cfg in "4096 1024 1024" "1024 4096 1024" "4096 1024 128" "1024 4096 128" "4096 128 1024" "128 4096 1024"; do
  set -- $cfg
  echo "LBO=$1 SBO=$2 KSTEP=$3: $(SF_MN_LBO=$1 SF_MN_SBO=$2 SF_MN_KSTEP=$3 python tools/mn_probe.py 2>&1 | sed -n 2,3p | tr '\n' ' ')"
done
