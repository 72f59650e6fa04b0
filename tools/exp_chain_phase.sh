export KZ_EXPERIMENTS=1
P="python tools/prof_case.py"
echo "== c4shape RKAB bs2000"; KZ_PHASE_TIMING=1 $P --m 80000 --n 2000 --variant rkab --q 64 --bs 2000 --budget 3 --solves 1 2>&1 | grep "kz chain\|us/it" | sed 's/ host.*//'
echo "== c4shape RKAB C=1"; KZ_CHAIN_PAIR=1 $P --m 80000 --n 2000 --variant rkab --q 64 --bs 2000 --budget 3 --solves 2 2>&1 | grep "us/it" | sed 's/ host.*//'
echo "== c4shape RK"; KZ_PHASE_TIMING=1 $P --m 80000 --n 2000 --variant rk --q 1 --budget 20000 --solves 1 2>&1 | grep "kz chain\|us/it" | sed 's/ host.*//'
echo "== c3 RKAB"; KZ_PHASE_TIMING=1 $P --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 --scheme distributed --budget 2 --solves 1 2>&1 | grep "kz chain\|us/it" | sed 's/ host.*//'
for st in 2 3 4 6 8; do echo "== c4shape RKAB stages=$st"; KZ_CHAIN_STAGES=$st $P --m 80000 --n 2000 --variant rkab --q 64 --bs 2000 --budget 3 --solves 2 2>&1 | grep "us/it" | tail -1 | sed 's/ host.*//'; done
