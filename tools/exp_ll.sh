#!/bin/bash
cd "$(dirname "$0")/.."
P="python tools/prof_case.py"
$P --m 160000 --n 20000 --gen counter --variant rka --q 64 --scheme distributed --budget 400 --solves 3 2>&1 | grep 'us/it' | sed 's/ host.*//'
$P --m 80000 --n 2000 --variant rka --q 512 --budget 500 --solves 2 2>&1 | grep 'us/it' | sed 's/ host.*//'
$P --workload c1 --solves 2 2>&1 | grep 'us/it' | sed 's/ host.*//'
