#!/bin/bash
# Per-kernel counts of the Blackwell-native SASS mnemonics (tcgen05 MMA / TMEM / TMA / bulk copies /
# packed fp32) in the in-tree librsvd.so (B200_PROFILING.md "What proves a Blackwell-native kernel").
LIB=${1:-paper_2202_07235_b200/librsvd.so}
cuobjdump -sass $LIB | awk '
/Function :/ { if (name != "") report(); name = $3; delete c; next }
{ for (i = 1; i <= NF; i++) { t = $i; sub(/\..*/, "", t);
    if (t ~ /^(UTCHMMA|UTCQMMA|UTCBAR|UTCATOMSWS|LDTM|STTM|UTMALDG|UTMASTG|UTMAPF|UBLKCP|FFMA2|FADD2|FMUL2|DMMA|DFMA|HMMA)$/) c[t]++ } }
function report() { s = ""; for (k in c) s = s sprintf(" %s=%d", k, c[k]); if (s != "") printf "%-70s%s\n", substr(name, 1, 70), s }
END { report() }' | sort
