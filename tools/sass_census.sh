# SASS opcode census per object of libpswa_cuda.so (cuobjdump -sass): the
# tcgen05 / TMA / TMEM / legacy-MMA instructions that prove which hardware
# paths each kernel file uses (B200_PROFILING.md: UTCHMMA = tcgen05.mma,
# UTMALDG = TMA tensor load, UBLKCP = bulk copy, LDTM = tcgen05.ld,
# HMMA = mma.sync, LDSM = ldmatrix, MUFU = special functions).
cd "$(dirname "$0")/../paper_2605_20977_b200/build" || exit 1
printf "%-22s" object; for op in UTCHMMA UTCBAR UTMALDG UTMAPF UBLKCP LDTM HMMA LDSM MOVM MUFU SYNCS DMUL; do printf "%9s" $op; done; echo
for f in cuda_*.o; do
  /usr/local/cuda/bin/cuobjdump -sass "$f" > /tmp/sass_$$.txt 2>/dev/null
  printf "%-22s" "${f%.o}"
  for op in UTCHMMA UTCBAR UTMALDG UTMAPF UBLKCP LDTM HMMA LDSM MOVM MUFU SYNCS DMUL; do
    printf "%9s" "$(grep -cE "[[:space:]]$op([. ]|$)" /tmp/sass_$$.txt)"
  done
  echo
done
rm -f /tmp/sass_$$.txt
