F=cache/magnitude_4096x4096_s0.5_seed1.ecsr
python scripts/probe.py $F 12 fast,acc,copy
for T in 4096 16384 32768; do ECSR_B200_TILE=$T python scripts/probe.py $F 12 fast,acc; done
ECSR_B200_DEBUG=1 python scripts/probe.py $F 12 acc
ECSR_B200_DEBUG=1 ECSR_B200_TILE=32768 python scripts/probe.py $F 12 acc
