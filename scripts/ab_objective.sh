A="|"; B="QSV_PLAN_OBJECTIVE=time QSV_MODEL_STAGE=0 QSV_MODEL_FLOOR=65|"; C="QSV_PLAN_OBJECTIVE=time|"; D="QSV_PLAN_OBJECTIVE=time QSV_MODEL_STAGE=6|"
STEPS=5 bash scripts/sweep.sh "$A" "$B" "$C" "$D" "$A" "$B" "$C" "$D" "$A" "$B" "$C" "$D"
STEPS=3 bash scripts/sweep.sh "|--qubits 32" "QSV_PLAN_OBJECTIVE=time QSV_MODEL_STAGE=0 QSV_MODEL_FLOOR=65|--qubits 32" "QSV_PLAN_OBJECTIVE=time|--qubits 32" "|--qubits 32" "QSV_PLAN_OBJECTIVE=time QSV_MODEL_STAGE=0 QSV_MODEL_FLOOR=65|--qubits 32" "QSV_PLAN_OBJECTIVE=time|--qubits 32"
