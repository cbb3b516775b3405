VARIANTS="default nocomp" MODELS="mixtral:q8q2 mixtral:f16q4 phi:f16q4" bash tools/cmp.sh
