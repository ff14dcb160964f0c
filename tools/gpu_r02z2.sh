bash tools/prof_one.sh C2P k_rollout_policy r02z_C2P
