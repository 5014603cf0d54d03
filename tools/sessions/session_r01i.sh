#!/bin/bash
tools/ab_session.sh r01i u1 pipe hoist pipe_hoist pipe_hoist_r80
